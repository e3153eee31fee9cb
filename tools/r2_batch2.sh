# round-2 batch 2: full GPU test suite on the current code, the c4 full chain (M = 8176, chi = 1e4,
# d = 4; Gamma regenerated on the device) and c5 chi = 1e4 bench lines, and the c3 full-chain parity
# with the reference's own F32 policy beside F64 (CPU-bound, in the background).
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/r2b2}; mkdir -p $o
(timeout 4200 python tests/parity_full.py --config c3 --samples 64 --f32 --out $o/c3_full_f32.json > $o/c3_f32.log 2>&1 &)
(time timeout 1500 python -m pytest tests -m gpu -q) > $o/pytest_gpu.log 2>&1
timeout 1800 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/bench_c4.json 2> $o/bench_c4.err
timeout 900 python bench.py --config c5_10000 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/bench_c5_10000.json 2> $o/bench_c5_10000.err
while pgrep -f "parity_full.py" > /dev/null; do sleep 10; done
ls -la $o
