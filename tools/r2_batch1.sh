# round-2 batch: full-chain c3 parity (CPU-bound, background, generated chain: little HBM) while the GPU
# runs the test suite, the drop-in adapter, the interior-site ncu captures and the new bench configs.
cd $GRAFT_REPO_ROOT
o=gpurun_out/r2c; mkdir -p $o
(timeout 2700 python tests/parity_full.py --config c3 --samples 64 --out $o/c3_full.json > $o/c3.log 2>&1 &)
(time timeout 1500 python -m pytest tests -m gpu -q -x) > $o/pytest_gpu.log 2>&1
oracle/_ref/adapter_test gpu > $o/adapter.log 2>&1
bash tools/ncu_site.sh $o/ncu > /dev/null 2>&1
timeout 900 python bench.py --config c5_8192 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/bench_c5_8192.json 2> $o/bench_c5_8192.err
timeout 900 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > $o/bench_c2.json 2> $o/bench_c2.err
timeout 900 python bench.py --config c5_1024 --steps 3 --warmup 3 --no-cpu-baseline --tp-exchange > $o/bench_c5_1024_tpx.json 2> $o/bench_c5_1024_tpx.err
while pgrep -f "parity_full.py" > /dev/null; do sleep 10; done
ls -la $o
