# round-2 batch 8: PRECISE on the generated supply -- tests, the c3 PRECISE bench line (Gamma hi + lo
# regenerated every pass: the 306 GB state never materialises) and the c3 full-chain parity of PRECISE
# against the chain's ORIGINAL values (the caller's-MPS contract), with the reference F32 policy beside.
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/r2b8}; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q -k "generated or synthetic" > $o/pytest.log 2>&1
(timeout 3300 python tests/parity_full.py --config c3 --samples 64 --mode precise --against original --out $o/c3_full_precise_original.json > $o/c3_precise.log 2>&1 &)
sleep 60
timeout 1200 python bench.py --config c3 --mode precise --supply generated --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/bench_c3_precise_generated.json 2> $o/bench_c3_precise_generated.err
while pgrep -f "parity_full.py" > /dev/null; do sleep 10; done
ls -la $o
