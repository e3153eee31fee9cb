# A/B of two builds of libmpsg (tools/bin/libmpsg_{a,b}.so): parity subset on b, then c3 / c2 /
# c5_256 benches, alternating runs.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab
MPSG_LIB_PATH=$GRAFT_REPO_ROOT/tools/bin/libmpsg_b.so timeout 900 python -m pytest tests -m gpu -x -q \
  -k "c1_strings or benchmark_bond_dims or host_streamed or randomized or invariants or slice_recompute" > gpurun_out/ab/pytest_b.log 2>&1
for cfg in c5_256 c2 c5_512 c3; do for r in 1 2; do for V in a b; do
  MPSG_LIB_PATH=$GRAFT_REPO_ROOT/tools/bin/libmpsg_$V.so timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 \
    --no-cpu-baseline --e2e resident --e2e-steps 1 > gpurun_out/ab/bench_${cfg}_${V}_$r.json 2> /dev/null
done; done; done
