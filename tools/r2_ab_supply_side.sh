# Regenerated supply: compression inline on the engine stream (default) vs on the low-priority copy
# stream (MPSG_SUPPLY_STREAM=side), with the engine streams at the greatest priority.  c5 chi=8192.
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/side}; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "generated or host_streamed or compact_3m" > $o/pytest.log 2>&1
for rep in 1 2; do
  for arm in inline side; do
    S=inline; [ $arm = side ] && S=side
    MPSG_SUPPLY_STREAM=$S timeout 900 python bench.py --config c5_8192 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/bench_c5_8192_${arm}_$rep.json 2> $o/bench_c5_8192_${arm}_$rep.err
  done
done
