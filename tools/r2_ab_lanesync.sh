# c3 two-lane ordering A/B: cross-lane event ordering of the contractions (default) vs none (the second
# lane's K1 may fill the first lane's tail wave).  Alternating runs.
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/lanesync}; mkdir -p $o
for rep in 1 2; do
  for arm in sync free; do
    S=1; [ $arm = free ] && S=0
    MPSG_LANE_SYNC=$S timeout 600 python bench.py --steps 5 --no-cpu-baseline --e2e resident --e2e-steps 1 > $o/bench_c3_${arm}_$rep.json 2> $o/bench_c3_${arm}_$rep.err
  done
done
for arm in sync free; do
  S=1; [ $arm = free ] && S=0
  MPSG_LANE_SYNC=$S timeout 600 python bench.py --config c5_1024 --no-cpu-baseline --e2e resident --e2e-steps 1 > $o/bench_c5_1024_${arm}.json 2> $o/bench_c5_1024_${arm}.err
done
