# 3M epilogue warps (4 / 8 / 16) at small chi, alternating runs.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/epi
for r in 1 2; do for cfg in c5_256 c2; do for E in 8 16 4; do
  MPSG_3M_EPI=$E timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --e2e resident --e2e-steps 1 \
    > gpurun_out/epi/bench_${cfg}_e${E}_$r.json 2> /dev/null
done; done; done
