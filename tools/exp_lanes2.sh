# Two lanes vs one at c5 chi = 1024 (3M) and chi = 4096 (4M).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/lanes2
for cfg in c5_1024 c5_4096; do for r in 1 2; do for L in 2 1; do
  MPSG_LANES=$L timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --e2e resident --e2e-steps 1 \
    > gpurun_out/lanes2/bench_${cfg}_l${L}_$r.json 2> /dev/null
done; done; done
