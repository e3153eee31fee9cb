# 3M vs 4M at small chi (c2, c5 chi = 256 / 512), alternating runs.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/m4small
for cfg in c2 c5_256 c5_512; do for r in 1 2; do for S in 4m 3m; do
  timeout 600 python bench.py --config $cfg --scheme $S --steps 5 --warmup 3 --no-cpu-baseline --e2e resident --e2e-steps 1 \
    > gpurun_out/m4small/bench_${cfg}_${S}_$r.json 2> /dev/null
done; done; done
