# c3 pass size A/B (samples per GPU per step; two lanes split it): 16384 vs 24576 vs 32768.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pass
for r in 1 2; do for P in 16384 32768 24576; do
  timeout 900 python bench.py --pass $P --steps 3 --warmup 3 --no-cpu-baseline --e2e resident --e2e-steps 1 \
    > gpurun_out/pass/bench_p${P}_$r.json 2> /dev/null
done; done
