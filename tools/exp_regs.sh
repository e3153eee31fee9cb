# A/B of two builds of libmpsg (tools/bin/libmpsg_{a,b}.so) on c3 / c2 / c5_256, alternating runs.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/regs
for cfg in c3 c2 c5_256; do for r in 1 2; do for V in a b; do
  MPSG_LIB_PATH=$GRAFT_REPO_ROOT/tools/bin/libmpsg_$V.so timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 \
    --no-cpu-baseline --e2e resident --e2e-steps 1 > gpurun_out/regs/bench_${cfg}_${V}_$r.json 2> /dev/null
done; done; done
