# Two pipeline lanes (the selection of one lane under the other lane's contraction) vs one, after
# the 3M kernel's register drop (128 regs: a selection block can now share an SM with it).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/lanes
for cfg in c5_256 c2 c5_512 c3; do for r in 1 2; do for L in 2 1; do
  MPSG_LANES=$L timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --e2e resident --e2e-steps 1 \
    > gpurun_out/lanes/bench_${cfg}_l${L}_$r.json 2> /dev/null
done; done; done
