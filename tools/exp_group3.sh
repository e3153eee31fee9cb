# Raster group = all Gamma tile pairs (the site's Gamma fits L2) vs 8 at c2 (12 pairs) and c5 chi=1024 (16).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/group3
for r in 1 2; do
  for v in "c2 8" "c2 12" "c5_1024 8" "c5_1024 16"; do set -- $v
    MPSG_3M_GROUP=$2 timeout 600 python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --e2e resident --e2e-steps 1 \
      > gpurun_out/group3/bench_$1_g$2_$r.json 2> /dev/null
  done
done
