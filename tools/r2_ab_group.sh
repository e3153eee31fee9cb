# c3 raster-group A/B on the final code (snake raster on): group 8 (default) vs 12 vs 16, alternating.
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/ab_group}; mkdir -p $o
for r in 1 2 3; do for g in 8 12 16; do
  MPSG_3M_GROUP=$g timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --e2e resident --e2e-steps 1 > $o/bench_c3_g${g}_$r.json 2> /dev/null
done; done
for f in $o/bench_*.json; do echo "$f $(python -c "import json; d=json.load(open('$f')); print(round(d['value']), d['clocks']['sm_mhz'], round(d['roofline']['frac'],3))" 2>&1 | tail -1)"; done
