# A/B of the select kernel's loop unrolling (tools/bin/libmpsg_{a,b}.so): parity subset on b, then
# c5_256 / c2 / c5_512 benches, alternating runs on one box.
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/ab_select}; mkdir -p $o
MPSG_LIB_PATH=$GRAFT_REPO_ROOT/tools/bin/libmpsg_b.so timeout 900 python -m pytest tests -m gpu -x -q \
  -k "c1_strings or benchmark_bond_dims or randomized or invariants or marginals or dead" > $o/pytest_b.log 2>&1
for cfg in c5_256 c2 c5_512; do for r in 1 2; do for V in a b; do
  MPSG_LIB_PATH=$GRAFT_REPO_ROOT/tools/bin/libmpsg_$V.so timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 \
    --no-cpu-baseline --e2e resident --e2e-steps 1 > $o/bench_${cfg}_${V}_$r.json 2> /dev/null
done; done; done
for f in $o/bench_*.json; do echo "$f $(python -c "import json; d=json.load(open('$f')); print(round(d['value']), d['clocks']['sm_mhz'], round(d['roofline']['gemm_share_of_step'],3))")"; done
