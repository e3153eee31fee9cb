# A/B of the K1 epilogue's temp stores: per-thread global stores vs TMA tensor stores from staging
# (MPSG_3M_TMA_STORE=1): parity subset with TMA stores, clock64 probes, then alternating bench runs.
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/ab_tma}; mkdir -p $o
MPSG_3M_TMA_STORE=1 timeout 900 python -m pytest tests -m gpu -x -q \
  -k "c1_strings or benchmark_bond_dims or randomized or invariants or host_streamed or tensor_parallel or generated or c3_shape or contract_site" > $o/pytest_tma.log 2>&1
for cfg in "24 256 4 65536" "24 512 6 32768" "24 2048 6 16384"; do set -- $cfg
  for T in 0 1; do MPSG_3M_TMA_STORE=$T MPSG_3M_FLAGS=32 timeout 300 python tools/perf_probe.py $1 $2 $3 $4 split $4 3 > $o/probe_$2_t$T.log 2>&1; done
done
for cfg in c5_256 c2 c5_512 c5_1024 c3; do for r in 1 2; do for T in 0 1; do
  MPSG_3M_TMA_STORE=$T timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 \
    --no-cpu-baseline --e2e resident --e2e-steps 1 > $o/bench_${cfg}_t${T}_$r.json 2> /dev/null
done; done; done
grep -H "prof3m\|interior" $o/probe_*.log
for f in $o/bench_*.json; do echo "$f $(python -c "import json; d=json.load(open('$f')); print(round(d['value']), d['clocks']['sm_mhz'], round(d['roofline']['gemm_share_of_step'],3), round(d['roofline']['frac'],3))" 2>&1 | tail -1)"; done
tail -2 $o/pytest_tma.log
