cd $GRAFT_REPO_ROOT
MPSG_3M_EPI=16 timeout 300 python -m pytest tests -m gpu -x -q --timeout 120 -k "c1_strings or benchmark_bond or randomized" 2>&1 | tail -2
b() { timeout 600 env $1 python bench.py --config $2 --no-cpu-baseline --steps 3 --e2e resident --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2 $1', round(d['value']), round(d['roofline']['issued_frac'],3), round(d['roofline']['gemm_share_of_step'],3), d['clocks']['sm_mhz'])"; }
for cfg in c5_256 c2 c3; do b MPSG_3M_EPI=8 $cfg; b MPSG_3M_EPI=16 $cfg; done
