cd $GRAFT_REPO_ROOT
b() { timeout 600 env $1 python bench.py --config $2 --no-cpu-baseline --steps 3 --e2e resident --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2 $1', round(d['value']), round(d['roofline']['issued_frac'],3), round(d['roofline']['gemm_share_of_step'],3), d['clocks']['sm_mhz'])"; }
for cfg in c2 c5_512 c5_256 c3; do b MPSG_3M_QUAD=0 $cfg; b MPSG_3M_QUAD=1 $cfg; done
