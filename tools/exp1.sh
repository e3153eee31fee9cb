cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -2
b() { timeout 300 env $1 python bench.py --config c2 $2 --no-cpu-baseline --steps 3 --e2e resident --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['gemm_share_of_step'], d['clocks']['sm_mhz'])"; }
echo "c2 plain"; b X=1 ""
echo "c2 displaced fused"; b X=1 "--displace 0.5"
echo "c2 displaced separate"; b MPSG_DISPLACE_SEPARATE=1 "--displace 0.5"
