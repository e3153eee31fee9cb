cd $GRAFT_REPO_ROOT
b() { timeout 600 env "$@" python bench.py --no-cpu-baseline --e2e resident --e2e-steps 1 --steps 4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['issued_frac'], d['roofline']['gemm_share_of_step'], d['clocks']['sm_mhz'], d['clocks']['power_w_median'])"; }
echo "epi8"; b MPSG_3M_EPI=8
echo "epi4"; b MPSG_3M_EPI=4
echo "epi4 max"; b MPSG_3M_EPI=4 MPSG_3M_MAX=1
echo "epi8 max"; b MPSG_3M_EPI=8 MPSG_3M_MAX=1
echo "epi8"; b MPSG_3M_EPI=8
