cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -2
for cfg in c2 c5_256 c5_512; do timeout 300 python bench.py --config $cfg --no-cpu-baseline --steps 3 --e2e resident --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['value'], d['roofline']['frac'], d['roofline']['gemm_share_of_step'], d['clocks']['sm_mhz'])"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"site_gemm|select_kernel" -s 300 -c 40 --csv --log-file gpurun_out/launches_c5_256.csv python bench.py --config c5_256 --steps 1 --warmup 1 --no-cpu-baseline --e2e resident --e2e-steps 0 > /dev/null 2>&1
