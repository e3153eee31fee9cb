cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "not c3_shape" 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:select_kernel -s 8 -c 3 --csv python tools/perf_probe.py 16 2048 6 16384 split 16384 3 2>/dev/null | grep -E "gpu__time|dram__" | awk -F'","' '{print $(NF-2), $NF}'
b() { timeout 600 python bench.py --config $1 --no-cpu-baseline --steps 3 --e2e resident --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']), round(d['roofline']['gemm_share_of_step'],3), d['clocks']['sm_mhz'])"; }
b c5_256; b c3
