cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 -k "scheme-4 or 4]" 2>&1 | tail -2
b() { timeout 600 python bench.py --config $1 --scheme 4m --no-cpu-baseline --steps 3 --e2e resident --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 4m', round(d['value']), round(d['roofline']['issued_frac'],3), d['clocks']['sm_mhz'])"; }
b c3; b c5_4096; b c2
