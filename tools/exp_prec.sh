cd $GRAFT_REPO_ROOT
timeout 1300 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -2
b() { timeout 600 python bench.py --config $1 --mode $2 --no-cpu-baseline --steps 3 --e2e resident --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['value']), round(d['roofline']['frac'],3), round(d['roofline']['issued_frac'],3), d['clocks']['sm_mhz'])"; }
b c2 split; b c2 precise; b c5_1024 split; b c5_1024 precise
