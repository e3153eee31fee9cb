cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -2
for e in 0 1e-6 1e-4; do timeout 300 python bench.py --config c3 --schedule-eps $e --no-cpu-baseline --steps 2 --e2e resident --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 eps $e', d['value'], d['roofline']['frac'], d['config']['bond_schedule'], d['clocks']['sm_mhz'])"; done
