cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
