# HEAD check on one B200: GPU tests, smoke, default bench line.
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/r2check}; mkdir -p $o
(time timeout 1500 python -m pytest tests -m gpu -q -x) > $o/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1
timeout 900 python bench.py > $o/bench_c3.json 2> $o/bench_c3.err
ls -la $o
