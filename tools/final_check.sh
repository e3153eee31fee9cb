# Round-end check on one B200: GPU tests, smoke, the default bench line, and the ncu launch list of
# one c3 step (contraction + selection kernels).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
(time timeout 1500 python -m pytest tests -m gpu -q) > gpurun_out/final/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/final/bench_c3.json 2> gpurun_out/final/bench_c3.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"site_gemm|select_kernel" -c 2048 --csv \
  --log-file gpurun_out/final/launches_c3.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e resident --e2e-steps 1 \
  > /dev/null 2>&1
