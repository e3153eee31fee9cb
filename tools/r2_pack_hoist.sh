# Regenerated supply after hoisting the generator's per-column operands out of colmax / pack:
# identity tests, the launch list of the regeneration kernels at chi = 8192, the c5 chi=8192 bench.
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/packhoist}; mkdir -p $o
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "generated or compression or compact_3m" > $o/pytest.log 2>&1
MPSG_PROBE_SUPPLY=generated timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:"colmax|colfinish|pack_kernel|synth" --launch-count 60 \
  python tools/perf_probe.py 12 8192 4 8192 split 8192 3 > $o/launches_gen.csv 2> $o/launches_gen.err
timeout 1200 python bench.py --config c5_8192 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/bench_c5_8192.json 2> $o/bench_c5_8192.err
