# Compression of regenerated sites with the fp32 fast path (no f64 conversions): identity tests and the
# interior launch list at chi = 8192.
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/packbatch}; mkdir -p $o
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "generated or compression or compact_3m or precise" > $o/pytest.log 2>&1
MPSG_PROBE_SUPPLY=generated timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:"colmax|pack_kernel" --launch-skip 16 --launch-count 8 --log-file $o/launches_interior.csv \
  python tools/perf_probe.py 24 8192 4 8192 split 8192 3 > /dev/null 2>&1
timeout 1200 python bench.py --config c5_8192 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/bench_c5_8192.json 2> $o/bench_c5_8192.err
