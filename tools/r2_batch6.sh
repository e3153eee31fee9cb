# round-2 batch 6: fp32 quantize_pair for fp32-exact sources (bit-identical planes): supply / parity
# tests, the compression launch list at chi = 8192 and the c5 chi = 8192 bench line.
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/r2b6}; mkdir -p $o
timeout 1200 python -m pytest tests -m gpu -q -k "generated or streamed or mpsb or precise or decode or synthetic or host_streamed or parity_at" > $o/pytest.log 2>&1
MPSG_PROBE_SUPPLY=generated timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:"colmax|colfinish|pack_kernel|synth" --launch-count 100 \
  python tools/perf_probe.py 24 8192 4 8192 split 8192 3 > $o/launches_gen.csv 2> $o/launches_gen.err
timeout 900 python bench.py --config c5_8192 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/bench_c5_8192.json 2> $o/bench_c5_8192.err
ls -la $o
