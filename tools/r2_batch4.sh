# round-2 batch 4: compression kernels without f64 divisions + half2 plane stores (bit-identical
# planes): the supply tests, the generated / resident A/B at chi = 8192 and the launch list; the
# parallel-reader file supply bench line.
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/r2b4}; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q -k "generated or streamed or mpsb or grid or decode or precise or host_streamed or synthetic" > $o/pytest.log 2>&1
MPSG_PROBE_SUPPLY=generated timeout 600 python tools/perf_probe.py 24 8192 4 8192 split 8192 3 > $o/probe_gen.log 2>&1
MPSG_PROBE_SUPPLY=resident timeout 600 python tools/perf_probe.py 24 8192 4 8192 split 8192 3 > $o/probe_res.log 2>&1
MPSG_PROBE_SUPPLY=generated timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:"colmax|colfinish|pack_kernel|synth" --launch-count 100 \
  python tools/perf_probe.py 24 8192 4 8192 split 8192 3 > $o/launches_gen.csv 2> $o/launches_gen.err
timeout 900 python bench.py --config c5_1024 --supply file --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/bench_c5_1024_file.json 2> $o/bench_c5_1024_file.err
ls -la $o
