# Generated supply at chi = 8192: launch list (duration, DRAM) of the library's own kernels over a
# 24-site chain (regeneration kernels beside the contraction), and a resident / generated A/B.
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/regen}; mkdir -p $o
MPSG_PROBE_SUPPLY=generated timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:"site_gemm|select_kernel|colmax|colfinish|pack_kernel|synth|sum_plane|init_env|draws" --launch-count 400 \
  python tools/perf_probe.py 24 8192 4 8192 split 8192 3 > $o/launches_gen.csv 2> $o/launches_gen.err
ls -la $o
