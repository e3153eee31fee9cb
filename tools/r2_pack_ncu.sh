# Interior-site compression kernels of the regenerated supply at chi = 8192 (launch list with DRAM
# bytes, and one full capture of pack_kernel)
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/packncu}; mkdir -p $o
MPSG_PROBE_SUPPLY=generated timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:"colmax|pack_kernel" --launch-skip 16 --launch-count 8 --log-file $o/launches_interior.csv \
  python tools/perf_probe.py 24 8192 4 8192 split 8192 3 > /dev/null 2>&1
MPSG_PROBE_SUPPLY=generated timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"pack_kernel" --launch-skip 10 --launch-count 1 -o $o/pack_full \
  python tools/perf_probe.py 24 8192 4 8192 split 8192 3 > /dev/null 2>&1
ls -la $o
