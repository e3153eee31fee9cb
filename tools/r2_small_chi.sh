# Small-chi breakdown: per-kernel launch lists (ncu gpu__time_duration + DRAM bytes) of the sweep
# kernels at chi = 256 (d=4, 65536 rows) and chi = 512 (d=6, 32768 rows), plus the per-site probe times.
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/small}; mkdir -p $o
for c in "256 4 65536" "512 6 32768"; do
  set -- $c
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"site_gemm|select|init_env" -c 120 --csv \
    --log-file $o/launches_$1.csv python tools/perf_probe.py 16 $1 $2 $3 split $3 3 > /dev/null 2>&1
done
