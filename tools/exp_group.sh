# Raster-group experiment for the 3M contraction: DRAM bytes per interior c3 launch (ncu) and the
# c3 bench at Gamma groups of 8 / 16 / 24 tile pairs (alternating runs on one box).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/group
for G in 8 16 24; do
  MPSG_3M_GROUP=$G timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:site_gemm_3m -s 8 -c 1 --csv --log-file gpurun_out/group/dram_g$G.csv \
    python tools/perf_probe.py 16 2048 6 16384 split 16384 3 > /dev/null 2>&1
done
for r in 1 2; do for G in 8 16 24; do
  MPSG_3M_GROUP=$G timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e resident --e2e-steps 1 \
    > gpurun_out/group/bench_g${G}_$r.json 2> /dev/null
done; done
