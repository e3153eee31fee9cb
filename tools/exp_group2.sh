# DRAM bytes of one interior c3 launch of the 3M contraction vs the Gamma raster group (ncu).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/group2
for G in 1 2 4 6 8 12; do
  MPSG_3M_GROUP=$G timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum --clock-control none \
    -k regex:site_gemm_3m -s 8 -c 1 --csv --log-file gpurun_out/group2/dram_g$G.csv \
    python tools/perf_probe.py 16 2048 6 16384 split 16384 3 > /dev/null 2>&1
done
