cd $GRAFT_REPO_ROOT
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct"
for cfg in "16 0" "16 64" "8 0" "32 0" "16 256" "48 0"; do set -- $cfg
  MPSG_3M_GROUP=$1 MPSG_3M_FLAGS=$2 timeout 300 ncu $M --clock-control none -k regex:site_gemm_3m -s 12 -c 1 --csv --log-file gpurun_out/dram_g$1_f$2.csv python tools/perf_probe.py 24 2048 6 16384 split 16384 3 > gpurun_out/dram_g$1_f$2.log 2>&1
done
