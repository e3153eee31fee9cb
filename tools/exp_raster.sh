# A/B of the 3M raster (MPSG_3M_RASTER: 0 = round-1 order, 1 = snake over sample tiles, 3 = snake +
# the second lane's groups last-to-first) and raster group size (MPSG_3M_GROUP, Gamma tile pairs):
# DRAM bytes of site 10's two lane launches (pass 16384 -> 2 x 8192 rows, c3 interior shape) under
# ncu, and c3 bench lines alternating on one box.
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/raster}; mkdir -p $o
for rg in "0 8" "3 8" "3 12" "3 16"; do
  set -- $rg
  MPSG_3M_RASTER=$1 MPSG_3M_GROUP=$2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:site_gemm_3m --launch-skip 20 --launch-count 8 --csv \
    python tools/perf_probe.py 32 2048 6 16384 split 16384 3 > $o/ncu_r$1_g$2.csv 2> $o/ncu_r$1_g$2.err
done
for rep in 1 2; do
  for rg in "0 8" "3 8" "3 16"; do
    set -- $rg
    MPSG_3M_RASTER=$1 MPSG_3M_GROUP=$2 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e resident --e2e-steps 1 \
      > $o/bench_c3_r$1_g$2_$rep.json 2> $o/bench_c3_r$1_g$2_$rep.err
  done
done
ls $o
