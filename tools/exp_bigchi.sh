# chi = 8192 / 1e4 interior sites: Gamma supply (resident / host-streamed / regenerated) and raster group
# size, per-site device time of a 40-site chain (perf_probe), plus ncu DRAM of an interior launch.
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/bigchi}; mkdir -p $o
for sup in resident generated stream; do
  MPSG_PROBE_SUPPLY=$sup timeout 900 python tools/perf_probe.py 40 8192 4 8192 split 8192 3 > $o/probe_8192_$sup.log 2>&1
done
for g in 2 4 16; do
  MPSG_3M_GROUP=$g MPSG_PROBE_SUPPLY=resident timeout 900 python tools/perf_probe.py 40 8192 4 8192 split 8192 3 > $o/probe_8192_resident_g$g.log 2>&1
done
for g in 0 2 4; do
  if [ $g = 0 ]; then unset MPSG_3M_GROUP; else export MPSG_3M_GROUP=$g; fi
  MPSG_PROBE_SUPPLY=resident timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:site_gemm_3m --launch-skip 40 --launch-count 4 --csv \
    python tools/perf_probe.py 40 8192 4 8192 split 8192 3 > $o/ncu_8192_g$g.csv 2> $o/ncu_8192_g$g.err
done
unset MPSG_3M_GROUP
ls $o
