# round-2 batch 3: storage-streamed MPSB supply (tests + c5 chi=1024 bench line from an f16 file), and
# the raster-group sweep at chi = 8192 (per-site device time of a 40-site chain + ncu DRAM / L2 of
# interior launches) -- the large-chi K1 issues at 0.71 of the sustained rate per clock.
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/r2b3}; mkdir -p $o
timeout 600 python -m pytest tests -m gpu -q -k "streamed or mpsb" > $o/pytest_file.log 2>&1
timeout 900 python bench.py --config c5_1024 --supply file --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/bench_c5_1024_file.json 2> $o/bench_c5_1024_file.err
for g in 0 1 2 4 16; do
  if [ $g = 0 ]; then unset MPSG_3M_GROUP; else export MPSG_3M_GROUP=$g; fi
  timeout 600 python tools/perf_probe.py 40 8192 4 8192 split 8192 3 > $o/probe_8192_g$g.log 2>&1
done
unset MPSG_3M_GROUP
for g in 0 2; do
  if [ $g = 0 ]; then unset MPSG_3M_GROUP; else export MPSG_3M_GROUP=$g; fi
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:site_gemm_3m --launch-skip 40 --launch-count 2 --csv \
    python tools/perf_probe.py 40 8192 4 8192 split 8192 3 > $o/ncu_8192_g$g.csv 2> $o/ncu_8192_g$g.err
done
unset MPSG_3M_GROUP
ls -la $o
