# Launch lists (ncu gpu__time_duration) of a 16-site chi=256 d=4 chain, 65536 samples: temp vs recompute.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/slice4
for S in 1 2; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"site_gemm|select|permute|zero_dead" -c 100 --csv \
    --log-file gpurun_out/slice4/launches_s$S.csv python tools/perf_probe.py 16 256 4 65536 split 65536 3 $S > /dev/null 2>&1
done
