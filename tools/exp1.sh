cd $GRAFT_REPO_ROOT
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
for cfg in "8 0" "8 64" "16 64" "32 64" "4 64"; do set -- $cfg
  MPSG_3M_GROUP=$1 MPSG_3M_FLAGS=$2 timeout 300 ncu $M --clock-control none -k regex:site_gemm_3m -s 12 -c 1 --csv --log-file gpurun_out/dram2_g$1_f$2.csv python tools/perf_probe.py 24 2048 6 16384 split 16384 3 > /dev/null 2>&1
done
b() { timeout 600 env $1 python bench.py --no-cpu-baseline --steps 3 --e2e resident --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value']), d['clocks']['sm_mhz'])"; }
b "MPSG_3M_FLAGS=0"; b "MPSG_3M_FLAGS=64 MPSG_3M_GROUP=16"; b "MPSG_3M_FLAGS=0"
