# Round-2 closing sweep on one B200 (after the selection / compact-3M / compression changes): GPU tests,
# smoke, the c3 headline with the CPU reference, c2 and the resident c5 sweep, the ncu launch list of
# one c3 step.  (c5 chi >= 8192 and c4 come from tools/r2_pack_fast.sh.)
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/r2final3}; mkdir -p $o
(time timeout 1500 python -m pytest tests -m gpu -q) > $o/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1
timeout 900 python bench.py > $o/bench_c3.json 2> $o/bench_c3.err
for cfg in c2 c5_256 c5_512 c5_1024 c5_2048 c5_4096; do
  timeout 900 python bench.py --config $cfg --no-cpu-baseline > $o/bench_$cfg.json 2> $o/bench_$cfg.err
done
timeout 600 python bench.py --config c2 --displace 0.5 --e2e resident --no-cpu-baseline > $o/bench_c2_displaced.json 2> /dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"site_gemm|select" -c 2048 --csv \
  --log-file $o/launches_c3.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e resident --e2e-steps 1 > /dev/null 2>&1
ls -la $o
