# Round-2 final sweep on one B200: GPU tests + smoke, every bench configuration BASELINE.json names
# that fits one GPU (c3 headline with the CPU reference, c2, the c5 chi sweep incl. 8192 / 1e4
# regenerated, the full c4 chain), the variants (GBS displacement, dynamic bonds, SINGLE, GRID-class
# SINGLE, the storage-streamed file supply), the ncu launch list of one c3 step and full captures of
# the interior c3 site kernels.
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/r2sweep}; mkdir -p $o
(time timeout 1500 python -m pytest tests -m gpu -q) > $o/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1
timeout 900 python bench.py > $o/bench_c3.json 2> $o/bench_c3.err
for cfg in c2 c5_256 c5_512 c5_1024 c5_2048 c5_4096; do
  timeout 900 python bench.py --config $cfg --no-cpu-baseline > $o/bench_$cfg.json 2> $o/bench_$cfg.err
done
for cfg in c5_8192 c5_10000; do
  timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/bench_$cfg.json 2> $o/bench_$cfg.err
done
timeout 600 python bench.py --config c2 --displace 0.5 --e2e resident --no-cpu-baseline > $o/bench_c2_displaced.json 2> /dev/null
timeout 600 python bench.py --config c3 --schedule-eps 1e-4 --e2e resident --no-cpu-baseline > $o/bench_c3_sched1e-4.json 2> /dev/null
timeout 600 python bench.py --config c3 --mode single --e2e resident --no-cpu-baseline > $o/bench_c3_single.json 2> /dev/null
timeout 900 python bench.py --config c5_1024 --supply file --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/bench_c5_1024_file.json 2> $o/bench_c5_1024_file.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"site_gemm|select_kernel" -c 2048 --csv \
  --log-file $o/launches_c3.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e resident --e2e-steps 1 > /dev/null 2>&1
bash tools/ncu_site.sh $o/ncu > /dev/null 2>&1
timeout 2400 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/bench_c4.json 2> $o/bench_c4.err
ls -la $o
