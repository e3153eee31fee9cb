cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sweep_final2
timeout 900 python bench.py > gpurun_out/sweep_final2/bench_c3.json 2> gpurun_out/sweep_final2/bench_c3.err
for cfg in c2 c5_256 c5_512 c5_1024 c5_2048 c5_4096; do
  timeout 600 python bench.py --config $cfg --e2e resident > gpurun_out/sweep_final2/bench_$cfg.json 2> gpurun_out/sweep_final2/bench_$cfg.err
done
timeout 600 python bench.py --config c2 --displace 0.5 --e2e resident --no-cpu-baseline > gpurun_out/sweep_final2/bench_c2_displaced.json 2> /dev/null
timeout 600 python bench.py --config c3 --schedule-eps 1e-4 --e2e resident --no-cpu-baseline > gpurun_out/sweep_final2/bench_c3_sched1e-4.json 2> /dev/null
timeout 600 python bench.py --config c3 --mode single --e2e resident --no-cpu-baseline > gpurun_out/sweep_final2/bench_c3_single.json 2> /dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:site_gemm_3m -s 8 -c 1 -o gpurun_out/sweep_final2/prof3m_c3 python tools/perf_probe.py 16 2048 6 16384 split 16384 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:select_kernel -s 8 -c 1 -o gpurun_out/sweep_final2/prof_select_c3 python tools/perf_probe.py 16 2048 6 16384 split 16384 3 > /dev/null 2>&1
for f in gpurun_out/sweep_final2/*.json; do echo "$f $(python -c "import json; d=json.load(open('$f')); print(d['value'], d['config'].get('scheme'), round(d['roofline']['frac'],3), round(d['roofline']['issued_frac'],3), round(d['roofline']['gemm_share_of_step'],3), d['clocks']['sm_mhz'], (d.get('cpu_baseline') or {}).get('value'), d['e2e']['value'], d['e2e'].get('mode'))" 2>&1 | tail -1)"; done
