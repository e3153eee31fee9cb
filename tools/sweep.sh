cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sweep
for cfg in c2 c5_256 c5_512 c5_1024 c5_2048 c5_4096; do
  timeout 600 python bench.py --config $cfg --e2e resident > gpurun_out/sweep/bench_$cfg.json 2> gpurun_out/sweep/bench_$cfg.err
done
timeout 600 python bench.py --config c3 --mode single --e2e resident --no-cpu-baseline > gpurun_out/sweep/bench_c3_single.json 2> gpurun_out/sweep/bench_c3_single.err
timeout 600 python bench.py --config c3 --scheme 4m --e2e resident --no-cpu-baseline > gpurun_out/sweep/bench_c3_4m.json 2> gpurun_out/sweep/bench_c3_4m.err
for f in gpurun_out/sweep/*.json; do echo "$f $(python -c "import json; d=json.load(open('$f')); print(d['value'], d['config'].get('scheme'), d['roofline']['frac'], d['roofline']['issued_frac'], d['roofline']['gemm_share_of_step'], d['clocks']['sm_mhz'], (d.get('cpu_baseline') or {}).get('value'))" 2>&1 | tail -1)"; done
