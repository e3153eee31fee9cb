cd $GRAFT_REPO_ROOT
for sc in 4m 3m; do
timeout 1500 python bench.py --config c4s --scheme $sc --steps 3 --warmup 2 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_c4s_$sc.json 2> gpurun_out/bench_c4s_$sc.err
python -c "import json; d=json.load(open('gpurun_out/bench_c4s_$sc.json')); print('$sc', d['value'], d['roofline']['issued_frac'], d['clocks']['sm_mhz'], d['host_link'], d['e2e']['value'])"
done
