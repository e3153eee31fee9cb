# round-2 batch 5: supply compression inline on the engine stream (default) vs the side stream, at
# chi = 8192 (24-site chain, regenerated vs resident) and the c5 chi = 8192 bench line.
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/r2b5}; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q -k "generated or streamed or mpsb" > $o/pytest.log 2>&1
for rep in 1 2; do
MPSG_PROBE_SUPPLY=generated timeout 600 python tools/perf_probe.py 24 8192 4 8192 split 8192 3 > $o/probe_gen_inline_$rep.log 2>&1
MPSG_SUPPLY_STREAM=side MPSG_PROBE_SUPPLY=generated timeout 600 python tools/perf_probe.py 24 8192 4 8192 split 8192 3 > $o/probe_gen_side_$rep.log 2>&1
MPSG_PROBE_SUPPLY=resident timeout 600 python tools/perf_probe.py 24 8192 4 8192 split 8192 3 > $o/probe_res_$rep.log 2>&1
done
timeout 900 python bench.py --config c5_8192 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/bench_c5_8192.json 2> $o/bench_c5_8192.err
ls -la $o
