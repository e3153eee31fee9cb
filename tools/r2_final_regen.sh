# Closing regenerated-supply lines on the final code: c5 chi=8192 / 1e4 and the full c4 chain.
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/finalregen}; mkdir -p $o
timeout 1200 python bench.py --config c5_8192 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/bench_c5_8192.json 2> $o/bench_c5_8192.err
timeout 1200 python bench.py --config c5_10000 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/bench_c5_10000.json 2> $o/bench_c5_10000.err
timeout 2400 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/bench_c4.json 2> $o/bench_c4.err
