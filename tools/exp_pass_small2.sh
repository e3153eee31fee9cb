# Larger passes at c2 / c5 chi=512 (default 32768) vs 65536, alternating runs.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pass_small2
for r in 1 2; do
  for v in "c2 32768" "c2 65536" "c5_512 32768" "c5_512 65536"; do set -- $v
    timeout 600 python bench.py --config $1 --pass $2 --steps 3 --warmup 3 --no-cpu-baseline --e2e resident --e2e-steps 1 \
      > gpurun_out/pass_small2/bench_$1_p$2_$r.json 2> /dev/null
  done
done
