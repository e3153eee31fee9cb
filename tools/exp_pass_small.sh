# Pass size at small chi (the environment of a smaller pass can stay in L2 between the selection that
# writes it and the next contraction): c5 chi=256 and c2, alternating runs.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pass_small
for r in 1 2; do
  for v in "c5_256 65536" "c5_256 16384" "c5_256 8192" "c2 32768" "c2 8192" "c2 4096"; do set -- $v
    timeout 600 python bench.py --config $1 --pass $2 --steps 3 --warmup 3 --no-cpu-baseline --e2e resident --e2e-steps 1 \
      > gpurun_out/pass_small/bench_$1_p$2_$r.json 2> /dev/null
  done
done
