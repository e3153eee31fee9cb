# select-kernel live-counter aggregation: launch list at chi = 256 / 512 + c5_256 / c2 / c5_512 bench lines
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/live}; mkdir -p $o
bash tools/r2_small_chi.sh $o
for c in c5_256 c2 c5_512; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $o/bench_$c.json 2> $o/bench_$c.err
done
