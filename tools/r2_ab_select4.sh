# select4 (four rows per warp) vs legacy select: identity test, launch lists, bench A/B (alternating)
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/sel4}; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "select_fast_path or slice_recompute or c1_strings or randomized" > $o/pytest.log 2>&1
bash tools/r2_small_chi.sh $o
for rep in 1 2; do
  for arm in fast legacy; do
    L=0; [ $arm = legacy ] && L=1
    for c in c5_256 c2 c5_512; do
      MPSG_SELECT_LEGACY=$L timeout 600 python bench.py --config $c --no-cpu-baseline > $o/bench_${c}_${arm}_$rep.json 2> $o/bench_${c}_${arm}_$rep.err
    done
  done
done
