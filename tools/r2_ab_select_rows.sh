# select_rows (R rows per warp, slices in registers) and programmatic dependent launch A/B:
# identity test, launch list at chi = 256 / 512, alternating bench runs (legacy / rows / rows + PDL)
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/selrows}; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "select_fast_path or slice_recompute or c1_strings or randomized or near_boundary" > $o/pytest.log 2>&1
MPSG_PDL=0 bash tools/r2_small_chi.sh $o
for rep in 1 2; do
  for arm in legacy rows pdl; do
    L=0; P=0; [ $arm = legacy ] && L=1; [ $arm = pdl ] && P=1
    for c in c5_256 c2 c5_512; do
      MPSG_SELECT_LEGACY=$L MPSG_PDL=$P timeout 600 python bench.py --config $c --no-cpu-baseline > $o/bench_${c}_${arm}_$rep.json 2> $o/bench_${c}_${arm}_$rep.err
    done
  done
done
