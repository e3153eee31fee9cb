# Compact 3M (only [Gr, Gi] resident; Gs re-formed per site in the slot ring): identity tests and the
# c5 chi=4096 bench (AUTO picks compact 3M; MPSG_COMPACT_3M=0 keeps the resident 4M state).
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/compact}; mkdir -p $o
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "compact_3m or select_fast_path or host_streamed" > $o/pytest.log 2>&1
for rep in 1 2; do
  for arm in compact m4; do
    C=1; [ $arm = m4 ] && C=0
    MPSG_COMPACT_3M=$C timeout 900 python bench.py --config c5_4096 --no-cpu-baseline --e2e-steps 1 > $o/bench_c5_4096_${arm}_$rep.json 2> $o/bench_c5_4096_${arm}_$rep.err
  done
done
