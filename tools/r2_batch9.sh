# round-2 batch 9: select-kernel unrolling A/B, then PRECISE on the generated supply at c3 (bench line
# + full-chain parity against the chain's original values).
cd $GRAFT_REPO_ROOT
bash tools/r2_ab_select.sh gpurun_out/ab_select > gpurun_out/ab_select_summary.txt 2>&1
o=gpurun_out/r2b9; mkdir -p $o
timeout 1200 python bench.py --config c3 --mode precise --supply generated --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/bench_c3_precise_generated.json 2> $o/bench_c3_precise_generated.err
timeout 3000 python tests/parity_full.py --config c3 --samples 64 --mode precise --against original --out $o/c3_full_precise_original.json > $o/c3_precise.log 2>&1
ls -la $o
