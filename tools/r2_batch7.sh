# round-2 batch 7: pack unrolling check (supply tests + launch list), the C++ adapter (storage-streamed
# file executor), and the c2 full-chain parity against the chain's ORIGINAL values (PRECISE, and SPLIT
# for the fp16 format's own effect) with the reference's F32 policy beside it.
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/r2b7}; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q -k "generated or streamed or mpsb or synthetic or adapter" > $o/pytest.log 2>&1
oracle/_ref/adapter_test gpu > $o/adapter.log 2>&1
MPSG_PROBE_SUPPLY=generated timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:"colmax|colfinish|pack_kernel|synth" --launch-count 100 \
  python tools/perf_probe.py 24 8192 4 8192 split 8192 3 > $o/launches_gen.csv 2> $o/launches_gen.err
timeout 1800 python tests/parity_full.py --config c2 --samples 1024 --mode precise --against original --f32 --out $o/c2_full_precise_original.json > $o/c2_precise.log 2>&1
timeout 1800 python tests/parity_full.py --config c2 --samples 1024 --mode split --against original --out $o/c2_full_split_original.json > $o/c2_split_orig.log 2>&1
ls -la $o
