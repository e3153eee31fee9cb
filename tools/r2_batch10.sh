# round-2 batch 10: parity at the c4 bond dimension against the reference -- a 64-site chain of the
# c4 shape (chi = 1e4 for ~50 sites, both edges), generated supply, 64 samples, with the reference's
# F32 policy beside it.
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/r2b10}; mkdir -p $o
timeout 3000 python tests/parity_full.py --config c4 --sites 64 --samples 64 --f32 --out $o/c4s64_full.json > $o/c4s64.log 2>&1
ls -la $o
