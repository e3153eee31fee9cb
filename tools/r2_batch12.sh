# round-2 batch 12: full-chain parity across the c5 chi sweep (chi = 256 / 1024 with 3M, 4096 with the
# 4M scheme AUTO picks there) with the reference's F32 policy beside it, and the full c3 job
# (N = 1e6: 62 passes of 16384) on the final code.
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/r2b12}; mkdir -p $o
timeout 1200 python bench.py --steps 62 --warmup 3 --no-cpu-baseline --e2e resident --e2e-steps 1 > $o/c3_full_job_1e6.json 2> $o/c3_full_job.err
timeout 1200 python tests/parity_full.py --config c5_256 --samples 1024 --f32 --out $o/c5_256_full.json > $o/c5_256.log 2>&1
timeout 1200 python tests/parity_full.py --config c5_1024 --samples 256 --f32 --out $o/c5_1024_full.json > $o/c5_1024.log 2>&1
timeout 2400 python tests/parity_full.py --config c5_4096 --samples 16 --scheme 4m --f32 --out $o/c5_4096_4m_full.json > $o/c5_4096.log 2>&1
ls -la $o
