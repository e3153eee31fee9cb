cd $GRAFT_REPO_ROOT
timeout 1700 python tools/parity_diag.py 24 2048 6 256 3 gpurun_out/diag3m_b.npz 2>&1 | tail -1
timeout 1700 python tools/parity_diag.py 24 2048 6 256 4 gpurun_out/diag4m_b.npz 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -2
