cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none -k regex:site_gemm_pair -s 8 -c 1 -o gpurun_out/prof4m_c3 python tools/perf_probe.py 16 2048 6 16384 split 16384 4 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:site_gemm_3m -s 8 -c 1 -o gpurun_out/prof3m_precise python tools/perf_probe.py 16 1024 4 32768 precise 32768 3 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
