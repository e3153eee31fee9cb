# ncu --set full of the c3 site kernels exactly as the default bench launches them: an interior site
# (chiL = chiR = 2048, d = 6) of a 32-site chain, pass 16384 split into the two pipeline lanes of 8192
# rows each.  Launches 20, 21 of site_gemm_3m_kernel are site 10's two lane launches (the first 10
# sites are skipped: the left edge ramps 1, 6, 36, 216, 1296, 2048 over sites 0-4).
cd $GRAFT_REPO_ROOT
out=${1:-gpurun_out/ncu_site}
mkdir -p $out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:site_gemm_3m --launch-skip 20 --launch-count 2 \
  -o $out/k1_c3_interior python tools/perf_probe.py 32 2048 6 16384 split 16384 3 > $out/k1.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:select_kernel --launch-skip 20 --launch-count 2 \
  -o $out/k2_c3_interior python tools/perf_probe.py 32 2048 6 16384 split 16384 3 > $out/k2.log 2>&1
ls -la $out
