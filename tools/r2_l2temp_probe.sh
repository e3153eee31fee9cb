# Is the small-chi K1 epilogue bound by the SM's store path or by the temp stream's DRAM write-back?
# clock64 probes (flags 32) + per-site times for: stores to temp (0), no stores (64), stores into an
# L2-resident 8-tile region (128).  Timing-only switches (64 / 128 give wrong samples).
cd $GRAFT_REPO_ROOT
o=${1:-gpurun_out/l2temp}; mkdir -p $o
for c in "256 4 65536" "512 6 32768"; do
  set -- $c
  for f in 32 96 160 32; do
    echo "== chi=$1 flags=$f" >> $o/probe.log
    MPSG_3M_FLAGS=$f timeout 300 python tools/perf_probe.py 16 $1 $2 $3 split $3 3 2>&1 | grep -v "first rows\|^ \[\|histogram" >> $o/probe.log
  done
done
