cd $GRAFT_REPO_ROOT
P="python tools/perf_probe.py 64 2048 6 16384 split 16384 3"
for f in 0 1 2; do echo "== 3M flags $f"
  nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader -lms 100 > /tmp/clk_$f.csv &
  SP=$!
  MPSG_3M_FLAGS=$f $P 2>&1 | grep -E "interior|rep 2"
  kill $SP
  sort -t, -k2 -n -r /tmp/clk_$f.csv | head -30 | awk -F, '{c+=$1; p+=$2; n++} END {print "top-30 power samples: clock", c/n, "MHz power", p/n, "W"}'
done
echo "== 4M"
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader -lms 100 > /tmp/clk_4.csv &
SP=$!
python tools/perf_probe.py 64 2048 6 16384 split 16384 4 2>&1 | grep -E "interior|rep 2"
kill $SP
sort -t, -k2 -n -r /tmp/clk_4.csv | head -30 | awk -F, '{c+=$1; p+=$2; n++} END {print "top-30 power samples: clock", c/n, "MHz power", p/n, "W"}'
