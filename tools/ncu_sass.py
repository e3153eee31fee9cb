"""Per-SASS-instruction warp-stall samples of an ncu report (top N), with the stall reasons.

usage: python tools/ncu_sass.py report.ncu-rep [N] [grep-pattern]
"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
pat = re.compile(sys.argv[3]) if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, out = None, []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0"))
    except ValueError:
        continue
    if pat and not pat.search(d["Source"]):
        continue
    st = sorted(((k[6:], int(v)) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k
                 and v.isdigit() and int(v) > 0), key=lambda x: -x[1])[:3]
    out.append((s, d["Address"], d["Source"].strip()[:60], st))
tot = sum(o[0] for o in out) or 1
for s, a, src, st in sorted(out, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}% {a} {src:60s} {st}")
