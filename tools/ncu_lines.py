"""Top source lines by warp-stall samples from an ncu report (run here, no GPU).

usage: python tools/ncu_lines.py report.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
fname, hdr, out = "?", None, []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0] not in ("", "Function Name"):
        d = dict(zip(hdr, r))
        try:
            s = int(d.get("Warp Stall Sampling (All Samples)", "0"))
        except ValueError:
            continue
        stalls = {k[6:]: int(v) for k, v in zip(hdr, r) if k.startswith("stall_") and v.isdigit() and int(v) > 0}
        out.append((s, fname, r[0], r[1][:90], sorted(stalls.items(), key=lambda x: -x[1])[:3]))
tot = sum(o[0] for o in out) or 1
for s, f, ln, src, st in sorted(out, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}% {f}:{ln} {src}  {st}")
