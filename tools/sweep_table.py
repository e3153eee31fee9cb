"""Markdown table of a bench sweep directory (one JSON line per file): python tools/sweep_table.py DIR"""
import glob
import json
import os
import sys

ORDER = ["c3", "c3_sched1e-4", "c3_single", "c2", "c2_displaced", "c5_256", "c5_512", "c5_1024", "c5_2048",
         "c5_4096", "c5_8192", "c5_10000", "c4", "c5_1024_file"]


def main(d):
    rows = {}
    for f in glob.glob(os.path.join(d, "bench_*.json")):
        try:
            line = [x for x in open(f).read().splitlines() if x.startswith("{")][-1]
            rows[os.path.basename(f)[6:-5]] = json.loads(line)
        except Exception:
            continue
    print("| config | samples/s | e2e samples/s | K1 frac alg. / issued (sustained peak) | issued/clock vs cuBLAS | K1 share | SM MHz | Γ supply |")
    print("|---|---|---|---|---|---|---|---|")
    for k in ORDER + sorted(set(rows) - set(ORDER)):
        if k not in rows:
            continue
        r = rows[k]
        rf = r["roofline"]
        sup = r["config"].get("gamma_residency", "")
        sup = "HBM" if sup == "HBM" else sup.split(" (")[0].split(":")[0]
        print(f"| {k} | {r['value']:,.1f} | {r['e2e']['value']:,.1f} ({r['e2e'].get('mode')}) | "
              f"{rf['frac']:.3f} / {rf['issued_frac']:.3f} | {rf.get('issued_frac_at_equal_clock') or 0:.2f} | "
              f"{rf['gemm_share_of_step']:.2f} | {r['clocks']['sm_mhz']:.0f} | {sup} |")


if __name__ == "__main__":
    main(sys.argv[1])
