"""Summarise an ncu report: key throughput metrics of every captured kernel (run here, no GPU).

usage: python tools/ncu_summary.py report.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "tc_smem_wavefronts_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct_rt",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "launch__grid_size": "grid",
    "launch__registers_per_thread": "regs",
}


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")][:80]}
        for i, h in enumerate(hdr):
            if h in KEYS:
                d[KEYS[h]] = f"{vals[i]} {units[i]}".strip()
        out.append(d)
    return out


if __name__ == "__main__":
    res = summarise(sys.argv[1])
    for d in res:
        print(json.dumps(d, indent=1))
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
