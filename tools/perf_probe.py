"""Perf probe: per-site device times and algorithmic TFLOP/s for a synthetic chain.

usage: python tools/perf_probe.py M CHI D N [mode] [pass] [scheme 0|3|4] [slice 0|1|2]
MPSG_PROBE_SUPPLY=generated|stream|resident (default resident) selects the Gamma supply.
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_20064_b200 as P  # noqa: E402
from paper_2512_20064_b200.synthetic import build_synthetic  # noqa: E402

M, chi, d, N = (int(x) for x in sys.argv[1:5])
mode = {"single": P.Mode.SINGLE, "precise": P.Mode.PRECISE}.get(sys.argv[5] if len(sys.argv) > 5 else "split", P.Mode.SPLIT)
ps = int(sys.argv[6]) if len(sys.argv) > 6 else 0
scheme = int(sys.argv[7]) if len(sys.argv) > 7 else 0
slice_ = int(sys.argv[8]) if len(sys.argv) > 8 else 0
t = time.time()
supply = os.environ.get("MPSG_PROBE_SUPPLY", "resident")
smp, lams = build_synthetic(M, chi, d, mode=mode, pass_samples=ps or N, record_site_times=True, scheme=scheme,
                           slice=slice_, generated=supply == "generated",
                           host_stream_slots=3 if supply == "stream" else 0)
print(f"build {time.time()-t:.1f}s state {smp.state_bytes/1e9:.2f} GB scheme {int(smp.scheme)} supply {supply}", flush=True)
bonds = smp.bond_dims
rows = torch.empty((N, M), dtype=torch.uint8, device="cuda")
for rep in range(3):
    st = P.RunStats()
    torch.cuda.synchronize()
    t = time.time()
    out = smp.sample(0, N, 7, stats=st)
    el = time.time() - t
    flops = 8.0 * N * sum(bonds[i] * bonds[i + 1] * d for i in range(M))
    ss = np.array(st.site_seconds)
    print(f"rep {rep}: {el:.3f}s  {N/el:.0f} samples/s  alg {flops/el/1e12:.1f} TF/s  issued {st.issued_mma_flops/el/1e12:.1f} TF/s"
          f"  sum(site) {ss.sum():.3f}s  dead {st.dead_samples}", flush=True)
if int(os.environ.get("MPSG_3M_FLAGS", "0")) & 32:
    import ctypes
    buf = (ctypes.c_ulonglong * 8)()
    P.sampler._lib.lib().mpsg_debug_prof3m(buf, 8)
    u = max(buf[4], 1)
    print(f"prof3m per unit (cycles): epi wait {buf[0]/u:.0f} epi busy {buf[1]/u:.0f} epi to-release {buf[5]/u:.0f}"
          f" | per CTA-pair unit: mma slot-wait {2*buf[2]/u:.0f} mma full-wait {2*buf[3]/u:.0f}  units {buf[4]}", flush=True)
full = [i for i in range(M) if bonds[i] == chi and bonds[i + 1] == chi]
if full:
    i = full[len(full) // 2]
    f_site = 8.0 * N * chi * chi * d
    print(f"interior site {i}: {ss[i]*1e3:.2f} ms -> alg {f_site/ss[i]/1e12:.1f} TF/s", flush=True)
print("first rows", out[:2], flush=True)
print("outcome histogram site 10:", np.bincount(out[:, min(10, M - 1)], minlength=d), flush=True)
