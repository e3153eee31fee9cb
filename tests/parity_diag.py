"""Diagnostic (needs a B200 and oracle/_ref): dump GPU vs reference marginals at the c3 shape.

usage: python tests/parity_diag.py M CHI D N SCHEME out.npz
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import oracle as O  # noqa: E402  (test infrastructure: the checker)
import paper_2512_20064_b200 as P  # noqa: E402
from paper_2512_20064_b200.synthetic import build_synthetic  # noqa: E402
from concurrent.futures import ThreadPoolExecutor  # noqa: E402

m, chi, d, n, scheme = (int(x) for x in sys.argv[1:6])
pol = P.PrecisionPolicy(scaling=P.ScalingMode.PER_SAMPLE_MAX)
smp, lams = build_synthetic(m, chi, d, seed=5, policy=pol, scheme=scheme)
dec = O.Mps(d, list(smp.bond_dims), [smp.decoded_gamma(i) for i in range(m)], list(lams))
rs = O.RefState(dec)
rows = rs.sample_range(0, n, 7, threads=16)
chunks = [c for c in np.array_split(np.arange(n), 16) if len(c)]
with ThreadPoolExecutor(16) as ex:
    ref = np.concatenate(list(ex.map(lambda idx: rs.marginals_forced(rows[idx]), chunks)))
with ThreadPoolExecutor(16) as ex:
    f32 = np.concatenate(list(ex.map(lambda idx: rs.marginals_forced(rows[idx], compute=O.F32), chunks)))
gm = smp.marginals(0, rows)
np.savez_compressed(sys.argv[6], ref=ref, f32=f32, gpu=gm, rows=rows, bonds=np.array(smp.bond_dims))
big = ref >= 1e-3
print("gpu max rel", (np.abs(gm - ref)[big] / ref[big]).max(), "ref-F32 max rel", (np.abs(f32 - ref)[big] / ref[big]).max())
