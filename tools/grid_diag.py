"""GRID-mode diagnostic: per-site marginal error of the GPU GRID path vs the compiled reference's
reduced policy (and the policy vs F64), and the decoded Gamma vs round_scalar."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import oracle as O  # noqa: E402

import paper_2512_20064_b200 as P  # noqa: E402

case, comp, scal = sys.argv[1], sys.argv[2], sys.argv[3]
z = np.load(f"{ROOT}/tests/golden/{case}.npz")
mps = O.load_npz_mps(z)
cp = {"F16": O.F16, "TF32": O.TF32}[comp]
sc = {"PSM": O.SCALE_PER_SAMPLE, "NONE": O.SCALE_NONE}[scal]
pol = P.PrecisionPolicy(compute=getattr(P.Precision, comp),
                        scaling={"PSM": P.ScalingMode.PER_SAMPLE_MAX, "NONE": P.ScalingMode.NONE}[scal])
st = P.MpsState(mps.num_sites, mps.phys_dim, list(mps.bond_dims), list(mps.gammas), list(mps.lambdas))
smp = P.GpuSampler(st, pol)
L = O.ref()
for i in range(mps.num_sites):
    g = mps.gammas[i]
    want = np.vectorize(lambda x: L.ref_round_scalar(float(x), cp))(g.real) + \
        1j * np.vectorize(lambda x: L.ref_round_scalar(float(x), cp))(g.imag)
    dec = smp.decoded_gamma(i)
    nbad = int((dec != want).sum())
    if nbad:
        print("site", i, "decoded != round_scalar at", nbad, "of", g.size)
n = 1000
rs = O.RefState(mps)
rows = rs.sample_range(0, n, 7, compute=cp, scaling=sc, threads=8)
rm = rs.marginals_forced(rows, compute=cp, scaling=sc)
fm = rs.marginals_forced(rows, compute=O.F64, scaling=sc)
gm = smp.marginals(0, rows)
for i in range(mps.num_sites):
    big = rm[:, i, :] >= 1e-3
    e = np.abs(gm[:, i, :][big] - rm[:, i, :][big]) / rm[:, i, :][big]
    f = np.abs(fm[:, i, :][big] - rm[:, i, :][big]) / fm[:, i, :][big]
    print(f"site {i:2d}: grid-vs-policy max {e.max():.2e} median {np.median(e):.2e} | policy-vs-f64 max {f.max():.2e} median {np.median(f):.2e}")
