"""Worker for the engine A/B identity tests (test_select_fast_path_identical,
test_compact_3m_store_identical): samples a set of chains and writes rows, teacher-forced marginals,
counters and state sizes to an npz.  The tests run it under two settings of an engine switch
(MPSG_SELECT_LEGACY, MPSG_COMPACT_3M -- read once per process) and compare the files bit for bit."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402
import paper_2512_20064_b200 as P  # noqa: E402
from paper_2512_20064_b200.synthetic import build_synthetic  # noqa: E402

out, gold = sys.argv[1], sys.argv[2]
res = {}
pol = P.PrecisionPolicy(scaling=P.ScalingMode.PER_SAMPLE_MAX)


def record(tag, smp, n, seed, first=0):
    st = P.RunStats()
    rows = smp.sample(first, n, seed, stats=st)
    res[tag + "_rows"] = rows
    res[tag + "_stats"] = np.array([st.contraction_macs, st.dead_samples, st.measure_weight_macs,
                                    st.near_boundary_draws], dtype=np.uint64)
    # teacher-forced marginals along the recorded strings (forced path, marginals written)
    res[tag + "_marg"] = smp.marginals(first, rows[: min(n, 300)])


for m, chi, d, n, ps, mode in [(10, 256, 4, 2000, 0, P.Mode.SPLIT), (8, 512, 6, 1100, 384, P.Mode.SPLIT),
                               (6, 1024, 4, 900, 512, P.Mode.SPLIT), (8, 256, 8, 700, 0, P.Mode.SINGLE),
                               (6, 256, 3, 600, 256, P.Mode.PRECISE)]:
    smp, _ = build_synthetic(m, chi, d, seed=13, policy=pol, mode=mode, pass_samples=ps)
    record(f"syn_{m}_{chi}_{d}_{int(mode)}", smp, n, 7, first=5)
    res[f"syn_{m}_{chi}_{d}_{int(mode)}_state_bytes"] = np.array([smp.state_bytes], dtype=np.uint64)
    smp.close()
g0 = np.zeros((1, 2, 2), complex)  # a chain where some samples die (test_gpu_parity._dead_chain)
g0[0, 0, 0], g0[0, 1, 1] = 1.0, 0.8
g1 = np.zeros((2, 2, 2), complex)
g1[0, :, :] = [[0.5, 0.2j], [0.3, 0.4]]
g2 = np.zeros((2, 1, 2), complex)
g2[:, 0, :] = [[1.0, 0.5], [0.25, 1.0]]
dead = O.Mps(2, [1, 2, 2, 1], [g0, g1, g2])
dead.lambdas = [np.array([0.8, 0.6]), np.array([0.9, 0.4359]), np.ones(1)]
for name in ("c1", "c1b", "dead"):
    mps = dead if name == "dead" else O.load_npz_mps(np.load(f"{gold}/{name}.npz"))
    st = P.MpsState(mps.num_sites, mps.phys_dim, list(mps.bond_dims), list(mps.gammas), list(mps.lambdas))
    smp = P.GpuSampler(st, pol, pass_samples=384)
    record(name, smp, 1000, 7)
    smp.close()
np.savez(out, **res)
