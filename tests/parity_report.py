"""Parity report (needs a B200): the CUDA sweep against the CPU oracle on the same decoded MPS and
seed, with the north-star counts -- per-site marginals (teacher-forced along the oracle's strings)
within 1e-4 relative, outcome strings identical except draws within 1e-6 of a CDF boundary, which
are counted and reported.

    python tests/parity_report.py [out.json]

Test infrastructure (it imports the oracle); the same checks run as assertions in
test_gpu_parity.py.  Cases: the reference's random_mps(16, 32, 4, 42) (c1) and its lambda-decay
variant (c1b) from tests/golden, and device-generated chains at the c2 / c3 / c5 bond dimensions
(short M so the f64 oracle finishes in seconds), each under the 3M and the 4M contraction.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import oracle as O  # noqa: E402

import paper_2512_20064_b200 as P  # noqa: E402
from paper_2512_20064_b200.synthetic import build_synthetic  # noqa: E402

EPS_BOUNDARY = 1e-6
GOLD = os.path.join(ROOT, "tests", "golden")


def boundary_distance(marg_row, u):
    cum = np.cumsum(marg_row)[:-1]
    return float(np.min(np.abs(cum - u))) if cum.size else 1.0


def report(name, smp, dec, n, seed, scheme):
    t0 = time.time()
    ref_rows, ref_marg, _ = O.orc_sample_range(dec, 0, n, seed, want_marginals=True)
    gpu_rows = smp.sample(0, n, seed)
    gm = smp.marginals(0, ref_rows)
    live = ref_marg >= 0
    big = live & (ref_marg >= 1e-3)
    small = live & (ref_marg < 1e-3)
    rel = np.abs(gm[big] - ref_marg[big]) / ref_marg[big]
    # every (sample, site) draw of the oracle's own path: how many fall within EPS of a boundary
    m = dec.num_sites
    near = 0
    pairs = 0
    for s in range(n):
        for i in range(m):
            if ref_rows[s, i] == P.DEAD_OUTCOME:
                break
            pairs += 1
            u = O.orc().orc_uniform(seed, O.MEASURE_STREAM, s, i)
            if boundary_distance(ref_marg[s, i], u) < EPS_BOUNDARY:
                near += 1
    diff = np.nonzero((gpu_rows != ref_rows).any(axis=1))[0]
    explained, first_sites = 0, []
    for s in diff:
        i = int(np.argmax(gpu_rows[s] != ref_rows[s]))
        first_sites.append(i)
        u = O.orc().orc_uniform(seed, O.MEASURE_STREAM, int(s), i)
        if boundary_distance(ref_marg[s, i], u) < EPS_BOUNDARY:
            explained += 1
    return {
        "case": name, "scheme": scheme, "samples": n, "sites": m, "phys_dim": dec.phys_dim,
        "max_bond": int(max(dec.bond_dims)), "seed": seed, "draws_checked": pairs,
        "draws_within_1e-6_of_boundary": near,
        "strings_differing": int(len(diff)), "differences_explained_by_boundary_draws": explained,
        "unexplained_differences": int(len(diff)) - explained,
        "marginals_checked": int(big.sum() + small.sum()),
        "max_marginal_rel_err_p_ge_1e-3": float(rel.max()) if rel.size else 0.0,
        "max_marginal_abs_err_p_lt_1e-3": float(np.abs(gm[small] - ref_marg[small]).max()) if small.any() else 0.0,
        "pass": bool((rel.max() if rel.size else 0) < 1e-4 and len(diff) == explained),
        "seconds": round(time.time() - t0, 1),
    }


def report_ref(name, smp, dec, n, seed, scheme, threads=None):
    """Same checks against the reference itself (oracle/_ref, compiled from the reference's sources),
    multi-threaded: rows from ref_sample_range, teacher-forced marginals from ref_marginals_forced in
    parallel chunks -- for chains too large for the single-threaded C restatement."""
    from concurrent.futures import ThreadPoolExecutor
    t0 = time.time()
    threads = threads or os.cpu_count() or 1
    rs = O.RefState(dec)
    ref_rows = rs.sample_range(0, n, seed, threads=threads)
    chunks = np.array_split(np.arange(n), threads)
    with ThreadPoolExecutor(threads) as ex:
        parts = list(ex.map(lambda idx: rs.marginals_forced(ref_rows[idx]), [c for c in chunks if len(c)]))
    ref_marg = np.concatenate(parts)
    with ThreadPoolExecutor(threads) as ex:  # the reference's own F32 policy on the same strings
        f32_marg = np.concatenate(list(ex.map(lambda idx: rs.marginals_forced(ref_rows[idx], compute=O.F32),
                                              [c for c in chunks if len(c)])))
    gpu_rows = smp.sample(0, n, seed)
    gm = smp.marginals(0, ref_rows)
    live = ref_marg >= 0
    big = live & (ref_marg >= 1e-3)
    rel = np.abs(gm[big] - ref_marg[big]) / ref_marg[big]
    diff = np.nonzero((gpu_rows != ref_rows).any(axis=1))[0]
    explained = 0
    for s_ in diff:
        i = int(np.argmax(gpu_rows[s_] != ref_rows[s_]))
        u = O.orc().orc_uniform(seed, O.MEASURE_STREAM, int(s_), i)
        if boundary_distance(ref_marg[s_, i], u) < EPS_BOUNDARY:
            explained += 1
    # per-site classes: interior (full chi on both bonds) vs the right edge (chiR < chiL)
    b = list(dec.bond_dims)
    cmax = max(b)
    inner = [i for i in range(dec.num_sites) if b[i] == cmax and b[i + 1] == cmax]
    redge = [i for i in range(dec.num_sites) if b[i + 1] < b[i]]

    def cls_max(mg, sites):
        if not sites:
            return 0.0
        sel = big[:, sites, :]
        e = np.abs(mg[:, sites, :] - ref_marg[:, sites, :])[sel] / ref_marg[:, sites, :][sel]
        return float(e.max()) if e.size else 0.0
    extra = {"max_rel_err_interior_sites": cls_max(gm, inner), "max_rel_err_right_edge_sites": cls_max(gm, redge),
             "reference_f32_policy_max_rel_err_interior": cls_max(f32_marg, inner),
             "reference_f32_policy_max_rel_err_right_edge": cls_max(f32_marg, redge),
             "right_edge_sites": redge}
    return {**extra, "case": name, "scheme": scheme, "oracle": "reference (oracle/_ref, threaded)", "samples": n,
            "sites": dec.num_sites, "phys_dim": dec.phys_dim, "max_bond": int(max(dec.bond_dims)),
            "seed": seed, "draws_checked": int((ref_rows != P.DEAD_OUTCOME).sum()),
            "strings_differing": int(len(diff)), "differences_explained_by_boundary_draws": explained,
            "unexplained_differences": int(len(diff)) - explained,
            "marginals_checked": int(live.sum()),
            "max_marginal_rel_err_p_ge_1e-3": float(rel.max()) if rel.size else 0.0,
            "pass": bool((rel.max() if rel.size else 0) < 1e-4 and len(diff) == explained),
            "seconds": round(time.time() - t0, 1)}


def main():
    pol = P.PrecisionPolicy(scaling=P.ScalingMode.PER_SAMPLE_MAX)
    out = []
    for scheme in (P.Scheme.M3, P.Scheme.M4):
        tag = "3M" if scheme == P.Scheme.M3 else "4M"
        for case in ("c1", "c1b"):
            z = np.load(os.path.join(GOLD, f"{case}.npz"))
            mps = O.load_npz_mps(z)
            st = P.MpsState(mps.num_sites, mps.phys_dim, list(mps.bond_dims), list(mps.gammas),
                            list(mps.lambdas))
            smp = P.GpuSampler(st, pol, scheme=scheme)
            dec = O.Mps(mps.phys_dim, list(mps.bond_dims), [smp.decoded_gamma(i) for i in range(mps.num_sites)],
                        list(mps.lambdas))
            out.append(report(case, smp, dec, int(z["n"]), int(z["seed"]), tag))
            smp.close()
            print(json.dumps(out[-1]), flush=True)
        for (m, chi, d, n) in ((10, 512, 6, 64), (10, 2048, 6, 16), (12, 1024, 4, 32)):
            smp, lams = build_synthetic(m, chi, d, seed=11, policy=pol, scheme=int(scheme))
            dec = O.Mps(d, list(smp.bond_dims), [smp.decoded_gamma(i) for i in range(m)], list(lams))
            out.append(report(f"synthetic M={m} chi={chi} d={d}", smp, dec, n, 7, tag))
            smp.close()
            print(json.dumps(out[-1]), flush=True)
    # MPSG_MODE_PRECISE against the ORIGINAL chains (not the decoded ones)
    for case in ("c1", "c1b"):
        z = np.load(os.path.join(GOLD, f"{case}.npz"))
        mps = O.load_npz_mps(z)
        st = P.MpsState(mps.num_sites, mps.phys_dim, list(mps.bond_dims), list(mps.gammas), list(mps.lambdas))
        smp = P.GpuSampler(st, pol, mode=P.Mode.PRECISE)
        r = report(case + " (original MPS)", smp, mps, int(z["n"]), int(z["seed"]), "3M PRECISE")
        out.append(r)
        smp.close()
        print(json.dumps(out[-1]), flush=True)
    if O.have_ref():  # the c3 bond dimension over a 24-site chain (19 sites at chi = 2048)
        for scheme in (P.Scheme.M3, P.Scheme.M4):
            tag = "3M" if scheme == P.Scheme.M3 else "4M"
            m, chi, d, n = 24, 2048, 6, 256
            smp, lams = build_synthetic(m, chi, d, seed=5, policy=pol, scheme=int(scheme))
            dec = O.Mps(d, list(smp.bond_dims), [smp.decoded_gamma(i) for i in range(m)], list(lams))
            out.append(report_ref(f"c3 shape M={m} chi={chi} d={d}", smp, dec, n, 7, tag))
            smp.close()
            print(json.dumps(out[-1]), flush=True)
    path = sys.argv[1] if len(sys.argv) > 1 else None
    if path:
        with open(path, "w") as f:
            json.dump(out, f, indent=1)
    print("ALL PASS" if all(r["pass"] for r in out) else "FAILURES", flush=True)


if __name__ == "__main__":
    main()
