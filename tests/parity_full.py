"""Full-length parity on a benchmark chain (needs a B200; test infrastructure -- imports the oracle).

    python tests/parity_full.py --config c2 --samples 1024 --out profiles/r2_parity/c2_full.json
    python tests/parity_full.py --config c3 --samples 64 --f32 --out profiles/r2_parity/c3_full.json
    python tests/parity_full.py --config c2 --samples 1024 --mode precise --against original --f32 \
        --out profiles/r2_parity/c2_full_precise_original.json

The chain is the benchmark's own synthetic chain (bench.py: build_synthetic(M, chi, d, seed=42)) at
its full length.  The GPU sweep (through the C ABI) is compared with the reference itself
(oracle/_ref, compiled from /root/reference/proj/src) run on the same decoded Gamma and measurement
seed, site by site (oracle.RefSiteSweep: the reference's contract_site -> measurement_draws ->
measure -> scale_rows_inplace, sampler.cpp:140-158, threaded over sample chunks), so chains whose
complex128 Gamma exceeds host memory (c3: 409 GB) can be checked: one decoded site at a time.

Per site it records the reference's conditional distribution along its own outcome prefix and the
GPU's teacher-forced distribution along the same prefix (mpsg_marginals), and counts the draws that
lie within 1e-6 of an interior CDF boundary on the reference's path (the north star's exclusion
rule).  Reported: per-site max relative error (p >= 1e-3) split into left-edge (bond growing),
interior (full chi) and right-edge (bond shrinking) sites, the absolute error below p = 1e-3,
differing outcome strings and whether each is explained by a near-boundary draw at its first
differing site, and the GPU's own device-side near-boundary counter.  --f32 also runs the
reference's F32 compute policy teacher-forced along the same strings (the fp32-class envelope).
"""
import argparse
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

CONFIGS = {"c2": (256, 512, 6), "c3": (1024, 2048, 6), "c5_256": (512, 256, 4), "c5_1024": (512, 1024, 4),
           "c5_4096": (512, 4096, 4),
           "c4": (8176, 10000, 4)}  # c4 with --sites N: an N-site chain of the c4 shape (chi = 1e4 in the middle)
EPS = 1e-6


def site_classes(bonds):
    m = len(bonds) - 1
    cmax = max(bonds)
    left = [i for i in range(m) if bonds[i + 1] > bonds[i]]
    inner = [i for i in range(m) if bonds[i] == cmax and bonds[i + 1] == cmax]
    right = [i for i in range(m) if bonds[i + 1] < bonds[i]]
    return left, inner, right


def run(config, n, seed=7, mps_seed=42, threads=None, f32=False, scheme=0, m_override=0, log=print,
        generated=True, mode="split", against="decoded"):
    m, chi, d = CONFIGS[config]
    if m_override:
        m = m_override
    t0 = time.time()
    pol = P.PrecisionPolicy(scaling=P.ScalingMode.PER_SAMPLE_MAX)
    # generated=True: the same chain (tests/test_gpu_parity.py::test_generated_supply_equals_resident_chain)
    # held as its generators -- a few hundred MB of HBM instead of the resident state (c3: 153 GB)
    # against="original": the reference runs on the chain's own values (the generator's complex64
    # sites, widened to f64) instead of the device's decoded Gamma -- the caller's-MPS contract that
    # MPSG_MODE_PRECISE (AUTO at F64 / F32) targets
    pmode = {"split": P.Mode.SPLIT, "precise": P.Mode.PRECISE}[mode]
    host = None
    if against == "original" and not generated:
        smp, lams, host = build_synthetic(m, chi, d, seed=mps_seed, policy=pol, scheme=scheme, mode=pmode,
                                          keep_host=True)
    else:  # generated: the original sites come from the generator on demand (original_gamma)
        smp, lams = build_synthetic(m, chi, d, seed=mps_seed, policy=pol, scheme=scheme, mode=pmode,
                                    generated=generated)
    original = against == "original"
    bonds = list(smp.bond_dims)
    scheme_name = ("3M" if smp.scheme == P.Scheme.M3 else "4M") + " " + smp.mode.name
    t_build = time.time() - t0
    st = P.RunStats()
    gpu_rows = smp.sample(0, n, seed, stats=st)
    # the reference, site by site on the decoded Gamma
    ref = O.RefSiteSweep(0, n, seed, threads=threads, eps=EPS)
    r32 = O.RefSiteSweep(0, n, seed, compute=O.F32, threads=threads, eps=EPS) if f32 else None
    ref_rows = np.empty((n, m), np.uint8)
    ref_marg = np.empty((n, m, d), np.float64)
    f32_marg = np.empty((n, m, d), np.float64) if f32 else None
    near = np.zeros((n, m), bool)
    t1 = time.time()
    for i in range(m):
        g = host[i] if host is not None else (smp.original_gamma(i) if original else smp.decoded_gamma(i))
        o, mg, nb = ref.site(i, g, lams[i])
        ref_rows[:, i], ref_marg[:, i], near[:, i] = o, mg, nb
        if f32:
            _, mg32, _ = r32.site(i, g, lams[i], forced=o)
            f32_marg[:, i] = mg32
        del g
        if i % 64 == 0 or i == m - 1:
            log(f"  site {i}/{m}  {time.time() - t1:.0f} s")
    t_ref = time.time() - t1
    gm = smp.marginals(0, ref_rows)
    smp.close()

    live = ref_marg >= 0
    big = live & (ref_marg >= 1e-3)
    small = live & (ref_marg < 1e-3)
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.where(big, np.abs(gm - ref_marg) / np.where(big, ref_marg, 1.0), 0.0)
        rel32 = np.where(big, np.abs(f32_marg - ref_marg) / np.where(big, ref_marg, 1.0), 0.0) if f32 else None
    per_site = rel.max(axis=(0, 2))
    per_site32 = rel32.max(axis=(0, 2)) if f32 else None
    left, inner, right = site_classes(bonds)

    def cmax(a, sites):
        return float(a[sites].max()) if sites else 0.0

    diff = np.nonzero((gpu_rows != ref_rows).any(axis=1))[0]
    details, explained = [], 0
    for s in diff:
        i = int(np.argmax(gpu_rows[s] != ref_rows[s]))
        ok = bool(near[s, i])
        explained += ok
        u = O.orc().orc_uniform(seed, O.MEASURE_STREAM, int(s), i)
        cum = np.cumsum(ref_marg[s, i])[:-1]
        details.append({"sample": int(s), "first_site": i, "gpu": int(gpu_rows[s, i]), "ref": int(ref_rows[s, i]),
                        "draw": u, "boundary_distance": float(np.min(np.abs(cum - u))) if cum.size else 1.0,
                        "explained": ok})
    out = {
        "config": config, "M": m, "chi": chi, "d": d, "samples": n, "mps_seed": mps_seed, "seed": seed,
        "scheme": scheme_name,
        "oracle": ("reference (oracle/_ref), site-streamed " +
                   ("original (generator) Gamma" if original else "decoded Gamma") +
                   ", F64 + PerSampleMax, threaded"),
        "gamma_supply": "generated (regenerated on the device)" if generated else "resident",
        "draws_checked": int(live[:, :, 0].sum()),
        "near_boundary_draws_reference_path": int(near.sum()),
        "near_boundary_draws_gpu_device_counter": int(st.near_boundary_draws),
        "strings_differing": int(len(diff)), "differences_explained_by_boundary_draws": int(explained),
        "unexplained_differences": int(len(diff)) - int(explained), "differences": details[:50],
        "marginals_checked": int(live.sum()),
        "max_rel_err_p_ge_1e-3": float(per_site.max()),
        "max_rel_err_left_edge_sites": cmax(per_site, left),
        "max_rel_err_interior_sites": cmax(per_site, inner),
        "max_rel_err_right_edge_sites": cmax(per_site, right),
        "right_edge_sites": right, "left_edge_sites": left,
        "max_abs_err_p_lt_1e-3": float(np.abs(gm[small] - ref_marg[small]).max()) if small.any() else 0.0,
        "per_site_max_rel_err": [float(x) for x in per_site],
        "dead_samples_gpu": int((gpu_rows[:, -1] == P.DEAD_OUTCOME).sum()),
        "dead_samples_ref": int((ref_rows[:, -1] == P.DEAD_OUTCOME).sum()),
        "contraction_macs_ref": ref.contraction_macs, "contraction_macs_gpu": int(st.contraction_macs),
        "seconds": {"build": round(t_build, 1), "reference": round(t_ref, 1), "total": round(time.time() - t0, 1)},
        "threads": threads or os.cpu_count(),
    }
    if f32:
        out.update({"reference_f32_policy_max_rel_err_interior": cmax(per_site32, inner),
                    "reference_f32_policy_max_rel_err_right_edge": cmax(per_site32, right),
                    "reference_f32_policy_max_rel_err_left_edge": cmax(per_site32, left),
                    "reference_f32_policy_per_site_max_rel_err": [float(x) for x in per_site32]})
    out["pass_interior_1e-4"] = out["max_rel_err_interior_sites"] < 1e-4
    out["pass_strings"] = out["unexplained_differences"] == 0
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--samples", type=int, default=1024)
    ap.add_argument("--sites", type=int, default=0, help="override M (0: the config's full chain)")
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--f32", action="store_true")
    ap.add_argument("--scheme", default="auto", choices=["auto", "3m", "4m"])
    ap.add_argument("--supply", default="generated", choices=["generated", "resident"])
    ap.add_argument("--mode", default="split", choices=["split", "precise"])
    ap.add_argument("--against", default="decoded", choices=["decoded", "original"],
                    help="original: the reference on the chain's own values (PRECISE's contract)")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    scheme = {"auto": 0, "3m": 3, "4m": 4}[a.scheme]
    r = run(a.config, a.samples, threads=a.threads or None, f32=a.f32, scheme=scheme, m_override=a.sites,
            log=lambda s: print(s, file=sys.stderr, flush=True), generated=a.supply == "generated",
            mode=a.mode, against=a.against)
    txt = json.dumps(r, indent=1)
    if a.out:
        os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
        with open(a.out, "w") as f:
            f.write(txt)
    short = {k: v for k, v in r.items() if not isinstance(v, list) and k != "differences"}
    print(json.dumps(short))


if __name__ == "__main__":
    main()
