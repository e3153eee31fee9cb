"""TEST INFRASTRUCTURE ONLY — regenerate tests/golden/ from the compiled reference.

Run here (where /root/reference exists):  python oracle/gen_golden.py
Every number in tests/golden/ comes from oracle/_ref/libmpsamp_ref.so, i.e. the unmodified
reference sources compiled by oracle/Makefile.  The reference ships no tests or fixtures
(SURVEY.md §4), so these goldens are the pinned known answers for the hot path:

  rng_kat.json      rng::mix64 / key / uniform (rng.hpp:12-37) incl. the survey's KATs (§8c)
  round_kat.json    round_scalar F32/TF32/F16 (precision.cpp:23-50)
  c1.npz            random_mps(16, 32, 4, 42) (mps.cpp:129) Gamma/Lambda + outcome matrices
                    (sample_batch, sampler.cpp:164) for seed 7, N=1000 under several policies,
                    teacher-forced marginals, contraction MACs
  c1b.npz           same chain with lambda_decay = 4/chi = 0.125
  small.npz         a few tiny edge-case chains (d=2/3/5/7, chi 1..8) with outcomes
  decay.npz         decay_chain / branching_decay_chain outcomes (underflow rows)
  schemes.json      serial == DP(p1=4) == single-site TP(2x2) == double-site TP(2x4) hashes
"""
from __future__ import annotations

import json
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import oracle as O  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def mps_to_npz_dict(mps: O.Mps, prefix: str = "") -> dict:
    d = {prefix + "bond_dims": np.array(mps.bond_dims, np.int64),
         prefix + "phys_dim": np.array(mps.phys_dim)}
    for i, (g, lam) in enumerate(zip(mps.gammas, mps.lambdas)):
        d[f"{prefix}gamma_{i}"] = g
        d[f"{prefix}lambda_{i}"] = lam
    return d


def rng_kat() -> dict:
    L = O.ref()
    keys = []
    for seed, sample, site in [(7, 0, 0), (7, 0, 1), (7, 1, 0), (0, 0, 0), (123456789, 999999, 1023),
                               (2**64 - 1, 2**63 + 5, 77), (42, 12345, 8175), (7, 999999, 0)]:
        k = L.ref_rng_key(seed, O.MEASURE_STREAM, sample, site)
        u = L.ref_rng_uniform(seed, O.MEASURE_STREAM, sample, site)
        keys.append({"seed": seed, "sample": sample, "site": site, "key": f"{k:016x}", "u": u.hex()})
    mix = [{"z": z, "mix64": f"{L.ref_mix64(z):016x}"} for z in [0, 1, 2, 0xDEADBEEF, 2**64 - 1]]
    return {"stream": O.MEASURE_STREAM, "keys": keys, "mix64": mix}


def round_kat() -> dict:
    L = O.ref()
    rng = np.random.default_rng(5)
    xs = [0.0, -0.0, 1.0, 1.0 + 2**-11, 1.0 + 3 * 2**-11, 65504.0, 65520.0, 2**-14, 2**-24, 2**-25,
          3 * 2**-26, 1e-30, 3.0e38, 3.5e38, 1 / 3]
    xs += list(rng.standard_normal(40) * 10.0 ** rng.integers(-9, 9, 40))
    out = []
    for x in xs:
        out.append({"x": float(x).hex(), "f32": L.ref_round_scalar(x, O.F32).hex(),
                    "tf32": L.ref_round_scalar(x, O.TF32).hex(), "f16": L.ref_round_scalar(x, O.F16).hex()})
    return {"cases": out}


def chain_goldens(mps: O.Mps, n: int, seed: int) -> dict:
    rs = O.RefState(mps)
    d = mps_to_npz_dict(mps)
    for tag, compute, scaling in [("f64_psm", O.F64, O.SCALE_PER_SAMPLE), ("f64_none", O.F64, O.SCALE_NONE),
                                  ("tf32_psm", O.TF32, O.SCALE_PER_SAMPLE), ("f16_psm", O.F16, O.SCALE_PER_SAMPLE)]:
        out, macs, dead = rs.sample_batch(n, seed, compute=compute, scaling=scaling)
        d[f"out_{tag}"] = out
        d[f"hash_{tag}"] = np.array(O.fnv1a(out), np.uint64)
        d[f"macs_{tag}"] = np.array(macs, np.uint64)
        d[f"dead_{tag}"] = np.array(dead, np.uint64)
    d["seed"] = np.array(seed)
    d["n"] = np.array(n)
    nf = min(n, 64)
    d["marg_f64"] = rs.marginals_forced(d["out_f64_psm"][:nf])
    return d


def small_chains() -> dict:
    out = {}
    cases = [(6, 8, 2, 3), (5, 4, 3, 11), (4, 8, 5, 12), (3, 16, 7, 13), (8, 1, 2, 14), (2, 64, 3, 15)]
    for j, (m, chi, dd, s) in enumerate(cases):
        mps = O.ref_random_mps(m, chi, dd, s)
        rs = O.RefState(mps)
        res, _, _ = rs.sample_batch(300, 99 + j)
        out.update(mps_to_npz_dict(mps, f"c{j}_"))
        out[f"c{j}_out"] = res
        out[f"c{j}_seed"] = np.array(99 + j)
    out["ncases"] = np.array(len(cases))
    return out


def decay_goldens() -> dict:
    out = {}
    mps = O.ref_decay_chain(60, 3, 1.0)
    rs = O.RefState(mps)
    for tag, compute, scaling in [("f64_none", O.F64, O.SCALE_NONE), ("f16_none", O.F16, O.SCALE_NONE),
                                  ("f16_psm", O.F16, O.SCALE_PER_SAMPLE)]:
        res, _, dead = rs.sample_batch(200, 3, compute=compute, scaling=scaling)
        out[f"decay_{tag}"] = res
        out[f"decay_dead_{tag}"] = np.array(dead)
    out.update(mps_to_npz_dict(mps, "decay_"))
    return out


def schemes() -> dict:
    mps = O.ref_random_mps(16, 32, 4, 42)
    rs = O.RefState(mps)
    res = {}
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "c1.mpsb").encode()
        assert O.ref().ref_save_mps(rs.h, path, O.F64) == 0
        for name, scheme, p1, p2 in [("serial", 0, 1, 1), ("dp4", 1, 4, 1), ("single_2x2", 2, 2, 2),
                                     ("double_2x4", 3, 2, 4)]:
            out = np.empty((1000, 16), np.uint8)
            rc = O.ref().ref_run_scheme(path, scheme, 1000, 250, 77, p1, p2, 7, O.F64, O.SCALE_PER_SAMPLE,
                                        out.ctypes.data_as(O._pu8))
            assert rc == 0, O.ref().ref_last_error()
            res[name] = f"{O.fnv1a(out):016x}"
    return res


def main() -> None:
    os.makedirs(GOLD, exist_ok=True)
    with open(os.path.join(GOLD, "rng_kat.json"), "w") as f:
        json.dump(rng_kat(), f, indent=1)
    with open(os.path.join(GOLD, "round_kat.json"), "w") as f:
        json.dump(round_kat(), f, indent=1)
    np.savez_compressed(os.path.join(GOLD, "c1.npz"), **chain_goldens(O.ref_random_mps(16, 32, 4, 42), 1000, 7))
    np.savez_compressed(os.path.join(GOLD, "c1b.npz"),
                        **chain_goldens(O.ref_random_mps(16, 32, 4, 42, lambda_decay=4 / 32), 1000, 7))
    np.savez_compressed(os.path.join(GOLD, "small.npz"), **small_chains())
    np.savez_compressed(os.path.join(GOLD, "decay.npz"), **decay_goldens())
    with open(os.path.join(GOLD, "schemes.json"), "w") as f:
        json.dump(schemes(), f, indent=1)
    print("goldens written to", GOLD)


if __name__ == "__main__":
    main()
