"""The CPU oracle (oracle/mpsamp_oracle.c) pinned against the reference's own outputs.

Golden vectors in tests/golden/ were produced by the compiled reference (oracle/gen_golden.py);
when oracle/_ref is present the restatement is also cross-checked live on random inputs.
"""
import json
import os

import numpy as np
import pytest

import oracle as O


def load_mps(npz, prefix=""):
    bonds = [int(x) for x in npz[prefix + "bond_dims"]]
    m = len(bonds) - 1
    mps = O.Mps(int(npz[prefix + "phys_dim"]), bonds)
    for i in range(m):
        mps.gammas.append(npz[f"{prefix}gamma_{i}"])
        mps.lambdas.append(npz[f"{prefix}lambda_{i}"])
    return mps


def test_rng_kat(gold):
    kat = json.load(open(os.path.join(gold, "rng_kat.json")))
    L = O.orc()
    for c in kat["keys"]:
        k = L.orc_key(c["seed"], kat["stream"], c["sample"], c["site"])
        assert f"{k:016x}" == c["key"]
        assert L.orc_uniform(c["seed"], kat["stream"], c["sample"], c["site"]) == float.fromhex(c["u"])
    for c in kat["mix64"]:
        assert f"{L.orc_mix64(c['z']):016x}" == c["mix64"]
    # SURVEY.md §8c known answers
    assert L.orc_key(7, O.MEASURE_STREAM, 0, 0) == 0xEA0DDC510138B7A2
    assert L.orc_mix64(0) == 0xE220A8397B1DCDAF


def test_round_kat(gold):
    kat = json.load(open(os.path.join(gold, "round_kat.json")))
    L = O.orc()
    for c in kat["cases"]:
        x = float.fromhex(c["x"])
        for tag, p in (("f32", O.F32), ("tf32", O.TF32), ("f16", O.F16)):
            got = L.orc_round_scalar(x, p)
            want = float.fromhex(c[tag])
            assert got == want or (np.isnan(got) and np.isnan(want)), (x, tag, got, want)


@pytest.mark.parametrize("name", ["c1", "c1b"])
@pytest.mark.parametrize("tag,compute,scaling", [("f64_psm", O.F64, O.SCALE_PER_SAMPLE),
                                                 ("f64_none", O.F64, O.SCALE_NONE),
                                                 ("tf32_psm", O.TF32, O.SCALE_PER_SAMPLE),
                                                 ("f16_psm", O.F16, O.SCALE_PER_SAMPLE)])
def test_chain_golden(gold, name, tag, compute, scaling):
    z = np.load(os.path.join(gold, f"{name}.npz"))
    mps = load_mps(z)
    rows, macs = O.orc_sample_range(mps, 0, int(z["n"]), int(z["seed"]), compute, scaling)
    assert np.array_equal(rows, z[f"out_{tag}"])
    assert O.fnv1a(rows) == int(z[f"hash_{tag}"])
    assert macs == int(z[f"macs_{tag}"])


def test_c1_hash_matches_survey(gold):
    z = np.load(os.path.join(gold, "c1.npz"))
    assert int(z["hash_f64_psm"]) == 0x991D873B454AB515
    assert int(z["hash_tf32_psm"]) == 0x8A7DA8296A6DCE27
    assert list(z["out_f64_psm"][0]) == [0] * 10 + [1, 0, 0, 0, 2, 2]
    assert int(z["macs_f64_psm"]) == 45_600_000


def test_forced_marginals_golden(gold):
    z = np.load(os.path.join(gold, "c1.npz"))
    mps = load_mps(z)
    forced = z["out_f64_psm"][:64]
    _, marg, _ = O.orc_sample_range(mps, 0, 64, 7, forced=forced, want_marginals=True)
    np.testing.assert_allclose(marg, z["marg_f64"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(marg.sum(-1), 1.0, atol=1e-12)


def test_small_chains_golden(gold):
    z = np.load(os.path.join(gold, "small.npz"))
    for j in range(int(z["ncases"])):
        mps = load_mps(z, f"c{j}_")
        rows, _ = O.orc_sample_range(mps, 0, 300, int(z[f"c{j}_seed"]))
        assert np.array_equal(rows, z[f"c{j}_out"]), j


def test_decay_golden(gold):
    z = np.load(os.path.join(gold, "decay.npz"))
    mps = load_mps(z, "decay_")
    for tag, compute, scaling in [("f64_none", O.F64, O.SCALE_NONE), ("f16_none", O.F16, O.SCALE_NONE),
                                  ("f16_psm", O.F16, O.SCALE_PER_SAMPLE)]:
        rows, _ = O.orc_sample_range(mps, 0, 200, 3, compute, scaling)
        assert np.array_equal(rows, z[f"decay_{tag}"]), tag
        dead = int((rows[:, -1] == O.DEAD).sum())
        assert dead == int(z[f"decay_dead_{tag}"])


def test_capped_bond_dims():
    assert O.capped_bond_dims(16, 4, 32) == [1, 4, 16] + [32] * 11 + [16, 4, 1]
    b = O.capped_bond_dims(1024, 6, 2048)
    assert b[:6] == [1, 6, 36, 216, 1296, 2048] and b[-6:] == [2048, 1296, 216, 36, 6, 1]


def test_batching_invariance():
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "c1.npz"))
    mps = load_mps(z)
    full = z["out_f64_psm"]
    a, _ = O.orc_sample_range(mps, 300, 77, 7)
    assert np.array_equal(a, full[300:377])


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")
def test_live_cross_check_random():
    rng = np.random.default_rng(0)
    for trial in range(4):
        m, chi, d = int(rng.integers(2, 9)), int(rng.integers(1, 24)), int(rng.integers(2, 6))
        mps = O.ref_random_mps(m, chi, d, int(rng.integers(1 << 30)), lambda_decay=0.3)
        rs = O.RefState(mps)
        for compute in (O.F64, O.F32, O.F16):
            want, _, _ = rs.sample_batch(200, 11 + trial, compute=compute)
            got, _ = O.orc_sample_range(mps, 0, 200, 11 + trial, compute=compute)
            assert np.array_equal(want, got), (trial, compute)
        forced = want
        np.testing.assert_allclose(O.orc_sample_range(mps, 0, 200, 1, forced=forced, want_marginals=True)[1],
                                   rs.marginals_forced(forced), rtol=1e-12, atol=1e-15)
