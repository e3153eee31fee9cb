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


def test_site_streaming_sweep_equals_reference_sampler(gold):
    """oracle.RefSiteSweep (the reference's per-site body driven one site at a time, threaded over
    sample chunks; used for the full-length c2 / c3 parity) reproduces the reference's own
    sample_micro_serial rows and teacher-forced marginals bit for bit, for F64 and F32, free-running
    and teacher-forced, and its near-boundary flags equal a direct count on the same CDFs."""
    if not O.have_ref():
        pytest.skip("oracle/_ref not built")
    for name in ("c1", "c1b"):
        mps = O.load_npz_mps(np.load(os.path.join(gold, f"{name}.npz")))
        rs = O.RefState(mps)
        for compute in (O.F64, O.F32):
            rows = rs.sample_range(0, 1000, 7, compute=compute, threads=4)
            marg = rs.marginals_forced(rows, compute=compute)
            sw = O.RefSiteSweep(0, 1000, 7, compute=compute, threads=3, eps=1e-3)
            tf = O.RefSiteSweep(0, 1000, 7, compute=compute, threads=2)
            for i in range(mps.num_sites):
                o, mg, near = sw.site(i, mps.gammas[i], mps.lambdas[i])
                assert np.array_equal(o, rows[:, i]), (name, compute, i)
                np.testing.assert_array_equal(mg, marg[:, i])
                u = np.array([O.orc().orc_uniform(7, O.MEASURE_STREAM, n, i) for n in range(1000)])
                cum = np.cumsum(mg, axis=1)[:, :-1]
                want = (np.abs(cum - u[:, None]) < 1e-3).any(axis=1) & (mg[:, 0] >= 0)
                assert np.array_equal(near, want), (name, i)
                o2, mg2, _ = tf.site(i, mps.gammas[i], mps.lambdas[i], forced=rows[:, i])
                assert np.array_equal(o2, rows[:, i])
                np.testing.assert_array_equal(mg2, marg[:, i])
            assert sw.contraction_macs == 1000 * sum(mps.bond_dims[i] * mps.bond_dims[i + 1] * mps.phys_dim
                                                     for i in range(mps.num_sites))


# ---- GBS displacement (SPEC.md gbs-ops; the reference's src/gbs.cpp is absent) ---------------
def test_displacement_closed_form_kats():
    """expm_displacement: mu = 0 -> identity; n = 2 closed form; the closed form
    L U e^{-|mu|^2/2} equals the exact Fock-basis matrix elements of D(mu) (expm of the generator at
    a 60-level cutoff, leading n x n block); vs the exact expm of the generator truncated at n = 10,
    1000 random |mu| <= 1, the leading 4 x 4 block (the levels a d = 4 site samples) agrees within
    the paper's 0.2% (§4.1) -- the difference is the generator's truncation, not the
    closed form."""
    from scipy.linalg import expm
    assert np.array_equal(O.orc_displacement(0.0, 6), np.eye(6))
    mu = 0.3
    want = np.exp(-mu * mu / 2) * np.array([[1, -mu], [mu, 1 - mu * mu]])
    np.testing.assert_allclose(O.orc_displacement(mu, 2), want, rtol=1e-15, atol=1e-16)
    rng = np.random.default_rng(1)
    n, big_n = 10, 60
    a10 = np.diag(np.sqrt(np.arange(1, n)), 1)
    a60 = np.diag(np.sqrt(np.arange(1, big_n)), 1)
    worst_exact = worst_trunc = 0.0
    for j in range(1000):
        m = rng.uniform(0, 1) * np.exp(2j * np.pi * rng.uniform())
        d = O.orc_displacement(m, n)
        if j < 50:
            exact = expm(m * a60.T - np.conj(m) * a60)[:n, :n]
            worst_exact = max(worst_exact, np.abs(d - exact).max())
        trunc = expm(m * a10.T - np.conj(m) * a10)[:4, :4]
        sel = np.abs(trunc) > 1e-3
        worst_trunc = max(worst_trunc, (np.abs(d[:4, :4] - trunc)[sel] / np.abs(trunc)[sel]).max())
    assert worst_exact < 1e-12, worst_exact
    assert worst_trunc < 2e-3, worst_trunc
    # first-order sanity: D(mu) -> I + mu a^dag - conj(mu) a
    eps = 1e-6 * (1 + 1j)
    np.testing.assert_allclose(O.orc_displacement(eps, 5), np.eye(5) + eps * np.diag(np.sqrt(np.arange(1, 5)), -1)
                               - np.conj(eps) * np.diag(np.sqrt(np.arange(1, 5)), 1), atol=1e-11)


def test_displaced_sampler_hook(gold):
    """The displacement hook sits between contract_site and measure (sampler.cpp:143): mu = 0 gives
    the undisplaced outcomes; a per-sample loop applying D(mu[n, i]) to temp matches the hook."""
    z = np.load(f"{gold}/c1b.npz")
    mps = O.load_npz_mps(z)
    n, m = 200, mps.num_sites
    base, _ = O.orc_sample_range(mps, 0, n, 7)
    zero, _ = O.orc_sample_range(mps, 0, n, 7, mu=np.zeros((n, m), complex))
    assert np.array_equal(base, zero)
    rng = np.random.default_rng(4)
    mu = 0.5 * (rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m)))
    rows, marg, _ = O.orc_sample_range(mps, 0, n, 7, want_marginals=True, mu=mu)
    assert (rows != base).any()
    # marginals of sample 0 at site 0 by hand: D applied to Gamma_0[0, b, :], weights sum_b L^2 |.|^2
    t = mps.gammas[0][0] @ O.orc_displacement(mu[0, 0], mps.phys_dim).T
    w = (mps.lambdas[0][:, None] ** 2 * np.abs(t) ** 2).sum(axis=0)
    np.testing.assert_allclose(marg[0, 0], w / w.sum(), rtol=1e-12)
