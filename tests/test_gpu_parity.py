"""GPU parity: the CUDA sweep (through the C ABI) against the CPU oracle on the same MPS and seed.

The oracle consumes the *decoded* compressed Gamma (mpsg_decoded_gamma), i.e. exactly the values
the GPU samples.  Tolerances (north star, BASELINE.json):
  * per-site marginals: relative 1e-4 (absolute 1e-7 for p < 1e-3);
  * outcome strings identical except draws within EPS_BOUNDARY of a CDF boundary, which are
    counted and reported (north-star rule: 1e-6).
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

MARG_RTOL = 1e-4
MARG_ATOL_SMALL = 1e-7
EPS_BOUNDARY = 1e-6
# Right-edge sites (chiR < chiL) of long chains: pinned bound on the marginal relative error against
# the f64 reference (measured on the full c2 / c3 chains, profiles/r2_parity/).
RIGHT_EDGE_RTOL = 2e-3
# sharded vs unsharded sweep: identical contraction; only the exchanged per-rank weight partials are
# rounded to fp32 (relative 2^-24 each)
TP_RTOL = 1e-6


@pytest.fixture(scope="module")
def pkg():
    import paper_2512_20064_b200 as P
    if P.sampler._lib.lib().mpsg_device_count() == 0:
        pytest.fail("no B200 visible to libmpsg (GPU test on a non-GPU host)")
    return P


def to_state(P, mps: O.Mps):
    return P.MpsState(mps.num_sites, mps.phys_dim, list(mps.bond_dims), list(mps.gammas), list(mps.lambdas))


def decoded_mps(smp, mps: O.Mps) -> O.Mps:
    out = O.Mps(mps.phys_dim, list(mps.bond_dims))
    for i in range(mps.num_sites):
        out.gammas.append(smp.decoded_gamma(i))
        out.lambdas.append(mps.lambdas[i])
    return out


def boundary_distance(marg_row: np.ndarray, u: float) -> float:
    """Distance of draw u to the nearest interior CDF boundary of one site's distribution."""
    cum = np.cumsum(marg_row)[:-1]
    return float(np.min(np.abs(cum - u))) if cum.size else 1.0


def compare_strings(gpu_rows, ref_rows, marg_ref, seed, first=0, eps=EPS_BOUNDARY):
    """Returns (#differing samples, #explained by boundary draws).  A sample's string may differ
    only from the first site whose draw lies within eps of a reference CDF boundary."""
    diff = np.nonzero((gpu_rows != ref_rows).any(axis=1))[0]
    explained = 0
    for n in diff:
        i = int(np.argmax(gpu_rows[n] != ref_rows[n]))
        u = O.orc().orc_uniform(seed, O.MEASURE_STREAM, first + int(n), i)
        if boundary_distance(marg_ref[n, i], u) < eps:
            explained += 1
    return len(diff), explained


def test_device_rng_bit_exact(pkg):
    L = O.orc()
    for seed, first, site in [(7, 0, 0), (7, 0, 1), (123456789, 999990, 1023), (2**64 - 1, 2**63, 5)]:
        got = pkg.device_draws(seed, first, 64, site)
        want = np.array([L.orc_uniform(seed, O.MEASURE_STREAM, first + j, site) for j in range(64)])
        assert np.array_equal(got, want)
    assert pkg.device_draws(7, 0, 1, 0)[0] == 0.91427399614005611


def test_decode_close_to_input(pkg, gold):
    z = np.load(f"{gold}/c1b.npz")
    mps = O.load_npz_mps(z)
    smp = pkg.GpuSampler(to_state(pkg, mps))
    for i in range(mps.num_sites):
        g, dg = mps.gammas[i], smp.decoded_gamma(i)
        # per-column relative error <= fp16 half-ulp of the column max (plus subnormal floor)
        colmax = np.maximum(np.abs(g.real), np.abs(g.imag)).max(axis=0, keepdims=True)
        err = np.maximum(np.abs(g.real - dg.real), np.abs(g.imag - dg.imag))
        assert (err <= colmax * 2.0 ** -10 + 1e-300).all(), i


@pytest.mark.parametrize("scheme", [3, 4])
@pytest.mark.parametrize("mode", ["split", "single"])
def test_contract_site_numerics(pkg, gold, mode, scheme):
    z = np.load(f"{gold}/c1b.npz")
    mps = O.load_npz_mps(z)
    smp = pkg.GpuSampler(to_state(pkg, mps), mode=pkg.Mode.SPLIT if mode == "split" else pkg.Mode.SINGLE,
                         scheme=pkg.Scheme(scheme))
    rng = np.random.default_rng(3)
    tol = 2e-6 if mode == "split" else 2e-3
    for i in [0, 1, 2, 5, 13, 14, 15]:
        gd = smp.decoded_gamma(i)
        cl = gd.shape[0]
        env = rng.standard_normal((300, cl)) + 1j * rng.standard_normal((300, cl))
        got = smp.contract_site(i, env)
        want = np.einsum("nl,lrk->nrk", env, gd)
        scale = np.abs(want).max(axis=(1, 2), keepdims=True)
        rel = (np.abs(got - want) / scale).max()
        assert rel < tol, (i, rel)


@pytest.mark.parametrize("scheme,mode", [(3, 1), (4, 1), (3, 0)])
@pytest.mark.parametrize("name", ["c1", "c1b"])
def test_c1_strings_and_marginals(pkg, gold, name, scheme, mode):
    """mode 1 = SPLIT (the benchmark's), 0 = AUTO (F64 compute: PRECISE, the state fits)."""
    z = np.load(f"{gold}/{name}.npz")
    mps = O.load_npz_mps(z)
    n, seed = int(z["n"]), int(z["seed"])
    smp = pkg.GpuSampler(to_state(pkg, mps), pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX),
                         scheme=pkg.Scheme(scheme), mode=pkg.Mode(mode))
    assert smp.mode == (pkg.Mode.PRECISE if mode == 0 else pkg.Mode.SPLIT)
    dec = decoded_mps(smp, mps)
    ref_rows, ref_marg, _ = O.orc_sample_range(dec, 0, n, seed, want_marginals=True)
    gpu_rows = smp.sample(0, n, seed)
    # teacher-forced GPU marginals along the reference's own outcome strings
    gpu_marg = smp.marginals(0, ref_rows)
    live = ref_marg >= 0
    big = live & (ref_marg >= 1e-3)
    small = live & (ref_marg < 1e-3)
    rel = np.abs(gpu_marg[big] - ref_marg[big]) / ref_marg[big]
    assert rel.max() < MARG_RTOL, rel.max()
    assert np.abs(gpu_marg[small] - ref_marg[small]).max() < MARG_ATOL_SMALL
    ndiff, explained = compare_strings(gpu_rows, ref_rows, ref_marg, seed)
    assert ndiff == explained, (ndiff, explained)


def test_c1_sample_batch_api(pkg, gold):
    """sample_batch through the reference-shaped API; batching plan must not change outcomes."""
    z = np.load(f"{gold}/c1.npz")
    mps = O.load_npz_mps(z)
    st = to_state(pkg, mps)
    opts = pkg.SamplerOptions(policy=pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX), seed=7)
    a = pkg.sample_batch(st, pkg.BatchPlan(1000, 0, 5000), opts)
    opts.pass_samples = 128
    b = pkg.sample_batch(st, pkg.BatchPlan(1000, 300, 77), opts)
    assert np.array_equal(a.outcomes, b.outcomes)
    assert a.dead_count() == 0
    smp = pkg.GpuSampler(st, opts.policy)
    part = smp.sample(300, 77, 7)
    assert np.array_equal(part, a.outcomes[300:377])


def test_cpp_dropin_adapter_gpu():
    """mpsg_mpsamp::sample_batch (C++ drop-in, built against the reference headers) on the B200."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "adapter_test")
    if not os.path.exists(exe):
        pytest.skip("adapter_test not built (needs the reference headers at build time)")
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=120)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("p2", [2, 3])
def test_tensor_parallel_local(pkg, gold, p2):
    """Column-sharded Gamma + per-site exchange (p2 ranks on one device, in-process exchange):
    rows identical on every rank and equal to the unsharded sweep except boundary draws;
    marginals within 1e-4 of the oracle."""
    from paper_2512_20064_b200.parallel import TensorParallelLocal
    z = np.load(f"{gold}/c1b.npz")
    mps = O.load_npz_mps(z)
    st = to_state(pkg, mps)
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    tp = TensorParallelLocal(st, p2, policy=pol)
    one = pkg.GpuSampler(st, pol)
    for i in range(mps.num_sites):
        assert np.array_equal(tp.decoded_gamma(i), one.decoded_gamma(i)), i
    rows = tp.sample(0, 1000, 7)
    for r in rows[1:]:
        assert np.array_equal(r, rows[0])
    dec = decoded_mps(one, mps)
    ref_rows, ref_marg, _ = O.orc_sample_range(dec, 0, 1000, 7, want_marginals=True)
    ndiff, explained = compare_strings(rows[0], ref_rows, ref_marg, 7)
    assert ndiff == explained, (ndiff, explained)
    marg = tp.marginals(0, ref_rows)[0]
    big = ref_marg >= 1e-3
    assert (np.abs(marg[big] - ref_marg[big]) / ref_marg[big]).max() < MARG_RTOL
    # block-aligned shards: the sharded sweep accumulates the unsharded sweep's K blocks in order,
    # so rows are identical and marginals differ only by the fp32 rounding of the exchanged weights
    assert np.array_equal(rows[0], one.sample(0, 1000, 7))
    gm = one.marginals(0, ref_rows)
    assert (np.abs(marg[big] - gm[big]) / gm[big]).max() < TP_RTOL
    tp.close()
    one.close()


@pytest.mark.parametrize("slots,scheme", [(2, 4), (3, 4), (2, 3)])
def test_host_streamed_gamma(pkg, gold, slots, scheme):
    """Gamma kept in pinned host memory and streamed through `slots` device buffers: identical rows
    to the HBM-resident sweep, across several passes (the load sequence wraps around the chain)."""
    z = np.load(f"{gold}/c1b.npz")
    mps = O.load_npz_mps(z)
    st = to_state(pkg, mps)
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    res = pkg.GpuSampler(st, pol, pass_samples=256, scheme=pkg.Scheme(scheme))
    stm = pkg.GpuSampler(st, pol, pass_samples=256, host_stream_slots=slots, scheme=pkg.Scheme(scheme))
    for i in (0, 7, 15):
        assert np.array_equal(stm.decoded_gamma(i), res.decoded_gamma(i))
    a = res.sample(0, 1000, 7)
    stats = pkg.RunStats()
    b = stm.sample(0, 1000, 7, stats=stats)
    assert np.array_equal(a, b)
    assert np.array_equal(stm.sample(123, 77, 7), a[123:200])
    if scheme == 3:  # 3M streams Gr, Gi only (Gs re-formed on the device): 2/3 of the planes' bytes
        assert stm.state_bytes * 3 == res.state_bytes * 2


def test_host_streamed_gamma_precise(pkg, gold):
    """PRECISE mode with Gamma streamed from pinned host memory (hi and lo Gr, Gi planes copied, both
    sum planes re-formed on the device): identical rows and decoded tensors to the resident sweep."""
    z = np.load(f"{gold}/c1b.npz")
    mps = O.load_npz_mps(z)
    st = to_state(pkg, mps)
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    res = pkg.GpuSampler(st, pol, pass_samples=256, mode=pkg.Mode.PRECISE)
    stm = pkg.GpuSampler(st, pol, pass_samples=256, mode=pkg.Mode.PRECISE, host_stream_slots=2)
    for i in range(mps.num_sites):
        assert np.array_equal(stm.decoded_gamma(i), res.decoded_gamma(i))
    assert np.array_equal(stm.sample(0, 700, 7), res.sample(0, 700, 7))
    assert stm.state_bytes * 6 == res.state_bytes * 4


def test_mpsb_files_roundtrip(pkg, gold, tmp_path):
    """MPSB files written by the reference load into the GPU state (F64 and F16 storage), a GPU state
    saves to a file the reference loads back bit-exactly, and corrupt payloads raise IoError."""
    z = np.load(f"{gold}/c1.npz")
    mps = O.load_npz_mps(z)
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    base = pkg.GpuSampler(to_state(pkg, mps), pol)
    want = base.sample(0, 500, 7)
    f64 = str(tmp_path / "c1_f64.mpsb")
    O.ref_save_mps(mps, f64, O.F64)
    assert np.array_equal(pkg.GpuSampler.from_file(f64, pol).sample(0, 500, 7), want)
    f16 = str(tmp_path / "c1_f16.mpsb")
    O.ref_save_mps(mps, f16, O.F16)
    # c1's Gamma spans 1e-14..1e10: F16 storage overflows to inf, and like the reference at F64
    # (contract.cpp:117-119) the GPU path refuses the non-finite tensor
    with pytest.raises(pkg.NumericError):
        pkg.GpuSampler.from_file(f16, pol)
    mb = O.load_npz_mps(np.load(f"{gold}/c1b.npz"))
    O.ref_save_mps(mb, f16, O.F16)
    m16 = O.ref_load_mps(f16)  # the F16-rounded values the file holds
    a = pkg.GpuSampler.from_file(f16, pol)
    b = pkg.GpuSampler(to_state(pkg, m16), pol)
    for i in range(mps.num_sites):
        assert np.array_equal(a.decoded_gamma(i), b.decoded_gamma(i))
    assert np.array_equal(a.sample(0, 500, 7), b.sample(0, 500, 7))
    out = str(tmp_path / "ours.mpsb")
    base.save(out, pkg.Precision.F64)
    back = O.ref_load_mps(out)
    for i in range(mps.num_sites):
        assert np.array_equal(back.gammas[i], base.decoded_gamma(i))
        assert np.array_equal(back.lambdas[i], mps.lambdas[i])
    res = pkg.run_data_parallel(f64, pkg.BatchPlan(500), 1, pkg.SamplerOptions(policy=pol, seed=7))
    assert np.array_equal(res.batch.outcomes, want)
    res = pkg.run_serial(f64, pkg.BatchPlan(500), pkg.SamplerOptions(policy=pol, seed=7), from_storage=True)
    assert np.array_equal(res.batch.outcomes, want)
    raw = bytearray(open(f64, "rb").read())
    raw[-100] ^= 0x40  # flip a bit in the last site's payload
    bad = str(tmp_path / "bad.mpsb")
    open(bad, "wb").write(bytes(raw))
    with pytest.raises(pkg.IoError, match="checksum"):
        pkg.GpuSampler.from_file(bad, pol)


@pytest.mark.parametrize("storage,scheme,mode", [("F64", 3, "AUTO"), ("F32", 4, "AUTO"), ("F16", 3, "AUTO"),
                                                  ("F64", 4, "GRID")])
def test_mpsb_file_streamed_equals_resident(pkg, gold, tmp_path, storage, scheme, mode):
    """mpsg_create_from_file_streamed (the reference's SiteStream, mps_io.cpp:294-350, as a per-pass
    supply): the site payloads are re-read from storage, checksum-verified and compressed on the device
    every pass, and the samples, marginals and decoded Gamma equal the resident state built from the
    same file bit for bit -- over several passes (the load sequence wraps the chain) and several calls."""
    mb = O.load_npz_mps(np.load(f"{gold}/c1b.npz"))
    path = str(tmp_path / f"c1b_{storage}.mpsb")
    O.ref_save_mps(mb, path, getattr(O, storage))
    comp = pkg.Precision.F16 if mode == "GRID" else pkg.Precision.F64
    pol = pkg.PrecisionPolicy(compute=comp, scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    kw = dict(scheme=pkg.Scheme(scheme) if mode != "GRID" else pkg.Scheme.AUTO, pass_samples=256)
    res = pkg.GpuSampler.from_file(path, pol, **kw)
    st = pkg.GpuSampler.from_file(path, pol, streamed=True, host_stream_slots=2 if scheme == 4 else 0, **kw)
    assert pkg.sampler._lib.lib().mpsg_scheme(st._h) == pkg.sampler._lib.lib().mpsg_scheme(res._h)
    assert pkg.sampler._lib.lib().mpsg_mode(st._h) == pkg.sampler._lib.lib().mpsg_mode(res._h)
    for i in (0, 7, mb.num_sites - 1):
        assert np.array_equal(st.decoded_gamma(i), res.decoded_gamma(i)), i
    for first, n in ((0, 700), (3, 300)):  # 700 = three passes of 256 rows
        rows = st.sample(first, n, 7)
        assert np.array_equal(rows, res.sample(first, n, 7))
        assert np.array_equal(st.marginals(first, rows), res.marginals(first, rows))
    res.close()
    st.close()


def test_generated_precise_and_original_values(pkg):
    """A generated handle in MPSG_MODE_PRECISE (6 planes regenerated every pass) samples exactly like
    the resident PRECISE handle of the same chain, and mpsg_generated_site_values returns the chain's
    own (uncompressed) values -- the sites build_synthetic materialises for the resident handle."""
    from paper_2512_20064_b200.synthetic import build_synthetic
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    kw = dict(seed=5, policy=pol, mode=pkg.Mode.PRECISE, pass_samples=512)
    res, _, host = build_synthetic(10, 256, 4, keep_host=True, **kw)
    gen, _ = build_synthetic(10, 256, 4, generated=True, **kw)
    assert pkg.sampler._lib.lib().mpsg_mode(gen._h) == int(pkg.Mode.PRECISE)
    for i in range(10):
        assert np.array_equal(gen.original_gamma(i), host[i]), i
        assert np.array_equal(gen.decoded_gamma(i), res.decoded_gamma(i)), i
    rows = gen.sample(0, 1200, 7)
    assert np.array_equal(rows, res.sample(0, 1200, 7))
    assert np.array_equal(gen.marginals(0, rows[:64]), res.marginals(0, rows[:64]))
    res.close()
    gen.close()


def test_mpsb_file_streamed_two_devices(pkg, gold, tmp_path):
    """A storage-streamed handle driving two device contexts (here both on GPU 0), each with its own
    reader threads and slot ring over the same file, splits the samples and returns the resident
    handle's rows."""
    mb = O.load_npz_mps(np.load(f"{gold}/c1b.npz"))
    path = str(tmp_path / "c1b.mpsb")
    O.ref_save_mps(mb, path, O.F32)
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    res = pkg.GpuSampler.from_file(path, pol, pass_samples=256)
    st = pkg.GpuSampler.from_file(path, pol, devices=[0, 0], pass_samples=256, streamed=True)
    assert np.array_equal(st.sample(0, 1500, 11), res.sample(0, 1500, 11))
    res.close()
    st.close()


def test_mpsb_file_streamed_corrupt_payload(pkg, gold, tmp_path):
    """A payload whose checksum fails surfaces as IoError from the sampling call that reads it."""
    mb = O.load_npz_mps(np.load(f"{gold}/c1b.npz"))
    path = str(tmp_path / "c1b.mpsb")
    O.ref_save_mps(mb, path, O.F64)
    raw = bytearray(open(path, "rb").read())
    raw[-100] ^= 0x40  # a Gamma scalar of the last site
    open(path, "wb").write(bytes(raw))
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    st = pkg.GpuSampler.from_file(path, pol, streamed=True)  # header + Lambda only: accepted
    with pytest.raises(pkg.IoError, match="checksum"):
        st.sample(0, 64, 7)
    st.close()


def test_bond_schedule(pkg, gold):
    """sample_batch with a BondSchedule (sampler.cpp:173-176): the truncated chain, sampled on the GPU,
    matches the oracle on the same truncated (decoded) chain."""
    z = np.load(f"{gold}/c1b.npz")
    mps = O.load_npz_mps(z)
    chi = [1, 4, 16, 24, 32, 20, 32, 32, 12, 32, 32, 32, 32, 28, 16, 4, 1]
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    opts = pkg.SamplerOptions(policy=pol, seed=7, schedule=pkg.BondSchedule(chi, 32))
    got = pkg.sample_batch(to_state(pkg, mps), pkg.BatchPlan(1000), opts).outcomes
    trunc = O.ref_apply_schedule(mps, chi, 32)
    smp = pkg.GpuSampler(to_state(pkg, trunc), pol)
    assert np.array_equal(smp.sample(0, 1000, 7), got)
    ref_rows, ref_marg, _ = O.orc_sample_range(decoded_mps(smp, trunc), 0, 1000, 7, want_marginals=True)
    ndiff, explained = compare_strings(got, ref_rows, ref_marg, 7)
    assert ndiff == explained, (ndiff, explained)


def _synthetic(pkg, m, chi, d, **kw):
    from paper_2512_20064_b200.synthetic import build_synthetic
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    smp, lams = build_synthetic(m, chi, d, seed=11, policy=pol, **kw)
    return smp, lams, pol


@pytest.mark.parametrize("m,chi,d,n,scheme", [(10, 512, 6, 48, 3), (10, 512, 6, 48, 4), (10, 2048, 6, 12, 3),
                                              (10, 2048, 6, 12, 4)])
def test_parity_at_benchmark_bond_dims(pkg, m, chi, d, n, scheme):
    """Device-generated chains at the c2 / c3 bond dimensions (short M so the f64 oracle is quick):
    teacher-forced marginals within 1e-4 and identical strings (boundary draws excepted)."""
    smp, lams, _ = _synthetic(pkg, m, chi, d, scheme=scheme)
    dec = O.Mps(d, list(smp.bond_dims), [smp.decoded_gamma(i) for i in range(m)], list(lams))
    ref_rows, ref_marg, _ = O.orc_sample_range(dec, 0, n, 7, want_marginals=True)
    gpu_rows = smp.sample(0, n, 7)
    gm = smp.marginals(0, ref_rows)
    big = ref_marg >= 1e-3
    rel = np.abs(gm[big] - ref_marg[big]) / ref_marg[big]
    assert rel.max() < MARG_RTOL, rel.max()
    ndiff, explained = compare_strings(gpu_rows, ref_rows, ref_marg, 7)
    assert ndiff == explained, (ndiff, explained)


def test_invariants_at_chi2048(pkg):
    """Size-independent properties on a chi=2048, d=6 chain (c3 bond dimension): outcomes do not depend
    on the pass size, on host streaming, or on tensor-parallel sharding; site-0 frequencies follow the
    exact site-0 distribution (chi-square)."""
    from paper_2512_20064_b200.parallel import TensorParallelLocal
    m, chi, d = 16, 2048, 6
    a, lams, pol = _synthetic(pkg, m, chi, d, pass_samples=512)  # 3M (auto)
    rows = a.sample(0, 4096, 3)
    b, _, _ = _synthetic(pkg, m, chi, d, pass_samples=4096, host_stream_slots=2, scheme=3)
    assert np.array_equal(b.sample(0, 4096, 3), rows)
    # the 4M kernel on the same decoded tensor: only CDF-boundary draws may differ
    c, _, _ = _synthetic(pkg, m, chi, d, pass_samples=4096, scheme=4)
    assert (c.sample(0, 4096, 3) != rows).any(axis=1).sum() <= 4
    assert np.array_equal(a.sample(1000, 300, 3), rows[1000:1300])
    # exact site-0 distribution from the decoded tensor (sampler.cpp:83-90 with env = 1)
    g0 = a.decoded_gamma(0)[0]
    w = (lams[0][:, None] ** 2 * np.abs(g0) ** 2).sum(axis=0)
    p = w / w.sum()
    cnt = np.bincount(rows[:, 0], minlength=d)
    live = p * len(rows) > 5
    chi2 = (((cnt - p * len(rows)) ** 2) / (p * len(rows)))[live].sum()
    assert chi2 < 40.0, (chi2, cnt, p)
    # tensor-parallel (p2 = 2 ranks on this device) on a state built from the decoded tensors
    st = pkg.MpsState(m, d, list(a.bond_dims), [a.decoded_gamma(i) for i in range(m)], list(lams))
    tp = TensorParallelLocal(st, 2, policy=pol)
    one = pkg.GpuSampler(st, pol)
    t = tp.sample(0, 512, 3)
    assert np.array_equal(t[0], t[1])
    ref = one.sample(0, 512, 3)
    assert np.array_equal(t[0], ref)  # block-aligned shards: the unsharded K order
    tp.close()


def test_edge_decay_chain_golden(pkg, gold):
    """decay_chain (mps.cpp:183-196): the reference's own outcomes (F64, no scaling) reproduced; the
    GPU renormalises every site so nothing dies where F16-without-scaling would (decay.npz)."""
    z = np.load(f"{gold}/decay.npz")
    mps = O.load_npz_mps(z, "decay_")
    smp = pkg.GpuSampler(to_state(pkg, mps), pkg.PrecisionPolicy())
    rows = smp.sample(0, 200, 3)
    assert np.array_equal(rows, z["decay_f64_none"])
    assert int((rows[:, -1] == pkg.DEAD_OUTCOME).sum()) == 0


def test_edge_structural_dead_paths(pkg):
    """Outcome 1 at site 0 leads to an all-zero environment at site 1: those samples are dead
    (0xFF) from site 1 on (sampler.cpp:94-98), exactly as the oracle says."""
    g0 = np.zeros((1, 2, 2), complex)
    g0[0, 0, 0] = 1.0
    g0[0, 1, 1] = 0.8
    g1 = np.zeros((2, 2, 2), complex)  # row l=1 is zero: env [0, x] from outcome 1 dies here
    g1[0, :, :] = [[0.5, 0.2j], [0.3, 0.4]]
    g2 = np.zeros((2, 1, 2), complex)
    g2[:, 0, :] = [[1.0, 0.5], [0.25, 1.0]]
    mps = O.Mps(2, [1, 2, 2, 1], [g0, g1, g2])
    mps.lambdas = [np.array([0.8, 0.6]), np.array([0.9, 0.4359]), np.ones(1)]
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    smp = pkg.GpuSampler(to_state(pkg, mps), pol)
    dec = decoded_mps(smp, mps)
    ref, _ = O.orc_sample_range(dec, 0, 2000, 5)
    got = smp.sample(0, 2000, 5)
    assert np.array_equal(got, ref)
    dead = got[:, -1] == pkg.DEAD_OUTCOME
    assert 0 < dead.sum() < 2000
    assert (got[dead, 0] == 1).all() and (got[dead, 1:] == pkg.DEAD_OUTCOME).all()


def test_edge_small_odd_chains(pkg, gold):
    """d in {2,3,5,7}, chi 1..64, short chains (small.npz shapes): GPU == oracle on the decoded Gamma."""
    z = np.load(f"{gold}/small.npz")
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    for j in range(int(z["ncases"])):
        mps = O.load_npz_mps(z, f"c{j}_")
        smp = pkg.GpuSampler(to_state(pkg, mps), pol)
        seed = int(z[f"c{j}_seed"])
        ref, marg, _ = O.orc_sample_range(decoded_mps(smp, mps), 0, 300, seed, want_marginals=True)
        got = smp.sample(0, 300, seed)
        ndiff, explained = compare_strings(got, ref, marg, seed)
        assert ndiff == explained, (j, ndiff, explained)


def test_edge_phys_dim_one_and_huge_index(pkg):
    """d = 1 (every outcome 0) and a single sample at a global index near 2^64 (keyed RNG)."""
    g = [np.ones((1, 1, 1), complex) * 0.5 for _ in range(4)]
    mps = O.Mps(1, [1, 1, 1, 1, 1], g, [np.ones(1)] * 4)
    smp = pkg.GpuSampler(to_state(pkg, mps))
    assert (smp.sample(0, 10, 1) == 0).all()
    z = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "c1.npz"))
    m1 = O.load_npz_mps(z)
    s1 = pkg.GpuSampler(to_state(pkg, m1), pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX))
    first = 2**64 - 3
    got = s1.sample(first, 2, 7)
    ref, _ = O.orc_sample_range(decoded_mps(s1, m1), first, 2, 7)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("scaling", [0, 2])
def test_decay_trace_matches_reference(pkg, gold, scaling):
    """RunStats.decay_trace / decay_probe (sampler.cpp:149-153, 207-216): mean |env| per site before
    scaling, in the reference's own scaling, vs the compiled reference on the same (decoded) chains."""
    if not O.have_ref():
        pytest.skip("oracle/_ref not available")
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode(scaling))
    for name, prefix in (("c1b", ""), ("decay", "decay_")):
        mps = O.load_npz_mps(np.load(f"{gold}/{name}.npz"), prefix)
        smp = pkg.GpuSampler(to_state(pkg, mps), pol)
        dec = decoded_mps(smp, mps)
        want = O.RefState(dec).decay_probe(500, seed=1, scaling=scaling)
        got = np.array(pkg.decay_probe(to_state(pkg, dec), pol, 500, seed=1))
        np.testing.assert_allclose(got, want, rtol=2e-5, atol=0)


def test_multi_device_handle_threads(pkg, gold):
    """mpsg_create with several devices (one host thread + stream + replica each) splits the range
    contiguously; listing device 0 twice exercises that path on a single-GPU box."""
    z = np.load(f"{gold}/c1b.npz")
    st = to_state(pkg, O.load_npz_mps(z))
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    one = pkg.GpuSampler(st, pol).sample(0, 1000, 7)
    two = pkg.GpuSampler(st, pol, devices=[0, 0], pass_samples=256).sample(0, 1000, 7)
    assert np.array_equal(one, two)
    res = pkg.sample_batch(st, pkg.BatchPlan(1000), pkg.SamplerOptions(policy=pol, seed=7), devices=[0, 0])
    assert np.array_equal(res.outcomes, one)


# ---- GBS displacement site transform (SPEC.md gbs-ops, hook position sampler.cpp:143) ---------
def test_displacement_matrix_device_matches_oracle(pkg):
    rng = np.random.default_rng(2)
    for n in (1, 2, 4, 6, 10, 16):
        for _ in range(5):
            mu = complex(*rng.uniform(-1.2, 1.2, 2))
            # f64 on both sides; device vs host libm (exp, lgamma) differ in the last bits
            np.testing.assert_allclose(pkg.displacement_matrix(mu, n), O.orc_displacement(mu, n),
                                       rtol=1e-10, atol=1e-11)


@pytest.mark.parametrize("scheme", [3, 4])
def test_displaced_sampling_parity(pkg, gold, scheme):
    """Per-sample displacement D(mu[n, i]) between contraction and measurement: strings and
    teacher-forced marginals vs the oracle with the same mu (c1b, d = 4); mu = 0 reproduces the
    undisplaced sweep exactly."""
    z = np.load(f"{gold}/c1b.npz")
    mps = O.load_npz_mps(z)
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    smp = pkg.GpuSampler(to_state(pkg, mps), pol, scheme=pkg.Scheme(scheme), pass_samples=256)
    n, m = 1000, mps.num_sites
    zero = smp.sample(0, n, 7, mu=np.zeros((n, m), complex))
    assert np.array_equal(zero, smp.sample(0, n, 7))
    rng = np.random.default_rng(9)
    mu = 0.6 * (rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m)))
    dec = decoded_mps(smp, mps)
    ref_rows, ref_marg, _ = O.orc_sample_range(dec, 0, n, 7, want_marginals=True, mu=mu)
    gpu_rows = smp.sample(0, n, 7, mu=mu)
    assert (gpu_rows != zero).any()
    gm = smp.marginals(0, ref_rows, mu=mu)
    big = ref_marg >= 1e-3
    rel = np.abs(gm[big] - ref_marg[big]) / ref_marg[big]
    assert rel.max() < MARG_RTOL, rel.max()
    ndiff, explained = compare_strings(gpu_rows, ref_rows, ref_marg, 7)
    assert ndiff == explained, (ndiff, explained)
    # the reference-shaped API: SamplerOptions.site_transform = Displacement(mu)
    opts = pkg.SamplerOptions(policy=pol, seed=7, site_transform=pkg.Displacement(mu), scheme=pkg.Scheme(scheme))
    assert np.array_equal(pkg.sample_batch(to_state(pkg, mps), pkg.BatchPlan(n), opts).outcomes, gpu_rows)


def test_displaced_sampling_bench_dims_and_tp(pkg):
    """chi = 512, d = 6 device-generated chain with displacement: parity vs the oracle; the
    tensor-parallel sweep (p2 = 2, one device) agrees with the unsharded one."""
    from paper_2512_20064_b200.parallel import TensorParallelLocal
    smp, lams, pol = _synthetic(pkg, 8, 512, 6)
    m, n, d = 8, 48, 6
    rng = np.random.default_rng(3)
    mu = 0.5 * (rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m)))
    dec = O.Mps(d, list(smp.bond_dims), [smp.decoded_gamma(i) for i in range(m)], list(lams))
    ref_rows, ref_marg, _ = O.orc_sample_range(dec, 0, n, 7, want_marginals=True, mu=mu)
    gpu_rows = smp.sample(0, n, 7, mu=mu)
    gm = smp.marginals(0, ref_rows, mu=mu)
    big = ref_marg >= 1e-3
    assert (np.abs(gm[big] - ref_marg[big]) / ref_marg[big]).max() < MARG_RTOL
    ndiff, explained = compare_strings(gpu_rows, ref_rows, ref_marg, 7)
    assert ndiff == explained, (ndiff, explained)
    st = pkg.MpsState(m, d, list(dec.bond_dims), list(dec.gammas), list(dec.lambdas))
    tp = TensorParallelLocal(st, 2, policy=pol)
    t = tp.sample(0, n, 7, mu=mu)
    assert np.array_equal(t[0], t[1])
    # the sharded displacement runs as its own kernel (fused into the selection when unsharded)
    assert (t[0] != gpu_rows).any(axis=1).sum() <= 1
    tp.close()


def test_dynamic_bond_schedule_ragged_chain(pkg):
    """A device-generated chi = 512 chain truncated by dynamic_bond_schedule (ragged, non-monotone
    per-site GEMM shapes, padded K / N tiles): parity vs the oracle on the same truncated chain."""
    cfg = pkg.TruncationFilter(chi_max=512, eps_center=2e-2, edge_factor=4.0)
    smp, lams, _ = _synthetic(pkg, 10, 512, 6, schedule=cfg)
    b = smp.bond_dims
    assert max(b) < 512 and len(set(b[2:-2])) > 1
    dec = O.Mps(6, list(b), [smp.decoded_gamma(i) for i in range(10)], list(lams))
    ref_rows, ref_marg, _ = O.orc_sample_range(dec, 0, 64, 7, want_marginals=True)
    gpu_rows = smp.sample(0, 64, 7)
    gm = smp.marginals(0, ref_rows)
    big = ref_marg >= 1e-3
    assert (np.abs(gm[big] - ref_marg[big]) / ref_marg[big]).max() < MARG_RTOL
    ndiff, explained = compare_strings(gpu_rows, ref_rows, ref_marg, 7)
    assert ndiff == explained, (ndiff, explained)


@pytest.mark.parametrize("scheme", [3, 4])
def test_randomized_shapes(pkg, scheme):
    """Seeded fuzz over chain shapes: random M, d, ragged bonds (1..300, not capped), pass sizes and
    scaling modes; every chain must match the oracle on the decoded tensors (strings up to boundary
    draws, teacher-forced marginals within 1e-4)."""
    rng = np.random.default_rng(1234 + scheme)
    for case in range(16):
        m = int(rng.integers(2, 9))
        d = int(rng.integers(1, 13))
        bonds = [1] + [int(rng.integers(1, 301)) for _ in range(m - 1)] + [1]
        gam, lam = [], []
        for i in range(m):
            cl, cr = bonds[i], bonds[i + 1]
            g = (rng.standard_normal((cl, cr, d)) + 1j * rng.standard_normal((cl, cr, d))) / np.sqrt(cl * d)
            gam.append(g)
            l = np.sort(rng.uniform(0.05, 1.0, cr))[::-1]
            if case % 5 == 4 and cr > 2:
                l[cr // 2:] = 0.0  # zero-weight columns (Lambda_r = 0 is legal, mps.cpp:31-35)
            lam.append(l / np.linalg.norm(l))
        mps = O.Mps(d, bonds, gam, lam)
        scaling = [0, 2][case % 2]
        pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode(scaling))
        n = int(rng.integers(1, 400))
        smp = pkg.GpuSampler(to_state(pkg, mps), pol, scheme=pkg.Scheme(scheme),
                             pass_samples=int(rng.choice([128, 256, 1024])))
        dec = decoded_mps(smp, mps)
        seed = int(rng.integers(0, 2**63))
        ref_rows, ref_marg, _ = O.orc_sample_range(dec, 0, n, seed, scaling=scaling, want_marginals=True)
        got = smp.sample(0, n, seed)
        ndiff, explained = compare_strings(got, ref_rows, ref_marg, seed)
        assert ndiff == explained, (case, m, d, bonds, ndiff, explained)
        gm = smp.marginals(0, ref_rows)
        big = ref_marg >= 1e-3
        if big.any():
            rel = (np.abs(gm[big] - ref_marg[big]) / ref_marg[big]).max()
            assert rel < MARG_RTOL, (case, m, d, bonds, rel)
        smp.close()


@pytest.mark.parametrize("scheme", [3, 4])
def test_single_mode_within_reference_f16_envelope(pkg, gold, scheme):
    """SINGLE (one fp16 pass, compute = TF32 / F16 policies): its marginal error vs the f64 oracle stays
    within the error envelope of the reference's own F16 compute policy (the oracle's emulated-F16
    contraction, precision.cpp:23-50 / contract.cpp:53-81) on the same decoded chain."""
    z = np.load(f"{gold}/c1b.npz")
    mps = O.load_npz_mps(z)
    pol = pkg.PrecisionPolicy(compute=pkg.Precision.F16, scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    smp = pkg.GpuSampler(to_state(pkg, mps), pol, mode=pkg.Mode.SINGLE, scheme=pkg.Scheme(scheme))
    dec = decoded_mps(smp, mps)
    n = 500
    ref_rows, ref_marg, _ = O.orc_sample_range(dec, 0, n, 7, want_marginals=True)
    _, f16_marg, _ = O.orc_sample_range(dec, 0, n, 7, compute=O.F16, forced=ref_rows, want_marginals=True)
    gm = smp.marginals(0, ref_rows)
    big = ref_marg >= 1e-3
    err_gpu = (np.abs(gm[big] - ref_marg[big]) / ref_marg[big]).max()
    err_f16 = (np.abs(f16_marg[big] - ref_marg[big]) / ref_marg[big]).max()
    assert err_gpu <= max(2.0 * err_f16, 1e-3), (err_gpu, err_f16)


# GPU GRID vs the reference's own reduced policy: both round every operand onto the same grid
# (decoded Gamma == round_scalar bit for bit) and differ only in fp32 accumulation order (~1e-7 on a
# marginal), which now and then moves an environment entry across a rounding boundary of the 11-bit
# grid (one grid ulp, 2^-11; a few % of the marginals downstream of it, profiles/r2_grid/).
GRID_MEDIAN_RTOL = 1e-6   # typical marginal: fp32 accumulation noise (the policy itself: ~1e-4 vs F64)
GRID_FLIP_FRAC = 0.05     # marginals off by more than 1e-5 (downstream of a grid-ulp flip)


@pytest.mark.parametrize("case,compute,scaling", [("c1b", "F16", "PER_SAMPLE_MAX"), ("c1b", "F16", "NONE"),
                                                  ("c1b", "TF32", "PER_SAMPLE_MAX"), ("c1", "TF32", "PER_SAMPLE_MAX"),
                                                  ("c1", "TF32", "NONE")])
def test_grid_mode_reproduces_reference_reduced_policy(pkg, gold, case, compute, scaling):
    """MPSG_MODE_GRID (AUTO at compute = F16 / TF32) against the compiled reference running the same
    policy on the ORIGINAL chain (contract_block_reduced, contract.cpp:43-82: round_scalar on Gamma and
    on every environment, float accumulation): outcome strings identical except draws near a CDF
    boundary, marginals (teacher-forced on the reference's strings) within GRID_RTOL -- 20x inside the
    policy's own deviation from F64, which SINGLE only matches as an envelope."""
    if not O.have_ref():
        pytest.skip("oracle/_ref not available")
    z = np.load(f"{gold}/{case}.npz")
    mps = O.load_npz_mps(z)
    cp = {"F16": O.F16, "TF32": O.TF32}[compute]
    sc = {"PER_SAMPLE_MAX": O.SCALE_PER_SAMPLE, "NONE": O.SCALE_NONE}[scaling]
    pol = pkg.PrecisionPolicy(compute=getattr(pkg.Precision, compute), scaling=getattr(pkg.ScalingMode, scaling))
    smp = pkg.GpuSampler(to_state(pkg, mps), pol)
    assert pkg.sampler._lib.lib().mpsg_mode(smp._h) == int(pkg.Mode.GRID)
    n = 1000
    rs = O.RefState(mps)
    ref_rows = rs.sample_range(0, n, 7, compute=cp, scaling=sc, threads=8)
    ref_marg = rs.marginals_forced(ref_rows, compute=cp, scaling=sc)
    f64_marg = rs.marginals_forced(ref_rows, compute=O.F64, scaling=sc)
    rows = smp.sample(0, n, 7)
    gm = smp.marginals(0, ref_rows)
    live = (ref_marg >= 0).all(axis=2)  # sites where the reference sample is alive
    big = (ref_marg >= 1e-3) & live[:, :, None]
    e = np.abs(gm[big] - ref_marg[big]) / ref_marg[big]
    f = np.abs(f64_marg[big] - ref_marg[big]) / f64_marg[big]
    print(f"{case} {compute} {scaling}: GPU grid vs reference policy median {np.median(e):.2e} max {e.max():.2e} "
          f"(>1e-5: {(e > 1e-5).mean():.3f}); policy vs F64 median {np.median(f):.2e} max {f.max():.2e}")
    if scaling == "PER_SAMPLE_MAX":
        assert np.median(e) < GRID_MEDIAN_RTOL and np.median(e) < np.median(f) / 100
        assert (e > 1e-5).mean() < GRID_FLIP_FRAC
        assert e.max() < 0.5 * f.max()
    else:  # unscaled environments decay into coarser binades (F16: subnormals): flips weigh more
        assert np.median(e) < np.median(f) / 20
        assert e.max() < f.max()
    # sites 0, 1 see identical operands (site 0's env is 1, site 1's is site 0's rounded row)
    b01 = big[:, :2, :]
    e01 = np.abs(gm[:, :2, :][b01] - ref_marg[:, :2, :][b01]) / ref_marg[:, :2, :][b01]
    assert e01.max() < 1e-6, e01.max()
    # the decoded Gamma is round_scalar(Gamma) component-wise, bit for bit (precision.cpp:23-50)
    rnd = np.vectorize(lambda x: O.ref().ref_round_scalar(float(x), cp))
    for i in (0, mps.num_sites // 2):
        assert np.array_equal(smp.decoded_gamma(i), rnd(mps.gammas[i].real) + 1j * rnd(mps.gammas[i].imag))
    # strings: a differing string must have its first difference at a draw within 1e-4 of the
    # reference policy's CDF boundary (the grid-ulp flips above move a CDF by ~1e-5)
    ndiff, explained = compare_strings(rows, ref_rows, ref_marg, 7, eps=1e-4)
    assert ndiff == explained and ndiff <= n // 50, (ndiff, explained)
    smp.close()


def test_grid_mode_decay_chain_golden(pkg, gold):
    """decay_chain (mps.cpp:183-196) under the reference's F16 policy (goldens from the compiled
    reference): without scaling the F16 environment underflows and every sample dies at site 8,
    with PerSampleMax none does -- GRID reproduces both outcome matrices, deaths included."""
    z = np.load(f"{gold}/decay.npz")
    mps = O.load_npz_mps(z, "decay_")
    for key, sc in (("decay_f16_none", pkg.ScalingMode.NONE), ("decay_f16_psm", pkg.ScalingMode.PER_SAMPLE_MAX)):
        pol = pkg.PrecisionPolicy(compute=pkg.Precision.F16, scaling=sc)
        smp = pkg.GpuSampler(to_state(pkg, mps), pol)
        rows = smp.sample(0, 200, 3)
        assert np.array_equal(rows, z[key]), (key, int((rows != z[key]).any(axis=1).sum()))
        smp.close()


def test_grid_mode_f16_overflow_is_numeric_error(pkg, gold):
    """c1's Gamma reaches 1e10: on the F16 grid it overflows (round_scalar -> inf, precision.cpp:46-47);
    the reference then propagates inf / NaN, GRID refuses the state with NumericError."""
    z = np.load(f"{gold}/c1.npz")
    mps = O.load_npz_mps(z)
    pol = pkg.PrecisionPolicy(compute=pkg.Precision.F16, scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    with pytest.raises(pkg.NumericError):
        pkg.GpuSampler(to_state(pkg, mps), pol)
    smp = pkg.GpuSampler(to_state(pkg, mps), pol, mode=pkg.Mode.SINGLE)  # SINGLE keeps its scaled format
    assert smp.sample(0, 8, 7).shape == (8, mps.num_sites)
    smp.close()


@pytest.mark.parametrize("scheme", [3, 4])
def test_c3_shape_parity_vs_reference_f32_envelope(pkg, scheme):
    """The c3 bond dimension over a 20-site chain (15 sites at chi = 2048), against the compiled
    reference itself (threaded): outcome strings identical (boundary draws excepted); interior-site
    marginals within 1e-4; right-edge sites (chiR < chiL), where every fp32-class contraction
    amplifies the environment's accumulated rounding through the cancellation of the narrowing bonds,
    within 10x the reference's own F32 policy on the same strings."""
    if not O.have_ref():
        pytest.skip("oracle/_ref not available")
    from concurrent.futures import ThreadPoolExecutor
    m, chi, d, n = 20, 2048, 6, 128
    smp, lams, _ = _synthetic(pkg, m, chi, d, scheme=scheme)
    dec = O.Mps(d, list(smp.bond_dims), [smp.decoded_gamma(i) for i in range(m)], list(lams))
    rs = O.RefState(dec)
    rows = rs.sample_range(0, n, 7, threads=16)
    chunks = [c for c in np.array_split(np.arange(n), 16) if len(c)]
    with ThreadPoolExecutor(16) as ex:
        ref = np.concatenate(list(ex.map(lambda idx: rs.marginals_forced(rows[idx]), chunks)))
        f32 = np.concatenate(list(ex.map(lambda idx: rs.marginals_forced(rows[idx], compute=O.F32), chunks)))
    got = smp.sample(0, n, 7)
    ndiff, explained = compare_strings(got, rows, ref, 7)
    assert ndiff == explained, (ndiff, explained)
    gm = smp.marginals(0, rows)
    b = list(smp.bond_dims)
    big = ref >= 1e-3

    def worst(mg, sites):
        sel = big[:, sites, :]
        return (np.abs(mg[:, sites, :] - ref[:, sites, :])[sel] / ref[:, sites, :][sel]).max()
    inner = [i for i in range(m) if b[i] == chi and b[i + 1] == chi]
    redge = [i for i in range(m) if b[i + 1] < b[i]]
    assert worst(gm, inner) < MARG_RTOL
    assert worst(gm, redge) < max(MARG_RTOL, 10.0 * worst(f32, redge)), (worst(gm, redge), worst(f32, redge))


def test_precise_mode_vs_original_mps(pkg, gold):
    """MPSG_MODE_PRECISE (Gamma hi + lo planes): the decoded tensor matches the caller's f64 Gamma to
    ~2^-23, so the GPU agrees with the reference run on the *original* MPS (not the decoded one):
    marginals within 1e-4 and identical strings; the default format (fp16 Gamma, 2^-12) does not
    reach that against the original on c1b."""
    z = np.load(f"{gold}/c1b.npz")
    mps = O.load_npz_mps(z)
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    smp = pkg.GpuSampler(to_state(pkg, mps), pol, mode=pkg.Mode.PRECISE)
    worst = 0.0
    for i in range(mps.num_sites):
        g, dg = mps.gammas[i], smp.decoded_gamma(i)
        colmax = np.maximum(np.abs(g.real), np.abs(g.imag)).max(axis=0, keepdims=True)
        err = np.maximum(np.abs(g.real - dg.real), np.abs(g.imag - dg.imag))
        worst = max(worst, float((err / np.where(colmax > 0, colmax, 1)).max()))
    print("precise decode: max |err| / column max", worst)
    assert worst < 2.0 ** -16, worst
    n = 1000
    ref_rows, ref_marg, _ = O.orc_sample_range(mps, 0, n, 7, want_marginals=True)  # the ORIGINAL chain
    got = smp.sample(0, n, 7)
    ndiff, explained = compare_strings(got, ref_rows, ref_marg, 7)
    assert ndiff == explained, (ndiff, explained)
    gm = smp.marginals(0, ref_rows)
    big = ref_marg >= 1e-3
    rel = (np.abs(gm[big] - ref_marg[big]) / ref_marg[big]).max()
    print("precise vs original: max marginal rel err", rel)
    assert rel < MARG_RTOL, rel
    # the default (fp16 Gamma) handle, same comparison against the original chain, for contrast
    dflt = pkg.GpuSampler(to_state(pkg, mps), pol, mode=pkg.Mode.SPLIT)
    rel_d = (np.abs(dflt.marginals(0, ref_rows)[big] - ref_marg[big]) / ref_marg[big]).max()
    print("default (fp16 Gamma) vs original: max marginal rel err", rel_d)
    assert rel_d > rel


def test_tensor_parallel_at_c4_bond_dimension(pkg):
    """The c4 shape (chi = 1e4, d = 4; three sites at the full bond) built directly as two column-
    sharded ranks (device-generated, same seed) on this GPU with the in-process exchange and two
    pipeline lanes: both ranks produce identical rows, equal to the unsharded sampler's except draws
    at a CDF boundary, and their marginals agree with it to F32-class accuracy."""
    import threading
    from paper_2512_20064_b200.synthetic import build_synthetic
    m, chi, d, n = 16, 10000, 4, 1024
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    one, _ = build_synthetic(m, chi, d, seed=3, policy=pol, pass_samples=n)
    assert max(one.bond_dims) == chi
    ranks = [build_synthetic(m, chi, d, seed=3, policy=pol, pass_samples=n, tp_size=2, tp_rank=r)[0]
             for r in range(2)]
    pkg.sampler.connect_local(ranks)
    out = [None, None]
    marg = [None, None]
    ref_rows = one.sample(0, n, 9)

    def run(r):
        out[r] = ranks[r].sample(0, n, 9)
        marg[r] = ranks[r].marginals(0, ref_rows)
    ts = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert np.array_equal(out[0], out[1])
    assert np.array_equal(out[0], ref_rows)  # block-aligned shards: the unsharded K order
    gm = one.marginals(0, ref_rows)
    big = gm >= 1e-3
    assert (np.abs(marg[0][big] - gm[big]) / gm[big]).max() < TP_RTOL
    for s in ranks + [one]:
        s.close()


def test_sample_device_rows_and_stats(pkg, gold):
    """mpsg_sample_device (rows written to device memory, the bench's device-timed path) equals the
    host-rows call; RunStats carries the reference's contraction_macs formula (contract.cpp:97-100)."""
    import torch
    z = np.load(f"{gold}/c1b.npz")
    mps = O.load_npz_mps(z)
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    smp = pkg.GpuSampler(to_state(pkg, mps), pol, pass_samples=256)
    st = pkg.RunStats()
    host = smp.sample(5, 700, 7, stats=st)
    dev = torch.empty((700, mps.num_sites), dtype=torch.uint8, device="cuda")
    smp.sample_device(5, 700, 7, dev.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(dev.cpu().numpy(), host)
    b = mps.bond_dims
    assert st.contraction_macs == 700 * sum(b[i] * b[i + 1] * mps.phys_dim for i in range(mps.num_sites))
    assert st.issued_mma_flops > 0 and st.d2h_bytes == 700 * mps.num_sites


def test_runstats_counters_match_reference(pkg, gold):
    """RunStats / FlopCounters (sampler.hpp:46-54, contract.hpp:12-25): contraction MACs over every
    sample, measure's weight MACs and pipeline ops over the live ones only, dead samples — equal to
    the reference's own counters, on c1b and on a chain where samples die (structural zeros)."""
    if not O.have_ref():
        pytest.skip("oracle/_ref not available")
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    g0 = np.zeros((1, 2, 2), complex)
    g0[0, 0, 0], g0[0, 1, 1] = 1.0, 0.8
    g1 = np.zeros((2, 2, 2), complex)
    g1[0, :, :] = [[0.5, 0.2j], [0.3, 0.4]]
    g2 = np.zeros((2, 1, 2), complex)
    g2[:, 0, :] = [[1.0, 0.5], [0.25, 1.0]]
    dying = O.Mps(2, [1, 2, 2, 1], [g0, g1, g2], [np.array([0.8, 0.6]), np.array([0.9, 0.4359]), np.ones(1)])
    for mps in (O.load_npz_mps(np.load(f"{gold}/c1b.npz")), dying):
        smp = pkg.GpuSampler(to_state(pkg, mps), pol)
        dec = decoded_mps(smp, mps)
        n = 777
        ref_rows, want, dead = O.RefState(dec).sample_batch_stats(n, 7)
        st = pkg.RunStats()
        rows = smp.sample(0, n, 7, stats=st)
        assert np.array_equal(rows, ref_rows)
        assert st.contraction_macs == want["contraction_macs"]
        assert st.measure_weight_macs == want["measure_weight_macs"]
        assert st.measure_pipeline_ops == want["measure_pipeline_ops"]
        assert st.dead_samples == dead
        smp.close()


def _dead_chain():
    g0 = np.zeros((1, 2, 2), complex)
    g0[0, 0, 0] = 1.0
    g0[0, 1, 1] = 0.8
    g1 = np.zeros((2, 2, 2), complex)
    g1[0, :, :] = [[0.5, 0.2j], [0.3, 0.4]]
    g2 = np.zeros((2, 1, 2), complex)
    g2[:, 0, :] = [[1.0, 0.5], [0.25, 1.0]]
    mps = O.Mps(2, [1, 2, 2, 1], [g0, g1, g2])
    mps.lambdas = [np.array([0.8, 0.6]), np.array([0.9, 0.4359]), np.ones(1)]
    return mps


@pytest.mark.parametrize("case", ["c1", "c1b", "dead", "chi512_passes", "chi2048", "precise", "single",
                                  "stream"])
def test_slice_recompute_identical_to_temp(pkg, gold, case):
    """The slice-recompute path (weights-only contraction, rows bucketed by outcome, 1/d slice GEMM
    writing the next environment) produces exactly the temp path's outcome strings and counters:
    same arithmetic per element, only the row order inside the device changes.  Covers forced
    recompute at every site, dead samples, several passes with a ragged last pass, PRECISE, SINGLE
    and a host-streamed state."""
    from paper_2512_20064_b200.synthetic import build_synthetic
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    n, seed = 1000, 7

    def make(slice_):
        if case in ("c1", "c1b", "dead", "precise", "single"):
            mps = _dead_chain() if case == "dead" else O.load_npz_mps(np.load(f"{gold}/{'c1b' if case == 'c1b' else 'c1'}.npz"))
            mode = {"precise": pkg.Mode.PRECISE, "single": pkg.Mode.SINGLE}.get(case, pkg.Mode.AUTO)
            return pkg.GpuSampler(to_state(pkg, mps), pol, mode=mode, pass_samples=384, slice=slice_)
        chi, m = (512, 12) if case != "chi2048" else (2048, 8)
        kw = dict(pass_samples=384) if case == "chi512_passes" else {}
        if case == "stream":
            chi, m, kw = 512, 10, dict(host_stream_slots=2)
        smp, _ = build_synthetic(m, chi, 6, seed=11, policy=pol, slice=int(slice_), **kw)
        return smp

    temp = make(pkg.Slice.TEMP)
    st_t = pkg.RunStats()
    want = temp.sample(0, n, seed, stats=st_t)
    temp.close()
    for sl in (pkg.Slice.RECOMPUTE,):
        smp = make(sl)
        st = pkg.RunStats()
        got = smp.sample(0, n, seed, stats=st)
        assert np.array_equal(got, want), (case, sl, int((got != want).any(axis=1).sum()))
        assert st.contraction_macs == st_t.contraction_macs and st.dead_samples == st_t.dead_samples
        assert st.measure_weight_macs == st_t.measure_weight_macs
        assert np.array_equal(smp.sample(217, 301, seed), want[217:518])
        smp.close()
    if case == "dead":
        assert 0 < (want[:, -1] == pkg.DEAD_OUTCOME).sum() < n


def test_host_streamed_two_lanes_displaced(pkg):
    """chi = 1024 (two pipeline lanes) with Gamma streamed through 2 device slots, plain and with the
    fused displacement selection (which reads the slot's column info): identical rows to the
    HBM-resident sweep over several passes."""
    from paper_2512_20064_b200.synthetic import build_synthetic
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    m, chi, d, n = 8, 1024, 4, 1200
    res, _ = build_synthetic(m, chi, d, seed=5, policy=pol, pass_samples=512)
    stm, _ = build_synthetic(m, chi, d, seed=5, policy=pol, pass_samples=512, host_stream_slots=2)
    rng = np.random.default_rng(9)
    mu = 0.4 * (rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m)))
    assert np.array_equal(stm.sample(0, n, 7), res.sample(0, n, 7))
    assert np.array_equal(stm.sample(0, n, 7, mu=mu), res.sample(0, n, 7, mu=mu))
    stm.close()
    res.close()


# ---- round 2: boundary-draw accounting, full-length chains, per-device state, boundary checks ----
def test_near_boundary_counter_matches_reference_path(pkg, gold):
    """The device counter of draws within 1e-6 of an interior CDF boundary (mpsg_stats.
    near_boundary_draws) against the reference's own path (oracle.RefSiteSweep on the decoded c1
    chain): 1e6 samples x 16 sites give ~100 such draws.  Every differing outcome string is
    explained by a near-boundary draw at its first differing site."""
    if not O.have_ref():
        pytest.skip("oracle/_ref not available")
    z = np.load(f"{gold}/c1.npz")
    mps = O.load_npz_mps(z)
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    smp = pkg.GpuSampler(to_state(pkg, mps), pol)
    dec = decoded_mps(smp, mps)
    n, seed = 1_000_000, 7
    st = pkg.RunStats()
    got = smp.sample(0, n, seed, stats=st)
    sw = O.RefSiteSweep(0, n, seed, threads=16)
    ref_rows = np.empty_like(got)
    near = np.zeros(got.shape, bool)
    for i in range(mps.num_sites):
        o, _, nb = sw.site(i, dec.gammas[i], dec.lambdas[i])
        ref_rows[:, i], near[:, i] = o, nb
    diff = np.nonzero((got != ref_rows).any(axis=1))[0]
    for s in diff:
        i = int(np.argmax(got[s] != ref_rows[s]))
        assert near[s, i], (s, i)
    ref_near = int(near.sum())
    assert ref_near >= 20  # the statistic is informative at this size
    # the device counts along its own path; paths agree except after the (rare) boundary flips
    assert abs(int(st.near_boundary_draws) - ref_near) <= 2 + 16 * len(diff), (st.near_boundary_draws, ref_near)


def test_full_c2_chain_parity(pkg):
    """The full benchmark c2 chain (M = 256, chi = 512, d = 6, build_synthetic seed 42) at reduced N
    against the reference itself, site-streamed (tests/parity_full.py): strings identical except
    near-boundary draws; interior and left-edge marginals within 1e-4; the right edge within the
    pinned bound RIGHT_EDGE_RTOL (the narrowing bonds amplify the environment's
    accumulated fp32-class rounding)."""
    if not O.have_ref():
        pytest.skip("oracle/_ref not available")
    import parity_full
    r = parity_full.run("c2", 48, threads=16, f32=True, log=lambda s: None)
    assert r["unexplained_differences"] == 0, r["differences"]
    assert r["max_rel_err_interior_sites"] < MARG_RTOL, r["max_rel_err_interior_sites"]
    assert r["max_rel_err_left_edge_sites"] < MARG_RTOL, r["max_rel_err_left_edge_sites"]
    assert r["max_rel_err_right_edge_sites"] < RIGHT_EDGE_RTOL, r["max_rel_err_right_edge_sites"]
    assert r["contraction_macs_gpu"] == r["contraction_macs_ref"]


def test_multi_device_handle_two_gpus(pkg, gold):
    """A handle over two distinct devices: per-device kernel attributes (dynamic shared memory
    opt-in, cluster occupancy) and the displacement factorial table must be set up on each device.
    Rows (plain and displaced) equal the single-device ones.  Needs >= 2 GPUs."""
    if pkg.sampler._lib.lib().mpsg_device_count() < 2:
        pytest.skip("needs two B200s")
    z = np.load(f"{gold}/c1b.npz")
    st = to_state(pkg, O.load_npz_mps(z))
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    mu = (np.random.default_rng(3).normal(size=(2000, st.num_sites)) * 0.3).astype(np.complex128)
    one = pkg.GpuSampler(st, pol)
    two = pkg.GpuSampler(st, pol, devices=[0, 1], pass_samples=256)
    assert np.array_equal(one.sample(0, 2000, 7), two.sample(0, 2000, 7))
    assert np.array_equal(one.sample(0, 2000, 7, mu=mu), two.sample(0, 2000, 7, mu=mu))
    # the second device alone (its own attribute / table setup)
    three = pkg.GpuSampler(st, pol, devices=[1])
    assert np.array_equal(one.sample(0, 2000, 7, mu=mu), three.sample(0, 2000, 7, mu=mu))


def test_boundary_input_validation(pkg, gold, tmp_path):
    """Teacher-forced outcomes must be < d or 0xFF; a site cannot be set again after the next one;
    a tensor-parallel handle cannot be saved as an MPSB file (it holds one column shard)."""
    import ctypes as C
    from paper_2512_20064_b200 import _lib
    from paper_2512_20064_b200.parallel import TensorParallelLocal
    z = np.load(f"{gold}/c1.npz")
    mps = O.load_npz_mps(z)
    st = to_state(pkg, mps)
    smp = pkg.GpuSampler(st)
    forced = np.zeros((4, mps.num_sites), np.uint8)
    forced[2, 5] = mps.phys_dim  # out of range
    with pytest.raises(pkg.ConfigError):
        smp.marginals(0, forced)
    forced[2, 5] = 0xFF
    smp.marginals(0, forced)
    # builder: re-setting site 0 after site 1
    L = _lib.lib()
    h = C.c_void_p()
    bd = (C.c_uint64 * (mps.num_sites + 1))(*mps.bond_dims)
    assert L.mpsg_builder_begin(mps.num_sites, mps.phys_dim, bd, None, None, None, 0, C.byref(h)) == 0
    g = [np.ascontiguousarray(x, np.complex128) for x in mps.gammas]
    lam = [np.ascontiguousarray(x, np.float64) for x in mps.lambdas]
    for i in (0, 1):
        assert L.mpsg_builder_set_site(h, i, g[i].ctypes.data_as(_lib._pd), 0, 0, lam[i].ctypes.data_as(_lib._pd)) == 0
    assert L.mpsg_builder_set_site(h, 0, g[0].ctypes.data_as(_lib._pd), 0, 0, lam[0].ctypes.data_as(_lib._pd)) == 2
    L.mpsg_destroy(h)
    tp = TensorParallelLocal(st, 2)
    with pytest.raises(pkg.ConfigError):
        tp.ranks[0].save(str(tmp_path / "x.mpsb"))
    tp.close()


# ---- generated supply: synthetic chains regenerated on the device every pass -----------------
@pytest.mark.parametrize("m,chi,d,scheme,pass_samples,sched", [
    (12, 256, 4, 3, 0, None), (10, 512, 6, 4, 0, None), (8, 1024, 4, 3, 1024, None),
    (14, 256, 4, 3, 0, 1e-3)])
def test_generated_supply_equals_resident_chain(pkg, m, chi, d, scheme, pass_samples, sched):
    """A generated handle (base isometries + per-site spectra; every site regenerated and compressed
    on the device into the slot ring on every pass) holds exactly the chain build_synthetic
    materialises: identical decoded Gamma, identical rows (several passes, two lanes at chi = 1024,
    ragged dynamic bonds) and identical RunStats counters."""
    from paper_2512_20064_b200.synthetic import build_synthetic
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    schedule = (pkg.TruncationFilter(chi_max=chi, eps_center=sched, edge_factor=100.0) if sched else None)
    kw = dict(seed=13, policy=pol, scheme=scheme, pass_samples=pass_samples, schedule=schedule)
    res, lams = build_synthetic(m, chi, d, **kw)
    gen, lams2 = build_synthetic(m, chi, d, generated=True, **kw)
    assert res.bond_dims == gen.bond_dims
    for i in range(m):
        assert np.array_equal(res.decoded_gamma(i), gen.decoded_gamma(i)), i
    n = 3000
    st1, st2 = pkg.RunStats(), pkg.RunStats()
    a = res.sample(0, n, 7, stats=st1)
    b = gen.sample(0, n, 7, stats=st2)
    assert np.array_equal(a, b)
    assert st1.contraction_macs == st2.contraction_macs and st1.measure_weight_macs == st2.measure_weight_macs
    assert np.array_equal(gen.sample(0, n, 7), b)  # second call: the ring restarts cleanly
    mg = gen.marginals(0, a[:64])
    np.testing.assert_array_equal(mg, res.marginals(0, a[:64]))
    # the generators (a few chi x d chi complex64 bases) undercut the resident planes once the chain
    # holds more full-chi sites than it has bases (c4: 11 GB of bases for a 13-20 TB chain)
    if sum(1 for i in range(m) if res.bond_dims[i] == chi and res.bond_dims[i + 1] == chi) >= 8:
        assert gen.state_bytes < res.state_bytes


def test_generated_supply_parity_vs_reference(pkg):
    """The regenerated chain against the reference on its decoded tensors (c3 bond dimension)."""
    if not O.have_ref():
        pytest.skip("oracle/_ref not available")
    from paper_2512_20064_b200.synthetic import build_synthetic
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    m, chi, d, n = 10, 2048, 6, 16
    smp, lams = build_synthetic(m, chi, d, seed=3, policy=pol, generated=True)
    dec = O.Mps(d, list(smp.bond_dims), [smp.decoded_gamma(i) for i in range(m)], list(lams))
    ref_rows, ref_marg, _ = O.orc_sample_range(dec, 0, n, 7, want_marginals=True)
    got = smp.sample(0, n, 7)
    ndiff, explained = compare_strings(got, ref_rows, ref_marg, 7)
    assert ndiff == explained
    gm = smp.marginals(0, ref_rows)
    big = ref_marg >= 1e-3
    assert (np.abs(gm[big] - ref_marg[big]) / ref_marg[big]).max() < MARG_RTOL


def test_generated_supply_rejects_nonfinite(pkg):
    """A zero in Lambda_i makes Gamma_i infinite (1 / Lambda): the regenerated site fails the
    compression's finiteness check and the call raises NumericError (contract.cpp:117-119)."""
    import ctypes as C
    from paper_2512_20064_b200 import _lib
    import torch
    L = _lib.lib()
    bonds = [1, 4, 1]
    h = C.c_void_p()
    bd = (C.c_uint64 * 3)(*bonds)
    assert L.mpsg_generated_begin(2, 4, bd, None, None, None, 0, 5, C.byref(h)) == 0
    b0 = torch.eye(1, 16, dtype=torch.complex64, device="cuda")
    b1 = torch.zeros(4, 4, dtype=torch.complex64, device="cuda")
    b1[:, 0] = 1.0
    ids = []
    for t in (b0, b1):
        bid = C.c_int()
        assert L.mpsg_generated_add_base(h, C.c_void_p(t.data_ptr()), 1, t.shape[0], t.shape[1], C.byref(bid)) == 0
        ids.append(bid.value)
    lam0 = np.array([1.0, 0.5, 0.25, 0.0])
    lam1 = np.ones(1)
    assert L.mpsg_generated_set_site(h, 0, ids[0], lam0.ctypes.data_as(_lib._pd)) == 0
    assert L.mpsg_generated_set_site(h, 1, ids[1], lam1.ctypes.data_as(_lib._pd)) == 0
    assert L.mpsg_builder_finish(h) == 0
    rows = np.empty((8, 2), np.uint8)
    assert L.mpsg_sample(h, 7, 0, 8, rows.ctypes.data_as(_lib._pu8), None) == 3  # MPSG_ERR_NUMERIC
    L.mpsg_destroy(h)


@pytest.mark.parametrize("scheme", [3, 4])
def test_nccl_one_rank_group_exchange(pkg, gold, scheme):
    """The tensor-parallel data plane through NCCL on one GPU: a one-rank group (tp_size 1 connected
    with mpsg_tp_connect_nccl) runs the partial-weight all-gather, the strided environment all-gather
    (grouped ncclBroadcast of the re / im planes; 3M re-forms its s planes after it) and the lane-1
    communicator split -- and samples what the plain handle samples (the exchanged partials are
    rounded to fp32, so only a draw within ~1e-7 of a boundary could differ)."""
    z = np.load(f"{gold}/c1b.npz")
    mps = O.load_npz_mps(z)
    st = to_state(pkg, mps)
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    plain = pkg.GpuSampler(st, pol, scheme=scheme).sample(0, 4000, 7)
    smp = pkg.GpuSampler(st, pol, scheme=scheme, pass_samples=1024)
    smp.connect_nccl(pkg.sampler.nccl_unique_id())
    got = smp.sample(0, 4000, 7)
    assert (got != plain).any(axis=1).sum() <= 1
    dec = decoded_mps(smp, mps)
    ref_rows, ref_marg, _ = O.orc_sample_range(dec, 0, 1000, 7, want_marginals=True)
    gm = smp.marginals(0, ref_rows)
    big = ref_marg >= 1e-3
    assert (np.abs(gm[big] - ref_marg[big]) / ref_marg[big]).max() < MARG_RTOL
    smp.close()


def test_nccl_one_rank_group_generated_chi1024(pkg):
    """Same at chi = 1024 with two pipeline lanes (lane 1's communicator split from lane 0's) over a
    generated (regenerated-per-pass) chain."""
    from paper_2512_20064_b200.synthetic import build_synthetic
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    a, _ = build_synthetic(8, 1024, 4, seed=5, policy=pol, generated=True, pass_samples=2048)
    b, _ = build_synthetic(8, 1024, 4, seed=5, policy=pol, generated=True, pass_samples=2048)
    b.connect_nccl(pkg.sampler.nccl_unique_id())
    x, y = a.sample(0, 4096, 7), b.sample(0, 4096, 7)
    assert (x != y).any(axis=1).sum() <= 1


# ---- multi-rank paths through libmpsg (gloo process group; ranks share the one GPU) --------------
def _dp_gpu_worker(rank, world, port, gold, q):
    import os
    import torch.distributed as dist
    import paper_2512_20064_b200 as P
    from paper_2512_20064_b200.parallel import run_data_parallel
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    z = np.load(os.path.join(gold, "c1.npz"))
    mps = O.load_npz_mps(z)
    st = P.MpsState(mps.num_sites, mps.phys_dim, list(mps.bond_dims), list(mps.gammas), list(mps.lambdas))
    smp = P.GpuSampler(st, P.PrecisionPolicy(scaling=P.ScalingMode.PER_SAMPLE_MAX), mode=P.Mode.SPLIT)
    out = run_data_parallel(smp.sample, 0, 5000, 7, mps.num_sites)
    if rank == 0:
        q.put(out)
    smp.close()
    dist.destroy_process_group()


def test_data_parallel_two_ranks_libmpsg(pkg, gold):
    """parallel.run_data_parallel with two processes, each sampling its share on the GPU through
    libmpsg (gloo for the final gather): the merged rows equal one process's sweep."""
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_dp_gpu_worker, args=(r, 2, port, gold, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = q.get(timeout=300)
    for p in ps:
        p.join(120)
    assert all(p.exitcode == 0 for p in ps)
    z = np.load(f"{gold}/c1.npz")
    st = to_state(pkg, O.load_npz_mps(z))
    one = pkg.GpuSampler(st, pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX),
                         mode=pkg.Mode.SPLIT).sample(0, 5000, 7)
    assert np.array_equal(got, one)


def test_torchrun_bench_two_ranks_shared_device():
    """bench.py under torchrun with two ranks (MPSG_BENCH_SHARE_DEVICE=1: both on GPU 0, gloo):
    whole-job value over both ranks, max-over-ranks timing, one JSON line from rank 0; the
    reference arm prints from rank 0 only."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MPSG_BENCH_SHARE_DEVICE="1")
    def cmd(port, *extra):
        return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(root, "bench.py"),
                "--gpus", "2", "--config", "c2", "--steps", "2", "--warmup", "3", *extra]
    r = subprocess.run(cmd(29517, "--no-cpu-baseline", "--e2e", "resident", "--e2e-steps", "1"),
                       capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["parallelism"] == "dp2"
    assert d["gpu_launches"] > 0 and d["e2e"]["value"] > 0
    r = subprocess.run(cmd(29518, "--impl", "reference", "--ref-seconds", "1"),
                       capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1 and json.loads(lines[0])["impl"] == "reference"


def test_select_fast_path_identical(pkg, gold, tmp_path):
    """The four-rows-per-warp selection (select4_kernel, the default for plain sampling passes with
    d <= 8) against the one-warp-per-row select_kernel (MPSG_SELECT_LEGACY=1): identical outcome
    strings, teacher-forced marginals and RunStats counters (incl. the near-boundary count) on
    synthetic chains at chi = 256 / 512 / 1024 (one and two pipeline lanes, ragged passes, d = 3, 4,
    6, 8), SPLIT / SINGLE / PRECISE, the c1 / c1b goldens and a chain where samples die."""
    import os
    import subprocess
    import sys
    worker = os.path.join(os.path.dirname(__file__), "select_identity_worker.py")
    files = {}
    for arm, legacy in (("fast", "0"), ("legacy", "1")):
        env = dict(os.environ, MPSG_SELECT_LEGACY=legacy)
        files[arm] = str(tmp_path / f"{arm}.npz")
        r = subprocess.run([sys.executable, worker, files[arm], str(gold)], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    a, b = np.load(files["fast"]), np.load(files["legacy"])
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        assert a[k].dtype == b[k].dtype and np.array_equal(a[k], b[k], equal_nan=True), k
    assert (a["dead_rows"][:, -1] == pkg.DEAD_OUTCOME).any()


def _worker_arms(gold, tmp_path, var, arms):
    import os
    import subprocess
    import sys
    worker = os.path.join(os.path.dirname(__file__), "select_identity_worker.py")
    out = {}
    for arm, val in arms:
        f = str(tmp_path / f"{arm}.npz")
        r = subprocess.run([sys.executable, worker, f, str(gold)], env=dict(os.environ, **{var: val}),
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
        out[arm] = np.load(f)
    return out


def test_compact_3m_store_identical(pkg, gold, tmp_path):
    """Compact 3M (only [Gr, Gi] resident in HBM; every site copied into the slot ring and its Gs
    plane re-formed there -- AUTO's choice when the 3-plane state does not fit but the 2-plane one
    does, e.g. c5 chi = 4096) forced on every chain (MPSG_COMPACT_3M=2) against the resident
    3-plane state (=0): identical rows, marginals and counters; the resident store is 2/3 of the
    3-plane one for the SPLIT / SINGLE synthetic chains (PRECISE and the AUTO c1 chains keep their
    own state)."""
    r = _worker_arms(gold, tmp_path, "MPSG_COMPACT_3M", (("compact", "2"), ("resident", "0")))
    a, b = r["compact"], r["resident"]
    assert sorted(a.files) == sorted(b.files)
    compacted = 0
    for k in a.files:
        if k.endswith("_state_bytes"):
            if int(a[k][0]) != int(b[k][0]):
                assert 3 * int(a[k][0]) == 2 * int(b[k][0]), k
                compacted += 1
            continue
        assert a[k].dtype == b[k].dtype and np.array_equal(a[k], b[k], equal_nan=True), k
    assert compacted >= 4


@pytest.mark.parametrize("chi,d", [(256, 4), (512, 6)])
def test_generated_compression_equals_array_compression(pkg, chi, d):
    """The regenerated supply's compression (SynthSrc: generator values straight into colmax / pack,
    fp32 quantize_pair) against the array path (the same site values materialised as complex128 by
    mpsg_generated_site_values, compressed with the f64 quantize_pair): identical decoded Gamma at
    every site, so hoisting the generator's per-column operands out of the row loops changed no bit."""
    from paper_2512_20064_b200.synthetic import build_synthetic
    pol = pkg.PrecisionPolicy(scaling=pkg.ScalingMode.PER_SAMPLE_MAX)
    m = 8
    gen, lams = build_synthetic(m, chi, d, seed=21, policy=pol, generated=True, pass_samples=512)
    gammas = [gen.original_gamma(i) for i in range(m)]
    st = pkg.MpsState(m, d, list(gen.bond_dims), gammas, [np.asarray(x, float) for x in lams])
    arr = pkg.GpuSampler(st, pol, mode=pkg.Mode.SPLIT, pass_samples=512)
    for i in range(m):
        assert np.array_equal(gen.decoded_gamma(i), arr.decoded_gamma(i)), i
    assert np.array_equal(gen.sample(0, 700, 7), arr.sample(0, 700, 7))
    gen.close()
    arr.close()


def test_gamma_store_reported(pkg):
    """mpsg_gamma_store names where each handle's compressed Gamma lives (resident in HBM, pinned host
    memory streamed per site, regenerated on the device); the compact store is covered by
    test_compact_3m_store_identical (its state is 2/3 of the 3-plane bytes)."""
    from paper_2512_20064_b200.synthetic import build_synthetic
    res, _ = build_synthetic(6, 256, 4, seed=3)
    host, _ = build_synthetic(6, 256, 4, seed=3, host_stream_slots=2)
    gen, _ = build_synthetic(6, 256, 4, seed=3, generated=True)
    assert (res.gamma_store, host.gamma_store, gen.gamma_store) == ("resident", "host", "generated")
    assert np.array_equal(host.sample(0, 300, 7), res.sample(0, 300, 7))
    for s in (res, host, gen):
        s.close()
