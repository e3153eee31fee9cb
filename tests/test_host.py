"""CPU tests: the C ABI library, the host-side mirror of the reference interface, and the
multi-rank data-parallel driver (gloo, world_size 2)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_2512_20064_b200 as P
from paper_2512_20064_b200 import _lib
from paper_2512_20064_b200.parallel import balanced_partition, rank_range, run_data_parallel

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---- C ABI ------------------------------------------------------------------------------------
def header_symbols():
    txt = open(os.path.join(ROOT, "include", "mpsg.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(mpsg_[a-z_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
    assert {name for name, _, _ in _lib.SIGNATURES} == set(syms)


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out
    sass = os.popen(f"cuobjdump -sass {_lib.LIB_PATH} 2>/dev/null").read()
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass  # tcgen05 + TMA + TMEM


def test_abi_basics_without_gpu():
    L = _lib.lib()
    assert L.mpsg_abi_version() == _lib.ABI_VERSION == 5
    if L.mpsg_device_count() == 0:
        # no CPU fallback: a compute call fails loudly with the CUDA code
        out = np.empty(4)
        assert L.mpsg_device_draws(1, 0, 4, 0, out.ctypes.data_as(_lib._pd)) == _lib.MPSG_ERR_CUDA
        assert "device" in _lib.last_error()


def _begin(bonds, d=2, policy=(0, 0, 0)):
    L = _lib.lib()
    h = C.c_void_p()
    bd = (C.c_uint64 * len(bonds))(*bonds)
    pol = _lib.Policy(*policy)
    rc = L.mpsg_builder_begin(len(bonds) - 1, d, bd, C.byref(pol), None, None, 0, C.byref(h))
    if rc == 0:
        L.mpsg_destroy(h)
    return rc


def test_abi_config_validation_precedes_device():
    # MpsState::validate (mps.cpp:12-38) and PrecisionPolicy::validate (precision.cpp:98-102)
    assert _begin([2, 2]) == _lib.MPSG_ERR_CONFIG            # boundary bonds must be 1
    assert _begin([1, 4, 1], d=0) == _lib.MPSG_ERR_CONFIG     # phys_dim >= 1
    assert _begin([1, 4, 1], policy=(0, 2, 0)) == _lib.MPSG_ERR_CONFIG  # tf32 storage
    assert _begin([1, 0, 1]) == _lib.MPSG_ERR_CONFIG          # zero bond
    assert _begin([1, 4, 1], d=300) == _lib.MPSG_ERR_CONFIG   # u8 outcomes


def test_abi_scheme_option_validated_before_device():
    """mpsg_options.scheme: only AUTO / 3M / 4M are accepted (ConfigError before any device work)."""
    L = _lib.lib()
    bd = (C.c_uint64 * 3)(1, 4, 1)
    pol = _lib.Policy(0, 0, 0)
    for bad in (1, 2, 5, -1):
        h = C.c_void_p()
        opt = _lib.Options(scheme=bad)
        assert L.mpsg_builder_begin(2, 2, bd, C.byref(pol), C.byref(opt), None, 0, C.byref(h)) == _lib.MPSG_ERR_CONFIG
    assert L.mpsg_scheme(None) == 0
    assert [int(x) for x in P.Scheme] == [0, 3, 4]


def test_abi_slice_option_validated_before_device():
    """mpsg_options.slice: only AUTO / TEMP / RECOMPUTE are accepted (ConfigError before device work)."""
    L = _lib.lib()
    bd = (C.c_uint64 * 3)(1, 4, 1)
    pol = _lib.Policy(0, 0, 0)
    for bad in (3, -1, 7):
        h = C.c_void_p()
        opt = _lib.Options(slice=bad)
        assert L.mpsg_builder_begin(2, 2, bd, C.byref(pol), C.byref(opt), None, 0, C.byref(h)) == _lib.MPSG_ERR_CONFIG
    assert [int(x) for x in P.Slice] == [0, 1, 2]


def test_options_struct_layout_matches_header(tmp_path):
    """The ctypes mirrors of mpsg_options / mpsg_stats have the header's layout (gcc offsetof)."""
    import subprocess
    fields = [f for f, _ in _lib.Options._fields_]
    sfields = [f for f, _ in _lib.Stats._fields_]
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "mpsg.h"\nint main(void){\n'
                   + "".join(f'printf("%zu ", offsetof(mpsg_options, {f}));' for f in fields)
                   + 'printf("%zu\\n", sizeof(mpsg_options));'
                   + "".join(f'printf("%zu ", offsetof(mpsg_stats, {f}));' for f in sfields)
                   + 'printf("%zu\\n", sizeof(mpsg_stats)); return 0;}\n')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    lines = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    want_o = [getattr(_lib.Options, f).offset for f in fields] + [C.sizeof(_lib.Options)]
    want_s = [getattr(_lib.Stats, f).offset for f in sfields] + [C.sizeof(_lib.Stats)]
    assert [int(x) for x in lines[0].split()] == want_o
    assert [int(x) for x in lines[1].split()] == want_s


# ---- host mirror of the reference interface ----------------------------------------------------
def test_batch_plan_normalize_matches_reference():
    p = P.BatchPlan(1000, 0, 5000)
    p.normalize()
    assert (p.total_samples, p.macro_batch, p.micro_batch) == (1000, 1000, 1000)
    p = P.BatchPlan(1000, 300, 0)
    p.normalize()
    assert (p.macro_batch, p.micro_batch, p.macro_count()) == (300, 300, 4)
    with pytest.raises(P.ConfigError):
        P.BatchPlan(0).normalize()


def test_policy_and_enums():
    assert P.Precision.from_string("tf32") == P.Precision.TF32
    assert P.ScalingMode.from_string("per-sample-max") == P.ScalingMode.PER_SAMPLE_MAX
    with pytest.raises(P.ConfigError):
        P.Precision.from_string("bf16")
    with pytest.raises(P.ConfigError):
        P.PrecisionPolicy(storage=P.Precision.TF32).validate()


def test_mps_state_validation(gold):
    z = np.load(os.path.join(gold, "c1.npz"))
    mps = O.load_npz_mps(z)
    st = P.MpsState(mps.num_sites, mps.phys_dim, list(mps.bond_dims), list(mps.gammas), list(mps.lambdas))
    st.validate()
    bad = P.MpsState(st.num_sites, st.phys_dim, list(st.bond_dims), list(st.gammas), list(st.lambdas))
    bad.lambdas[3] = bad.lambdas[3][::-1].copy()
    with pytest.raises(P.NumericError):
        bad.validate()
    bad = P.MpsState(st.num_sites, st.phys_dim, [2] + list(st.bond_dims[1:]), list(st.gammas), list(st.lambdas))
    with pytest.raises(P.DimensionError):
        bad.validate()


def test_capped_bond_dims_matches_oracle():
    for m, d, chi in [(16, 4, 32), (1024, 6, 2048), (8176, 4, 10000), (5, 7, 3)]:
        assert P.capped_bond_dims(m, d, chi) == O.capped_bond_dims(m, d, chi)


def test_sample_batch_rejects_out_of_scope_options(gold):
    z = np.load(os.path.join(gold, "c1.npz"))
    mps = O.load_npz_mps(z)
    st = P.MpsState(mps.num_sites, mps.phys_dim, list(mps.bond_dims), list(mps.gammas), list(mps.lambdas))
    with pytest.raises(P.ConfigError):
        P.sample_batch(st, P.BatchPlan(10), P.SamplerOptions(site_transform=lambda *a: None))


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")
def test_apply_schedule_matches_reference(gold):
    """BondSchedule truncation (sampler.cpp:218-246) restated on the host == the reference's."""
    z = np.load(os.path.join(gold, "c1.npz"))
    mps = O.load_npz_mps(z)
    st = P.MpsState(mps.num_sites, mps.phys_dim, list(mps.bond_dims), list(mps.gammas), list(mps.lambdas))
    chi = [1, 4, 9, 20, 32, 17, 32, 32, 5, 32, 32, 32, 32, 32, 16, 4, 1]
    got = P.apply_schedule(st, P.BondSchedule(chi, 32))
    want = O.ref_apply_schedule(mps, chi, 32)
    assert got.bond_dims == want.bond_dims
    for a, b in zip(got.gammas, want.gammas):
        assert np.array_equal(a, b)
    for a, b in zip(got.lambdas, want.lambdas):
        assert np.array_equal(a, b)
    sched = P.BondSchedule(chi, 32)
    assert abs(sched.compute_ratio() - sum(chi[i] * chi[i + 1] for i in range(16)) / (16 * 32 * 32)) < 1e-15


def test_mpsb_header_errors_are_io_errors(tmp_path):
    """read_mps_info (mps_io.cpp:212-254) failures surface as IoError before any device work."""
    bad = tmp_path / "bad.mpsb"
    bad.write_bytes(b"NOPE" + bytes(40))
    with pytest.raises(P.IoError):
        P.GpuSampler.from_file(str(bad))
    with pytest.raises(P.IoError):
        P.GpuSampler.from_file(str(tmp_path / "missing.mpsb"))


# ---- data-parallel driver ----------------------------------------------------------------------
def test_balanced_partition_matches_reference():
    assert balanced_partition(10, 4) == [(0, 3), (3, 6), (6, 8), (8, 10)]
    assert rank_range(100, 7, 2, 3) == (105, 2)


def _dp_worker(rank, world, port, gold, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    z = np.load(os.path.join(gold, "c1.npz"))
    mps = O.load_npz_mps(z)
    # per-rank sampler = the CPU oracle (this test checks the orchestration, not the kernels)
    fn = lambda f, n, s: O.orc_sample_range(mps, f, n, s)[0]  # noqa: E731
    out = run_data_parallel(fn, 0, 1000, 7, mps.num_sites)
    if rank == 0:
        q.put(O.fnv1a(out))
    dist.destroy_process_group()


def test_data_parallel_gloo_world2(gold):
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_dp_worker, args=(r, 2, port, gold, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
    assert all(p.exitcode == 0 for p in ps)
    assert q.get(timeout=5) == 0x991D873B454AB515  # == serial reference (tests/golden/c1.npz)


ADAPTER = os.path.join(ROOT, "oracle", "_ref", "adapter_test")


@pytest.mark.skipif(not os.path.exists(ADAPTER), reason="adapter_test needs the reference headers to build")
def test_cpp_dropin_adapter_cpu():
    """include/mpsg_mpsamp.hpp compiled against the reference headers: validation and error mapping."""
    import subprocess
    r = subprocess.run([ADAPTER, "cpu"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr


def test_dynamic_bond_schedule_spec_examples():
    """dynamic_bond_schedule / entanglement_entropy (SPEC.md gbs-ops examples, Table 1)."""
    assert P.entanglement_entropy([1.0]) == 0.0
    assert abs(P.entanglement_entropy([2 ** -0.5, 2 ** -0.5]) - np.log(2)) < 1e-15
    with pytest.raises(P.NumericError):
        P.entanglement_entropy([0.5, 0.5])
    m = 12
    # product state: chi = 1 everywhere
    s = P.dynamic_bond_schedule([np.array([1.0, 0.0, 0.0, 0.0])] * m, P.TruncationFilter(chi_max=4, eps_center=1e-9))
    assert s.per_site_chi == [1] * (m + 1)
    assert abs(s.compute_ratio() - 1.0 / 16) < 1e-15
    # flat spectrum, no budget: chi_max everywhere, step ratio 100%
    s = P.dynamic_bond_schedule([np.ones(16) / 4.0] * m, P.TruncationFilter(chi_max=16, eps_center=0.0))
    assert s.per_site_chi[1:-1] == [16] * (m - 1) and s.step_ratio() == 1.0
    # area-law spectra, edge-aggressive budgets: comp ratio < 1, equivalent chi < chi_max, budgets
    # nonincreasing toward the centre, smaller eps never lowers chi (schedule monotonicity)
    rng = np.random.default_rng(0)
    lams = []
    for b in range(1, m):
        rate = 0.05 + 0.3 * abs(b - m / 2) / (m / 2)  # entanglement peaked at the centre
        lam = np.exp(-rate * np.arange(64)) * (1 + 0.01 * rng.uniform(size=64))
        lam = np.sort(lam)[::-1]
        lams.append(lam / np.linalg.norm(lam))
    lams.append(np.ones(1))
    cfg = P.TruncationFilter(chi_max=64, eps_center=1e-8, edge_factor=100.0)
    eps = [cfg.eps(b, m) for b in range(m + 1)]
    assert min(eps) == eps[m // 2] and all(eps[b] >= eps[b + 1] for b in range(m // 2))
    s = P.dynamic_bond_schedule(lams, cfg)
    assert s.compute_ratio() < 1.0 and s.equivalent_chi() < 64
    tighter = P.dynamic_bond_schedule(lams, P.TruncationFilter(chi_max=64, eps_center=1e-10, edge_factor=100.0))
    assert all(a >= b for a, b in zip(tighter.per_site_chi, s.per_site_chi))
    for b in range(1, m):  # the rule itself: minimal k with discarded weight <= eps_b
        k, lam = s.per_site_chi[b], lams[b - 1]
        assert (lam[k:] ** 2).sum() <= eps[b] + 1e-18
        assert k == 1 or (lam[k - 1:] ** 2).sum() > eps[b]


def test_file_executors_reject_schedule_and_foreign_transforms(tmp_path):
    """run_serial / run_data_parallel (file-backed) raise ConfigError for a bond schedule -- the
    file state is built site by site on the device and not truncated, as in the C++ adapter -- and
    for site transforms other than the GBS Displacement, before touching a device."""
    opts = P.SamplerOptions(schedule=P.BondSchedule([1, 2, 1], 2))
    with pytest.raises(P.ConfigError):
        P.sampler.run_data_parallel(str(tmp_path / "none.mpsb"), P.BatchPlan(10), 1, opts)
    with pytest.raises(P.ConfigError):
        P.sampler.run_serial(str(tmp_path / "none.mpsb"), P.BatchPlan(10), P.SamplerOptions(site_transform=len))


def test_displacement_transform_host_checks():
    """Displacement (the GBS SiteTransform): shape checks on the host; other site transforms are
    rejected like the reference's TP executor rejects options it cannot run (ConfigError)."""
    d = P.Displacement(np.zeros((10, 4), complex))
    assert d.amplitudes(2, 5, 4).shape == (5, 4)
    with pytest.raises(P.DimensionError):
        d.amplitudes(8, 5, 4)  # beyond the batch
    with pytest.raises(P.DimensionError):
        d.amplitudes(0, 5, 3)  # wrong site count
    mps = P.MpsState(2, 2, [1, 2, 1], [np.ones((1, 2, 2), complex), np.ones((2, 1, 2), complex)],
                     [np.array([0.8, 0.6]), np.ones(1)])
    with pytest.raises(P.ConfigError):
        P.sample_batch(mps, P.BatchPlan(4), P.SamplerOptions(site_transform=lambda *a: None))


def test_file_streamed_entry_without_gpu(tmp_path):
    """mpsg_create_from_file_streamed parses the MPSB header and Lambda on the host (IoError for a
    missing or foreign file) and fails loudly with MPSG_ERR_CUDA where no B200 is visible."""
    L = _lib.lib()
    h = C.c_void_p()
    assert L.mpsg_create_from_file_streamed(str(tmp_path / "none.mpsb").encode(), None, None, None, 0,
                                            C.byref(h)) == _lib.MPSG_ERR_IO
    junk = tmp_path / "junk.mpsb"
    junk.write_bytes(b"NOTMPSB" * 8)
    assert L.mpsg_create_from_file_streamed(str(junk).encode(), None, None, None, 0, C.byref(h)) == _lib.MPSG_ERR_IO
    if L.mpsg_device_count() == 0 and O.have_ref():
        mps = O.ref_random_mps(4, 4, 2, 5)
        path = str(tmp_path / "small.mpsb")
        O.ref_save_mps(mps, path, O.F64)
        assert L.mpsg_create_from_file_streamed(path.encode(), None, None, None, 0, C.byref(h)) == _lib.MPSG_ERR_CUDA


def test_tp_partition_block_aligned():
    """Tensor-parallel column shards (engine.cu part_range / parallel.tp_partition): contiguous,
    covering [0, extent), every boundary on a K-block multiple, at most one partial (last non-empty)
    shard, balanced to within one block, and the identity for one rank -- the alignment that makes a
    sharded contraction accumulate the unsharded K blocks in order."""
    from paper_2512_20064_b200.parallel import tp_granule, tp_partition
    assert tp_granule(3) == 64 and tp_granule(4) == 32
    for extent in (1, 4, 16, 63, 64, 65, 100, 512, 1296, 2048, 4095, 10000):
        for parts in (1, 2, 3, 4, 8):
            for gran in (32, 64):
                sh = tp_partition(extent, parts, gran)
                assert len(sh) == parts and sh[0][0] == 0 and sh[-1][1] == extent
                for (b0, e0), (b1, e1) in zip(sh, sh[1:]):
                    assert e0 == b1 and b0 <= e0
                if parts == 1:
                    assert sh == [(0, extent)]
                    continue
                widths = [e - b for b, e in sh]
                assert all(b % gran == 0 for b, _ in sh if b < extent)
                full = -(-(-(-extent // parts)) // gran) * gran
                last = max(i for i, w in enumerate(widths) if w > 0)  # the last non-empty shard
                assert all(w == full for w in widths[:last]) and 0 < widths[last] <= full
                assert all(w == 0 for w in widths[last + 1:])


def test_grid_mode_config_checks_precede_device():
    """MPSG_MODE_GRID reproduces the TF32 / F16 compute policies only: with compute F64 / F32, with
    tensor parallelism, GlobalMax scaling or the decay trace it is a ConfigError (checked before any
    device is touched); a valid GRID request reaches the device check (MPSG_ERR_CUDA here)."""
    L = _lib.lib()
    if L.mpsg_device_count() != 0:
        pytest.skip("device present: the no-device code path is not reachable")
    bd = (C.c_uint64 * 3)(1, 4, 1)

    def begin(compute, scaling=2, tp=1, trace=0):
        h = C.c_void_p()
        pol = _lib.Policy(compute, 0, scaling)
        opt = _lib.Options(4, 0, 0, tp, 0, 0, trace, 0, 0)
        return L.mpsg_builder_begin(2, 2, bd, C.byref(pol), C.byref(opt), None, 0, C.byref(h))

    assert begin(0) == _lib.MPSG_ERR_CONFIG            # F64 compute
    assert begin(1) == _lib.MPSG_ERR_CONFIG            # F32 compute
    assert begin(3, tp=2) == _lib.MPSG_ERR_CONFIG      # tensor parallelism
    assert begin(3, scaling=1) == _lib.MPSG_ERR_CONFIG  # GlobalMax
    assert begin(2, trace=1) == _lib.MPSG_ERR_CONFIG   # decay trace
    assert begin(3) == _lib.MPSG_ERR_CUDA and begin(2) == _lib.MPSG_ERR_CUDA
