"""TEST INFRASTRUCTURE ONLY — ctypes front for the CPU checkers.

Two libraries, both built by ``oracle/Makefile`` (``make -C oracle``):

* ``oracle/liboracle.so``       — the plain-C restatement (``mpsamp_oracle.c``), always buildable;
* ``oracle/_ref/libmpsamp_ref.so`` — the unmodified reference compiled from /root/reference
  (``ref_capi.cpp`` wraps its public API).  Present here and, as a prebuilt file, on the GPU box.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may import this module.
The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libmpsamp_ref.so")

F64, F32, TF32, F16 = 0, 1, 2, 3
SCALE_NONE, SCALE_GLOBAL, SCALE_PER_SAMPLE = 0, 1, 2
DEAD = 0xFF
MEASURE_STREAM = 0x6D656173

_u64, _sz, _dbl, _int = C.c_uint64, C.c_size_t, C.c_double, C.c_int
_pd = C.POINTER(C.c_double)
_pu8 = C.POINTER(C.c_uint8)


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load(path: str):
    if not os.path.exists(path):
        build()
    return C.CDLL(path)


_orc = None
_ref = None


def orc():
    global _orc
    if _orc is None:
        _orc = _load(ORC_PATH)
        L = _orc
        L.orc_mix64.restype = _u64
        L.orc_mix64.argtypes = [_u64]
        L.orc_key.restype = _u64
        L.orc_key.argtypes = [_u64] * 4
        L.orc_uniform.restype = _dbl
        L.orc_uniform.argtypes = [_u64] * 4
        L.orc_round_scalar.restype = _dbl
        L.orc_round_scalar.argtypes = [_dbl, _int]
        L.orc_sample_range.restype = _int
        L.orc_sample_range.argtypes = [_sz, _sz, C.POINTER(_sz), C.POINTER(_pd), C.POINTER(_pd),
                                       _u64, _sz, _u64, _int, _int, _pu8, _pu8, _pd,
                                       C.POINTER(_u64)]
        L.orc_sample_range_displaced.restype = _int
        L.orc_sample_range_displaced.argtypes = [_sz, _sz, C.POINTER(_sz), C.POINTER(_pd), C.POINTER(_pd),
                                                 _u64, _sz, _u64, _int, _int, _pu8, _pd, _pu8, _pd,
                                                 C.POINTER(_u64)]
        L.orc_displacement.argtypes = [_dbl, _dbl, _sz, _pd]
        L.orc_capped_bond_dims.argtypes = [_sz, _sz, _sz, C.POINTER(_sz)]
        L.orc_fnv1a.restype = _u64
        L.orc_fnv1a.argtypes = [_pu8, _sz]
        L.orc_site_step.restype = _u64
        L.orc_site_step.argtypes = [_pd, _sz, _sz, _sz, _pd, _sz, _u64]
    return _orc


def have_ref() -> bool:
    if not os.path.exists(REF_PATH) and os.path.isdir("/root/reference/proj/src"):
        build()
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        if not have_ref():
            raise RuntimeError("oracle/_ref/libmpsamp_ref.so not built")
        L = C.CDLL(REF_PATH)
        _ref = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_mix64.restype = _u64
        L.ref_mix64.argtypes = [_u64]
        L.ref_rng_key.restype = _u64
        L.ref_rng_key.argtypes = [_u64] * 4
        L.ref_rng_uniform.restype = _dbl
        L.ref_rng_uniform.argtypes = [_u64] * 4
        L.ref_round_scalar.restype = _dbl
        L.ref_round_scalar.argtypes = [_dbl, _int]
        L.ref_mps_random.restype = C.c_void_p
        L.ref_mps_random.argtypes = [_sz, _sz, _sz, _u64, _dbl, _dbl]
        L.ref_mps_decay_chain.restype = C.c_void_p
        L.ref_mps_decay_chain.argtypes = [_sz, _sz, _dbl]
        L.ref_mps_branching_decay_chain.restype = C.c_void_p
        L.ref_mps_branching_decay_chain.argtypes = [_sz, _dbl]
        L.ref_mps_from_arrays.restype = C.c_void_p
        L.ref_mps_from_arrays.argtypes = [_sz, _sz, C.POINTER(_sz), C.POINTER(_pd), C.POINTER(_pd)]
        L.ref_mps_free.argtypes = [C.c_void_p]
        for f in ("ref_mps_num_sites", "ref_mps_phys_dim"):
            getattr(L, f).restype = _sz
            getattr(L, f).argtypes = [C.c_void_p]
        L.ref_mps_bond.restype = _sz
        L.ref_mps_bond.argtypes = [C.c_void_p, _sz]
        L.ref_mps_gamma.argtypes = [C.c_void_p, _sz, _pd]
        L.ref_mps_lambda.argtypes = [C.c_void_p, _sz, _pd]
        L.ref_mps_validate.restype = _int
        L.ref_mps_validate.argtypes = [C.c_void_p]
        L.ref_sample_batch.restype = _int
        L.ref_sample_batch.argtypes = [C.c_void_p, _u64, _u64, _u64, _u64, _int, _int, _pu8,
                                       C.POINTER(_u64), C.POINTER(_u64)]
        L.ref_sample_range.restype = _int
        L.ref_sample_range.argtypes = [C.c_void_p, _u64, _u64, _u64, _int, _int, _int, _pu8]
        L.ref_marginals_forced.restype = _int
        L.ref_marginals_forced.argtypes = [C.c_void_p, _u64, _int, _int, _pu8, _pd]
        L.ref_time_site_step.restype = _dbl
        L.ref_time_site_step.argtypes = [C.c_void_p, _sz, _u64, _int, _int, C.POINTER(_u64)]
        L.ref_save_mps.restype = _int
        L.ref_save_mps.argtypes = [C.c_void_p, C.c_char_p, _int]
        L.ref_mps_load.restype = C.c_void_p
        L.ref_mps_load.argtypes = [C.c_char_p]
        L.ref_mps_apply_schedule.restype = C.c_void_p
        L.ref_mps_apply_schedule.argtypes = [C.c_void_p, C.POINTER(_sz), _sz, _sz]
        L.ref_sample_batch_scheduled.restype = _int
        L.ref_sample_batch_scheduled.argtypes = [C.c_void_p, _u64, _u64, _int, C.POINTER(_sz), _sz, _sz, _pu8]
        L.ref_decay_probe.restype = _int
        L.ref_decay_probe.argtypes = [C.c_void_p, _int, _int, _u64, _u64, _pd]
        L.ref_run_scheme.restype = _int
        L.ref_run_scheme.argtypes = [C.c_char_p, _int, _u64, _u64, _u64, _sz, _sz, _u64, _int,
                                     _int, _pu8]
    return _ref


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check_ref(rc: int) -> None:
    if rc != 0:
        raise OracleError(rc, ref().ref_last_error().decode())


@dataclass
class Mps:
    """Host MPS in the reference layout: gammas[i] complex128 (chiL, chiR, d), lambdas[i] f64."""

    phys_dim: int
    bond_dims: list
    gammas: list = field(default_factory=list)
    lambdas: list = field(default_factory=list)

    @property
    def num_sites(self) -> int:
        return len(self.gammas)

    def arrays(self):
        g = [np.ascontiguousarray(x, dtype=np.complex128) for x in self.gammas]
        lam = [np.ascontiguousarray(x, dtype=np.float64) for x in self.lambdas]
        gp = (_pd * len(g))(*[x.ctypes.data_as(_pd) for x in g])
        lp = (_pd * len(lam))(*[x.ctypes.data_as(_pd) for x in lam])
        bd = (_sz * len(self.bond_dims))(*self.bond_dims)
        return (g, lam), bd, gp, lp


def ref_random_mps(m, chi, d, seed, level_damping=0.2, lambda_decay=0.8) -> Mps:
    h = ref().ref_mps_random(m, chi, d, seed, level_damping, lambda_decay)
    if not h:
        raise OracleError(2, ref().ref_last_error().decode())
    try:
        return _mps_from_handle(h)
    finally:
        ref().ref_mps_free(h)


def ref_decay_chain(m, d, decades) -> Mps:
    h = ref().ref_mps_decay_chain(m, d, decades)
    try:
        return _mps_from_handle(h)
    finally:
        ref().ref_mps_free(h)


def _mps_from_handle(h) -> Mps:
    L = ref()
    m, d = L.ref_mps_num_sites(h), L.ref_mps_phys_dim(h)
    bonds = [L.ref_mps_bond(h, i) for i in range(m + 1)]
    mps = Mps(d, bonds)
    for i in range(m):
        g = np.empty((bonds[i], bonds[i + 1], d), np.complex128)
        L.ref_mps_gamma(h, i, g.ctypes.data_as(_pd))
        lam = np.empty(bonds[i + 1], np.float64)
        L.ref_mps_lambda(h, i, lam.ctypes.data_as(_pd))
        mps.gammas.append(g)
        mps.lambdas.append(lam)
    return mps


class RefState:
    """The reference's own MpsState built from host arrays (ref_capi.cpp ref_mps_from_arrays)."""

    def __init__(self, mps: Mps):
        self._keep, bd, gp, lp = mps.arrays()
        self.mps = mps
        self.h = ref().ref_mps_from_arrays(mps.num_sites, mps.phys_dim, bd, gp, lp)

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_mps_free(self.h)

    def validate(self) -> None:
        _check_ref(ref().ref_mps_validate(self.h))

    def sample_batch(self, n, seed, n1=0, n2=5000, compute=F64, scaling=SCALE_PER_SAMPLE):
        out = np.empty((n, self.mps.num_sites), np.uint8)
        macs, dead = _u64(), _u64()
        _check_ref(ref().ref_sample_batch(self.h, n, n1, n2, seed, compute, scaling,
                                          out.ctypes.data_as(_pu8), C.byref(macs), C.byref(dead)))
        return out, macs.value, dead.value

    def sample_batch_stats(self, n, seed, compute=F64, scaling=SCALE_PER_SAMPLE):
        """sample_batch with RunStats: (rows, {contraction_macs, displacement_macs,
        measure_weight_macs, measure_pipeline_ops}, dead_samples)."""
        out = np.empty((n, self.mps.num_sites), np.uint8)
        c4 = (_u64 * 4)()
        dead = _u64()
        L = ref()
        L.ref_sample_batch_stats.argtypes = [C.c_void_p, _u64, _u64, _int, _int, _pu8, C.POINTER(_u64),
                                             C.POINTER(_u64)]
        L.ref_sample_batch_stats.restype = _int
        _check_ref(L.ref_sample_batch_stats(self.h, n, seed, compute, scaling, out.ctypes.data_as(_pu8), c4,
                                            C.byref(dead)))
        names = ("contraction_macs", "displacement_macs", "measure_weight_macs", "measure_pipeline_ops")
        return out, dict(zip(names, list(c4))), dead.value

    def sample_range(self, first, count, seed, compute=F64, scaling=SCALE_PER_SAMPLE, threads=None):
        threads = threads or os.cpu_count() or 1
        out = np.empty((count, self.mps.num_sites), np.uint8)
        _check_ref(ref().ref_sample_range(self.h, first, count, seed, compute, scaling, threads,
                                          out.ctypes.data_as(_pu8)))
        return out

    def marginals_forced(self, forced: np.ndarray, compute=F64, scaling=SCALE_PER_SAMPLE):
        forced = np.ascontiguousarray(forced, np.uint8)
        n, m = forced.shape
        marg = np.empty((n, m, self.mps.phys_dim), np.float64)
        _check_ref(ref().ref_marginals_forced(self.h, n, compute, scaling,
                                              forced.ctypes.data_as(_pu8), marg.ctypes.data_as(_pd)))
        return marg

    def decay_probe(self, count, seed=1, compute=F64, scaling=SCALE_NONE):
        out = np.empty(self.mps.num_sites, np.float64)
        _check_ref(ref().ref_decay_probe(self.h, compute, scaling, count, seed, out.ctypes.data_as(_pd)))
        return out

    def time_site_step(self, site, count, threads, reps=1):
        macs = _u64()
        s = ref().ref_time_site_step(self.h, site, count, threads, reps, C.byref(macs))
        return s, macs.value


def orc_displacement(mu: complex, n: int) -> np.ndarray:
    """expm_displacement closed form: D(mu) = exp(-|mu|^2/2) L U, n x n."""
    out = np.empty((n, n), np.complex128)
    orc().orc_displacement(float(np.real(mu)), float(np.imag(mu)), n, out.ctypes.data_as(_pd))
    return out


def orc_sample_range(mps: Mps, first, count, seed, compute=F64, scaling=SCALE_PER_SAMPLE,
                     forced=None, want_marginals=False, mu=None):
    """Plain-C restatement of detail::sample_micro_serial (sampler.cpp:129-162); mu (count, M)
    complex applies the GBS displacement D(mu[n, i]) as the site transform (sampler.cpp:143)."""
    keep, bd, gp, lp = mps.arrays()
    m, d = mps.num_sites, mps.phys_dim
    rows = np.empty((count, m), np.uint8)
    marg = np.empty((count, m, d), np.float64) if want_marginals else None
    f = None
    if forced is not None:
        forced = np.ascontiguousarray(forced, np.uint8)
        f = forced.ctypes.data_as(_pu8)
    macs = _u64()
    mu_p = None
    if mu is not None:
        mu = np.ascontiguousarray(mu, np.complex128)
        assert mu.shape == (count, m)
        mu_p = mu.ctypes.data_as(_pd)
    rc = orc().orc_sample_range_displaced(m, d, bd, gp, lp, first, count, seed, compute, scaling, f, mu_p,
                                          rows.ctypes.data_as(_pu8),
                                          marg.ctypes.data_as(_pd) if marg is not None else None,
                                          C.byref(macs))
    if rc != 0:
        raise OracleError(rc, "oracle numeric error (non-finite input)")
    return (rows, marg, macs.value) if want_marginals else (rows, macs.value)


def fnv1a(buf: np.ndarray) -> int:
    b = np.ascontiguousarray(buf, np.uint8)
    return orc().orc_fnv1a(b.ctypes.data_as(_pu8), b.size)


def capped_bond_dims(m, d, chi):
    out = (_sz * (m + 1))()
    orc().orc_capped_bond_dims(m, d, chi, out)
    return list(out)


def load_npz_mps(npz, prefix: str = "") -> Mps:
    """Mps from a tests/golden/*.npz fixture (keys bond_dims, phys_dim, gamma_i, lambda_i)."""
    bonds = [int(x) for x in npz[prefix + "bond_dims"]]
    mps = Mps(int(npz[prefix + "phys_dim"]), bonds)
    for i in range(len(bonds) - 1):
        mps.gammas.append(npz[f"{prefix}gamma_{i}"])
        mps.lambdas.append(npz[f"{prefix}lambda_{i}"])
    return mps


def orc_time_site_step(gamma: np.ndarray, lam: np.ndarray, count: int):
    """Port CPU probe: one site step for `count` samples on one thread -> (seconds, complex MACs)."""
    import time as _t
    g = np.ascontiguousarray(gamma, np.complex128)
    lam = np.ascontiguousarray(lam, np.float64)
    cl, cr, d = g.shape
    t0 = _t.perf_counter()
    macs = orc().orc_site_step(g.ctypes.data_as(_pd), cl, cr, d, lam.ctypes.data_as(_pd), count, 7)
    return _t.perf_counter() - t0, macs


def ref_load_mps(path: str) -> Mps:
    h = ref().ref_mps_load(path.encode())
    if not h:
        raise OracleError(4, ref().ref_last_error().decode())
    try:
        return _mps_from_handle(h)
    finally:
        ref().ref_mps_free(h)


def ref_save_mps(mps: Mps, path: str, storage: int = F64) -> None:
    rs = RefState(mps)
    _check_ref(ref().ref_save_mps(rs.h, path.encode(), storage))


def ref_apply_schedule(mps: Mps, chi: list, chi_max: int) -> Mps:
    rs = RefState(mps)
    arr = (_sz * len(chi))(*chi)
    h = ref().ref_mps_apply_schedule(rs.h, arr, len(chi), chi_max)
    if not h:
        raise OracleError(2, ref().ref_last_error().decode())
    try:
        return _mps_from_handle(h)
    finally:
        ref().ref_mps_free(h)


class RefSiteSweep:
    """The reference's per-site sweep body (ref_capi.cpp ref_sweep_*: contract_site ->
    measurement_draws -> measure -> scale_rows_inplace, sampler.cpp:140-158) driven one site at a
    time, threaded over contiguous sample chunks.  For full-length parity on chains whose complex128
    Gamma does not fit in host memory (c3: 409 GB): the caller passes one decoded Gamma_i per call.

    site(i, gamma, lam) -> (outcomes (count,) u8, marginals (count, d) f64, near (count,) bool);
    with forced (count,) u8 the outcome column is imposed (teacher forcing)."""

    def __init__(self, first, count, seed, compute=F64, scaling=SCALE_PER_SAMPLE, threads=None, eps=1e-6):
        L = ref()
        L.ref_sweep_begin.restype = C.c_void_p
        L.ref_sweep_begin.argtypes = [_u64, _u64, _u64, _int, _int, _int]
        L.ref_sweep_site.restype = _int
        L.ref_sweep_site.argtypes = [C.c_void_p, _sz, _pd, _sz, _sz, _sz, _pd, _pu8, _dbl, _pu8, _pd, _pu8]
        L.ref_sweep_macs.restype = _u64
        L.ref_sweep_macs.argtypes = [C.c_void_p]
        L.ref_sweep_end.argtypes = [C.c_void_p]
        self.count, self.eps = int(count), float(eps)
        self.h = L.ref_sweep_begin(first, count, seed, compute, scaling, threads or os.cpu_count() or 1)

    def site(self, i, gamma: np.ndarray, lam: np.ndarray, forced=None):
        g = np.ascontiguousarray(gamma, np.complex128)
        lam = np.ascontiguousarray(lam, np.float64)
        chil, chir, d = g.shape
        out = np.empty(self.count, np.uint8)
        marg = np.empty((self.count, d), np.float64)
        near = np.zeros(self.count, np.uint8)
        fp = None
        if forced is not None:
            forced = np.ascontiguousarray(forced, np.uint8)
            fp = forced.ctypes.data_as(_pu8)
        _check_ref(ref().ref_sweep_site(self.h, i, g.ctypes.data_as(_pd), chil, chir, d, lam.ctypes.data_as(_pd),
                                        fp, self.eps, out.ctypes.data_as(_pu8), marg.ctypes.data_as(_pd),
                                        near.ctypes.data_as(_pu8)))
        return out, marg, near.astype(bool)

    @property
    def contraction_macs(self) -> int:
        return int(ref().ref_sweep_macs(self.h))

    def close(self):
        if getattr(self, "h", None):
            ref().ref_sweep_end(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
