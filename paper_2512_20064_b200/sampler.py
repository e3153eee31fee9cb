"""Host-side mirror of the reference's sampling interface (``mpsamp``), backed by libmpsg.so.

Names, argument meaning and error behaviour follow the reference headers so that code written
against ``mpsamp::sample_batch`` reads the same here:

=========================  ======================================================================
this module                reference (proj/include/mpsamp/…)
=========================  ======================================================================
``Precision``              ``enum class Precision``           precision.hpp:15
``ScalingMode``            ``enum class ScalingMode``         precision.hpp:17
``PrecisionPolicy``        ``struct PrecisionPolicy``         precision.hpp:27-33 (validate :98-102)
``MpsState``               ``struct MpsState``                mps.hpp:14-22 (validate mps.cpp:12-38)
``BatchPlan``              ``struct BatchPlan``               sampler.hpp:22-31 (normalize sampler.cpp:20-25)
``SamplerOptions``         ``struct SamplerOptions``          sampler.hpp:75-81
``SampleBatch``            ``struct SampleBatch``             sampler.hpp:33-44
``RunStats``               ``struct RunStats``                sampler.hpp:46-54
``sample_batch``           ``sample_batch``                   sampler.hpp:84-85 (sampler.cpp:164-205)
``sample_micro_serial``    ``detail::sample_micro_serial``    sampler.hpp:103-104
``Error`` & subclasses     ``errors.hpp:8-27``
=========================  ======================================================================

The compute runs on the B200 through the C ABI; this layer only validates, marshals pointers and
maps return codes onto the exception hierarchy.
"""
from __future__ import annotations

import ctypes as C
import enum
import time
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib

DEAD_OUTCOME = 0xFF  # sampler.hpp:17


# ---- errors.hpp:8-27 -----------------------------------------------------------------------
class Error(RuntimeError):
    """mpsamp::Error"""


class ConfigError(Error):
    """mpsamp::ConfigError (exit code 2)"""


class DimensionError(ConfigError):
    """mpsamp::DimensionError"""


class NumericError(Error):
    """mpsamp::NumericError (exit code 3)"""


class IoError(Error):
    """mpsamp::IoError (exit code 4)"""


class DeviceError(Error):
    """CUDA / NCCL failure (no reference counterpart; the reference has no device)."""


def _check(rc: int) -> None:
    if rc == _lib.MPSG_OK:
        return
    msg = _lib.last_error()
    cls = {_lib.MPSG_ERR_CONFIG: ConfigError, _lib.MPSG_ERR_NUMERIC: NumericError,
           _lib.MPSG_ERR_IO: IoError, _lib.MPSG_ERR_CUDA: DeviceError}.get(rc, Error)
    if cls is ConfigError and ("shape" in msg or "length" in msg or "bond" in msg or "dimension" in msg):
        cls = DimensionError
    raise cls(msg)


# ---- precision.hpp ---------------------------------------------------------------------------
class Precision(enum.IntEnum):
    F64 = 0
    F32 = 1
    TF32 = 2
    F16 = 3

    @staticmethod
    def from_string(s: str) -> "Precision":  # precision.cpp:78-84
        m = {"f64": Precision.F64, "f32": Precision.F32, "tf32": Precision.TF32, "f16": Precision.F16}
        if s not in m:
            raise ConfigError("unknown precision tag: " + s)
        return m[s]


class ScalingMode(enum.IntEnum):
    NONE = 0
    GLOBAL_MAX = 1
    PER_SAMPLE_MAX = 2

    @staticmethod
    def from_string(s: str) -> "ScalingMode":  # precision.cpp:86-91
        m = {"none": ScalingMode.NONE, "global-max": ScalingMode.GLOBAL_MAX,
             "per-sample-max": ScalingMode.PER_SAMPLE_MAX}
        if s not in m:
            raise ConfigError("unknown scaling mode: " + s)
        return m[s]


@dataclass
class PrecisionPolicy:
    compute: Precision = Precision.F64
    storage: Precision = Precision.F64
    scaling: ScalingMode = ScalingMode.NONE

    def validate(self) -> None:  # precision.cpp:98-102
        if self.storage == Precision.TF32:
            raise ConfigError("storage precision must be one of f64/f32/f16")


class Mode(enum.IntEnum):
    """GPU contraction precision; AUTO picks PRECISE for F64/F32 compute when its
    state fits (else SPLIT) and GRID for TF32/F16 (SINGLE where GRID does not apply)."""
    AUTO = 0
    SPLIT = 1
    SINGLE = 2
    PRECISE = 3  # SPLIT + Gamma hi / lo planes: samples the caller's Gamma to ~2^-23 (3M only)
    GRID = 4     # the TF32 / F16 compute policies on their own operand grids (round_scalar, 4M only)


class Slice(enum.IntEnum):
    """How the chosen slice reaches the next environment (mpsg.h MPSG_SLICE_*): TEMP materialises
    all d outcomes of the contraction and gathers one; RECOMPUTE emits only the Born weights, buckets
    the samples by drawn outcome and recomputes the chosen slices with a 1/d-size GEMM (identical
    outcomes, no temp round trip, measured 15-32% slower); AUTO = TEMP."""
    AUTO = 0
    TEMP = 1
    RECOMPUTE = 2


class Scheme(enum.IntEnum):
    """Complex decomposition of the contraction: Gauss 3M (Gamma planes
    Gr, Gi, Gr+Gi) or 4M (Gr, Gi); AUTO = 3M when Gamma is resident and the state fits."""
    AUTO = 0
    M3 = 3
    M4 = 4


# ---- mps.hpp ---------------------------------------------------------------------------------
@dataclass
class MpsState:
    """gammas[i]: complex128 (bond[i], bond[i+1], d); lambdas[i]: float64 (bond[i+1],)."""

    num_sites: int = 0
    phys_dim: int = 0
    bond_dims: list = field(default_factory=list)
    gammas: list = field(default_factory=list)
    lambdas: list = field(default_factory=list)

    def validate(self) -> None:  # mps.cpp:12-38
        if self.num_sites == 0:
            raise DimensionError("mps has no sites")
        if self.phys_dim < 1:
            raise DimensionError("mps physical dimension must be >= 1")
        if len(self.bond_dims) != self.num_sites + 1:
            raise DimensionError("bond_dims length mismatch")
        if self.bond_dims[0] != 1 or self.bond_dims[-1] != 1:
            raise DimensionError("boundary bonds must be 1")
        if len(self.gammas) != self.num_sites or len(self.lambdas) != self.num_sites:
            raise DimensionError("site tensor count mismatch")
        for i in range(self.num_sites):
            g = self.gammas[i]
            if g.ndim != 3 or g.shape != (self.bond_dims[i], self.bond_dims[i + 1], self.phys_dim):
                raise DimensionError("gamma shape disagrees with bond dimension chain")
            lam = np.asarray(self.lambdas[i])
            if lam.shape != (self.bond_dims[i + 1],):
                raise DimensionError("lambda length disagrees with bond dimension chain")
            if (lam < 0).any():
                raise NumericError("lambda entries must be nonnegative")
            if lam.size > 1 and (np.diff(lam) > 0).any():
                raise NumericError("lambda vectors must be nonincreasing")


def capped_bond_dims(num_sites: int, phys_dim: int, chi_max: int) -> list:
    """mps.cpp:78-88: min(d^i, d^(M-i), chi_max) (double arithmetic, truncated)."""
    def p(e):  # std::pow(double, double), +inf on overflow
        try:
            return float(phys_dim) ** e
        except OverflowError:
            return float("inf")

    return [int(min(p(i), p(num_sites - i), float(chi_max))) for i in range(num_sites + 1)]


# ---- sampler.hpp -----------------------------------------------------------------------------
@dataclass
class BatchPlan:
    total_samples: int = 0
    macro_batch: int = 0
    micro_batch: int = 5000

    def normalize(self) -> None:  # sampler.cpp:20-25
        if self.total_samples == 0:
            raise ConfigError("batch plan: total samples must be >= 1")
        if self.macro_batch == 0 or self.macro_batch > self.total_samples:
            self.macro_batch = self.total_samples
        if self.micro_batch == 0:
            self.micro_batch = 5000
        if self.micro_batch > self.macro_batch:
            self.micro_batch = self.macro_batch

    def macro_count(self) -> int:
        return (self.total_samples + self.macro_batch - 1) // self.macro_batch

    @staticmethod
    def simple(n: int, n2: int = 5000) -> "BatchPlan":
        p = BatchPlan(n, n, n2)
        p.normalize()
        return p


@dataclass
class SamplerOptions:
    policy: PrecisionPolicy = field(default_factory=PrecisionPolicy)
    seed: int = 0
    schedule: Optional[object] = None        # BondSchedule: applied to the state before upload
    site_transform: Optional[object] = None  # SiteTransform hook: a Displacement, else ConfigError
    record_decay_trace: bool = False
    mode: Mode = Mode.AUTO
    pass_samples: int = 0
    scheme: Scheme = Scheme.AUTO


@dataclass
class SampleBatch:
    num_samples: int = 0
    num_sites: int = 0
    phys_dim: int = 0
    seed: int = 0
    outcomes: np.ndarray = None  # (N, M) uint8

    def outcome(self, sample: int, site: int) -> int:
        return int(self.outcomes[sample, site])

    def dead_count(self) -> int:  # sampler.cpp:40-47
        return int((self.outcomes[:, -1] == DEAD_OUTCOME).sum())


@dataclass
class RunStats:
    device_seconds: float = 0.0
    decay_trace: list = field(default_factory=list)
    contraction_macs: int = 0
    measure_weight_macs: int = 0
    dead_samples: int = 0
    site_seconds: list = field(default_factory=list)
    total_seconds: float = 0.0
    issued_mma_flops: int = 0
    displacement_macs: int = 0
    measure_pipeline_ops: int = 0
    near_boundary_draws: int = 0   # draws within 1e-6 of an interior CDF boundary (device-counted)
    h2d_bytes: int = 0
    d2h_bytes: int = 0


# ---- the device-resident sampler -------------------------------------------------------------
class GpuSampler:
    """A compressed MPS resident on one or more B200s (libmpsg handle)."""

    def __init__(self, mps: MpsState, policy: Optional[PrecisionPolicy] = None, mode: Mode = Mode.AUTO,
                 devices: Optional[Sequence[int]] = None, pass_samples: int = 0,
                 record_site_times: bool = False, tp_size: int = 1, tp_rank: int = 0,
                 host_stream_slots: int = 0, record_decay_trace: bool = False,
                 scheme: Scheme = Scheme.AUTO, slice: Slice = Slice.AUTO):
        L = _lib.lib()
        mps.validate()
        self.policy = policy or PrecisionPolicy()
        self.policy.validate()
        self.num_sites, self.phys_dim = mps.num_sites, mps.phys_dim
        self.bond_dims = list(mps.bond_dims)
        self._h = C.c_void_p()
        bonds = (C.c_uint64 * len(mps.bond_dims))(*mps.bond_dims)
        g = [np.ascontiguousarray(x, np.complex128) for x in mps.gammas]
        lam = [np.ascontiguousarray(x, np.float64) for x in mps.lambdas]
        view = _lib.MpsView(mps.num_sites, mps.phys_dim, bonds,
                            (_lib._pd * len(g))(*[x.ctypes.data_as(_lib._pd) for x in g]),
                            (_lib._pd * len(lam))(*[x.ctypes.data_as(_lib._pd) for x in lam]))
        pol = _lib.Policy(int(self.policy.compute), int(self.policy.storage), int(self.policy.scaling))
        opt = _lib.Options(int(mode), int(pass_samples), int(record_site_times), int(tp_size), int(tp_rank),
                           int(host_stream_slots), int(record_decay_trace), int(scheme), int(slice))
        self.tp_size, self.tp_rank = tp_size, tp_rank
        devs, nd = self._devices(devices)
        _check(L.mpsg_create(C.byref(view), C.byref(pol), C.byref(opt), devs, nd, C.byref(self._h)))

    @classmethod
    def from_file(cls, path: str, policy: Optional[PrecisionPolicy] = None, mode: Mode = Mode.AUTO,
                  devices: Optional[Sequence[int]] = None, pass_samples: int = 0,
                  record_site_times: bool = False, host_stream_slots: int = 0,
                  scheme: Scheme = Scheme.AUTO, slice: Slice = Slice.AUTO,
                  record_decay_trace: bool = False, streamed: bool = False) -> "GpuSampler":
        """Build the device state from an MPSB file (the reference's format, mps_io.hpp:17-24).
        streamed=True keeps only the header and Lambda: every pass re-reads the site payloads from
        storage (checksum-verified) and compresses them on the device -- the reference's SiteStream
        (mps_io.cpp:294-350) for chains beyond device and host memory (mpsg_create_from_file_streamed)."""
        L = _lib.lib()
        policy = policy or PrecisionPolicy()
        policy.validate()
        pol = _lib.Policy(int(policy.compute), int(policy.storage), int(policy.scaling))
        opt = _lib.Options(int(mode), int(pass_samples), int(record_site_times), 1, 0, int(host_stream_slots),
                           int(record_decay_trace), int(scheme), int(slice))
        devs, nd = cls._devices(devices)
        h = C.c_void_p()
        create = L.mpsg_create_from_file_streamed if streamed else L.mpsg_create_from_file
        _check(create(path.encode(), C.byref(pol), C.byref(opt), devs, nd, C.byref(h)))
        m, d, bonds = _read_mpsb_shape(path)
        self = cls.from_builder(h, m, d, bonds, policy)
        return self

    def save(self, path: str, storage: Precision = Precision.F64) -> None:
        """save_mps (mps_io.cpp:167-210) of the decoded state."""
        _check(_lib.lib().mpsg_save_file(self._h, path.encode(), int(storage)))

    @staticmethod
    def _devices(devices):
        if not devices:
            return None, 0
        arr = (C.c_int * len(devices))(*devices)
        return arr, len(devices)

    @classmethod
    def from_builder(cls, handle: C.c_void_p, num_sites: int, phys_dim: int, bond_dims: list,
                     policy: PrecisionPolicy) -> "GpuSampler":
        self = cls.__new__(cls)
        self._h = handle
        self.tp_size, self.tp_rank = 1, 0
        self.num_sites, self.phys_dim, self.bond_dims = num_sites, phys_dim, list(bond_dims)
        self.policy = policy
        return self

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            _lib.lib().mpsg_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def connect_nccl(self, unique_id: bytes) -> None:
        """Join the tensor-parallel NCCL communicator (see mpsg_tp_connect_nccl)."""
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        _check(_lib.lib().mpsg_tp_connect_nccl(self._h, buf))

    @property
    def state_bytes(self) -> int:
        return int(_lib.lib().mpsg_state_bytes(self._h))

    def sample(self, first: int, count: int, seed: int, stats: Optional[RunStats] = None,
               out: Optional[np.ndarray] = None, mu: Optional[np.ndarray] = None) -> np.ndarray:
        """detail::sample_micro_serial over global samples [first, first+count); mu (count, M)
        complex applies the GBS displacement D(mu[n, i]) as the site transform (sampler.cpp:143)."""
        rows = out if out is not None else np.empty((count, self.num_sites), np.uint8)
        st = _lib.Stats()
        site_s = None
        trace = np.zeros(self.num_sites, np.float64)
        st.decay_trace = trace.ctypes.data_as(_lib._pd)
        if stats is not None:
            site_s = np.zeros(self.num_sites, np.float64)
            st.site_seconds = site_s.ctypes.data_as(_lib._pd)
        if mu is None:
            _check(_lib.lib().mpsg_sample(self._h, seed, first, count, rows.ctypes.data_as(_lib._pu8),
                                          C.byref(st)))
        else:
            mu = self._mu(mu, count)
            _check(_lib.lib().mpsg_sample_displaced(self._h, seed, first, count, mu.ctypes.data_as(_lib._pd),
                                                    rows.ctypes.data_as(_lib._pu8), C.byref(st)))
        if stats is not None:
            stats.contraction_macs += st.contraction_macs
            stats.measure_weight_macs += st.measure_weight_macs
            stats.dead_samples += st.dead_samples
            stats.total_seconds += st.seconds
            stats.issued_mma_flops += st.issued_mma_flops
            stats.displacement_macs += st.displacement_macs
            stats.measure_pipeline_ops += st.measure_pipeline_ops
            stats.near_boundary_draws += st.near_boundary_draws
            stats.h2d_bytes += st.h2d_bytes
            stats.d2h_bytes += st.d2h_bytes
            stats.site_seconds = list(np.asarray(stats.site_seconds or np.zeros(self.num_sites)) + site_s)
            stats.decay_trace = list(trace)
        return rows

    def sample_device(self, first: int, count: int, seed: int, rows_dev_ptr: int) -> None:
        _check(_lib.lib().mpsg_sample_device(self._h, seed, first, count, C.c_void_p(rows_dev_ptr), None))

    def marginals(self, first: int, forced: np.ndarray, mu: Optional[np.ndarray] = None) -> np.ndarray:
        forced = np.ascontiguousarray(forced, np.uint8)
        n = forced.shape[0]
        marg = np.empty((n, self.num_sites, self.phys_dim), np.float64)
        if mu is None:
            _check(_lib.lib().mpsg_marginals(self._h, first, n, forced.ctypes.data_as(_lib._pu8),
                                             marg.ctypes.data_as(_lib._pd)))
        else:
            mu = self._mu(mu, n)
            _check(_lib.lib().mpsg_marginals_displaced(self._h, first, n, forced.ctypes.data_as(_lib._pu8),
                                                       mu.ctypes.data_as(_lib._pd), marg.ctypes.data_as(_lib._pd)))
        return marg

    def _mu(self, mu, count):
        mu = np.ascontiguousarray(mu, np.complex128)
        if mu.shape != (count, self.num_sites):
            raise DimensionError(f"displacement amplitudes must be ({count}, {self.num_sites})")
        return mu

    @property
    def mode(self) -> Mode:
        """The precision mode this handle runs (MPSG_MODE_AUTO resolved: SPLIT, SINGLE or PRECISE)."""
        return Mode(_lib.lib().mpsg_mode(self._h))

    @property
    def scheme(self) -> Scheme:
        """The contraction scheme this handle runs (3M or 4M)."""
        return Scheme(_lib.lib().mpsg_scheme(self._h))

    @property
    def gamma_store(self) -> str:
        """Where the compressed Gamma lives: resident / compact (3M, [Gr, Gi] in HBM, Gs re-formed per
        site in device slots) / host / generated / file (mpsg_gamma_store)."""
        return {1: "resident", 2: "compact", 3: "host", 4: "generated", 5: "file"}.get(
            _lib.lib().mpsg_gamma_store(self._h), "none")

    def decoded_gamma(self, site: int) -> np.ndarray:
        b = self.bond_dims
        out = np.empty((b[site], b[site + 1], self.phys_dim), np.complex128)
        _check(_lib.lib().mpsg_decoded_gamma(self._h, site, out.ctypes.data_as(_lib._pd)))
        return out

    def original_gamma(self, site: int) -> np.ndarray:
        """A generated handle's own (uncompressed) site values: the generator evaluated in fp32,
        widened to complex128 (mpsg_generated_site_values) -- the chain the reference would hold."""
        b = self.bond_dims
        out = np.empty((b[site], b[site + 1], self.phys_dim), np.complex128)
        _check(_lib.lib().mpsg_generated_site_values(self._h, site, out.ctypes.data_as(_lib._pd)))
        return out

    def contract_site(self, site: int, env: np.ndarray) -> np.ndarray:
        env = np.ascontiguousarray(env, np.complex128)
        b = self.bond_dims
        out = np.empty((env.shape[0], b[site + 1], self.phys_dim), np.complex128)
        _check(_lib.lib().mpsg_contract_site(self._h, site, env.ctypes.data_as(_lib._pd), env.shape[0],
                                             out.ctypes.data_as(_lib._pd)))
        return out


def _read_mpsb_shape(path: str):
    import struct
    with open(path, "rb") as f:
        head = f.read(24)
        if head[:4] != b"MPSB":
            raise IoError("not an mps file: " + path)
        m, d = struct.unpack("<QQ", head[8:24])
        bonds = list(struct.unpack(f"<{m + 1}Q", f.read(8 * (m + 1))))
    return m, d, bonds


# ---- BondSchedule (mps.hpp:27-36, mps.cpp:40-76) and apply_schedule (sampler.cpp:218-246) ------
@dataclass
class BondSchedule:
    per_site_chi: list = field(default_factory=list)  # length M + 1
    chi_max: int = 0

    def compute_ratio(self) -> float:
        sites = len(self.per_site_chi) - 1
        work = sum(float(self.per_site_chi[i]) * self.per_site_chi[i + 1] for i in range(sites))
        return work / (sites * float(self.chi_max) * self.chi_max)

    def step_ratio(self) -> float:
        inner = self.per_site_chi[1:-1]
        return 0.0 if not inner else sum(1 for c in inner if c == self.chi_max) / len(inner)

    def equivalent_chi(self) -> float:
        inner = self.per_site_chi[1:-1]
        return 1.0 if not inner else float(np.sqrt(np.mean(np.square(np.array(inner, dtype=float)))))

    @staticmethod
    def full(bond_dims, chi_max: int) -> "BondSchedule":
        return BondSchedule(list(bond_dims), chi_max)


def entanglement_entropy(lam) -> float:
    """S = -sum L^2 ln L^2 with 0 ln 0 = 0 (SPEC.md gbs-ops entanglement_entropy; Fig. 6)."""
    p = np.square(np.asarray(lam, dtype=np.float64))
    norm = float(p.sum())
    if abs(norm - 1.0) > 1e-9:
        raise NumericError(f"entanglement_entropy: Lambda is not normalised (sum L^2 = {norm!r})")
    nz = p[p > 0]
    return float(-(nz * np.log(nz)).sum())


@dataclass
class TruncationFilter:
    """TruncationFilterConfig (SPEC.md gbs-ops): per-bond discarded-weight budgets eps_b with
    eps_b >= eps_center, equality at the centre bond and nonincreasing toward it (§3.4:
    "more aggressive at the edges").  eps_b = eps_center * (1 + edge_factor * x^edge_power) with
    x = |b - M/2| / (M/2) in [0, 1]; `budget` overrides the shape with any callable(b, M)."""

    chi_max: int
    eps_center: float = 1e-6
    edge_factor: float = 0.0
    edge_power: float = 2.0
    budget: Optional[object] = None

    def eps(self, bond: int, num_sites: int) -> float:
        if self.budget is not None:
            return float(self.budget(bond, num_sites))
        half = num_sites / 2.0
        x = abs(bond - half) / half if half > 0 else 0.0
        return self.eps_center * (1.0 + self.edge_factor * x ** self.edge_power)


def dynamic_bond_schedule(lambdas, cfg: TruncationFilter, bond_dims=None) -> BondSchedule:
    """dynamic_bond_schedule (SPEC.md gbs-ops, §3.4 / Table 1): bond b (between sites b-1
    and b, Lambda vector lambdas[b-1]) keeps the smallest k with sum_{j >= k} L[j]^2 <= eps_b, capped
    at chi_max (and at the state's own bond); boundary bonds are 1.  The result plugs into
    SamplerOptions.schedule / apply_schedule (sampler.cpp:173-176, 218-246)."""
    m = len(lambdas)
    chi = [1] * (m + 1)
    for b in range(1, m):
        lam = np.asarray(lambdas[b - 1], dtype=np.float64)
        if lam.size == 0:
            raise ConfigError("dynamic_bond_schedule: empty spectrum")
        if np.any(np.diff(lam) > 0):
            raise NumericError("dynamic_bond_schedule: Lambda must be nonincreasing")
        p = lam * lam
        tail = np.cumsum(p[::-1])[::-1]  # tail[k] = sum_{j >= k} L[j]^2
        eps = cfg.eps(b, m)
        ok = np.nonzero(np.append(tail, 0.0)[1:] <= eps)[0]  # discarded weight when keeping k + 1
        k = int(ok[0]) + 1 if ok.size else lam.size
        cap = cfg.chi_max if bond_dims is None else min(cfg.chi_max, int(bond_dims[b]))
        chi[b] = max(1, min(k, cap))
    return BondSchedule(chi, cfg.chi_max)


def apply_schedule(mps: MpsState, schedule: BondSchedule) -> MpsState:
    """Truncate gammas / lambdas to the schedule's per-site bonds (sampler.cpp:218-246)."""
    if len(schedule.per_site_chi) != len(mps.bond_dims):
        raise DimensionError("bond schedule length does not match state")
    bonds = [min(int(a), int(b)) for a, b in zip(schedule.per_site_chi, mps.bond_dims)]
    if any(b == 0 for b in bonds):
        raise DimensionError("bond schedule has a zero bond")
    bonds[0] = bonds[-1] = 1
    out = MpsState(mps.num_sites, mps.phys_dim, bonds)
    for i in range(mps.num_sites):
        cl, cr = bonds[i], bonds[i + 1]
        out.gammas.append(np.ascontiguousarray(mps.gammas[i][:cl, :cr, :]))
        out.lambdas.append(np.ascontiguousarray(np.asarray(mps.lambdas[i])[:cr]))
    return out


def decay_probe(mps: MpsState, policy: PrecisionPolicy, sample_count: int, seed: int = 1) -> list:
    """decay_probe (sampler.cpp:207-216): per-site mean |env| before scaling, on the B200."""
    stats = RunStats()
    sample_batch(mps, BatchPlan.simple(sample_count),
                 SamplerOptions(policy=policy, seed=seed, record_decay_trace=True), stats)
    return stats.decay_trace


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(_lib.lib().mpsg_nccl_unique_id(buf))
    return bytes(buf)


def connect_local(samplers: Sequence["GpuSampler"]) -> None:
    """Group tensor-parallel ranks living in this process (mpsg_tp_connect_local)."""
    arr = (C.c_void_p * len(samplers))(*[s._h.value for s in samplers])
    _check(_lib.lib().mpsg_tp_connect_local(arr, len(samplers)))


@dataclass
class Displacement:
    """The GBS displacement site transform (SPEC.md gbs-ops, §3.4): sample n is displaced by
    D(mu[n, i]) at site i, applied to the contracted site between contract_site and measure (the
    reference's SiteTransform hook, sampler.hpp:71-79, sampler.cpp:143).  mu: complex (N, M) over the
    global sample indices of the batch."""

    mu: np.ndarray

    def amplitudes(self, first: int, count: int, num_sites: int) -> np.ndarray:
        mu = np.asarray(self.mu)
        if mu.ndim != 2 or mu.shape[1] != num_sites or mu.shape[0] < first + count:
            raise DimensionError("Displacement.mu must be (N, M) covering the batch")
        return np.ascontiguousarray(mu[first:first + count], np.complex128)


def displacement_matrix(mu: complex, n: int) -> np.ndarray:
    """expm_displacement evaluated by the device generator: D(mu), n x n."""
    out = np.empty((n, n), np.complex128)
    _check(_lib.lib().mpsg_displacement_matrix(float(np.real(mu)), float(np.imag(mu)), n,
                                               out.ctypes.data_as(_lib._pd)))
    return out


def device_draws(seed: int, first: int, count: int, site: int) -> np.ndarray:
    """detail::measurement_draws (sampler.cpp:120-127) computed on the GPU."""
    out = np.empty(count, np.float64)
    _check(_lib.lib().mpsg_device_draws(seed, first, count, site, out.ctypes.data_as(_lib._pd)))
    return out


def sample_micro_serial(sampler: GpuSampler, first: int, count: int, opts: SamplerOptions,
                        rows: np.ndarray, stats: RunStats) -> None:
    """detail::sample_micro_serial (sampler.hpp:103-104) on a resident GpuSampler."""
    sampler.sample(first, count, opts.seed, stats=stats, out=rows)


def sample_batch(mps: MpsState, plan: BatchPlan, opts: SamplerOptions,
                 stats: Optional[RunStats] = None, devices: Optional[Sequence[int]] = None) -> SampleBatch:
    """mpsamp::sample_batch (sampler.cpp:164-205) on the B200.

    The batch plan is validated and normalised exactly like the reference; outcomes do not depend
    on N1/N2 (keyed RNG), so the GPU processes the whole range in passes of its own size.
    """
    mps.validate()
    opts.policy.validate()
    plan = BatchPlan(plan.total_samples, plan.macro_batch, plan.micro_batch)
    plan.normalize()
    if opts.schedule is not None:  # sampler.cpp:173-176
        mps = apply_schedule(mps, opts.schedule)
    mu = None
    if opts.site_transform is not None:
        if not isinstance(opts.site_transform, Displacement):
            raise ConfigError("site transforms other than the GBS Displacement are not supported by the GPU sweep")
        mu = opts.site_transform.amplitudes(0, plan.total_samples, mps.num_sites)
    t0 = time.perf_counter()
    smp = GpuSampler(mps, opts.policy, opts.mode, devices, opts.pass_samples,
                     record_site_times=stats is not None, record_decay_trace=opts.record_decay_trace,
                     scheme=opts.scheme)
    try:
        st = stats if stats is not None else RunStats()
        rows = smp.sample(0, plan.total_samples, opts.seed, stats=st, mu=mu)
    finally:
        smp.close()
    if stats is not None:
        stats.total_seconds = time.perf_counter() - t0
    return SampleBatch(plan.total_samples, mps.num_sites, mps.phys_dim, opts.seed, rows)


# ---- file-backed executors (parallel.hpp:24-52) ------------------------------------------------
@dataclass
class ParallelResult:
    batch: SampleBatch = None
    stats: RunStats = None


def run_serial(mps_path: str, plan: BatchPlan, opts: SamplerOptions, from_storage: bool = False) -> ParallelResult:
    """run_serial (parallel.cpp:232-238): load (or, from_storage, stream) the MPSB file and sample on
    one B200."""
    return run_data_parallel(mps_path, plan, 1, opts, from_storage=from_storage)


def run_data_parallel(mps_path: str, plan: BatchPlan, p1: int, opts: SamplerOptions,
                      devices: Optional[Sequence[int]] = None, from_storage: bool = False) -> ParallelResult:
    """run_data_parallel (parallel.cpp:240-330) on p1 B200s of this process: the file is read once
    (streamed site by site), every device keeps the compressed chain, each sweeps a contiguous
    share of the samples.  Outcomes equal the serial ones (keyed RNG).

    The site transform is applied per sample as in the reference's DP worker (parallel.cpp:291-308);
    the decay trace is recorded when asked.  A bond schedule raises ConfigError, as the C++ adapter
    does (include/mpsg_mpsamp.hpp): the file-backed state is built site by site on the device and
    is not truncated here -- truncate with apply_schedule and use sample_batch.  from_storage=True
    re-reads the payloads from the file on every pass instead of holding the chain
    (mpsg_create_from_file_streamed: chains beyond device and host memory)."""
    if p1 < 1:
        raise ConfigError("data parallel needs p1 >= 1")
    if opts.schedule is not None:
        raise ConfigError("file-backed executors do not apply bond schedules; use apply_schedule + sample_batch")
    if opts.site_transform is not None and not isinstance(opts.site_transform, Displacement):
        raise ConfigError("site transforms other than the GBS Displacement are not supported by the GPU sweep")
    opts.policy.validate()
    plan = BatchPlan(plan.total_samples, plan.macro_batch, plan.micro_batch)
    plan.normalize()
    devs = list(devices) if devices else list(range(p1))
    smp = GpuSampler.from_file(mps_path, opts.policy, opts.mode, devs, opts.pass_samples, scheme=opts.scheme,
                               record_decay_trace=opts.record_decay_trace, streamed=from_storage)
    try:
        st = RunStats()
        mu = (opts.site_transform.amplitudes(0, plan.total_samples, smp.num_sites)
              if opts.site_transform is not None else None)
        rows = smp.sample(0, plan.total_samples, opts.seed, stats=st, mu=mu)
    finally:
        smp.close()
    st.dead_samples = int((rows[:, -1] == DEAD_OUTCOME).sum())
    return ParallelResult(SampleBatch(plan.total_samples, smp.num_sites, smp.phys_dim, opts.seed, rows), st)
