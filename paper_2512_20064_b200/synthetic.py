"""Synthetic random right-canonical MPS at benchmark scale, generated on the device.

Same *form* as the reference generator ``random_mps`` (mps.cpp:129-181): bonds
``capped_bond_dims(M, d, chi)`` (mps.cpp:78-88); per-bond spectra Lambda_j ∝ exp(-decay j)(1 + U[0,
0.1]) sorted and unit-norm (mps.cpp:113-125); H_i with orthonormal rows built from a complex
Gaussian damped by ``level_damping**k`` per physical level (mps.cpp:156-165); and the telescoping
Gamma_i = diag(Lambda_{i-1}) H_i diag(Lambda_i)^-1 (mps.cpp:168-175), which makes the chain-rule
distribution a normalised |amplitude|^2.

Differences, for scale (SURVEY.md §7 hard part 4): the default ``lambda_decay`` is 4/chi (the
reference default 0.8 underflows for chi >~ 890); orthonormalisation is a device QR
(torch / cuSOLVER: generation-only library use, not the hot path) on a few base isometries per
bond shape, and each site gets its own H = H_base · diag(phase) with unit phases per column keyed
by (seed, site, column) with the reference's counter-based key chain (libmpsg's generator,
mpsg_synthetic_site), which keeps the rows orthonormal and every site distinct.  Because the phases
are keyed, a site can be regenerated on the device from its generator on every pass
(``generated=True``, mpsg_generated_*): chains beyond device and host memory (c4: M = 8176,
chi = 1e4, 13-20 TB compressed) are sampled from ~16 GB of base isometries.  The random stream is
torch's / the key chain's, not libstdc++'s, so values differ from ``random_mps`` — parity tests use
the reference generator itself (tests/golden) or feed the oracle the decoded tensors.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .sampler import GpuSampler, Mode, PrecisionPolicy, _check, capped_bond_dims


def random_lambda(gen, n: int, decay: float) -> np.ndarray:
    """mps.cpp:113-125 with numpy's generator."""
    lam = np.exp(-decay * np.arange(n)) * (1.0 + gen.uniform(0.0, 0.1, n))
    lam = np.sort(lam)[::-1]
    return lam / np.sqrt((lam * lam).sum())


def _isometry(torch, chil: int, cols: int, d: int, damping: float, gen, device):
    """(chil, cols) complex64 with orthonormal rows; columns j = r*d + k damped by damping**k."""
    x = torch.randn(cols, chil, dtype=torch.complex64, device=device, generator=gen)
    damp = torch.tensor([damping ** (j % d) for j in range(d)], dtype=torch.float32, device=device)
    x = x * damp.repeat(cols // d)[:, None]
    q, _ = torch.linalg.qr(x)  # (cols, chil), orthonormal columns
    return q.conj().T.contiguous()  # rows orthonormal


def _plan_bases(torch, bonds_full, d, level_damping, n_base, gen, device):
    """Base isometries per (chiL, chiR) shape of the full (untruncated) chain: min(n_base, number of
    sites with that shape) each, generated in chain order; site i uses base i mod that count."""
    m = len(bonds_full) - 1
    count = {}
    for i in range(m):
        key = (bonds_full[i], bonds_full[i + 1])
        count[key] = count.get(key, 0) + 1
    bases, which = {}, []
    for i in range(m):
        key = (bonds_full[i], bonds_full[i + 1])
        if key not in bases:
            bases[key] = [_isometry(torch, key[0], key[1] * d, d, level_damping, gen, device)
                          for _ in range(min(n_base, count[key]))]
        which.append((key, i % len(bases[key])))
    return bases, which


def _chain_setup(num_sites, chi, d, seed, lambda_decay, schedule):
    decay = 4.0 / chi if lambda_decay is None else lambda_decay
    bonds = capped_bond_dims(num_sites, d, chi)
    rng = np.random.default_rng(seed)
    lambdas = [random_lambda(rng, bonds[i + 1], decay) if i + 1 < num_sites else np.ones(1)
               for i in range(num_sites)]
    full_bonds = list(bonds)
    if schedule is not None:
        from .sampler import dynamic_bond_schedule
        bonds = [min(a, b) for a, b in zip(dynamic_bond_schedule(lambdas, schedule, full_bonds).per_site_chi,
                                           full_bonds)]
        bonds[0] = bonds[-1] = 1
        lambdas = [np.ascontiguousarray(lambdas[i][:bonds[i + 1]]) for i in range(num_sites)]
    return bonds, full_bonds, lambdas


def synthetic_site(base, rows: int, cols: int, d: int, lam_prev, lam, seed: int, site: int, out) -> None:
    """The generator of a synthetic site (mpsg_synthetic_site): out[l, j] = base[l, j] * phase_i[j] *
    lam_prev[l] / lam[j // d] for l < rows, j < cols (torch complex64 tensors on the current device;
    base may be wider than cols: its row stride is base.shape[1])."""
    lp = None if lam_prev is None else np.ascontiguousarray(lam_prev, np.float64)
    la = np.ascontiguousarray(lam, np.float64)
    _check(_lib.lib().mpsg_synthetic_site(C.c_void_p(base.data_ptr()), base.shape[1], rows, cols, d,
                                          None if lp is None else lp.ctypes.data_as(_lib._pd),
                                          la.ctypes.data_as(_lib._pd), seed, site, C.c_void_p(out.data_ptr())))


def build_synthetic(num_sites: int, chi: int, d: int, seed: int = 42, level_damping: float = 0.2,
                    lambda_decay: Optional[float] = None, policy: Optional[PrecisionPolicy] = None,
                    mode: Mode = Mode.SPLIT, devices: Optional[Sequence[int]] = None,
                    pass_samples: int = 0, n_base: int = 4, record_site_times: bool = False,
                    keep_host: bool = False, tp_size: int = 1, tp_rank: int = 0,
                    host_stream_slots: int = 0, scheme: int = 0, schedule=None, slice: int = 0,
                    generated: bool = False):
    """Build a GpuSampler holding a synthetic chain; returns (sampler, lambdas[, host gammas]).

    schedule: an optional TruncationFilter -- the chain is generated at the capped bonds and then
    truncated to dynamic_bond_schedule(lambdas) exactly like apply_schedule (sampler.cpp:218-246):
    Gamma_i[:chi_{i}, :chi_{i+1}, :] and Lambda_i[:chi_{i+1}] (ragged per-site GEMM shapes).

    The MPS is generated and compressed site by site on the first device, never materialised in
    host memory (c3: 102 GB compressed, 409 GB as complex128).  generated=True keeps only the
    generators (base isometries + per-site spectra; mpsg_generated_*) and the device regenerates
    every site on every pass -- the same chain, for chains beyond device and host memory (c4).
    The default mode is SPLIT: a synthetic chain is sampled under the decoded-Gamma contract, like the
    benchmark (MPSG_MODE_AUTO would pick PRECISE whenever its 6 planes fit)."""
    import torch

    policy = policy or PrecisionPolicy()
    bonds, full_bonds, lambdas = _chain_setup(num_sites, chi, d, seed, lambda_decay, schedule)
    dev0 = devices[0] if devices else 0
    device = torch.device("cuda", dev0)
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    L = _lib.lib()
    h = C.c_void_p()
    bd = (C.c_uint64 * (num_sites + 1))(*bonds)
    pol = _lib.Policy(int(policy.compute), int(policy.storage), int(policy.scaling))
    opt = _lib.Options(int(mode), int(pass_samples), int(record_site_times), int(tp_size), int(tp_rank),
                       int(host_stream_slots), 0, int(scheme), int(slice))
    devs, nd = GpuSampler._devices(devices)
    with torch.cuda.device(device):
        bases, which = _plan_bases(torch, full_bonds, d, level_damping, n_base, gen, device)
        if generated:
            _check(L.mpsg_generated_begin(num_sites, d, bd, C.byref(pol), C.byref(opt), devs, nd, seed, C.byref(h)))
        else:
            _check(L.mpsg_builder_begin(num_sites, d, bd, C.byref(pol), C.byref(opt), devs, nd, C.byref(h)))
        host = [] if keep_host else None
        try:
            ids = {}
            if generated:
                for key, lst in bases.items():
                    for b, t in enumerate(lst):
                        bid = C.c_int()
                        _check(L.mpsg_generated_add_base(h, C.c_void_p(t.data_ptr()), 1, t.shape[0], t.shape[1],
                                                         C.byref(bid)))
                        ids[(key, b)] = bid.value
                del bases  # the handle holds its own copies
                torch.cuda.empty_cache()
            buf = None
            for i in range(num_sites):
                cl, cr = bonds[i], bonds[i + 1]
                lam_np = np.ascontiguousarray(lambdas[i], np.float64)
                if generated:
                    _check(L.mpsg_generated_set_site(h, i, ids[which[i]], lam_np.ctypes.data_as(_lib._pd)))
                    continue
                key, b = which[i]
                base = bases[key][b]
                if buf is None or buf.numel() < cl * cr * d:
                    buf = torch.empty(max(cl * cr * d, 1), dtype=torch.complex64, device=device)
                g = buf[:cl * cr * d]
                synthetic_site(base, cl, cr * d, d, lambdas[i - 1] if i > 0 else None, lam_np, seed, i, g)
                _check(L.mpsg_builder_set_site(h, i, C.c_void_p(g.data_ptr()), 1, 1, lam_np.ctypes.data_as(_lib._pd)))
                if keep_host:
                    host.append(g.reshape(cl, cr, d).cpu().numpy().astype(np.complex128))
            _check(L.mpsg_builder_finish(h))
        except Exception:
            L.mpsg_destroy(h)
            raise
    smp = GpuSampler.from_builder(h, num_sites, d, bonds, policy)
    smp.tp_size, smp.tp_rank = tp_size, tp_rank
    return (smp, lambdas, host) if keep_host else (smp, lambdas)
