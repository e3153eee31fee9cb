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
bond shape, and each site gets its own H = H_base · diag(phase) with fresh random unit phases per
column, which keeps the rows orthonormal and every site distinct.  The random stream is torch's,
not libstdc++'s, so values differ from ``random_mps`` — parity tests use the reference generator
itself (tests/golden) or feed the oracle the decoded tensors.
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


def build_synthetic(num_sites: int, chi: int, d: int, seed: int = 42, level_damping: float = 0.2,
                    lambda_decay: Optional[float] = None, policy: Optional[PrecisionPolicy] = None,
                    mode: Mode = Mode.AUTO, devices: Optional[Sequence[int]] = None,
                    pass_samples: int = 0, n_base: int = 4, record_site_times: bool = False,
                    keep_host: bool = False, tp_size: int = 1, tp_rank: int = 0,
                    host_stream_slots: int = 0, scheme: int = 0, schedule=None, slice: int = 0):
    """Build a GpuSampler holding a synthetic chain; returns (sampler, lambdas[, host gammas]).

    schedule: an optional TruncationFilter -- the chain is generated at the capped bonds and then
    truncated to dynamic_bond_schedule(lambdas) exactly like apply_schedule (sampler.cpp:218-246):
    Gamma_i[:chi_{i}, :chi_{i+1}, :] and Lambda_i[:chi_{i+1}] (ragged per-site GEMM shapes).

    The MPS is generated and compressed site by site on the first device, never materialised in
    host memory (c3: 102 GB compressed, 409 GB as complex128)."""
    import torch

    policy = policy or PrecisionPolicy()
    decay = 4.0 / chi if lambda_decay is None else lambda_decay
    bonds = capped_bond_dims(num_sites, d, chi)
    dev0 = devices[0] if devices else 0
    device = torch.device("cuda", dev0)
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
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    bases = {}
    L = _lib.lib()
    h = C.c_void_p()
    bd = (C.c_uint64 * (num_sites + 1))(*bonds)
    pol = _lib.Policy(int(policy.compute), int(policy.storage), int(policy.scaling))
    opt = _lib.Options(int(mode), int(pass_samples), int(record_site_times), int(tp_size), int(tp_rank),
                       int(host_stream_slots), 0, int(scheme), int(slice))
    devs, nd = GpuSampler._devices(devices)
    _check(L.mpsg_builder_begin(num_sites, d, bd, C.byref(pol), C.byref(opt), devs, nd, C.byref(h)))
    host = [] if keep_host else None
    try:
        lam_prev = torch.ones(1, dtype=torch.float32, device=device)
        for i in range(num_sites):
            cl, cr = bonds[i], bonds[i + 1]
            fl, fr = full_bonds[i], full_bonds[i + 1]
            key = (fl, fr)
            if key not in bases:
                bases[key] = [_isometry(torch, fl, fr * d, d, level_damping, gen, device)
                              for _ in range(min(n_base, num_sites))]
            hb = bases[key][i % len(bases[key])][:cl, :cr * d]  # the scheduled truncation
            phase = torch.exp(2j * np.pi * torch.rand(cr * d, generator=gen, device=device,
                                                      dtype=torch.float32)).to(torch.complex64)
            lam = torch.as_tensor(lambdas[i], dtype=torch.float32, device=device)
            inv = (1.0 / lam).repeat_interleave(d)
            g = (hb * phase[None, :]) * lam_prev[:, None] * inv[None, :]
            g = g.contiguous()
            torch.cuda.synchronize(device)
            lam_np = np.ascontiguousarray(lambdas[i], np.float64)
            _check(L.mpsg_builder_set_site(h, i, C.c_void_p(g.data_ptr()), 1, 1,
                                           lam_np.ctypes.data_as(_lib._pd)))
            if keep_host:
                host.append(g.reshape(cl, cr, d).cpu().numpy().astype(np.complex128))
            lam_prev = lam
            del g
        _check(L.mpsg_builder_finish(h))
    except Exception:
        L.mpsg_destroy(h)
        raise
    smp = GpuSampler.from_builder(h, num_sites, d, bonds, policy)
    smp.tp_size, smp.tp_rank = tp_size, tp_rank
    return (smp, lambdas, host) if keep_host else (smp, lambdas)
