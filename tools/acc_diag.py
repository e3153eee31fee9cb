"""Diagnostic (needs a B200): contraction error sources at chi = 2048 (one site, random env).

Compares the GPU contraction (mpsg_contract_site) with f64, and numpy emulations of (a) the hi/lo
fp16 split of the environment alone and (b) IEEE fp32 accumulation, to locate the error budget.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_20064_b200 as P  # noqa: E402
from paper_2512_20064_b200.synthetic import build_synthetic  # noqa: E402

scheme = int(sys.argv[1]) if len(sys.argv) > 1 else 3
smp, lams = build_synthetic(12, 2048, 6, seed=5, scheme=scheme)
site = 5
g = smp.decoded_gamma(site)  # (2048, 2048, 6)
rng = np.random.default_rng(1)
n = 64
env = (rng.standard_normal((n, 2048)) + 1j * rng.standard_normal((n, 2048))) * np.exp(-2 * np.arange(2048) / 2048)
want = np.einsum("nl,lrk->nrk", env, g)
got = smp.contract_site(site, env)
scale = np.abs(want).max(axis=(1, 2), keepdims=True)
rel_elem = np.abs(got - want) / np.maximum(np.abs(want), 1e-30)
print("GPU: max |err|/rowmax", (np.abs(got - want) / scale).max(), " median per-element rel", np.median(rel_elem))
# (a) env represented as fp16 hi + fp16 lo of the fp32 value (per-sample power-of-two scaling as the engine)
mx = np.maximum(np.abs(env.real), np.abs(env.imag)).max(axis=1, keepdims=True)
sig = 2.0 ** (14 - np.ceil(np.log2(mx)))
def split(x):
    f = x.astype(np.float32)
    hi = f.astype(np.float16).astype(np.float32)
    lo = (f - hi).astype(np.float16).astype(np.float32)
    return hi.astype(np.float64) + lo.astype(np.float64)
e2 = (split((env * sig).real) + 1j * split((env * sig).imag)) / sig
wa = np.einsum("nl,lrk->nrk", e2, g)
print("split only: max |err|/rowmax", (np.abs(wa - want) / scale).max(), " median rel", np.median(np.abs(wa - want) / np.maximum(np.abs(want), 1e-30)))
# (b) IEEE fp32 accumulation (complex64 matmul, operands exact in fp32 where possible)
w32 = np.einsum("nl,lrk->nrk", env.astype(np.complex64), g.astype(np.complex64))
print("fp32 (numpy/BLAS): max |err|/rowmax", (np.abs(w32 - want) / scale).max(), " median rel", np.median(np.abs(w32 - want) / np.maximum(np.abs(want), 1e-30)))
