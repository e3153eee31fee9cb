"""Quick GPU bring-up probe (test infrastructure; prints, no asserts): RNG, one contraction, one c1
sweep against the oracle."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import oracle as O  # noqa: E402
import paper_2512_20064_b200 as P  # noqa: E402

print("devices", P.sampler._lib.lib().mpsg_device_count(), flush=True)
print("draw", P.device_draws(7, 0, 2, 0), flush=True)
z = np.load(os.path.join(ROOT, "tests/golden/c1b.npz"))
mps = O.load_npz_mps(z)
st = P.MpsState(mps.num_sites, mps.phys_dim, list(mps.bond_dims), list(mps.gammas), list(mps.lambdas))
for mode in (P.Mode.SPLIT, P.Mode.SINGLE):
    t = time.time()
    smp = P.GpuSampler(st, mode=mode)
    print("create", mode, time.time() - t, smp.state_bytes, flush=True)
    rng = np.random.default_rng(1)
    for i in (0, 1, 5, 15):
        gd = smp.decoded_gamma(i)
        env = rng.standard_normal((200, gd.shape[0])) + 1j * rng.standard_normal((200, gd.shape[0]))
        got = smp.contract_site(i, env)
        want = np.einsum("nl,lrk->nrk", env, gd)
        print(" site", i, "rel err", np.abs(got - want).max() / np.abs(want).max(), flush=True)
    t = time.time()
    rows = smp.sample(0, 1000, 7)
    print("sample", time.time() - t, rows[0], flush=True)
    dec = O.Mps(mps.phys_dim, list(mps.bond_dims), [smp.decoded_gamma(i) for i in range(16)], list(mps.lambdas))
    ref, marg, _ = O.orc_sample_range(dec, 0, 1000, 7, want_marginals=True)
    print("string diffs", int((rows != ref).any(1).sum()), flush=True)
    gm = smp.marginals(0, ref)
    live = marg > 1e-3
    print("marg max rel", (np.abs(gm[live] - marg[live]) / marg[live]).max(), flush=True)
