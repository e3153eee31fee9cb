"""Does per-kernel event timing (record_site_times = 2, the bench's value loop) cost time at small
chi?  Times sample_device() of one pass with torch events around the call for record_site_times
0 / 1 / 2 on the same chain.  usage: python tools/event_probe.py M CHI D N"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_20064_b200.synthetic import build_synthetic  # noqa: E402

M, chi, d, N = (int(x) for x in sys.argv[1:5])
rows = torch.empty((N, M), dtype=torch.uint8, device="cuda")
for rst in (0, 1, 2, 0, 2):
    smp, _ = build_synthetic(M, chi, d, pass_samples=N, record_site_times=rst)
    for _ in range(2):
        smp.sample_device(0, N, 7, rows.data_ptr())
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        smp.sample_device(0, N, 7, rows.data_ptr())
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(f"PDL={os.environ.get('MPSG_PDL', '0')} record_site_times={rst}: {ms:.2f} ms/pass, "
          f"{ms / M * 1e3:.1f} us/site, {N / ms * 1e3:.0f} samples/s", flush=True)
    smp.close()
