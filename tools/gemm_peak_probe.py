"""Sustained cuBLAS dense GEMM throughput and SM clock per input type (bf16 / fp16), measured like
the driver's MEASURED_PEAKS.json (torch.matmul 8192^3, 2*N^3 flops, back to back for 4 s) with the
nvidia-smi clock / power sampler of bench.py running.  The K1 contraction's MMAs are fp16 x fp16 ->
fp32; this tells whether the fp16 rate under the 1000 W cap differs from the bf16 peak the roofline
uses."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import ClockSampler  # noqa: E402

n = 8192
out = {}
for name, dt in (("bf16", torch.bfloat16), ("fp16", torch.float16), ("bf16_again", torch.bfloat16)):
    a = torch.randn(n, n, device="cuda", dtype=dt)
    b = torch.randn(n, n, device="cuda", dtype=dt)
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    clk = ClockSampler(0)
    clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    e0.record()
    it = 0
    while time.time() - t0 < 4.0:
        for _ in range(20):
            torch.matmul(a, b)
        it += 20
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    c = clk.stop()
    s = e0.elapsed_time(e1) / 1e3
    out[name] = {"tflops_sustained": 2 * n ** 3 * it / s / 1e12, "clocks": c}
    print(name, json.dumps(out[name]), flush=True)
    time.sleep(3)
print(json.dumps(out))
