#!/usr/bin/env python
"""Benchmark of the B200 MPS sampling sweep (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--pass P] [--impl ours|reference]

A *step* is one pass of the hot path — the full left-to-right sweep over all M sites (contract,
Born weights, keyed draw, gather + renormalise) — for P samples per GPU.  Inputs (the compressed
MPS) are resident in HBM before the timed region; the MPS (102 GB at c3) is far larger than L2,
so no flush is needed between steps.  `value` = samples/s of the whole job (all ranks), device
time from CUDA events on the engine's stream, max over ranks.  Multi-GPU: one process per GPU
(torchrun), data-parallel over disjoint global sample ranges with no data-path collective
(the keyed RNG makes outcomes partition-independent), so scaling is "weak".

--impl reference times the reference's own CPU sampler (oracle/_ref, the unmodified reference
compiled from its sources) on this host's cores for the same workload.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "samples/sec (M=1024, χ=2048) at 1/2/4/8 B200; % of tensor-core roofline"
CONFIGS = {
    "c1": dict(M=16, chi=32, d=4, job=1000, desc="c1: M=16, chi=32, d=4, N=1000"),
    "c2": dict(M=256, chi=512, d=6, job=100_000, desc="c2: M=256, chi=512, d=6, N=1e5 (whole MPS in HBM)"),
    "c3": dict(M=1024, chi=2048, d=6, job=1_000_000, desc="c3: M=1024, chi=2048, d=6, N=1e6 data-parallel"),
}
# c4 slice: the first 64 sites of the c4 chain shape (chi = 1e4, d = 4: 2.4 GB of 3M planes per
# interior site) on one GPU with Gamma streamed from pinned host memory -- the per-site work of the
# M = 8176 chain, which needs TP over 8 GPUs and 19.6 TB of host / disk storage
CONFIGS["c4s"] = dict(M=64, chi=10000, d=4, job=1_000_000, stream=3,
                      desc="c4 slice: M=64 sites of the c4 shape (chi=1e4, d=4), N=1e6, Gamma host-streamed")
# c4: the whole M = 8176 chain (13.1 TB as 4M planes, 19.6 TB as 3M) -- beyond HBM and host memory,
# so the sites are regenerated on the device from their generators every pass (mpsg_generated_*:
# ~16 GB of base isometries), on a side stream overlapping the contractions
CONFIGS["c4"] = dict(M=8176, chi=10000, d=4, job=1_000_000, generated=True, warm_pass=256,
                     desc="c4: M=8176, chi=1e4, d=4, N=1e6; Gamma regenerated on the device per site and pass")
for _chi in (256, 512, 1024, 2048, 4096, 8192, 10000):
    CONFIGS[f"c5_{_chi}"] = dict(M=512, chi=_chi, d=4, job=100_000, generated=_chi >= 8192,
                                 desc=f"c5: bond-dimension sweep M=512, chi={_chi}, d=4, N=1e5"
                                      + ("; Gamma regenerated on the device" if _chi >= 8192 else ""))
SLICE = {"auto": 0, "temp": 1, "recompute": 2}
DEFAULT_PASS = {"c1": 1000, "c2": 32768, "c3": 16384, "c5_256": 65536, "c5_512": 32768,
                "c5_1024": 32768, "c5_2048": 16384, "c5_4096": 8192, "c4s": 8192, "c4": 8192,
                "c5_8192": 8192, "c5_10000": 8192}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["bf16_tflops"], p["bf16_tflops_sustained"], p["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


def peak_clock_mhz():
    """Median SM clock under load while MEASURED_PEAKS.json's sustained bf16 figure was taken."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["clocks_under_load"]["sm_mhz_median"])
    except Exception:
        return None


def parity_report_path(config):
    """The committed full-chain parity report for this config (tests/parity_full.py), if any."""
    p = os.path.join("profiles", "r2_parity", f"{config}_full.json")
    if not os.path.exists(os.path.join(ROOT, p)):
        return None
    try:
        with open(os.path.join(ROOT, p)) as f:
            r = json.load(f)
        return {"path": p, "samples": r["samples"], "M": r["M"],
                "unexplained_string_differences": r["unexplained_differences"],
                "max_rel_err_interior": r["max_rel_err_interior_sites"],
                "max_rel_err_right_edge": r["max_rel_err_right_edge_sites"]}
    except Exception:
        return {"path": p}


def connect_tp(P, smp, tp, tp_rank, dist, force):
    """Joins this rank's handle to its tensor-parallel group's NCCL communicator (the unique id is
    made by the group's first rank and shared over the torch process group)."""
    if tp == 1 and not force:
        return
    uid = P.sampler.nccl_unique_id() if tp_rank == 0 else None
    if dist is not None:
        ids = [None] * dist.get_world_size()
        dist.all_gather_object(ids, uid)
        uid = ids[(dist.get_rank() // tp) * tp]
    smp.connect_nccl(uid)


def chain_macs(M, chi, d):
    from paper_2512_20064_b200.sampler import capped_bond_dims
    b = capped_bond_dims(M, d, chi)
    return sum(b[i] * b[i + 1] * d for i in range(M)), b


# ---------------------------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------------------------
def fp16_context(achieved, issued_tflops):
    """cuBLAS fp16 dense sustained throughput measured on a B200 of this pool with the
    MEASURED_PEAKS.json method (profiles/r2_gemm_peak/probe.log): fp16 runs ~5% slower than bf16
    under the 1000 W cap (lower clock), and K1 issues fp16 MMAs."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r2_gemm_peak", "probe.log")
    try:
        rec = json.loads(open(path).read().strip().splitlines()[-1])["fp16"]
    except Exception:
        return None
    pk = rec["tflops_sustained"]
    return {"peak": pk, "sm_mhz": rec["clocks"]["sm_mhz"], "source": "profiles/r2_gemm_peak/probe.log",
            "frac": achieved / pk if achieved else None,
            "issued_frac": issued_tflops / pk if issued_tflops else None}


class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = [l.split(", ") for l in self.lines if l and l[0].isdigit()]
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        pw = sorted(float(r[3]) for r in rows if r[3].replace(".", "").isdigit())
        mx = max(float(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in rows for j in range(4)
                          if len(r) > 5 + j and r[5 + j].strip() == "Active"})
        load = sorted(sm)[len(sm) // 2:] if sm else []
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(rows),
                "power_w_median": statistics.median(pw[len(pw) // 2:]) if pw else None}


# ---------------------------------------------------------------------------------------------
# CPU reference timing (oracle/_ref = the reference compiled from its own sources)
# ---------------------------------------------------------------------------------------------
def measure_link_gbs(device: int, nbytes: int = 1 << 30, reps: int = 4) -> float:
    """Pinned host -> device copy bandwidth (best of `reps`, CUDA events): the host-link roofline."""
    import torch
    src = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{device}")
    best = 0.0
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dst.copy_(src, non_blocking=True)
        b.record()
        b.synchronize()
        best = max(best, nbytes / (a.elapsed_time(b) * 1e-3) / 1e9)
    del src, dst
    return best


def host_mem_available() -> int:
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def cpu_reference_rate(chi: int, d: int, target_s: float = 8.0, threads: int | None = None):
    """Times the reference hot step (contract_site + measure + scale, sampler.cpp:140-158) on a
    full-chi interior site with all host threads; returns (complex MAC/s, threads, kind, sample)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ctypes as C

    import oracle as O

    threads = threads or os.cpu_count() or 1
    rng = np.random.default_rng(5)
    g = (rng.standard_normal((chi, chi, d)) + 1j * rng.standard_normal((chi, chi, d))) / np.sqrt(chi * d)
    lam = np.sort(rng.uniform(0.1, 1.0, chi))[::-1].copy()
    lam /= np.sqrt((lam * lam).sum())
    mps = O.Mps(d, [chi, chi], [g], [lam])
    if O.have_ref():
        kind = "reference"
        rs = O.RefState(mps)
        t1, m1 = rs.time_site_step(0, 1, threads)
        count = max(1, int(target_s / max(t1, 1e-3)))
        secs, macs = rs.time_site_step(0, count, threads)
    else:  # the plain-C restatement (oracle/mpsamp_oracle.c), one thread
        kind = "port"
        threads = 1
        t1, _ = O.orc_time_site_step(g, lam, 1)
        count = max(1, int(target_s / max(t1, 1e-3)))
        secs, macs = O.orc_time_site_step(g, lam, count)
    sample = (f"contract_site+measure+scale at one chi={chi}, d={d} interior site, {count} samples x "
              f"{threads} threads, extrapolated over the chain's complex MACs")
    return macs / secs, threads, kind, sample, secs


def run_reference_arm(args, cfg):
    """--impl reference: the reference CPU sampler on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    macs_per_sample, _ = chain_macs(cfg["M"], cfg["chi"], cfg["d"])
    vals = []
    for step in range(args.warmup + args.steps):
        rate, threads, kind, sample, secs = cpu_reference_rate(min(cfg["chi"], 4096), cfg["d"], target_s=args.ref_seconds)
        if step >= args.warmup:
            vals.append(rate / macs_per_sample)
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / v, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (random dense site)",
            "config": {"workload": cfg["desc"], "M": cfg["M"], "chi": cfg["chi"], "d": cfg["d"],
                       "parallelism": f"host threads x{threads}"},
            "cpu_baseline": {"value": v, "unit": "samples/s", "cores": threads, "kind": kind, "sample": sample},
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--pass", dest="pass_samples", type=int, default=0)
    ap.add_argument("--mode", default="split", choices=["split", "single", "precise"])
    ap.add_argument("--scheme", default="auto", choices=["auto", "3m", "4m"],
                    help="complex decomposition of the contraction (auto = 3M when the state fits)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--slice", default="auto", choices=sorted(SLICE),
                    help="chosen-slice path: recompute (weights-only contraction + bucketed 1/d slice GEMM), "
                         "temp (all d outcomes materialised), auto (= temp)")
    ap.add_argument("--ref-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--schedule-eps", type=float, default=0.0,
                    help="dynamic bond dimensions: truncate every bond to discarded weight <= eps "
                         "(dynamic_bond_schedule, edge budgets 100x the centre) before sampling")
    ap.add_argument("--displace", type=float, default=0.0,
                    help="GBS displacement site transform with mu ~ complex normal of this std per "
                         "(sample, site) (0 = none)")
    ap.add_argument("--e2e", default="auto", choices=["auto", "stream", "resident"],
                    help="end-to-end arm: 'stream' rebuilds the state in pinned host memory and streams the "
                         "compressed MPS H2D every step (auto: when host memory holds it for every local rank)")
    ap.add_argument("--stream-slots", type=int, default=0,
                    help="keep the compressed MPS in pinned host memory and stream it per site "
                         "through this many device slots (0 = resident in HBM)")
    ap.add_argument("--file-storage", default="f16", choices=["f64", "f32", "f16"],
                    help="--supply file: storage precision of the MPSB file written and streamed back")
    ap.add_argument("--supply", default="auto", choices=["auto", "resident", "generated", "file"],
                    help="generated: keep only the chain's generators and regenerate every site on the "
                         "device each pass (auto: the config's default -- c4, c5 chi >= 8192)")
    ap.add_argument("--tp", type=int, default=1,
                    help="tensor-parallel group size: consecutive ranks form a group holding column shards "
                         "of every Gamma_i (the even-site pattern, parallel.cpp:420-443) and exchange the "
                         "per-site partial weights and environment shards over NCCL; dp = world / tp")
    ap.add_argument("--tp-exchange", action="store_true",
                    help="with --tp 1: run the exchange data plane through a one-rank NCCL group anyway "
                         "(exercises the TP transport on a single GPU)")
    ap.add_argument("--warm-pass", type=int, default=0,
                    help="samples per warm-up step (0 = the timed pass size; c4 default 256: one full "
                         "pass takes minutes)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if not args.stream_slots and cfg.get("stream"):
        args.stream_slots = cfg["stream"]
    generated = args.supply == "generated" or (args.supply == "auto" and cfg.get("generated", False))
    if args.impl == "reference":
        run_reference_arm(args, cfg)
        return

    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: MPSG_BENCH_SHARE_DEVICE=1 puts every rank on device 0 with a gloo process group, so
    # the multi-rank bench path can be exercised on a one-GPU box (NCCL rejects two ranks per GPU)
    share = os.environ.get("MPSG_BENCH_SHARE_DEVICE") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2512_20064_b200 as P
    from paper_2512_20064_b200.synthetic import build_synthetic

    tp = max(1, args.tp)
    if world % tp:
        raise SystemExit(f"--tp {tp} must divide the world size {world}")
    dp, group, tp_rank = world // tp, rank // tp, rank % tp

    P_pass = args.pass_samples or DEFAULT_PASS[args.config]
    mode = {"split": P.Mode.SPLIT, "single": P.Mode.SINGLE, "precise": P.Mode.PRECISE}[args.mode]
    t0 = time.perf_counter()
    smp, _ = build_synthetic(cfg["M"], cfg["chi"], cfg["d"], seed=42, mode=mode, devices=[local],
                             pass_samples=P_pass, record_site_times=2, host_stream_slots=args.stream_slots,
                             policy=P.PrecisionPolicy(scaling=P.ScalingMode.PER_SAMPLE_MAX),
                             scheme={"auto": 0, "3m": 3, "4m": 4}[args.scheme], slice=SLICE[args.slice],
                             schedule=(P.TruncationFilter(chi_max=cfg["chi"], eps_center=args.schedule_eps,
                                                          edge_factor=100.0) if args.schedule_eps > 0 else None),
                             generated=generated, tp_size=tp, tp_rank=tp_rank)
    connect_tp(P, smp, tp, tp_rank, dist, args.tp_exchange)
    file_path = None
    if args.supply == "file":
        # the chain as an MPSB file (the reference's format), then a handle that re-reads it from
        # storage every pass (mpsg_create_from_file_streamed: reader thread, pinned staging, device
        # compression) -- the reference's SiteStream path for chains beyond device and host memory
        if tp > 1:
            raise SystemExit("--supply file: not with --tp")
        file_path = os.path.join(os.environ.get("MPSG_BENCH_DIR", "/tmp"), f"mpsg_bench_{args.config}_r{rank}.mpsb")
        smp.save(file_path, {"f64": P.Precision.F64, "f32": P.Precision.F32, "f16": P.Precision.F16}[args.file_storage])
        smp.close()
        smp = P.GpuSampler.from_file(file_path, P.PrecisionPolicy(scaling=P.ScalingMode.PER_SAMPLE_MAX), mode=mode,
                                     devices=[local], pass_samples=P_pass, record_site_times=2,
                                     scheme=P.Scheme({"auto": 0, "3m": 3, "4m": 4}[args.scheme]), streamed=True)
    scheme = "3M" if smp.scheme == P.Scheme.M3 else "4M"
    warm_pass = args.warm_pass or cfg.get("warm_pass", 0) or P_pass
    build_s = time.perf_counter() - t0
    macs_per_sample, bonds = chain_macs(cfg["M"], cfg["chi"], cfg["d"])
    sched_note = None
    if args.schedule_eps > 0:
        b = smp.bond_dims
        sched_macs = sum(b[i] * b[i + 1] * cfg["d"] for i in range(cfg["M"]))
        sched_note = (f"dynamic bonds, eps_center={args.schedule_eps:g} (edges x101): {sched_macs / macs_per_sample:.3f} "
                      f"of the full chain's MACs; max chi {max(b)}")
    rows_dev = torch.empty((P_pass, cfg["M"]), dtype=torch.uint8, device="cuda")

    mu_host = rows_host = None
    if args.displace > 0:
        rng = np.random.default_rng(1)
        mu_host = (args.displace * (rng.standard_normal((P_pass, cfg["M"]))
                                    + 1j * rng.standard_normal((P_pass, cfg["M"])))).astype(np.complex128)
        rows_host = np.empty((P_pass, cfg["M"]), np.uint8)

    def step(it):
        st = P.RunStats()
        first = (it * dp + group) * P_pass
        rows = smp.sample(first, P_pass, 7, stats=st, mu=mu_host)  # host rows; device time from events
        return st, rows

    def device_step(it, count=None):
        count = count or P_pass
        st = P.RunStats()
        first = (it * dp + group) * P_pass
        L = P.sampler._lib
        s = L.Stats()
        site = np.zeros(cfg["M"], np.float64)
        s.site_seconds = site.ctypes.data_as(L._pd)
        if mu_host is None:
            P.sampler._check(L.lib().mpsg_sample_device(smp._h, 7, first, count,
                                                        ctypes.c_void_p(rows_dev.data_ptr()), ctypes.byref(s)))
        else:  # GBS displacement site transform; device time from the engine's events
            P.sampler._check(L.lib().mpsg_sample_displaced(smp._h, 7, first, P_pass, mu_host.ctypes.data_as(L._pd),
                                                           rows_host.ctypes.data_as(L._pu8), ctypes.byref(s)))
        st.contraction_macs = s.contraction_macs
        st.issued_mma_flops = s.issued_mma_flops
        st.h2d = s.h2d_bytes
        st.site_seconds = site
        st.device_seconds = s.device_seconds
        return st, s

    for w in range(args.warmup):
        device_step(w, min(warm_pass, P_pass))
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    dev_s, gemm_s, gemm_flops, issued, launches, h2d, near = 0.0, 0.0, 0, 0, 0, 0, 0
    wall0 = time.perf_counter()
    for it in range(args.steps):
        st, s = device_step(args.warmup + it)
        dev_s += st.device_seconds if st.device_seconds > 0 else float(np.sum(st.site_seconds))
        gemm_s += s.gemm_seconds
        gemm_flops += s.gemm_flops
        issued += s.issued_mma_flops
        launches += s.kernel_launches
        h2d += s.h2d_bytes
        near += s.near_boundary_draws
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    clocks = clk.stop()
    t_max = dev_s
    if dist:
        tt = torch.tensor([dev_s], device="cpu" if share else "cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
        dist.barrier()

    # e2e through the C ABI with host buffers: rows D2H inside the timed region and, in the
    # streamed arm, the whole compressed MPS H2D from pinned host memory every step
    state_bytes = smp.state_bytes
    gamma_store = smp.gamma_store  # of the timed handle (the streamed e2e arm replaces smp below)
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    e2e_mode = args.e2e
    if e2e_mode == "auto":
        # a 3M state streams its Gr, Gi planes only (Gs is re-formed on the device): 2/3 of the bytes
        host_need = state_bytes * (2 / 3 if smp.scheme == P.Scheme.M3 and gamma_store == "resident" else 1)
        # several ranks pin their states at once: keep 40% of the host memory free then
        room = host_mem_available() * (1 / 1.15 if local_world == 1 else 0.6)
        e2e_mode = "stream" if (not args.stream_slots and room > host_need * local_world) \
            else "resident"
    if args.stream_slots:
        e2e_mode = "stream"
    if generated:
        e2e_mode = "generated"
    if file_path:
        e2e_mode = "file"
    e2e_h2d = 0
    if e2e_mode == "stream" and not args.stream_slots:
        smp.close()
        torch.cuda.empty_cache()
        t0 = time.perf_counter()
        smp, _ = build_synthetic(cfg["M"], cfg["chi"], cfg["d"], seed=42, mode=mode, devices=[local],
                                 pass_samples=P_pass, record_site_times=0, host_stream_slots=3,
                                 policy=P.PrecisionPolicy(scaling=P.ScalingMode.PER_SAMPLE_MAX),
                                 scheme={"auto": 0, "3m": 3, "4m": 4}[args.scheme], slice=SLICE[args.slice],
                                 schedule=(P.TruncationFilter(chi_max=cfg["chi"], eps_center=args.schedule_eps,
                                                              edge_factor=100.0) if args.schedule_eps > 0 else None),
                                 tp_size=tp, tp_rank=tp_rank)
        connect_tp(P, smp, tp, tp_rank, dist, args.tp_exchange)
        e2e_build_s = time.perf_counter() - t0
        step(args.warmup + args.steps)  # one untimed warm-up pass of the streamed state
    e2e_s = 0.0
    for it in range(args.e2e_steps):
        t = time.perf_counter()
        st_e2e, _ = step(args.warmup + args.steps + 1 + it)
        e2e_s += time.perf_counter() - t
        e2e_h2d += st_e2e.h2d_bytes
    e2e = P_pass * args.e2e_steps * dp / e2e_s if e2e_s > 0 else None
    if dist and e2e_s > 0:
        tt = torch.tensor([e2e_s], device="cpu" if share else "cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = P_pass * args.e2e_steps * dp / float(tt.item())

    value = P_pass * dp * args.steps / t_max
    burst, sustained, hbm, src = peaks()
    achieved = gemm_flops / gemm_s / 1e12 if gemm_s > 0 else None
    # north-star roofline: the slower of the GEMM at tensor peak and the Gamma bytes over the link
    # (host-streamed) -- per step, on this rank
    link = None
    if args.stream_slots and rank == 0:
        link_gbs = measure_link_gbs(local)
        t_tensor = gemm_flops / args.steps / (sustained * 1e12)
        t_link = h2d / args.steps / (link_gbs * 1e9)
        link = {"h2d_gb_per_step": h2d / args.steps / 1e9, "link_peak_gbs": link_gbs,
                "achieved_gbs": h2d / t_max / 1e9, "t_link_s": t_link, "t_tensor_s": t_tensor,
                "bound": "link" if t_link > t_tensor else "tensor"}
    supply = None
    if generated:
        # every pass regenerates each site of this rank's column shard: the generator reads its base
        # block twice (column maxima, then the packed planes) and writes the fp16 planes
        b = smp.bond_dims
        planes = 3 if scheme == "3M" else 2
        per_pass = 0
        for i in range(cfg["M"]):
            w = -(-b[i + 1] // tp)
            per_pass += 2 * 8 * b[i] * w * cfg["d"] + planes * 2 * b[i] * w * cfg["d"]
        t_tensor = gemm_flops / args.steps / (sustained * 1e12)
        t_hbm = per_pass / (hbm * 1e9)
        supply = {"kind": "generated on the device (mpsg_generated_*)", "bytes_per_step": per_pass,
                  "hbm_peak_gbs": hbm, "achieved_gbs": per_pass * args.steps / t_max / 1e9,
                  "t_supply_s_at_hbm_peak": t_hbm, "t_tensor_s_at_peak": t_tensor,
                  "bound": "hbm" if t_hbm > t_tensor else "tensor"}
    traffic = traffic_alg = traffic_src = None
    prof = os.path.join(ROOT, "profiles", f"traffic_{args.config}_{args.mode}_p{P_pass}.json")
    if os.path.exists(prof):
        with open(prof) as f:
            tj = json.load(f)
        if tj.get("kernel", "").startswith("site_gemm_3m") == (scheme == "3M"):
            traffic = tj.get("bytes_per_launch")
            traffic_alg = tj.get("algorithmic_bytes")
            traffic_src = os.path.relpath(prof, ROOT)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the reference's per-MAC rate is flat in chi at this size; a chi <= 4096 site keeps host memory
        # free for a host-streamed state (c4s)
        rate, threads, kind, sample, secs = cpu_reference_rate(min(cfg["chi"], 4096), cfg["d"],
                                                               target_s=args.ref_seconds)
        cpu = {"value": rate / macs_per_sample, "unit": "samples/s", "cores": threads, "kind": kind,
               "sample": sample, "seconds": round(secs, 2)}
    if rank == 0:
        pclk = peak_clock_mhz()
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": {"split": "f16 x (f16 hi + f16 lo) -> f32 accumulate; f64 CDF",
                      "single": "f16 x f16 -> f32 accumulate; f64 CDF",
                      "precise": "(f16 hi + f16 lo) x (f16 hi + f16 lo) -> f32 accumulate; f64 CDF"}[args.mode],
            "data": "synthetic random right-canonical MPS generated on device (seed 42), measurement seed 7",
            "config": {"workload": cfg["desc"] + f"; step = one sweep of {P_pass} samples/GPU over all M sites",
                       "M": cfg["M"], "chi": cfg["chi"], "d": cfg["d"], "pass_samples_per_gpu": P_pass,
                       "job_samples": cfg["job"], "job_seconds_at_value": cfg["job"] / value,
                       "mode": args.mode, "scheme": scheme, "slice": args.slice, "parallelism": f"dp{dp}" + (f"xtp{tp}" if tp > 1 or args.tp_exchange else ""),
                       "bond_schedule": sched_note,
                       "displacement": (f"GBS displacement D(mu) per (sample, site), mu ~ CN(0, {args.displace}^2)"
                                        if args.displace > 0 else None),
                       "l2": (f"inputs larger than L2 (compressed MPS {state_bytes / 1e9:.1f} GB)" if not generated
                              else "inputs larger than L2 (every site regenerated into 3 device slots of up to "
                                   f"{max(6 * cfg['chi'] * cfg['chi'] * cfg['d'], 1) / 1e9:.1f} GB)"),
                       "warmup_pass_samples": min(warm_pass, P_pass),
                       "gamma_residency": (f"pinned host memory, streamed per site through {args.stream_slots} "
                                           f"device slots ({h2d / args.steps / 1e9:.1f} GB H2D per step, "
                                           f"{h2d / t_max / 1e9:.1f} GB/s)") if args.stream_slots else
                                          ("regenerated on the device every pass from the chain's generators "
                                           f"({smp.state_bytes / 1e9:.1f} GB of base isometries in HBM), "
                                           "3 device slots, side stream") if generated else
                                          (f"streamed from storage every pass: MPSB {args.file_storage} file "
                                           f"({smp.state_bytes / 1e9:.1f} GB of Gamma scalars) re-read by a reader "
                                           "thread into pinned staging, uploaded and compressed on the device "
                                           f"into 3 slots ({h2d / t_max / 1e9:.1f} GB/s from the file)")
                                          if file_path else
                                          (f"HBM, compact 3M: the [Gr, Gi] planes ({state_bytes / 1e9:.1f} GB) "
                                           "resident, each site copied into 3 device slots and its Gs plane "
                                           "re-formed there on the copy stream (the 3-plane state does not fit)")
                                          if gamma_store == "compact" else "HBM",
                       "build_seconds": round(build_s, 1)},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": sustained, "unit": "TFLOP/s",
                         "frac": achieved / sustained if achieved else None, "traffic": traffic,
                         "traffic_algorithmic_bytes": traffic_alg, "traffic_source": traffic_src,
                         "peak_kind": f"bf16 dense sustained ({src})",
                         "kernel": ("site_gemm_3m_kernel" if scheme == "3M" else "site_gemm_pair_kernel")
                                   + " (tcgen05, all sites of the sweep)",
                         "flops_per_unit": "8*chiL*chiR*d per sample per site (the 4M count, = 8 x "
                                           "contraction_macs; 3M issues 6/8 of it per precision pass)",
                         "issued_tflops": issued / gemm_s / 1e12 if gemm_s > 0 else None,
                         "issued_frac": issued / gemm_s / 1e12 / sustained if gemm_s > 0 else None,
                         "frac_of_burst": achieved / burst if achieved else None,
                         # both the kernel and the sustained cuBLAS figure run at the 1000 W power cap:
                         # the issued rate per SM clock against cuBLAS's per clock separates issue
                         # efficiency from the operating clock the power cap leaves
                         "issued_frac_at_equal_clock": (issued / gemm_s / 1e12 / sustained * pclk / clocks["sm_mhz"]
                                                        if gemm_s > 0 and pclk and clocks and clocks.get("sm_mhz")
                                                        else None),
                         "peak_sm_mhz": pclk,
                         # the contraction's MMAs are fp16 (kind::f16): the same-method cuBLAS fp16
                         # figure under the same power cap, for context (frac above stays on bf16)
                         "fp16_sustained": fp16_context(achieved, issued / gemm_s / 1e12 if gemm_s > 0 else None),
                         "gemm_share_of_step": gemm_s / dev_s if dev_s > 0 else None},
            "cpu_baseline": cpu,
            "host_link": link,
            "gamma_supply": supply,
            "e2e": {"value": e2e, "unit": "samples/s", "h2d_bytes_per_step": e2e_h2d // max(args.e2e_steps, 1),
                    "d2h_bytes_per_step": P_pass * cfg["M"], "mode": e2e_mode,
                    "note": ("mpsg_sample (C ABI) with host output rows; the compressed MPS lives in pinned host "
                             "memory and is copied H2D site by site every step (3 device slots, copy stream "
                             "overlapping the kernels); wall clock per step, max over ranks")
                    if e2e_mode == "stream" else
                            ("mpsg_sample (C ABI) with host output rows (D2H inside the timed region); the "
                             "sites are regenerated on the device (no Gamma crosses the host link)")
                    if e2e_mode == "generated" else
                            ("mpsg_sample (C ABI) with host output rows (D2H inside the timed region); every "
                             "site is read from the MPSB file, uploaded and compressed inside the timed region")
                    if e2e_mode == "file" else
                            ("mpsg_sample (C ABI) with host output rows (D2H inside the timed region); the "
                             "compressed MPS stays resident in HBM (host memory cannot hold it for every rank)")},
            "clocks": clocks, "gpu_launches": launches, "wall_seconds": wall,
            # the north star's parity rule: draws within 1e-6 of an interior CDF boundary are counted
            # (on the device, this rank's timed steps) -- the only draws allowed to differ from the
            # reference; the full-chain comparison against the reference is tests/parity_full.py
            "parity": {"near_boundary_draws": near, "draws": P_pass * cfg["M"] * args.steps,
                       "eps": 1e-6, "full_chain_report": parity_report_path(args.config)},
        }
        print(json.dumps(line), flush=True)
    smp.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
