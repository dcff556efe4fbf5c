#!/usr/bin/env python
"""Benchmark of the DiLoCoX outer-synchronisation round (BASELINE.json metric).

One step = one outer-sync round of one worker per GPU: compress (warm-started rank-r power
iteration + q-bit stochastic quantisation) -> all-gather of the compressed factors (NCCL
over NVLink; no-op at N=1) + worker-0 warm-Q broadcast -> factor-space effective rank
(adaptive schedule) -> fused reconstruct / error feedback / delta staging / Nesterov
(one-step-delay overlapped mode). Workload: OPT-1.3B-shaped synthetic pseudo-gradients
(BASELINE configs[1]), rank-32 + int4, adaptive rank schedule, D = N workers.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "outer-sync ms/round & params/s (compress→allreduce→Nesterov), 1/2/4/8 GPU"
# bounded CPU sample: one whole OPT-1.3B attention projection (2048 x 2048) plus its bias
# (4 196 352 params), full reference round with the adaptive SVD. Every OPT-1.3B 2-D tensor
# has a short side of 2048, which sets the reference's per-parameter SVD cost (Gram a^2 b,
# Householder a^3); a narrower slab would overstate the CPU's throughput.
CPU_SAMPLE = [(2048, 2048), (2048,)]


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"
# dominant kernels timed with per-launch CUDA events (dlx_kernel_time)
KERNELS = ("k_o5", "k_tc_sweep_k1", "k_tc_sweep_k2", "k_outer_raw")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="opt-1.3b")
    ap.add_argument("--rank", type=int, default=32)
    ap.add_argument("--qbits", type=int, default=4)
    ap.add_argument("--no-adaptive", action="store_true")
    ap.add_argument("--hold-rank", action="store_true",
                    help="measure r' and run the controller every round but keep operating at "
                         "rank1 (default: the controller's rank is applied from the next round "
                         "on, engine.cpp:476-487, 506-507 — configs[1]'s adaptive schedule)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-held-rank", action="store_true",
                    help="skip the secondary rank-held (r1) measurement")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-compress", action="store_true",
                    help="dilocox-no-compress ablation: raw fp32 exchange (compress_raw)")
    ap.add_argument("--option", action="append", default=[], metavar="KEY=VALUE",
                    help="dlx_set_option before the run (A/B: e.g. cholqr_blocked=0)")
    ap.add_argument("--side-stream", type=int, default=None,
                    help="1/0: run the effective-rank measurement on a side stream (default: "
                         "on when N > 1, where the ranks split the eigenproblems)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks
class NvmlClockSampler:
    """SM clocks / throttle reasons sampled in-process through NVML (the fields of the
    profiling recipe's nvidia-smi clocks line) every 50 ms during the timed region, on rank 0
    only. Any clock query of a GPU measured a one-off stall of the rank driving it (NVML:
    ~15-25 ms per run; an nvidia-smi subprocess: 20-100 ms, on whichever rank it sampled);
    with every rank sampling, the slowest stall sets everyone's round at the next all-gather.
    DLX_CLOCKS=off disables sampling (the line then carries no clocks)."""

    BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
            "sw_power_cap": 0x4}

    def __init__(self, index: int | None):
        self.index = index
        self.samples = []  # (monotonic time, sm MHz, max MHz, reason bits)
        self.window = (0.0, float("inf"))
        self._stop = threading.Event()
        self.t = None

    def __enter__(self):
        if self.index is None:
            return self
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.mx = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
        except Exception:
            return self
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                sm = float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                rb = int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
                self.samples.append((time.monotonic(), sm, rb))
            except Exception:
                pass
            self._stop.wait(0.05)

    def wait_first(self, timeout=5.0):
        t = time.monotonic() + timeout
        while self.t is not None and not self.samples and time.monotonic() < t:
            time.sleep(0.01)

    def start(self):
        self.window = (time.monotonic(), float("inf"))

    def stop(self):
        self.window = (self.window[0], time.monotonic())

    def __exit__(self, *a):
        self._stop.set()
        if self.t is not None:
            self.t.join(timeout=1.0)

    def summary(self):
        inside = [x for x in self.samples if self.window[0] <= x[0] <= self.window[1]]
        reasons = sorted(n for n, b in self.BITS.items() if any(x[2] & b for x in inside))
        sm = [x[1] for x in inside]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": getattr(self, "mx", None), "reasons": reasons,
                "samples": len(sm), "source": "nvml"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, devices):
        # every rank samples its own GPU by index (-i <uuid> queries measured 100+ ms host
        # stalls of the CUDA process on that GPU)
        self.devices = devices
        self.proc = None
        self.lines = []  # (monotonic time, csv line)
        self.window = (0.0, float("inf"))

    def __enter__(self):
        if not self.devices:
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", ",".join(str(d) for d in self.devices),
                 f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def wait_first(self, timeout=5.0):
        t = time.monotonic() + timeout
        while self.proc and not self.lines and time.monotonic() < t:
            time.sleep(0.02)

    def start(self):
        self.window = (time.monotonic(), float("inf"))

    def stop(self):
        self.window = (self.window[0], time.monotonic())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        inside = [ln for t, ln in self.lines if self.window[0] <= t <= self.window[1]]
        for ln in inside:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 6:
                continue
            try:
                sm.append(float(p[0]))
                mx = max(mx, float(p[1]))
            except ValueError:
                continue
            for n, v in zip(names, p[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- reference arm
def cpu_reference_round_time(D: int, rounds: int, threads: int, warmup: int = 0):
    """Time the reference's own CPU round (oracle/_ref: compress per worker on
    min(D, threads) threads as parallel_over, allreduce_avg, measure_error, error feedback,
    staging, Nesterov, effective_rank) on the bounded sample. Returns (s/round, kind)."""
    import numpy as np
    from oracle.oracle import Oracle, Table, available
    kind = "reference" if available("reference") else "port"
    R = Oracle("reference" if kind == "reference" else "restatement")
    t = Table(CPU_SAMPLE)
    n = t.numel()
    anchor = (np.float32(0.02) * R.gaussian(R.stream(7, 0), n)[0]).astype(np.float32)
    local = np.stack([(anchor - np.float32(1e-3) * R.gaussian(R.stream(1, 10 + w), n)[0])
                      for w in range(D)]).astype(np.float32)
    pend = np.stack([anchor - local[w] for w in range(D)]).astype(np.float32)
    vel = np.zeros(n, np.float32)
    wq = np.zeros(2048 * 32, np.float32)
    wr = 0
    times = []
    for i in range(warmup + rounds):
        # warm-up rounds (allocator / caches) skip the adaptive SVD: only the timed ones matter
        adaptive = i >= warmup
        t0 = time.perf_counter()
        out = R.outer_round(t, D, 1, 2 + i, 32, 4, 0, 2, adaptive, 0.5, 32, 0.7, 0.9, False,
                            threads, anchor, vel, pend, local, wr, wq)
        if adaptive:
            times.append(time.perf_counter() - t0)
        wr = out["warm_rank"]
    return times, kind, n


def run_reference(args, world, rank):
    if rank != 0:
        return
    nproc = os.cpu_count() or 1
    D = world
    cores = min(D, nproc)
    times, kind, n = cpu_reference_round_time(D, args.steps, nproc, warmup=args.warmup)
    timed = times
    s = sum(timed) / len(timed)
    value = D * n / s
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "params/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": s * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.config} outer-sync round, D={D} workers, r=32, q=4, adaptive",
                   "sample": f"{CPU_SAMPLE} per worker ({n} params)", "threads": cores,
                   "nproc": nproc, "cpu_model": cpu_model()},
        "cpu_baseline": {"value": value, "unit": "params/s", "cores": cores, "kind": kind,
                         "sample": f"full reference round (compress r=32 q=4, allreduce_avg, "
                                   f"measure_error, error feedback, staging, Nesterov, "
                                   f"effective_rank) on {CPU_SAMPLE} x D={D} workers, "
                                   f"{args.warmup} warm-up rounds without the adaptive SVD",
                         "nproc": nproc, "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "params/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2506_21263_b200 import api, layouts
    from paper_2506_21263_b200.engine import OuterConfig, OuterSync

    torch.cuda.set_device(local_rank)
    # host-resident e2e leg: this rank's pinned buffers on its GPU's NUMA node
    numa_cpus = api.bind_host_to_device(local_rank) if os.environ.get("DLX_NUMA_BIND", "1") == "1" else []
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    dev = f"cuda:{local_rank}"
    ctx = api.Context(local_rank)
    for kv in args.option:
        k, v = kv.split("=", 1)
        api.set_option(k, int(v))
    table = layouts.CONFIGS[args.config]()
    L = api.Layout(ctx, table)
    P = L.total_params

    # synthetic state: anchor 0.02 N(0,1) (same on every rank), local = anchor - 1e-3 N(0,1)
    # drawn per worker; Tensor::gaussian-identical device generator
    anchor = L.empty(dev)
    api.fill_gaussian(L, anchor, 0.02, seed=7, tag=0xA7C4, worker=0)
    local = L.empty(dev)
    api.fill_gaussian(L, local, -1e-3, seed=1, tag=0xDA7A, worker=rank, base=anchor)
    torch.cuda.synchronize()

    cfg = OuterConfig(rank1=args.rank, qbits=args.qbits,
                      adaptive=not (args.no_adaptive or args.no_compress),
                      compress=not args.no_compress,
                      H1=125, window_c=5, tau=0.5, power_iters=2, seed=1, overlap=True,
                      hold_rank=args.hold_rank)
    eng = OuterSync(L, cfg, anchor, world=world, rank=rank, side_stream=None if args.side_stream is None else bool(args.side_stream))
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # clock sampling starts before the warm-up rounds (the summary keeps only the samples
    # inside the timed region): the first queries under load are where the sampled rank
    # stalls
    smi = os.environ.get("DLX_CLOCKS", "nvml0")  # nvml0 | nvml | smi | smi0 | off
    if smi.startswith("nvml"):
        sampler = NvmlClockSampler(local_rank if (smi == "nvml" or local_rank == 0) else None)
    else:
        sampler = ClockSampler([str(local_rank)] if smi == "smi" or
                               (smi == "smi0" and local_rank == 0) else None)
    sampler.__enter__()
    sampler.wait_first()
    # round 1 stages delta (no exchange, engine.cpp:473); then W warm-up rounds
    eng.step(local)
    for _ in range(args.warmup):
        eng.step(local)

    # ---------------- timed device region: K rounds, inputs resident in HBM (>> L2)
    eng.phase_events = []
    eng.side_events = []
    recs = []
    api.take_launch_count()
    api.set_option("kernel_events", 1)  # per-launch CUDA events on the launching stream
    for k in KERNELS:
        api.kernel_time(k)
    import gc
    gc.collect()
    gc.disable()  # a collector pause on one rank's host stalls every rank at the all-gather
    barrier()
    clocks = sampler
    clocks.start()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        recs.append(eng.step(local))
    t1.record(stream)
    barrier()
    clocks.stop()
    sampler.__exit__(None, None, None)
    gc.enable()
    eng.flush()  # held rank: the rounds' r' / controller suggestions were read back lazily
    launches = api.take_launch_count()
    ktimes = {k: api.kernel_time(k) for k in KERNELS}
    api.set_option("kernel_events", 0)
    ms = t0.elapsed_time(t1)
    if world > 1:
        m = torch.tensor([ms], device=dev)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        ms = float(m.item())
    ms_round = ms / args.steps
    value = world * P / (ms_round / 1e3)

    # per-phase device time (main stream) + effective rank (side stream)
    phases = {}
    ev = eng.phase_events
    exch = []  # per-round exchange time (all-gather incl. waiting for the other ranks)
    per_round = {}  # phase -> per-round device ms (DLX_BENCH_DETAIL=1 prints them)
    gaps = []  # device idle between one round's end and the next round's compress
    for (n0, e0), (n1, e1) in zip(ev, ev[1:]):
        if n0 == "end":
            if n1 == "compress":
                gaps.append(e0.elapsed_time(e1))
            continue
        t = e0.elapsed_time(e1)
        phases[n0] = phases.get(n0, 0.0) + t
        per_round.setdefault(n0, []).append(round(t, 3))
        if n0 == "exchange":
            exch.append(t)
    phases = {k: v / args.steps for k, v in phases.items()}
    if os.environ.get("DLX_BENCH_DETAIL") == "1":
        print(json.dumps({"rank": rank, "per_round_ms": per_round,
                          "r_t": [r.r_t for r in recs]}), file=sys.stderr, flush=True)
    if exch:
        phases["exchange_max"] = max(exch)
    if gaps:
        phases["inter_round_gap"] = sum(gaps) / args.steps
        phases["inter_round_gap_max"] = max(gaps)
    if eng.side_events and eng.side is not None:
        label = ("effective_rank (side stream, sharded)" if world > 1 else
                 "effective_rank (side stream, beside the operand prep)")
        phases[label] = sum(a.elapsed_time(b) for a, b in eng.side_events) / args.steps
    eng.phase_events = None
    phases_per_rank = None
    if world > 1:  # every rank's phase times (rank skew shows up as exchange time)
        names = sorted(phases)
        t = torch.tensor([phases[k] for k in names] + [ms / args.steps], dtype=torch.float64,
                         device=dev)
        allp = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allp, t)
        phases_per_rank = [{**{k: float(v) for k, v in zip(names, x.tolist())},
                            "round": float(x[-1])} for x in allp]

    # ---------------- roofline of the dominant kernel (CUDA events around each launch)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else \
        "fallback (B200_PROFILING.md)"
    iters = cfg.power_iters
    per_kernel = {}
    for k, (kms, kbytes, kn) in ktimes.items():
        if kn:
            per_kernel[k] = {"launches": kn, "ms_per_launch": kms / kn,
                             "bytes_per_launch": kbytes / kn,
                             "GBps": kbytes / (kms / 1e3) / 1e9 if kms > 0 else 0.0,
                             "share_of_step": kms / ms}
    dom = max(per_kernel, key=lambda k: per_kernel[k]["share_of_step"]) if per_kernel else None
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        t = prof.get("kernels", {}).get(dom)
        if t and prof.get("workload") == f"{args.config} r={args.rank} q={args.qbits} D={world}":
            traffic = t["dram_bytes_per_launch"]
    except Exception:
        pass
    achieved = per_kernel[dom]["GBps"] if dom else 0.0
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm_peak,
                "unit": "GB/s", "frac": achieved / hbm_peak, "peak_source": peak_src,
                "peak_note": ("the peak is a torch copy_ (one read + one write stream); the "
                              "TMA-streamed kernels can sit at or slightly above it (k_o5: 4 "
                              "reads + 3 writes); a pure TMA read stream tops out at 6.9-7.3 "
                              "TB/s (profiles/r02b_tma_read_bw.log)"),
                "traffic": traffic,
                "algorithmic_bytes_per_launch": per_kernel[dom]["bytes_per_launch"] if dom else None,
                "kernels": per_kernel,
                "phase_GBps": {k: (b * P / (phases[k] / 1e3) / 1e9) for k, b in
                               (("compress", 4.0 * (2 * iters + 1)), ("outer_update", 28.0))
                               if phases.get(k)}}

    # ---------------- end-to-end through the public API with host buffers
    # each step: H2D of the round's local parameters from pinned host memory -> round ->
    # D2H of the new anchor (theta_global) into pinned host memory (OuterSync.step_host:
    # the copies run on copy streams overlapping compress); optimiser state stays resident.
    h_local = torch.empty(L.slab_elems, dtype=torch.float32, pin_memory=True)
    h_local.copy_(local)
    h_anchor = torch.empty(L.slab_elems, dtype=torch.float32, pin_memory=True)
    ke = max(1, args.e2e_steps)
    eng.step_host(h_local, h_anchor)  # warm the copy streams / staging buffer
    eng.host_wait()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(ke):
        eng.step_host(h_local, h_anchor)
    eng.host_wait(stream)
    e1.record(stream)
    barrier()
    ms_e2e = e0.elapsed_time(e1)
    if world > 1:
        m = torch.tensor([ms_e2e], device=dev)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        ms_e2e = float(m.item())
    e2e_value = world * P / (ms_e2e / ke / 1e3)

    # ---------------- the same rounds at the configured rank r1, controller evaluated but not
    # applied (hold_rank): the per-round cost of the full-rank compress, for comparison
    held = None
    if not args.hold_rank and cfg.adaptive and not args.no_held_rank:
        eng.cfg.hold_rank = True
        eng.r_t = cfg.rank1
        for _ in range(args.warmup):
            eng.step(local)
        barrier()
        h0 = torch.cuda.Event(enable_timing=True)
        h1 = torch.cuda.Event(enable_timing=True)
        h0.record(stream)
        for _ in range(args.steps):
            eng.step(local)
        h1.record(stream)
        barrier()
        hms = h0.elapsed_time(h1)
        if world > 1:
            m = torch.tensor([hms], device=dev)
            dist.all_reduce(m, op=dist.ReduceOp.MAX)
            hms = float(m.item())
        eng.flush()
        held = {"rank": cfg.rank1, "ms_per_step": hms / args.steps,
                "value": world * P / (hms / args.steps / 1e3), "unit": "params/s",
                "note": "same rounds with the controller evaluated but the rank held at r1"}

    # ---------------- CPU baseline (rank 0, N=1 only): the reference round on a sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        times, kind, n = cpu_reference_round_time(1, 1, 1, warmup=1)
        s = sum(times) / len(times)
        cpu = {"value": n / s, "unit": "params/s", "cores": 1, "kind": kind,
               "sample": f"{len(times)} full reference round (compress r=32 q=4, allreduce_avg, "
                         f"measure_error, error feedback, staging, Nesterov, effective_rank) on "
                         f"{CPU_SAMPLE} ({n} params: one OPT-1.3B attention projection + bias), "
                         f"D=1, {sum(times):.1f} s; extrapolated to the whole model by parameter "
                         f"count ({P / n:.0f}x: {P / (n / s) / 60:.0f} min per worker-round)",
               "nproc": os.cpu_count(), "cpu_model": cpu_model(), "extrapolated": True}

    if rank == 0:
        rts = sorted({r.r_t for r in recs})
        line = {
            "metric": METRIC, "value": value, "unit": "params/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_round,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (Tensor::gaussian-identical device generator)",
            "config": {"workload": f"{args.config} outer-sync round (configs[1])" +
                                   (", dilocox-no-compress ablation" if args.no_compress else ""),
                       "params_per_worker": P, "workers": world, "rank1": args.rank,
                       "qbits": args.qbits, "rounding": "stochastic", "power_iters": iters,
                       "adaptive": cfg.adaptive, "tau": cfg.tau, "window_c": cfg.window_c,
                       "r_t_timed": rts, "r_prime_timed": [r.r_prime for r in recs],
                       "controller": ("evaluated every round, rank held at rank1 (r_next "
                                      f"suggested: {[r.r_next for r in recs]})" if args.hold_rank
                                      else "applied (r_t of round t+1 = adapt_compression of "
                                           "the r' window, engine.cpp:476-487)"),
                       "r_t_per_round": [r.r_t for r in recs],
                       "mode": "overlapped (one-step delay)", "parallelism": f"dp{world}",
                       "payload_bytes": recs[-1].payload_bytes if recs else None,
                       "l2": "inputs (>=5 GB slabs) larger than L2; no flush",
                       **({"options": args.option} if args.option else {}),
                       "phase_ms": phases,
                       **({"phase_ms_per_rank": phases_per_rank} if phases_per_rank else {})},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "params/s", "steps": ke,
                    "h2d_bytes_per_step": int(L.slab_elems * 4),
                    "d2h_bytes_per_step": int(L.slab_elems * 4),
                    "ms_per_step": ms_e2e / ke,
                    "host_cpus": (f"{len(numa_cpus)} CPUs local to the GPU (NVML affinity)"
                                  if numa_cpus else "unbound")},
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
            "comp_error": recs[-1].comp_error if recs else None,
            **({"rank_held": held} if held else {}),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
