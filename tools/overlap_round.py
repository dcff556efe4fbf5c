#!/usr/bin/env python
"""One-step-delay overlap at OPT-1.3B scale: round t's outer sync of delta^{t-1} starts
before round t's H inner AdamW steps (dlx_adamw_step over the 1.316 G-parameter slab):
compress on the main stream, then the NCCL exchange of the compressed factors and the
effective rank on a side stream concurrently with the inner steps (OuterSync.begin_round),
joined before the fused outer update (finish_round). Reports per round, max over ranks
(CUDA events):

  inner      H inner steps alone
  sync       begin + finish alone (serial)
  overlapped the same round with the sync on the side stream
  exposed    main-stream time spent waiting at the join (the sync not hidden)

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/overlap_round.py [--H 2]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--H", type=int, default=2)
    ap.add_argument("--rounds", type=int, default=6)
    ap.add_argument("--config", default="opt-1.3b")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    from paper_2506_21263_b200 import api, layouts
    from paper_2506_21263_b200.engine import OuterConfig, OuterSync
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    lr = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(lr)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{lr}"))
    ctx = api.Context(lr)
    L = api.Layout(ctx, layouts.CONFIGS[args.config]())
    dev = f"cuda:{lr}"
    anchor = L.empty(dev)
    api.fill_gaussian(L, anchor, 0.02, seed=7, tag=0xA7C4, worker=0)
    grads = L.empty(dev)
    api.fill_gaussian(L, grads, 1e-3, seed=3, tag=0x6AD5, worker=rank)
    cfg = OuterConfig(rank1=32, qbits=4, adaptive=True, hold_rank=True, H1=args.H)
    eng = OuterSync(L, cfg, anchor, world=world, rank=rank)
    opt = api.AdamWState(anchor)
    local = torch.empty_like(anchor)
    side = torch.cuda.Stream(device=dev)
    main = torch.cuda.current_stream()

    def inner():
        for _ in range(args.H):
            api.adamw_step(ctx, opt, local, grads)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        fn()
        e1.record(main)
        barrier()
        return e0.elapsed_time(e1)

    # warm-up: two rounds (the first stages only)
    for _ in range(3):
        local.copy_(eng.anchor)
        eng.begin_round(side)
        inner()
        eng.finish_round(local)
    res = {"inner": [], "sync": [], "overlapped": [], "exposed": []}
    for _ in range(args.rounds):
        local.copy_(eng.anchor)
        res["inner"].append(timed(inner))

        def serial():
            eng.begin_round(None)
            eng.finish_round(local)
        res["sync"].append(timed(serial))
        eng.overlap_events = []

        def over():
            local.copy_(eng.anchor)
            eng.begin_round(side)
            inner()
            eng.finish_round(local)
        res["overlapped"].append(timed(over))
        res["exposed"].append(sum(a.elapsed_time(b) for a, b in eng.overlap_events))
        eng.overlap_events = None
    out = {}
    for k, v in res.items():
        t = torch.tensor([sum(v) / len(v)], device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out[k + "_ms"] = float(t.item())
    if rank == 0:
        o = out
        o.update(n_gpus=world, H=args.H, config=args.config,
                 overlap_saving_ms=o["inner_ms"] + o["sync_ms"] - o["overlapped_ms"])
        print(json.dumps(o), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
