"""Inner training on the GPU around the outer-sync path: the reference's
mlp / synthetic-regression workload and its overlapped round loop, so a full DiLoCoX run —
H inner AdamW steps per round, then the one-step-delayed compressed outer sync — executes
with every parameter device-resident.

This is the caller on one side of the hot path, not the hot path: the dense forward /
backward of the toy MLP runs through torch (fp64 GEMMs, which the reference's fp64-
accumulating matmul calls for), the AdamW update through the fused `dlx_adamw_step` kernel
and the round through `OuterSync`.

Reference behaviour followed:
* batches: `next_batch` (data.cpp:161-190) — `batch` rows drawn with `RngStream::below`
  (rng.hpp:42-48) from the replica's stream `RngStream(seed, stream_key({0xda7a, i}))`
  (test_support.hpp:140-141), replica shard = `shard(train, D, i)` (data.cpp:130-137);
* model: `pipeline_forward_backward` for the mlp with M = 1 (model.cpp:272-359):
  z = matmul(x, W) + b (fp64 accumulation, fp32 result, then the fp32 bias add), tanh / relu
  between layers, linear output, `mse_head` (model.cpp:238-252), backward with
  `activation_backward` / `matmul_tn` / `bias_grad` (fp64 column sums) / `matmul_nt`;
* round: `reference_overlapped_run` (test_support.hpp:114-218) — each round every replica
  restarts from the anchor, runs h_t inner steps, then the outer sync of the previous
  round's delta (`OuterSync.round_overlapped`); h_t follows the adaptive schedule.
"""
from __future__ import annotations

import numpy as np
import torch

from . import api
from .engine import OuterConfig, OuterSync

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def _next_u64(state: int):
    """RngStream::next_u64 (rng.hpp:25-31): (new state, value)."""
    state = (state + GOLDEN) & M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return state, z ^ (z >> 31)


def below(state: int, n: int):
    """RngStream::below (rng.hpp:42-48): unbiased integer in [0, n) by rejection."""
    if n <= 1:
        return state, 0
    limit = M64 - (M64 % n)
    state, v = _next_u64(state)
    while v >= limit:
        state, v = _next_u64(state)
    return state, v % n


def mlp_table(widths):
    """build_model's ParamSet order for an mlp (model.cpp:75-87): w_l [in, out], b_l [out]."""
    t = []
    for l in range(len(widths) - 1):
        t.append((f"w{l + 1}", (widths[l], widths[l + 1])))
        t.append((f"b{l + 1}", (widths[l + 1],)))
    return t


class MLP:
    """Forward / backward of the reference mlp on a parameter slab (fp32, device)."""

    def __init__(self, layout: api.Layout, widths, activation: str = "tanh"):
        if activation not in ("tanh", "relu"):
            raise api._lib.ValidationError("activation must be tanh or relu")
        self.L = layout
        self.widths = list(widths)
        self.act = activation
        self.nl = len(widths) - 1
        offs, shapes = layout.offsets, layout.shapes
        self._views = [(int(offs[i]), shapes[i]) for i in range(layout.nt)]

    def _view(self, slab: torch.Tensor, i: int) -> torch.Tensor:
        o, s = self._views[i]
        return slab[o:o + int(np.prod(s))].view(*s)

    def forward_backward(self, params: torch.Tensor, x: torch.Tensor, y: torch.Tensor,
                         grads: torch.Tensor) -> float:
        """Loss (fp64, as mse_head) and the gradient slab written into `grads`."""
        ins, zs, acts = [], [], []
        h = x
        for l in range(self.nl):
            w, b = self._view(params, 2 * l), self._view(params, 2 * l + 1)
            ins.append(h)
            z = (h.double() @ w.double()).float() + b
            zs.append(z)
            if l + 1 < self.nl:
                a = torch.tanh(z) if self.act == "tanh" else torch.clamp_min(z, 0.0)
            else:
                a = z
            acts.append(a)
            h = a
        n = h.numel()
        diff = h.double() - y.double()
        loss = float((diff * diff).sum() / n)
        inv = torch.tensor(1.0, dtype=torch.float32) / float(n)  # 1.0f / (float)n
        dx = (2.0 * (h - y)) * inv.to(h.device)
        for l in range(self.nl - 1, -1, -1):
            if l + 1 < self.nl:
                a = acts[l]
                dx = dx * (1.0 - a * a) if self.act == "tanh" else torch.where(zs[l] > 0, dx, 0.0)
            gw, gb = self._view(grads, 2 * l), self._view(grads, 2 * l + 1)
            gw.copy_((ins[l].double().t() @ dx.double()).float())
            gb.copy_(dx.double().sum(0).float())
            if l > 0:
                dx = (dx.double() @ self._view(params, 2 * l).double().t()).float()
        return loss


class Replica:
    """One data-parallel replica's inner loop: its data shard, batch stream and AdamW."""

    def __init__(self, mlp: MLP, features: torch.Tensor, targets: torch.Tensor, seed: int,
                 index: int, hyper: api.AdamWHyper | None = None):
        self.mlp = mlp
        self.x, self.y = features, targets
        self.rng = api.rng_stream(seed, api.stream_key(0xDA7A, index))
        self.opt = None
        self.hyper = hyper or api.AdamWHyper()
        self.grads = None

    def next_batch(self, batch: int):
        """next_batch (data.cpp:161-190), regression branch."""
        n = self.x.shape[0]
        rows = []
        for _ in range(batch):
            self.rng, r = below(self.rng, n)
            rows.append(r)
        idx = torch.tensor(rows, dtype=torch.long, device=self.x.device)
        return self.x.index_select(0, idx), self.y.index_select(0, idx)

    def inner_steps(self, local: torch.Tensor, h: int, batch: int) -> float:
        """h AdamW steps on `local` in place; returns the last step's loss."""
        ctx = self.mlp.L.ctx
        if self.opt is None:
            self.opt = api.AdamWState(local, self.hyper)
            self.grads = torch.zeros_like(local)
        last = 0.0
        for _ in range(h):
            xb, yb = self.next_batch(batch)
            last = self.mlp.forward_backward(local, xb, yb, self.grads)
            api.adamw_step(ctx, self.opt, local, self.grads)
        return last


def shard(features: np.ndarray, targets: np.ndarray, D: int, i: int):
    """shard (data.cpp:130-137): contiguous n / D rows."""
    per = features.shape[0] // D
    return features[i * per:(i + 1) * per], targets[i * per:(i + 1) * per]


def train_overlapped(layout: api.Layout, mlp: MLP, anchor: torch.Tensor, replica: Replica,
                     cfg: OuterConfig, total_steps: int, batch: int, world: int = 1,
                     rank: int = 0, group=None, side_sync: bool = True, engine=None):
    """reference_overlapped_run (test_support.hpp:114-218) for this process's replica (one
    process per replica / GPU; world = D). Returns (final anchor slab, per-round losses of
    this replica, round records).

    side_sync: round t's sync of delta^{t-1} starts before round t's inner steps: compress on
    the main stream, then the NCCL exchange of the compressed factors and the effective rank
    on a side stream CONCURRENTLY with the inner steps (engine.begin_round), joined right
    before the fused outer update (engine.finish_round) — the one-step-delay overlap
    run_round_overlapped simulates in virtual time (engine.cpp:464-468). The results are
    identical to the serial order (same kernels, same inputs); only the schedule differs."""
    eng = engine or OuterSync(layout, cfg, anchor, world=world, rank=rank, group=group)
    sync_stream = torch.cuda.Stream(device=anchor.device) if side_sync else None
    local = torch.empty_like(anchor)
    steps, losses, recs = 0, [], []
    while steps < total_steps:
        h_used = min(eng.H_t, total_steps - steps)
        local.copy_(eng.anchor)  # continue_from_local = false
        eng.begin_round(sync_stream)
        losses.append(replica.inner_steps(local, h_used, batch))
        steps += h_used
        recs.append(eng.finish_round(local))
    torch.cuda.synchronize()
    return eng.anchor, losses, recs


def train_allreduce_per_step(layout: api.Layout, mlp: MLP, params: torch.Tensor,
                             replica: Replica, total_steps: int, batch: int, record_every: int,
                             world: int = 1, rank: int = 0, hyper: api.AdamWHyper | None = None,
                             exact: bool = True, group=None):
    """The per-step all-reduce baseline (run_allreduce_per_step, engine.cpp:517-591; mode
    allreduce-per-step): every inner step each worker computes its
    gradient on its own batch, the gradients are averaged across the D workers and ONE
    AdamW step updates the shared parameters (one optimiser state, engine.cpp:521).

    exact=True averages as the reference does — all-gather of the D gradient slabs through
    the library's NCCL communicator (dlx_comm_allgather) and the worker-order fp64 mean
    (dlx_mean_slabs, engine.cpp:559-570): bit-identical gradients on every rank and to the
    reference's mean. exact=False uses an NCCL all-reduce (sum, then x 1/D) — the fast
    collective a real DDP baseline uses (summation order differs from the reference's).

    Returns (params, per-record mean train losses over workers and steps — RoundRecord
    train_loss every `record_every` steps, engine.cpp:576-589)."""
    ctx = layout.ctx
    n = params.numel()
    opt = api.AdamWState(params, hyper or replica.hyper)
    grads = torch.zeros_like(params)
    mean = torch.empty_like(params)
    gathered = None
    if world > 1 and exact:
        api.ensure_comm(ctx, rank, world, group)
        gathered = torch.empty(world * n, dtype=torch.float32, device=params.device)
    losses, block, in_block, steps = [], 0.0, 0, 0
    while steps < total_steps:
        xb, yb = replica.next_batch(batch)
        loss = mlp.forward_backward(params, xb, yb, grads)
        if world > 1:
            import torch.distributed as dist
            if exact:
                api.comm_allgather(ctx, grads, gathered)
                api.mean_slabs(ctx, gathered, world, n, out=mean)
            else:
                mean.copy_(grads)
                dist.all_reduce(mean, group=group)
                mean.mul_(1.0 / world)
            lt = torch.tensor([loss], dtype=torch.float64, device=params.device)
            dist.all_reduce(lt, group=group)  # sum of the workers' losses (engine.cpp:575)
            loss_sum = float(lt.item())
        else:
            api.mean_slabs(ctx, grads, 1, n, out=mean)
            loss_sum = loss
        api.adamw_step(ctx, opt, params, mean)
        steps += 1
        in_block += 1
        block += loss_sum
        if steps % record_every == 0 or steps == total_steps:
            losses.append(block / (in_block * world))
            block, in_block = 0.0, 0
    torch.cuda.synchronize()
    return params, losses
