"""Device-resident outer-synchronisation engine: one process = one DiLoCoX worker = one GPU.

Mirrors the hot-path part of the reference engine (engine.cpp): RoundState (engine.hpp:114-132)
restricted to the outer state, collective_average (:215-263), stage_deltas (:266-276),
push_rank_window / adapt_compression (:278-308) and the round orderings
run_round_overlapped (:458-509) / run_round_sync (:423-456). Inner training is out of
scope: the caller hands in each round's local parameters (a device slab).

Exchange: the reference's "all-reduce" is a mean of per-worker reconstructions
(collective.cpp:17-46), so workers all-gather their compressed payloads (NCCL over NVLink
via torch.distributed) and every rank reconstructs the same Delta with K = D*r; worker 0's
float Q factors are broadcast as the next warm start (engine.cpp:498-501). The exchange and
the effective-rank measurement run on a side stream.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import api
from .api import NEAREST, OVERLAPPED, STOCHASTIC, SYNC, QuantSpec


def exchange(payload: torch.Tensor, gathered: torch.Tensor, warm_q: torch.Tensor | None,
             world: int, group=None) -> torch.Tensor:
    """The round's only data exchange (collective_average, engine.cpp:215-263): all-gather
    of every worker's compressed payload into `gathered` — worker w's bytes at
    [w * len(payload), (w + 1) * len(payload)), worker order = rank order, the order
    allreduce_avg sums in (collective.cpp:17-46) — and broadcast of worker 0's float Q
    factors as everyone's next warm start (engine.cpp:498-501). Byte-format agnostic; NCCL
    over NVLink on GPUs, gloo on CPU tensors."""
    if world == 1:
        return payload
    import torch.distributed as dist
    pb = payload.numel()
    g = gathered[:world * pb]
    dist.all_gather_into_tensor(g, payload, group=group)
    if warm_q is not None and warm_q.numel() > 0:
        dist.broadcast(warm_q, src=0, group=group)
    return g


@dataclass
class OuterConfig:
    """The config keys the path accepts (config.cpp:209-235); defaults engine.hpp:21-36,
    compress.hpp:21-27, optim.hpp:30-34."""
    rank1: int = 64
    qbits: int = 4
    rounding: int = STOCHASTIC
    power_iters: int = 2
    H1: int = 125
    adaptive: bool = True
    window_c: int = 5
    tau: float = 0.5
    H_min: int = 0
    outer_lr: float = 0.7
    outer_momentum: float = 0.9
    outer_classical: bool = False
    seed: int = 1
    overlap: bool = True      # dilocox (overlapped) vs dilocox-no-overlap (sync)
    compress: bool = True     # False: dilocox-no-compress ablation (raw fp32 exchange)
    measure_error: bool = True
    # benchmarking aid: run the adaptive measurement + controller every round but keep
    # operating at rank1 (the controller's choice is recorded in RoundRecord.r_next)
    hold_rank: bool = False
    # build every rank's device plan up front (OuterSync.prepare) when the controller is
    # applied, so a rank change does not stall the host between rounds
    prepare_ranks: bool = True
    # world == 1: measure the round's effective rank on the high-priority side stream, forked
    # after compress; the outer update's operand prep fills the SMs the eigenproblems' few
    # CTAs leave idle (bench, controller applied, 4 alternating runs each on one box: 10.44
    # vs 10.47 ms/round mean — within the box's clock noise, kept as the default)
    er_beside: bool = True

    def resolved_H_min(self) -> int:
        return self.H_min if self.H_min > 0 else (self.H1 + 9) // 10


_STAT_FIELDS = ("comp_error", "bound_violated", "err_buf_norm", "max_delta_norm", "nonfinite")


@dataclass
class RoundRecord:
    """Hot-path fields of RoundRecord (engine.hpp:74-95).

    comp_error / err_buf_norm describe THIS rank's worker (its own payload and error buffer);
    the reference's record reports worker 0 (engine.cpp:239, finish_record), so rank 0's
    records are the ones that follow reference semantics.

    The statistics the fused outer update reduces on the device (comp_error, bound_violated,
    err_buf_norm, max_delta_norm, nonfinite) are read back lazily: the engine does not wait
    for the round's main stream, so the host enqueues round t+1 while round t's outer update
    runs. Reading one of those fields (or resolve()) waits for the round's device work and
    raises NumericError if it produced non-finite parameters."""
    round: int = 0
    r_t: int = 0
    H_t: int = 0
    payload_bytes: float = 0.0
    omega_sq: float = 0.0
    averaged: bool = False
    _stats: dict = field(default_factory=dict, repr=False)
    _pending: object = field(default=None, repr=False)  # (event, host stats view, mode)
    # r', r_next, H_next: with the rank held (OuterConfig.hold_rank) the effective rank is
    # merged after the outer update and read back lazily; reading one of them drains it
    _ctl: dict = field(default_factory=lambda: {"r_prime": 0, "r_next": 0, "H_next": 0},
                       repr=False)
    _drain: object = field(default=None, repr=False)

    def _ctl_get(self, name):
        if self._drain is not None:
            self._drain()
        return self._ctl[name]

    r_prime = property(lambda self: self._ctl_get("r_prime"),
                       lambda self, v: self._ctl.__setitem__("r_prime", v))
    r_next = property(lambda self: self._ctl_get("r_next"),
                      lambda self, v: self._ctl.__setitem__("r_next", v))
    H_next = property(lambda self: self._ctl_get("H_next"),
                      lambda self, v: self._ctl.__setitem__("H_next", v))

    def resolve(self) -> "RoundRecord":
        if self._pending is not None:
            ev, st, mode = self._pending
            self._pending = None
            ev.synchronize()
            st = st.copy()
            d = {"comp_error": 0.0, "bound_violated": False, "err_buf_norm": 0.0,
                 "max_delta_norm": 0.0, "nonfinite": 0}
            if self.averaged:
                d["comp_error"] = float(st[0] / st[1]) if st[1] > 0 else 0.0
                d["bound_violated"] = self.omega_sq > 0 and d["comp_error"] > self.omega_sq
                d["err_buf_norm"] = math.sqrt(st[3])
                d["nonfinite"] = int(st[4])
                if mode == OVERLAPPED:
                    d["max_delta_norm"] = math.sqrt(st[2])
            self._stats.update(d)
            if d["nonfinite"]:
                from ._lib import NumericError
                raise NumericError(f"outer update produced {d['nonfinite']} non-finite parameters")
        return self

    def __getattr__(self, name):
        if name in _STAT_FIELDS:
            self.resolve()
            return self._stats.get(name, 0 if name == "nonfinite" else 0.0)
        raise AttributeError(name)


class OuterSync:
    ER_SLOTS = 8  # effective-rank results in flight (rank held: read back lazily)
    # per-round statistics in flight: the host may run this many rounds minus two ahead of
    # the device, so a host stall (a clock query, a scheduler hiccup) is absorbed by queued
    # rounds instead of idling the GPU and, at N > 1, every other rank at the next all-gather
    STATS_SLOTS = 8

    def __init__(self, layout: api.Layout, cfg: OuterConfig, anchor: torch.Tensor,
                 world: int = 1, rank: int = 0, group=None, side_stream: bool | None = None,
                 shard_effective_rank: bool = True):
        self.L = layout
        self.cfg = cfg
        self.world, self.rank, self.group = world, rank, group
        dev = anchor.device
        self.anchor = anchor
        self.velocity = torch.zeros_like(anchor)
        self.pending = torch.zeros_like(anchor)
        self.r_t = cfg.rank1
        self.H_t = cfg.H1
        self.round = 0
        self.has_pending = False
        self.window: list[int] = []
        self.warm_rank = 0
        qel = max(layout.q_factor_elems(cfg.rank1), 1)
        self.warm_q = torch.zeros(qel, dtype=torch.float32, device=dev)
        pb = layout.payload_bytes(cfg.rank1, cfg.qbits)
        self.payload = torch.zeros(pb, dtype=torch.uint8, device=dev)
        self.gathered = torch.zeros(world * pb, dtype=torch.uint8, device=dev)
        self.stats = torch.zeros(8, dtype=torch.float64, device=dev)
        self.draws = torch.zeros(1, dtype=torch.int64, device=dev)  # RNG draws of the last compress
        # Side stream for the effective-rank measurement. At world == 1 it is forked right
        # after compress (OuterConfig.er_beside), ahead of the outer update's operand prep on
        # the main stream, which overlaps it. (Launched after the persistent outer update
        # instead — ~215 KB of shared memory per SM — side kernels cannot co-reside and only
        # serialise behind it: measured 0.1-0.2 ms slower.) At world > 1 the eigenproblems are
        # split across the ranks (every rank holds the same all-gather buffer).
        if side_stream is None:
            side_stream = world > 1 or cfg.er_beside
        self.er_beside = world == 1 and cfg.er_beside and side_stream
        # high priority: the measurement's few CTAs are dispatched ahead of the outer update's
        # persistent grid, so the host learns r' (next round's rank) early in the round
        self.side = torch.cuda.Stream(device=dev, priority=-1) if side_stream else None
        if os.environ.get("DLX_ER_SHARD") == "0":  # experiments
            shard_effective_rank = False
        self.er_shards = world if (shard_effective_rank and world > 1) else 1
        self._bcast_work = None  # in-flight warm-start broadcast (waited before next compress)
        self._warm_elems = 0     # worker-0 Q elements gathered-but-not-yet-broadcast
        # worker sync through the library's own NCCL communicator (dlx_exchange: all-gather +
        # warm-Q broadcast on its side stream). torch.distributed only bootstraps it (ships
        # rank 0's unique id); DLX_LIB_NCCL=0 keeps the exchange in torch.distributed.
        self.lib_comm = (world > 1 and anchor.is_cuda and
                         os.environ.get("DLX_LIB_NCCL", "1") == "1")
        if self.lib_comm:
            api.ensure_comm(layout.ctx, rank, world, group)
        # warm-start broadcast right after the all-gather, before the outer update: 57 MB at
        # OPT-1.3B r=32 (~0.1 ms over NVLink); issued asynchronously it ran beside the outer
        # update's persistent grid and was the other source of multi-ms rank stalls
        self.bcast_sync = os.environ.get("DLX_BCAST_SYNC", "1") == "1"
        # per-round host copies of the device stats, double-buffered (records resolve lazily)
        self.stats_host = torch.zeros((self.STATS_SLOTS, 8), dtype=torch.float64,
                                      pin_memory=True)
        self._unresolved: list = []  # records whose device statistics are not read yet
        n2 = sum(1 for s in layout.shapes if len(s) == 2)
        self._n2 = n2
        # per-tensor effective ranks (as doubles) | energies: device results and host copy
        self.er_dev = torch.zeros(2 * max(n2, 1), dtype=torch.float64, device=dev)
        self.er_per = torch.zeros(max(n2, 1), dtype=torch.int32, device=dev)
        self.er_host = torch.zeros((self.ER_SLOTS, 2 * max(n2, 1)), dtype=torch.float64,
                                   pin_memory=True)
        self._er_fifo: list = []  # (record, event, host slot) awaiting their r'
        self._er_slot = 0
        self.last = RoundRecord()
        self.phase_events = None  # optional: list collecting (name, event) on the main stream
        self.side_events: list = []  # (start, end) of the effective rank on the side stream
        # host-resident parameter pipeline (step_host): copy streams + staging buffer
        self._h2d = self._d2h = None
        self._dev_local = None
        self._d2h_ev = None
        self._host_h2d_last = None
        self._pre_update: list = []  # events the next read of local / write of anchor waits on
        self._host_job = None        # per-step chunk schedule while step_host runs
        self.host_chunks = 8         # tensor groups of the chunked host pipeline
        self._groups = None
        self._begun = None           # begin_round state awaiting finish_round
        self.overlap_events = None   # optional: (before, after) of each finish_round join
        if (cfg.prepare_ranks and cfg.adaptive and not cfg.hold_rank and cfg.compress and
                anchor.is_cuda and self._n2):
            self.prepare()

    PREPARE_MAX_RANK = 64

    def prepare(self, ranks=None) -> None:
        """Build the device plans of every rank the adaptive schedule can reach (r1 down to 1,
        capped at PREPARE_MAX_RANK): plan tables, tensor-core tile lists, Gram jobs, the
        cold-start redo graph, effective-rank jobs and the outer update's shared-memory
        plan. The controller only moves r_t at round boundaries (engine.cpp:476-487,
        506-507) and each new rank would otherwise build all of that on the host between
        two rounds. Dry runs on the engine's own buffers, before round 1: compress of a
        noise-filled pending delta, the effective rank of an all-zero exchange, and a
        sync-mode outer update with a zero Delta and zero velocity — an exact no-op on the
        anchor and the pending delta (which is re-zeroed)."""
        cfg, L = self.cfg, self.L
        if self.round != 0:
            raise api._lib.ValidationError("prepare: only before the first round")
        if ranks is None:
            top = min(cfg.rank1, self.PREPARE_MAX_RANK)
            ranks = range(top, 0, -1)  # largest first: scratch buffers never grow afterwards
        api.fill_gaussian(L, self.pending, 1e-3, seed=0x5EED, tag=0x9E9A, worker=self.rank)
        nb = max(self._n2, 1)
        for r in ranks:
            pb = L.payload_bytes(r, cfg.qbits)
            qel = L.q_factor_elems(r)
            api.compress(L, self.pending, r, QuantSpec(cfg.qbits, cfg.rounding), None, 0,
                         cfg.power_iters, 0x1234, payload=self.payload[:pb],
                         q_out=self.warm_q[:max(qel, 1)])
            g = self.gathered[:self.world * pb] if self.world > 1 else self.payload[:pb]
            g.zero_()
            sharded = self.side is not None and self.er_shards > 1
            for shd in ((True, False) if sharded else (False,)):
                api.effective_rank_device(L, g, self.world, r, cfg.qbits, cfg.tau,
                                          shard=self.rank if shd else 0,
                                          nshards=self.er_shards if shd else 1,
                                          per=self.er_per, energy=self.er_dev[nb:])
            api.outer_update(L, g, self.world, r, cfg.qbits, self.pending, self.anchor, None,
                             self.velocity, cfg.outer_lr, cfg.outer_momentum,
                             cfg.outer_classical, mode=SYNC,
                             self_index=self.rank if cfg.measure_error else -1, stats=self.stats)
        self.pending.zero_()
        torch.cuda.synchronize(self.anchor.device)

    def _wait_pre_update(self):
        cur = torch.cuda.current_stream()
        for e in self._pre_update:
            cur.wait_event(e)
        self._pre_update = []

    def _ev(self, name: str):
        # NVTX marks of the round's phases on the host timeline (free without a tool)
        torch.cuda.nvtx.mark(f"dlx round {self.round}: {name}")
        if self.phase_events is None:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record(torch.cuda.current_stream())
        self.phase_events.append((name, e))
        return e

    # -- pieces -------------------------------------------------------------------------
    def _omega_sq(self, r: int) -> float:
        # size-weighted per-tensor bound with d = min(a, b) (engine.cpp:242-253)
        w = s = 0.0
        for sh in self.L.shapes:
            if len(sh) != 2:
                continue
            a, b = sh
            re = min(r, a, b)
            sz = a * b
            s += sz * (1.0 - (re / min(a, b)) * 2.0 ** (-self.cfg.qbits))
            w += sz
        return s / w if w > 0 else 0.0

    def _exchange(self, pb: int, qel: int):
        """All-gather payloads (the outer update waits for it); broadcast worker-0 Q (warm
        start) asynchronously — only the next round's compress needs it. NCCL over NVLink."""
        if self.world == 1:
            return self.payload[:pb]
        if self.lib_comm:
            # worker 0's Q is only needed if the next round is warm (same rank): its broadcast
            # waits until the controller has decided (_broadcast_warm, before the next
            # compress) — a rank change skips it
            self._warm_elems = qel
            return api.exchange(self.L.ctx, self.payload[:pb], self.gathered, None)
        if self.bcast_sync:
            return exchange(self.payload[:pb], self.gathered, self.warm_q[:qel] if qel else None,
                            self.world, self.group)
        g = exchange(self.payload[:pb], self.gathered, None, self.world, self.group)
        if qel > 0:
            import torch.distributed as dist
            self._bcast_work = dist.broadcast(self.warm_q[:qel], src=0, group=self.group,
                                              async_op=True)
        return g

    def _broadcast_warm(self, r: int):
        """Broadcast worker 0's float Q as everyone's warm start (engine.cpp:498-501) if this
        round uses it (warm_rank == r_t, compress.cpp:161); dropped on a rank change."""
        qel, self._warm_elems = self._warm_elems, 0
        if qel and self.warm_rank == r:
            api.exchange(self.L.ctx, self.payload[:0], self.gathered, self.warm_q[:qel])

    def _wait_bcast(self):
        if self.lib_comm:
            self.L.ctx.wait_warm()
            return
        if self._bcast_work is not None:
            self._bcast_work.wait()  # the current stream waits; the host does not
            self._bcast_work = None

    def _collective_average_raw(self, local: torch.Tensor | None, mode: int) -> RoundRecord:
        """dilocox-no-compress (engine.cpp:231-233): compress_raw payloads, reference-exact
        average (all-gather of the raw slabs, fp64 sum in worker order), fused epilogue;
        no measurement (adaptive needs compression, engine.cpp:50)."""
        L, cfg = self.L, self.cfg
        self._ev("compress")
        payload = api.compress_raw(L, self.pending)
        self._ev("exchange")
        if self.world > 1:
            import torch.distributed as dist
            if getattr(self, "_gathered_raw", None) is None:
                self._gathered_raw = torch.empty(self.world * L.slab_elems, dtype=torch.float32,
                                                 device=self.anchor.device)
            if self.lib_comm:
                api.comm_allgather(L.ctx, payload, self._gathered_raw)
            else:
                dist.all_gather_into_tensor(self._gathered_raw, payload, group=self.group)
            gathered = self._gathered_raw
        else:
            gathered = payload
        cur = torch.cuda.current_stream()
        self._ev("outer_update")
        self._wait_pre_update()
        api.outer_update_raw(L, gathered, self.world, self.pending, self.anchor, local,
                             self.velocity, cfg.outer_lr, cfg.outer_momentum, cfg.outer_classical,
                             mode=mode, self_index=self.rank if cfg.measure_error else -1,
                             stats=self.stats, stream=cur)
        self._ev("end")
        self.stats_host[self.round % self.STATS_SLOTS].copy_(self.stats, non_blocking=True)
        return RoundRecord(round=self.round, r_t=0, H_t=self.H_t, averaged=True,
                           payload_bytes=api.payload_bits_raw(L) / 8.0, omega_sq=0.0)

    def collective_average(self, local: torch.Tensor | None, mode: int) -> RoundRecord:
        """Compress (shared stream per round), exchange, measure, fused outer update."""
        if not self.cfg.compress:
            return self._collective_average_raw(local, mode)
        return self._sync_finish(self._sync_begin(early_rank=self._early_rank()), local, mode)

    EARLY_RANK_MAX_K = 128

    def _early_rank(self) -> bool:
        """Measure r' before the outer update (the host then has r_{t+1} while the outer
        update runs): always at N = 1; at N > 1 when the controller is applied and the
        eigenproblems are small (K = N r_t <= 128: measured faster at N = 2 and 4 than the
        host-side wait for r' after the outer update). Larger K (one CTA per tensor:
        ~1 ms at K = 128, ~3 ms at K = 256 whatever the shard size) stays beside the outer
        update on the side stream."""
        if self.side is None:
            return True
        return not self.cfg.hold_rank and self.world * self.r_t <= self.EARLY_RANK_MAX_K

    def _sync_begin(self, early_rank: bool, xstream=None) -> dict:
        """First half of collective_average (engine.cpp:215-263): compress of the pending
        delta (shared RNG stream per round, engine.cpp:226) on the CURRENT stream, then the
        exchange (all-gather of the payloads + worker-0 warm-Q broadcast) and — when
        `early_rank` — the unsharded effective rank, queued for the host before the outer
        update. With `xstream` the exchange and the measurement run on that stream (after the
        compress), so they proceed concurrently with whatever the current stream does next —
        the round's inner steps (one-step-delay overlap); the returned state carries the
        event finish_round joins."""
        cfg, L = self.cfg, self.L
        r, q = self.r_t, cfg.qbits
        pb = L.payload_bytes(r, q)
        qel = L.q_factor_elems(r)
        s0 = api.rng_stream(cfg.seed, api.stream_key(0xC09C, self.round))  # engine.cpp:226
        if self.lib_comm:
            self._broadcast_warm(r)
        self._wait_bcast()
        self._ev("compress")
        # compress in place over the warm buffer: each rank overwrites it with its own Q,
        # then rank 0's copy is broadcast (engine.cpp:498-501)
        api.compress(L, self.pending, r, QuantSpec(q, cfg.rounding),
                     self.warm_q if self.warm_rank == r else None, self.warm_rank,
                     cfg.power_iters, s0, payload=self.payload[:pb], q_out=self.warm_q[:max(qel, 1)],
                     draws=self.draws)
        rec = RoundRecord(round=self.round, r_t=r, H_t=self.H_t, averaged=True,
                          payload_bytes=L.payload_bits(r, q) / 8.0, omega_sq=self._omega_sq(r))
        measure = cfg.adaptive and self._n2 > 0
        main = torch.cuda.current_stream()
        st = dict(r=r, q=q, rec=rec, measure=measure, late_rank=measure and not early_rank)
        if xstream is not None:
            xstream.wait_stream(main)
        with torch.cuda.stream(xstream if xstream is not None else main):
            cur = torch.cuda.current_stream()
            self._ev("exchange")
            gathered = self._exchange(pb, qel)
            if measure and early_rank:
                # Unsharded measurement BEFORE the outer update: r' (and so the controller's
                # next rank, engine.cpp:476-487) reaches the host while the outer update still
                # runs, so applying the controller costs no host round trip on the device
                # timeline. (The persistent outer-update grid holds every SM, so a side stream
                # would only serialise behind it.)
                self._ev("effective_rank")
                if self.er_beside and xstream is None:
                    self.side.wait_stream(cur)
                    with torch.cuda.stream(self.side):
                        self._effective_rank(gathered, r, q, self.side, sharded=False)
                        self._queue_er(rec, self.side)
                    st["er_side"] = True
                else:
                    # at N > 1 the ranks split the eigenproblems and sum the per-tensor results
                    # right away (exact: one nonzero term per entry)
                    sharded = self.er_shards > 1
                    self._effective_rank(gathered, r, q, cur, sharded=sharded)
                    if sharded:
                        self._sum_er_shards()
                    self._queue_er(rec, cur)
            if xstream is not None:
                done = torch.cuda.Event(enable_timing=True)
                done.record(xstream)
                st["joined"] = done
        self.warm_rank = r
        st["gathered"] = gathered
        return st

    def _sync_finish(self, st: dict, local: torch.Tensor | None, mode: int) -> RoundRecord:
        """Second half: the fused outer update (error feedback, staging, Nesterov) on the
        current stream, plus the sharded effective rank beside it at N > 1."""
        cfg = self.cfg
        r, q, gathered, rec = st["r"], st["q"], st["gathered"], st["rec"]
        cur = torch.cuda.current_stream()
        side = self.side
        if st["late_rank"]:
            # sharded across the ranks, on a high-priority side stream beside the outer update
            side = side or cur
            side.wait_stream(cur)
            with torch.cuda.stream(side):
                self._effective_rank(gathered, r, q, side, sharded=True)
        self._ev("outer_update")
        self._outer_update(gathered, r, q, local, mode, cur)
        if st.get("er_side"):
            cur.wait_stream(self.side)
        self._ev("end")
        self.stats_host[self.round % self.STATS_SLOTS].copy_(self.stats, non_blocking=True)
        if st["late_rank"]:
            # the shards' per-tensor (k, energy) are summed AFTER the outer update, on the main
            # stream: no collective runs beside its persistent grid (an NCCL all-reduce there,
            # or a per-round CPU/gloo one, measured 20-260 ms rank stalls)
            cur.wait_stream(side)
            if self.er_shards > 1:
                self._sum_er_shards()
            self._queue_er(rec, cur)
        elif cfg.adaptive and cfg.compress and self._n2 == 0:
            # no 2-D tensor: effective_rank's aggregate is 1 (compress.cpp:333-339), pushed
            # every averaged round (engine.cpp:258-261, 480-482)
            rec.r_prime = 1
            self._push_window(1)
            rec.r_next, rec.H_next = self._adapt()
        return rec

    def _sum_er_shards(self):
        """Sum the ranks' per-tensor (k, energy) shards on the current stream: one nonzero
        term per entry, so the sum is exact and identical on every rank."""
        if self.lib_comm:
            api.comm_allreduce_sum_f64(self.L.ctx, self.er_dev)
        else:
            import torch.distributed as dist
            dist.all_reduce(self.er_dev, group=self.group)

    def _effective_rank(self, gathered, r: int, q: int, stream, sharded: bool):
        """Factor-space effective rank (dlx_effective_rank_shard) into er_dev; sharded: this
        rank measures only its 1/world of the tensors (the others read 0)."""
        cfg, L = self.cfg, self.L
        e0 = e1 = None
        if self.phase_events is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        nb = max(self._n2, 1)
        api.effective_rank_device(L, gathered, self.world, r, q, cfg.tau, stream=stream,
                                  shard=self.rank if (sharded and self.er_shards > 1) else 0,
                                  nshards=self.er_shards if sharded else 1, per=self.er_per,
                                  energy=self.er_dev[nb:])
        self.er_dev[:nb].copy_(self.er_per)
        if e0 is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(stream)
            self.side_events.append((e0, e1))

    def _queue_er(self, rec: RoundRecord, stream):
        """Copy the round's per-tensor (k, energy) to pinned host memory behind an event;
        the host resolves r' from it (lazily while the rank is held)."""
        if len(self._er_fifo) >= self.ER_SLOTS:
            self._drain_er(block=True, upto=1)
        slot = self._er_slot
        self._er_slot = (slot + 1) % self.ER_SLOTS
        self.er_host[slot].copy_(self.er_dev, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
        self._er_fifo.append((rec, ev, slot))
        rec._drain = lambda: self._drain_er(block=True)

    def _drain_er(self, block: bool, upto: int | None = None):
        """Resolve pending effective ranks in round order: r' into the window, then the
        controller's (r_next, H_next) for that round (engine.cpp:278-308)."""
        n = 0
        while self._er_fifo and (upto is None or n < upto):
            rec, ev, slot = self._er_fifo[0]
            if not block and not ev.query():
                break
            ev.synchronize()
            self._er_fifo.pop(0)
            h = self.er_host[slot].numpy()
            nb = max(self._n2, 1)
            er = api.effective_rank_reduce(self.L, h[:self._n2].astype(np.int32),
                                           h[nb:nb + self._n2], self.cfg.rank1)
            rec._drain = None
            rec.r_prime = er.aggregate
            self._push_window(er.aggregate)
            rec.r_next, rec.H_next = self._adapt()
            n += 1

    def flush(self):
        """Wait for every pending effective rank (RoundRecord r' / r_next / H_next)."""
        self._drain_er(block=True)

    def _outer_update(self, gathered, r: int, q: int, local, mode: int, cur):
        cfg, L = self.cfg, self.L
        kw = dict(mode=mode, self_index=self.rank if cfg.measure_error else -1,
                  stats=self.stats, stream=cur)
        job = self._host_job
        if job is None:
            self._wait_pre_update()
            api.outer_update(L, gathered, self.world, r, q, self.pending, self.anchor, local,
                             self.velocity, cfg.outer_lr, cfg.outer_momentum,
                             cfg.outer_classical, **kw)
            return
        # chunked host pipeline: each tensor group is updated as soon as its H2D copy has
        # landed, and its new anchor starts back to the host right after
        for e in job["prev"]:
            cur.wait_event(e)
        self._pre_update = []
        for (t0, t1, e0, e1), ev in zip(self._groups, job["h2d"]):
            cur.wait_event(ev)
            api.outer_update(L, gathered, self.world, r, q, self.pending, self.anchor, local,
                             self.velocity, cfg.outer_lr, cfg.outer_momentum,
                             cfg.outer_classical, tensors=(t0, t1), **kw)
            if job["out"] is not None:
                ue = torch.cuda.Event()
                ue.record(cur)
                self._d2h.wait_event(ue)
                with torch.cuda.stream(self._d2h):
                    job["out"][e0:e1].copy_(self.anchor[e0:e1], non_blocking=True)
        if job["out"] is not None:
            self._d2h_ev = torch.cuda.Event()
            self._d2h_ev.record(self._d2h)
        job["done"] = True

    def _finish(self, rec: RoundRecord, mode: int) -> RoundRecord:
        # no host wait on the main stream: the record resolves its device statistics when
        # read. Records older than STATS_SLOTS - 2 rounds are resolved here (their host stats
        # slot is about to be reused; a non-finite update surfaces within that many rounds).
        while self._unresolved and self._unresolved[0].round <= rec.round - (self.STATS_SLOTS - 2):
            self._unresolved.pop(0).resolve()
        if self.lib_comm:
            self.L.ctx.comm_check()  # surfaces an asynchronous NCCL failure (NcclError)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        rec._pending = (ev, self.stats_host[rec.round % self.STATS_SLOTS].numpy(), mode)
        self._unresolved.append(rec)
        self.last = rec
        return rec

    def _adapt(self):
        cfg = self.cfg
        if not cfg.adaptive or not cfg.compress:
            return self.r_t, self.H_t
        return api.adapt_compression(self.window, cfg.rank1, cfg.H1, cfg.window_c,
                                     cfg.resolved_H_min())

    def _apply_next(self, rec: RoundRecord, r_next: int, h_next: int):
        rec.r_next, rec.H_next = r_next, h_next
        if not self.cfg.hold_rank:
            self.r_t, self.H_t = r_next, h_next

    def _push_window(self, r_prime: int):
        self.window.append(r_prime)
        if len(self.window) > self.cfg.window_c:
            del self.window[:len(self.window) - self.cfg.window_c]

    # -- rounds -------------------------------------------------------------------------
    def round_overlapped(self, local: torch.Tensor) -> RoundRecord:
        """run_round_overlapped (engine.cpp:458-509) minus inner training: the sync of the
        previous round's delta, then staging of this round's delta against the pre-update
        anchor, then the one-step-delayed Nesterov step — all fused in one device pass."""
        if self._begun is None:
            self.begin_round()
        return self.finish_round(local)

    def begin_round(self, stream: torch.cuda.Stream | None = None) -> None:
        """Start round t's outer sync of delta^{t-1}: compress on the current stream, then
        the exchange of the compressed factors (NCCL) and the effective rank on `stream`
        (default: the current stream too). These read only the pending delta and the warm Q,
        so with a separate stream the exchange runs concurrently with the round's inner steps
        on the main stream: the one-step-delay overlap (engine.cpp:464-468).
        finish_round(local) joins it before the fused outer update."""
        if self._begun is not None:
            raise api._lib.ValidationError("begin_round: the previous round was not finished")
        self.round += 1
        st = None
        if self.has_pending and self.cfg.overlap and self.cfg.compress:
            if stream is None:
                st = self._sync_begin(early_rank=self._early_rank())
            else:
                # compress stays on the main stream (HBM-bound like the inner steps: sharing
                # the device with them measured slower than running it first); the exchange
                # and the measurement move to `stream` and overlap the inner steps
                st = self._sync_begin(early_rank=True, xstream=stream)
        self._begun = {"sync": st}

    def finish_round(self, local: torch.Tensor) -> RoundRecord:
        """Complete the round begun by begin_round with this round's local parameters."""
        if self._begun is None:
            self.begin_round()
        st = self._begun["sync"]
        self._begun = None
        if not self.cfg.overlap:
            self.round -= 1
            return self.round_sync(local)
        if self.has_pending:
            if st is None:  # no-compress ablation
                rec = self.collective_average(local, OVERLAPPED)
            else:
                if "joined" in st:
                    cur = torch.cuda.current_stream()
                    if self.overlap_events is not None:
                        w0 = torch.cuda.Event(enable_timing=True)
                        w0.record(cur)
                    cur.wait_event(st["joined"])
                    if self.overlap_events is not None:
                        w1 = torch.cuda.Event(enable_timing=True)
                        w1.record(cur)
                        self.overlap_events.append((w0, w1))
                rec = self._sync_finish(st, local, OVERLAPPED)
            # rank held: r' is not needed before the next round (read lazily); else wait
            self._drain_er(block=not self.cfg.hold_rank)
        else:
            rec = RoundRecord(round=self.round, r_t=self.r_t, H_t=self.H_t)
            self._wait_pre_update()
            api.stage_deltas(self.L, self.anchor, local, None, self.pending, None)
        r_next, h_next = self._adapt()
        self.has_pending = True
        rec = self._finish(rec, OVERLAPPED)
        self._apply_next(rec, r_next, h_next)
        return rec

    def round_sync(self, local: torch.Tensor) -> RoundRecord:
        """run_round_sync (engine.cpp:423-456): stage with the carried error, average the
        fresh delta, then Nesterov (pending carries e between rounds)."""
        self.round += 1
        self._wait_pre_update()
        api.stage_deltas(self.L, self.anchor, local, self.pending if self.has_pending else None,
                         self.pending, None)
        self.has_pending = True
        rec = self.collective_average(None, SYNC)
        r_next, h_next = self.r_t, self.H_t
        if self.cfg.adaptive and self.cfg.compress:
            self._drain_er(block=not self.cfg.hold_rank)
            r_next, h_next = self._adapt()
        rec = self._finish(rec, SYNC)
        self._apply_next(rec, r_next, h_next)
        return rec

    def step(self, local: torch.Tensor) -> RoundRecord:
        return self.round_overlapped(local) if self.cfg.overlap else self.round_sync(local)

    def _host_groups(self):
        """Contiguous tensor groups of ~equal slab size: (t0, t1, e0, e1) with slab element
        range [e0, e1) (the last group runs to the end of the slab)."""
        if self._groups is None:
            L = self.L
            nt = len(L.shapes)
            target = L.slab_elems / max(1, self.host_chunks)
            groups, t0 = [], 0
            for t in range(1, nt + 1):
                end = int(L.offsets[t]) if t < nt else L.slab_elems
                if t == nt or end - int(L.offsets[t0]) >= target:
                    groups.append((t0, t, int(L.offsets[t0]) if t0 else 0, end))
                    t0 = t
            self._groups = groups
        return self._groups

    def step_host(self, h_local: torch.Tensor, h_anchor_out: torch.Tensor | None = None
                  ) -> RoundRecord:
        """One round with the worker's local parameters in (pinned) host memory — the
        drop-in call a host-resident reference engine makes. The local parameters go to the
        device in tensor groups on a copy stream while compress runs (overlapped mode reads
        local only in the fused outer update); each group's outer update starts as soon as
        its copy has landed, and its new anchor goes back to `h_anchor_out` on a second copy
        stream right after, overlapping the remaining copies and the next round. host_wait()
        orders the caller's stream after the last D2H."""
        dev = self.anchor.device
        if self._h2d is None:
            self._h2d = torch.cuda.Stream(device=dev)
            self._d2h = torch.cuda.Stream(device=dev)
            self._dev_local = torch.empty_like(self.anchor)
        groups = self._host_groups()
        cur = torch.cuda.current_stream()
        self._h2d.wait_stream(cur)  # the previous round's reads of the staging buffer
        evs = []
        with torch.cuda.stream(self._h2d):
            for _, _, e0, e1 in groups:
                self._dev_local[e0:e1].copy_(h_local[e0:e1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self._h2d)
                evs.append(ev)
        self._host_h2d_last = evs[-1] if evs else None
        prev = [self._d2h_ev] if self._d2h_ev is not None else []
        self._pre_update = evs + prev  # for the un-chunked paths (staging round, sync mode)
        job = {"h2d": evs, "prev": prev, "out": h_anchor_out, "done": False}
        self._host_job = job if (self.cfg.overlap and self.cfg.compress) else None
        try:
            rec = self.step(self._dev_local)
        finally:
            self._host_job = None
        if h_anchor_out is not None and not job["done"]:
            self._d2h.wait_stream(cur)
            with torch.cuda.stream(self._d2h):
                h_anchor_out.copy_(self.anchor, non_blocking=True)
            self._d2h_ev = torch.cuda.Event()
            self._d2h_ev.record(self._d2h)
        return rec

    def host_wait(self, stream=None):
        """Make `stream` (default: current) wait for the last step_host D2H (device-side
        ordering only; the host does not block)."""
        if self._d2h_ev is not None:
            (stream or torch.cuda.current_stream()).wait_event(self._d2h_ev)

    def host_sync(self):
        """Block the host until the last step_host call's copies are done: afterwards the
        caller may overwrite the `h_local` it passed and read `h_anchor_out`. (step_host
        returns as soon as the work is enqueued; both host buffers are in use until then.)"""
        for e in self._pre_update:
            e.synchronize()
        if self._d2h_ev is not None:
            self._d2h_ev.synchronize()
        if self._host_h2d_last is not None:
            self._host_h2d_last.synchronize()
