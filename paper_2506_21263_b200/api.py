"""Host-side mirror of the reference compressor / worker-sync / outer-optimiser API
(reference proj/core: compress.hpp, collective.hpp, optim.hpp, engine.hpp) over
device-resident ParamSets. Every compute call goes through the C-ABI (include/dlx_b200.h);
torch is used only for device memory, streams and torch.distributed plumbing.

A ParamSet lives in one fp32 "slab" (a 1-D torch CUDA tensor) laid out by a Layout.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import check, lib

STOCHASTIC, NEAREST = 0, 1
OVERLAPPED, SYNC = 0, 1
GOLDEN = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


# ----------------------------------------------------------------------------- RNG (rng.hpp)
def _fmix(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _mix(z: int) -> int:
    return _fmix((z + GOLDEN) & M64)


def stream_key(*parts: int) -> int:
    """stream_key (rng.hpp:63-66)."""
    h = 0x100000001B3
    for p in parts:
        h = _mix(h ^ _mix(p & M64))
    return h


def rng_stream(seed: int, stream_id: int) -> int:
    """State of RngStream(seed, stream_id) after construction (rng.hpp:13-16)."""
    s = _mix((seed ^ GOLDEN) & M64)
    return _mix(s ^ _mix((stream_id + 0xBF58476D1CE4E5B9) & M64))


def _stream(s) -> C.c_void_p:
    if s is None:
        s = torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


# ----------------------------------------------------------------------------- context/layout
class Context:
    """One device context (dlx_ctx): workspaces and plan caches live here."""

    def __init__(self, device: int = 0):
        self.device = device
        h = C.c_void_p()
        check(lib().dlx_ctx_create(device, C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            lib().dlx_ctx_destroy(self.h)
            self.h = None

    # -- worker sync (dlx_comm_*; NCCL inside the library)
    def init_comm(self, rank: int, world: int, unique_id: bytes) -> None:
        """Join the D-worker communicator (collective: every rank calls it with rank 0's
        unique id)."""
        buf = C.create_string_buffer(bytes(unique_id), 128)
        check(lib().dlx_comm_init(self.h, rank, world, buf))
        self.rank, self.world = rank, world

    def comm_check(self) -> None:
        """Raise NcclError if the communicator reported an asynchronous failure."""
        check(lib().dlx_comm_check(self.h))

    def wait_warm(self, stream=None) -> None:
        check(lib().dlx_exchange_wait_warm(self.h, _stream(stream)))


def ensure_comm(ctx: Context, rank: int, world: int, group=None) -> None:
    """Give `ctx` the library's NCCL communicator for this D-worker group, bootstrapped
    through torch.distributed (rank 0's unique id is broadcast as an object); no-op if it
    already has one for `world` ranks or world == 1."""
    if world <= 1 or getattr(ctx, "world", 1) == world:
        return
    import torch.distributed as dist
    uid = [comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0, group=group)
    ctx.init_comm(rank, world, uid[0])


def comm_unique_id() -> bytes:
    """dlx_comm_unique_id: 128 opaque bytes rank 0 ships to every rank."""
    buf = C.create_string_buffer(128)
    check(lib().dlx_comm_unique_id(buf))
    return buf.raw


def exchange(ctx: Context, payload: torch.Tensor, gathered: torch.Tensor,
             warm_q: torch.Tensor | None, defer_warm: bool = False, stream=None) -> torch.Tensor:
    """dlx_exchange: all-gather of the payloads (worker order = rank order) + broadcast of
    worker 0's warm Q, on the library's side stream joined to `stream`."""
    pb = payload.numel()
    nw = gathered.numel() // max(pb, 1)
    wq = warm_q if (warm_q is not None and warm_q.numel() > 0) else None
    check(lib().dlx_exchange(ctx.h, _ptr(payload), pb, _ptr(gathered), _ptr(wq),
                             0 if wq is None else wq.numel(), 1 if defer_warm else 0,
                             _stream(stream)))
    return gathered[:nw * pb]


def comm_allgather(ctx: Context, send: torch.Tensor, recv: torch.Tensor, stream=None):
    check(lib().dlx_comm_allgather(ctx.h, _ptr(send), send.numel() * send.element_size(),
                                   _ptr(recv), _stream(stream)))
    return recv


def comm_allreduce_sum_f64(ctx: Context, buf: torch.Tensor, stream=None):
    assert buf.dtype == torch.float64
    check(lib().dlx_comm_allreduce_sum_f64(ctx.h, _ptr(buf), buf.numel(), _stream(stream)))
    return buf


@dataclass
class QuantSpec:
    """compress.hpp:21-27."""
    qbits: int = 4
    rounding: int = STOCHASTIC

    def levels(self) -> int:
        return (1 << (self.qbits - 1)) - 1


class Layout:
    """ParamSet tensor table (params.hpp:12-33) mapped onto one device slab."""

    def __init__(self, ctx: Context, table):
        self.ctx = ctx
        self.names = [n for n, _ in table]
        self.shapes = [tuple(int(d) for d in s) for _, s in table]
        if len(set(self.names)) != len(self.names):
            raise _lib.ValidationError("duplicate parameter name")
        nt = len(self.shapes)
        self.ndim = np.array([len(s) for s in self.shapes], np.int32)
        self.dims = np.zeros(2 * max(nt, 1), np.int64)
        for i, s in enumerate(self.shapes):
            self.dims[2 * i] = s[0]
            self.dims[2 * i + 1] = s[1] if len(s) == 2 else 1
        h = C.c_void_p()
        check(lib().dlx_layout_create(ctx.h, nt, self.ndim.ctypes.data_as(C.POINTER(C.c_int)),
                                      self.dims.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(h)))
        self.h = h
        self.nt = nt
        self.slab_elems = lib().dlx_layout_slab_elems(h)
        self.offsets = np.zeros(max(nt, 1), np.int64)
        check(lib().dlx_layout_offsets(h, self.offsets.ctypes.data_as(C.POINTER(C.c_int64))))
        self.numels = [int(np.prod(s)) for s in self.shapes]
        self.total_params = int(sum(self.numels))

    # -- slabs
    def empty(self, device=None) -> torch.Tensor:
        return torch.zeros(self.slab_elems, dtype=torch.float32,
                           device=device or f"cuda:{self.ctx.device}")

    def to_slab(self, arrays, device=None) -> torch.Tensor:
        host = np.zeros(self.slab_elems, np.float32)
        for i, a in enumerate(arrays):
            a = np.asarray(a, np.float32).reshape(-1)
            host[self.offsets[i]:self.offsets[i] + self.numels[i]] = a
        return torch.from_numpy(host).to(device or f"cuda:{self.ctx.device}")

    def from_slab(self, slab: torch.Tensor):
        host = slab.detach().cpu().numpy()
        return [host[self.offsets[i]:self.offsets[i] + self.numels[i]].reshape(self.shapes[i])
                for i in range(self.nt)]

    def pack(self, flat: np.ndarray, device=None) -> torch.Tensor:
        """Reference-order concatenation (no padding) -> padded slab."""
        out, o = [], 0
        for n in self.numels:
            out.append(flat[o:o + n])
            o += n
        return self.to_slab(out, device)

    def unpack(self, slab: torch.Tensor) -> np.ndarray:
        return np.concatenate([a.reshape(-1) for a in self.from_slab(slab)]) if self.nt else \
            np.zeros(0, np.float32)

    # -- geometry
    def payload_bytes(self, rank: int, qbits: int) -> int:
        n = lib().dlx_payload_bytes(self.h, rank, qbits)
        if n < 0:
            check(int(-n))
        return int(n)

    def payload_bits(self, rank: int, qbits: int) -> int:
        """payload_bits_formula (compress.cpp:92-114)."""
        return int(lib().dlx_payload_bits(self.h, rank, qbits))

    def segments(self, rank: int, qbits: int) -> np.ndarray:
        seg = np.zeros(4 * max(self.nt, 1), np.int64)
        check(lib().dlx_payload_segments(self.h, rank, qbits,
                                         seg.ctypes.data_as(C.POINTER(C.c_int64))))
        return seg.reshape(-1, 4)

    def factor_offsets(self, rank: int, side: int):
        off = np.zeros(max(self.nt, 1), np.int64)
        total = lib().dlx_factor_offsets(self.h, rank, side,
                                         off.ctypes.data_as(C.POINTER(C.c_int64)))
        if total < 0:
            check(int(-total))
        return off, int(total)

    def ranks(self, rank: int):
        return [min(rank, s[0], s[1]) if len(s) == 2 else 0 for s in self.shapes]

    def q_factor_elems(self, rank: int) -> int:
        return self.factor_offsets(rank, 1)[1]

    def factors_to_device(self, mats, rank: int, side: int, device=None) -> torch.Tensor:
        """List (per 2-D tensor, table order) of n x r row-major factors -> device buffer."""
        off, total = self.factor_offsets(rank, side)
        host = np.zeros(total, np.float32)
        k = 0
        for i, s in enumerate(self.shapes):
            if len(s) != 2:
                continue
            m = np.asarray(mats[k], np.float32)
            n, r = m.shape
            ld = (n + 31) // 32 * 32
            for j in range(r):
                host[off[i] + j * ld: off[i] + j * ld + n] = m[:, j]
            k += 1
        return torch.from_numpy(host).to(device or f"cuda:{self.ctx.device}")

    def factors_from_device(self, buf: torch.Tensor, rank: int, side: int):
        off, _ = self.factor_offsets(rank, side)
        host = buf.detach().cpu().numpy()
        out = []
        for i, s in enumerate(self.shapes):
            if len(s) != 2:
                continue
            n = s[side]
            r = min(rank, s[0], s[1])
            ld = (n + 31) // 32 * 32
            out.append(np.stack([host[off[i] + j * ld: off[i] + j * ld + n] for j in range(r)], 1))
        return out

    # -- wire format (compress.cpp:395-482)
    def serialize(self, payload: torch.Tensor, rank: int, qbits: int, names=None) -> bytes:
        host = payload.detach().cpu().numpy().astype(np.uint8, copy=False)
        nm = names if names is not None else self.names
        arr = (C.c_char_p * self.nt)(*[n.encode() for n in nm])
        args = [self.h, rank, qbits, arr, host.ctypes.data_as(C.c_void_p)]
        n = lib().dlx_serialize(*args, None, 0)
        if n < 0:
            check(int(-n))
        buf = np.zeros(n, np.uint8)
        lib().dlx_serialize(*args, buf.ctypes.data_as(C.c_void_p), n)
        return buf.tobytes()

    def parse(self, data: bytes, rank: int, qbits: int, device=None) -> torch.Tensor:
        src = np.frombuffer(data, np.uint8).copy()
        out = np.zeros(self.payload_bytes(rank, qbits), np.uint8)
        check(lib().dlx_parse(self.h, rank, qbits, src.ctypes.data_as(C.c_void_p), len(src),
                              out.ctypes.data_as(C.c_void_p)))
        return torch.from_numpy(out).to(device or f"cuda:{self.ctx.device}")

    def close(self):
        if self.h:
            lib().dlx_layout_destroy(self.h)
            self.h = None


# ----------------------------------------------------------------------------- compressor
@dataclass
class CompressResult:
    """compress.hpp:86-90 (payload + the float Q factors for the next warm start)."""
    payload: torch.Tensor
    q_factors: torch.Tensor
    draws: torch.Tensor  # device uint64: RNG draws consumed
    rank: int
    qbits: int


def fill_gaussian(layout: Layout, out: torch.Tensor, scale: float, seed: int, tag: int,
                  worker: int, base: torch.Tensor | None = None, stream=None):
    """out = base + scale * Tensor::gaussian, per-tensor streams
    RngStream(seed, stream_key({tag, worker, t})) — bit-identical to the reference."""
    check(lib().dlx_fill_gaussian(layout.ctx.h, layout.h, _ptr(out), _ptr(base), scale, seed,
                                  tag, worker, _stream(stream)))
    return out


def compress(layout: Layout, delta: torch.Tensor, rank: int, spec: QuantSpec,
             warm_q: torch.Tensor | None, warm_rank: int, power_iters: int, rng_state: int,
             payload: torch.Tensor | None = None, q_out: torch.Tensor | None = None,
             stream=None, draws: torch.Tensor | None = None) -> CompressResult:
    """compress (compress.cpp:146-183). q_out may alias warm_q (in-place warm refresh).
    draws (device int64[1], optional) receives the number of RNG draws consumed."""
    dev = delta.device
    if payload is None:
        payload = torch.empty(layout.payload_bytes(rank, spec.qbits), dtype=torch.uint8, device=dev)
    if q_out is None:
        q_out = torch.zeros(max(layout.q_factor_elems(rank), 1), dtype=torch.float32, device=dev)
    if draws is None:
        draws = torch.zeros(1, dtype=torch.int64, device=dev)
    check(lib().dlx_compress(layout.ctx.h, layout.h, _ptr(delta), rank, spec.qbits, spec.rounding,
                             power_iters, rng_state & M64, _ptr(warm_q), warm_rank, _ptr(payload),
                             _ptr(q_out), _ptr(draws), _stream(stream)))
    return CompressResult(payload, q_out, draws, rank, spec.qbits)


def quantize_factors(layout: Layout, p: torch.Tensor, q: torch.Tensor, delta: torch.Tensor,
                     rank: int, spec: QuantSpec, rng_state: int, cold: bool, stream=None):
    dev = delta.device
    payload = torch.zeros(layout.payload_bytes(rank, spec.qbits), dtype=torch.uint8, device=dev)
    draws = torch.zeros(1, dtype=torch.int64, device=dev)
    check(lib().dlx_quantize_factors(layout.ctx.h, layout.h, _ptr(p), _ptr(q), _ptr(delta), rank,
                                     spec.qbits, spec.rounding, rng_state & M64, int(cold),
                                     _ptr(payload), _ptr(draws), _stream(stream)))
    return payload, draws


def decompress(layout: Layout, payload: torch.Tensor, rank: int, qbits: int, stream=None):
    """decompress (compress.cpp:201-238) — reference-exact fp64 accumulation."""
    out = layout.empty(payload.device)
    check(lib().dlx_decompress(layout.ctx.h, layout.h, rank, qbits, _ptr(payload), _ptr(out),
                               _stream(stream)))
    return out


def allreduce_avg(layout: Layout, gathered: torch.Tensor, D: int, rank: int, qbits: int,
                  stream=None):
    """allreduce_avg (collective.cpp:17-46) given the all-gather buffer of D payloads."""
    out = layout.empty(gathered.device)
    check(lib().dlx_allreduce_avg(layout.ctx.h, layout.h, rank, qbits, D, _ptr(gathered),
                                  _ptr(out), _stream(stream)))
    return out


def outer_update(layout: Layout, gathered: torch.Tensor, D: int, rank: int, qbits: int,
                 pending: torch.Tensor, anchor: torch.Tensor, local: torch.Tensor | None,
                 velocity: torch.Tensor, gamma: float, beta: float, classical: bool = False,
                 mode: int = OVERLAPPED, self_index: int = -1, stats: torch.Tensor | None = None,
                 stream=None, tensors: tuple[int, int] | None = None):
    """Fused reconstruct + error feedback + stage + Nesterov (engine.cpp:254-276,
    optim.cpp:56-78). stats: device float64[8] (dlx_round_stats) or None. tensors=(t0, t1)
    restricts the update to layout tensors [t0, t1) (stats zeroed only when t0 == 0)."""
    if tensors is None:
        check(lib().dlx_outer_update(layout.ctx.h, layout.h, rank, qbits, D, _ptr(gathered),
                                     self_index, mode, _ptr(pending), _ptr(anchor), _ptr(local),
                                     _ptr(velocity), gamma, beta, int(classical), _ptr(stats),
                                     _stream(stream)))
    else:
        check(lib().dlx_outer_update_range(layout.ctx.h, layout.h, rank, qbits, D, _ptr(gathered),
                                           self_index, mode, _ptr(pending), _ptr(anchor),
                                           _ptr(local), _ptr(velocity), gamma, beta,
                                           int(classical), _ptr(stats), int(tensors[0]),
                                           int(tensors[1]), _stream(stream)))


@dataclass
class AdamWHyper:
    """optim.hpp:10-19."""
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.01
    warmup_steps: int = 0


class AdamWState:
    """make_adamw_state (optim.cpp:7-13): device m, v like the parameters, host step."""

    def __init__(self, params: torch.Tensor, hyper: AdamWHyper | None = None):
        self.m = torch.zeros_like(params)
        self.v = torch.zeros_like(params)
        self.step = 0
        self.hyper = hyper or AdamWHyper()
        self.nonfinite = torch.zeros(1, dtype=torch.int32, device=params.device)


def adamw_step(ctx: Context, state: AdamWState, params: torch.Tensor, grads: torch.Tensor,
               stream=None, raise_nonfinite: bool = False):
    """adamw_step (optim.cpp:15-47), in place on params / state (bit-exact).
    raise_nonfinite=True synchronises and raises NumericError on a non-finite gradient, as
    the reference does (otherwise the flag stays in state.nonfinite)."""
    h = state.hyper
    st = C.c_int64(state.step)
    check(lib().dlx_adamw_step(ctx.h, params.numel(), h.lr, h.beta1, h.beta2, h.eps,
                               h.weight_decay, h.warmup_steps, C.byref(st),
                               _ptr(params), _ptr(grads), _ptr(state.m), _ptr(state.v),
                               _ptr(state.nonfinite), _stream(stream)))
    state.step = st.value
    if raise_nonfinite and int(state.nonfinite.item()):
        state.nonfinite.zero_()
        from ._lib import NumericError
        raise NumericError("adamw_step: non-finite gradient")


def compress_raw(layout: Layout, delta: torch.Tensor) -> torch.Tensor:
    """compress_raw (compress.cpp:185-199): the payload of the no-compress ablation is the
    raw fp32 slab itself (32 bits per parameter)."""
    return delta


def payload_bits_raw(layout: Layout) -> int:
    """payload_bits_formula for RawDense payloads (compress.cpp:92-114): 32 n per tensor."""
    return 32 * int(layout.total_params)


def outer_update_raw(layout: Layout, gathered: torch.Tensor, D: int, pending: torch.Tensor,
                     anchor: torch.Tensor, local: torch.Tensor | None, velocity: torch.Tensor,
                     gamma: float, beta: float, classical: bool = False, mode: int = OVERLAPPED,
                     self_index: int = -1, stats: torch.Tensor | None = None, stream=None):
    """dilocox-no-compress: reference-exact allreduce_avg of D raw slabs (gathered back to
    back) fused with error feedback, staging and Nesterov."""
    check(lib().dlx_outer_update_raw(layout.ctx.h, layout.h, D, _ptr(gathered), self_index, mode,
                                     _ptr(pending), _ptr(anchor), _ptr(local), _ptr(velocity),
                                     gamma, beta, int(classical), _ptr(stats), _stream(stream)))


def measure_error(layout: Layout, payload: torch.Tensor, rank: int, qbits: int,
                  delta: torch.Tensor, stream=None) -> float:
    """measure_error (compress.cpp:246-262) on the device (synchronises for the result)."""
    out = torch.zeros(2, dtype=torch.float64, device=delta.device)
    check(lib().dlx_measure_error(layout.ctx.h, layout.h, rank, qbits, _ptr(payload), _ptr(delta),
                                  _ptr(out), _stream(stream)))
    num, den = out.tolist()
    return num / den if den > 0 else 0.0


def mean_slabs(ctx: Context, gathered: torch.Tensor, D: int, n: int, ld: int | None = None,
               out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Worker-order fp64 mean of D slabs (dlx_mean_slabs), bit-exact with the reference."""
    ld = n if ld is None else ld
    if out is None:
        out = torch.empty(n, dtype=torch.float32, device=gathered.device)
    check(lib().dlx_mean_slabs(ctx.h, n, ld, D, _ptr(gathered), _ptr(out), _stream(stream)))
    return out


def stage_deltas(layout: Layout, anchor, local, err, pending, norm_sq=None, stream=None):
    """stage_deltas (engine.cpp:266-276): pending = (anchor - local) + err."""
    check(lib().dlx_stage_deltas(layout.ctx.h, layout.h, _ptr(anchor), _ptr(local), _ptr(err),
                                 _ptr(pending), _ptr(norm_sq), _stream(stream)))


def nesterov_outer_step(ctx: Context, anchor: torch.Tensor, velocity: torch.Tensor,
                        delta: torch.Tensor, gamma: float = 0.7, beta: float = 0.9,
                        classical: bool = False, stream=None):
    """nesterov_outer_step (optim.cpp:56-78), in place on anchor / velocity."""
    check(lib().dlx_nesterov(ctx.h, anchor.numel(), gamma, beta, int(classical), _ptr(anchor),
                             _ptr(velocity), _ptr(delta), _stream(stream)))


@dataclass
class EffectiveRank:
    """compress.hpp:121-125."""
    aggregate: int = 1
    per_tensor: list = field(default_factory=list)
    all_zero: bool = False


def effective_rank_device(layout: Layout, gathered: torch.Tensor, D: int, rank: int,
                          qbits: int, tau: float, stream=None, shard: int = 0, nshards: int = 1,
                          per: torch.Tensor | None = None, energy: torch.Tensor | None = None):
    """Launch the factor-space effective rank; returns device (per_tensor, energy). With
    nshards > 1 only the 2-D tensors whose index % nshards == shard are measured and the
    other entries are zero (dlx_effective_rank_shard)."""
    n2 = sum(1 for s in layout.shapes if len(s) == 2)
    if per is None:
        per = torch.zeros(max(n2, 1), dtype=torch.int32, device=gathered.device)
    if energy is None:
        energy = torch.zeros(max(n2, 1), dtype=torch.float64, device=gathered.device)
    check(lib().dlx_effective_rank_shard(layout.ctx.h, layout.h, rank, qbits, D, _ptr(gathered),
                                         tau, shard, nshards, _ptr(per), _ptr(energy),
                                         _stream(stream)))
    return per, energy


def effective_rank_reduce(layout: Layout, per: np.ndarray, energy: np.ndarray,
                          r_max: int) -> EffectiveRank:
    per = np.ascontiguousarray(per, np.int32)
    energy = np.ascontiguousarray(energy, np.float64)
    agg, z = C.c_int(0), C.c_int(0)
    check(lib().dlx_effective_rank_reduce(layout.h, per.ctypes.data_as(C.POINTER(C.c_int)),
                                          energy.ctypes.data_as(C.POINTER(C.c_double)), r_max,
                                          C.byref(agg), C.byref(z)))
    names2 = [n for n, s in zip(layout.names, layout.shapes) if len(s) == 2]
    return EffectiveRank(agg.value, list(zip(names2, per.tolist())), bool(z.value))


def effective_rank(layout: Layout, gathered: torch.Tensor, D: int, rank: int, qbits: int,
                   tau: float, r_max: int, stream=None) -> EffectiveRank:
    """effective_rank (compress.cpp:306-344) of allreduce_avg(gathered), in factor space."""
    per, energy = effective_rank_device(layout, gathered, D, rank, qbits, tau, stream)
    n2 = sum(1 for s in layout.shapes if len(s) == 2)
    return effective_rank_reduce(layout, per.cpu().numpy()[:n2], energy.cpu().numpy()[:n2], r_max)


def adapt_compression(window, r1: int, H1: int, c: int, h_min: int):
    """adapt_compression (engine.cpp:294-308)."""
    w = np.ascontiguousarray(window if len(window) else [0], np.int32)
    r, h = C.c_int(0), C.c_int(0)
    check(lib().dlx_adapt_compression(w.ctypes.data_as(C.POINTER(C.c_int)), len(window), r1, H1,
                                      c, h_min, C.byref(r), C.byref(h)))
    return r.value, h.value


def omega_bound(r: int, d: int, q: int) -> float:
    """omega_bound (compress.cpp:240-244)."""
    v = lib().dlx_omega_bound(r, d, q)
    if v < 0:
        raise _lib.ValidationError("omega_bound: need 1 <= r <= d")
    return v


def bind_host_to_device(device: int) -> list[int]:
    """Pin the calling process to the CPUs NVML reports as local to `device` (its NUMA node)
    and return them. Call before allocating the pinned host buffers a host-resident caller
    hands to OuterSync.step_host: pinned pages land on the node of the allocating CPU, and
    with one process per GPU the 2 x 5.26 GB of copies per round otherwise cross the socket
    link for the GPUs on the other node. No-op (returns []) when NVML is unavailable."""
    import os
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(device)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = [64 * i + b for i, w in enumerate(words) for b in range(64) if (int(w) >> b) & 1]
        cpus = [c for c in cpus if c < os.cpu_count()]
        if cpus:
            os.sched_setaffinity(0, cpus)
        return cpus
    except Exception:
        return []


def take_launch_count() -> int:
    return int(lib().dlx_take_launch_count())


def set_option(key: str, value: int) -> None:
    """dlx_set_option: e.g. set_option("tensor_cores", 0) routes the power-iteration sweeps
    through the SIMT kernels (A/B testing)."""
    check(lib().dlx_set_option(key.encode(), int(value)))


def kernel_time(name: str):
    """dlx_kernel_time: (device ms, algorithmic bytes, launches) of the recorded launches of
    kernel `name` since the last call (needs set_option("kernel_events", 1))."""
    ms, by, n = C.c_double(0.0), C.c_double(0.0), C.c_int64(0)
    check(lib().dlx_kernel_time(name.encode(), C.byref(ms), C.byref(by), C.byref(n)))
    return ms.value, by.value, n.value


def debug_sweep(layout: Layout, rank: int, which: int, slab: torch.Tensor, fac_in: torch.Tensor,
                use_tc: bool, stream=None) -> torch.Tensor:
    """Test hook: one K1 (which=0, out = delta Q) or K2 (which=1, out = delta^T P) sweep."""
    side_out = 0 if which == 0 else 1
    out = torch.zeros(max(layout.factor_offsets(rank, side_out)[1], 1), dtype=torch.float32,
                      device=slab.device)
    check(lib().dlx_debug_sweep(layout.ctx.h, layout.h, rank, which, _ptr(slab), _ptr(fac_in),
                                _ptr(out), int(use_tc), _stream(stream)))
    return out
