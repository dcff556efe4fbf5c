"""ctypes front-end to the CPU checkers (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference``
leg may import this module. The product package never does.

Two backends export the same C interface (oracle/dlx_oracle.h):
  * ``restatement`` — oracle/liboracle.so, plain-C restatement (oracle/dlx_oracle.c)
  * ``reference``   — oracle/_ref/libdlxref.so, the reference proj/core compiled from
                      /root/reference by oracle/Makefile, behind oracle/ref_shim.cpp
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "restatement": os.path.join(HERE, "liboracle.so"),
    "reference": os.path.join(HERE, "_ref", "libdlxref.so"),
}

ERRORS = {1: "ValidationError", 2: "ShapeError", 3: "FormatError", 4: "NumericError",
          5: "IoError", 9: "Error"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, 'Error')}: {msg}")
        self.code = code
        self.kind = ERRORS.get(code, "Error")


def build(quiet: bool = True) -> None:
    """Build the checkers (make -C oracle). The reference part only builds where
    /root/reference exists; elsewhere the prebuilt _ref/ library is kept."""
    out = subprocess.run(["make", "-C", HERE, "all"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])
    if not quiet:
        print(out.stdout)


@dataclass
class Table:
    """Tensor table in reference ParamSet order: shapes are (a, b) or (n,)."""
    shapes: list

    @property
    def nt(self) -> int:
        return len(self.shapes)

    def arrays(self):
        ndim = np.array([len(s) for s in self.shapes], dtype=np.int32)
        dims = np.zeros(2 * self.nt, dtype=np.int64)
        for i, s in enumerate(self.shapes):
            dims[2 * i] = s[0]
            dims[2 * i + 1] = s[1] if len(s) == 2 else 1
        return ndim, dims

    def numel(self) -> int:
        return int(sum(int(np.prod(s)) for s in self.shapes))

    def ranks(self, rank: int) -> np.ndarray:
        return np.array([min(rank, s[0], s[1]) if len(s) == 2 else 0 for s in self.shapes],
                        dtype=np.int32)


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


class Oracle:
    def __init__(self, backend: str = "restatement"):
        path = LIBS[backend]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle backend {backend!r} not built: {path}")
        self.backend = backend
        L = self.lib = C.CDLL(path)
        u64p, i64, f32p, i32p = C.POINTER(C.c_uint64), C.c_int64, C.POINTER(C.c_float), C.POINTER(C.c_int)
        L.orc_last_error.restype = C.c_char_p
        L.orc_backend.restype = C.c_char_p
        L.orc_stream_key.restype = C.c_uint64
        L.orc_stream_key.argtypes = [u64p, C.c_int]
        L.orc_stream_init.restype = C.c_uint64
        L.orc_stream_init.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_next_u64.restype = C.c_uint64
        L.orc_next_u64.argtypes = [u64p]
        L.orc_gaussian.argtypes = [u64p, i64, f32p]
        L.orc_uniform.argtypes = [u64p, i64, C.c_float, C.c_float, f32p]
        L.orc_omega_bound.restype = C.c_double
        L.orc_payload_bits.restype = C.c_uint64
        L.orc_serialize.restype = C.c_int64
        L.orc_codes_count.restype = C.c_int64
        L.orc_scales_count.restype = C.c_int64
        L.orc_qfactor_count.restype = C.c_int64
        assert L.orc_backend().decode() == backend

    # -- helpers
    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(rc, self.lib.orc_last_error().decode())

    # -- RNG (rng.hpp)
    def stream_key(self, *parts) -> int:
        arr = (C.c_uint64 * len(parts))(*[p & 0xFFFFFFFFFFFFFFFF for p in parts])
        return self.lib.orc_stream_key(arr, len(parts))

    def stream(self, seed: int, stream_id: int) -> int:
        return self.lib.orc_stream_init(C.c_uint64(seed), C.c_uint64(stream_id))

    def next_u64(self, state: int, n: int = 1):
        st = C.c_uint64(state)
        out = [self.lib.orc_next_u64(C.byref(st)) for _ in range(n)]
        return out, st.value

    def gaussian(self, state: int, n: int):
        st = C.c_uint64(state)
        out = np.empty(n, np.float32)
        self.lib.orc_gaussian(C.byref(st), n, _p(out, C.c_float))
        return out, st.value

    def uniform(self, state: int, n: int, lo=-1.0, hi=1.0):
        st = C.c_uint64(state)
        out = np.empty(n, np.float32)
        self.lib.orc_uniform(C.byref(st), n, C.c_float(lo), C.c_float(hi), _p(out, C.c_float))
        return out, st.value

    # -- dense kernels (tensor.cpp)
    def matmul(self, a, b):
        a = np.ascontiguousarray(a, np.float32); b = np.ascontiguousarray(b, np.float32)
        c = np.empty((a.shape[0], b.shape[1]), np.float32)
        self._check(self.lib.orc_matmul(C.c_int64(a.shape[0]), C.c_int64(a.shape[1]),
                                        C.c_int64(b.shape[1]), _p(a, C.c_float), _p(b, C.c_float),
                                        _p(c, C.c_float)))
        return c

    def matmul_tn(self, a, b):
        a = np.ascontiguousarray(a, np.float32); b = np.ascontiguousarray(b, np.float32)
        c = np.empty((a.shape[1], b.shape[1]), np.float32)
        self._check(self.lib.orc_matmul_tn(C.c_int64(a.shape[0]), C.c_int64(a.shape[1]),
                                           C.c_int64(b.shape[1]), _p(a, C.c_float),
                                           _p(b, C.c_float), _p(c, C.c_float)))
        return c

    def matmul_nt(self, a, b):
        a = np.ascontiguousarray(a, np.float32); b = np.ascontiguousarray(b, np.float32)
        c = np.empty((a.shape[0], b.shape[0]), np.float32)
        self._check(self.lib.orc_matmul_nt(C.c_int64(a.shape[0]), C.c_int64(a.shape[1]),
                                           C.c_int64(b.shape[0]), _p(a, C.c_float),
                                           _p(b, C.c_float), _p(c, C.c_float)))
        return c

    def orthonormalize(self, m):
        m = np.ascontiguousarray(m, np.float32)
        out = np.empty_like(m)
        rep = C.c_int(0)
        self._check(self.lib.orc_orthonormalize(C.c_int64(m.shape[0]), C.c_int64(m.shape[1]),
                                                _p(m, C.c_float), _p(out, C.c_float),
                                                C.byref(rep)))
        return out, rep.value

    def singular_values(self, m):
        m = np.ascontiguousarray(m, np.float32)
        sv = np.empty(min(m.shape), np.float64)
        self._check(self.lib.orc_singular_values(C.c_int64(m.shape[0]), C.c_int64(m.shape[1]),
                                                 _p(m, C.c_float), _p(sv, C.c_double)))
        return sv

    # -- compressor (compress.cpp)
    def lowrank_approx(self, m, r, warm_q, iters, state):
        m = np.ascontiguousarray(m, np.float32)
        a, b = m.shape
        p = np.empty((a, r), np.float32); q = np.empty((b, r), np.float32)
        st = C.c_uint64(state)
        wq = None if warm_q is None else np.ascontiguousarray(warm_q, np.float32)
        self._check(self.lib.orc_lowrank_approx(
            C.c_int64(a), C.c_int64(b), _p(m, C.c_float), r,
            None if wq is None else _p(wq, C.c_float), iters, C.byref(st),
            _p(p, C.c_float), _p(q, C.c_float)))
        return p, q, st.value

    def quantize(self, x, qbits, rounding, state):
        x = np.ascontiguousarray(x, np.float32)
        codes = np.empty(x.size, np.int8)
        scale = C.c_float(0)
        st = C.c_uint64(state)
        self._check(self.lib.orc_quantize(_p(x, C.c_float), C.c_int64(x.size), qbits, rounding,
                                          C.byref(st), _p(codes, C.c_int8), C.byref(scale)))
        return codes, scale.value, st.value

    def compress(self, table: Table, data, rank, qbits, rounding, iters, state, warm_rank=0,
                 warm_q=None):
        ndim, dims = table.arrays()
        ranks = table.ranks(rank)
        data = np.ascontiguousarray(data, np.float32)
        codes = np.empty(self.lib.orc_codes_count(table.nt, _p(ndim, C.c_int), _p(dims, C.c_int64),
                                                  _p(ranks, C.c_int)), np.int8)
        scales = np.empty(self.lib.orc_scales_count(table.nt, _p(ndim, C.c_int),
                                                    _p(dims, C.c_int64), _p(ranks, C.c_int)),
                          np.float32)
        qf = np.zeros(max(1, self.lib.orc_qfactor_count(table.nt, _p(ndim, C.c_int),
                                                        _p(dims, C.c_int64), _p(ranks, C.c_int))),
                      np.float32)
        st = C.c_uint64(state)
        bits = C.c_uint64(0)
        got_ranks = np.zeros(table.nt, np.int32)
        wq = None if warm_q is None else np.ascontiguousarray(warm_q, np.float32)
        self._check(self.lib.orc_compress(
            table.nt, _p(ndim, C.c_int), _p(dims, C.c_int64), _p(data, C.c_float), rank, qbits,
            rounding, iters, warm_rank, None if wq is None else _p(wq, C.c_float), C.byref(st),
            _p(codes, C.c_int8), _p(scales, C.c_float), _p(qf, C.c_float),
            _p(got_ranks, C.c_int), C.byref(bits)))
        return dict(codes=codes, scales=scales, q=qf, ranks=got_ranks, bits=bits.value,
                    state=st.value)

    def decompress(self, table: Table, ranks, codes, scales):
        ndim, dims = table.arrays()
        ranks = np.ascontiguousarray(ranks, np.int32)
        out = np.empty(table.numel(), np.float32)
        codes = np.ascontiguousarray(codes, np.int8); scales = np.ascontiguousarray(scales, np.float32)
        self._check(self.lib.orc_decompress(table.nt, _p(ndim, C.c_int), _p(dims, C.c_int64),
                                            _p(ranks, C.c_int), _p(codes, C.c_int8),
                                            _p(scales, C.c_float), _p(out, C.c_float)))
        return out

    def allreduce_avg(self, table: Table, ranks, codes_list, scales_list):
        ndim, dims = table.arrays()
        ranks = np.ascontiguousarray(ranks, np.int32)
        D = len(codes_list)
        cl = [np.ascontiguousarray(c, np.int8) for c in codes_list]
        sl = [np.ascontiguousarray(s, np.float32) for s in scales_list]
        cp = (C.POINTER(C.c_int8) * D)(*[_p(c, C.c_int8) for c in cl])
        sp = (C.POINTER(C.c_float) * D)(*[_p(s, C.c_float) for s in sl])
        out = np.empty(table.numel(), np.float32)
        self._check(self.lib.orc_allreduce_avg(D, table.nt, _p(ndim, C.c_int), _p(dims, C.c_int64),
                                               _p(ranks, C.c_int), cp, sp, _p(out, C.c_float)))
        return out

    def measure_error(self, table: Table, delta, ranks, codes, scales) -> float:
        ndim, dims = table.arrays()
        ranks = np.ascontiguousarray(ranks, np.int32)
        delta = np.ascontiguousarray(delta, np.float32)
        err = C.c_double(0)
        self._check(self.lib.orc_measure_error(table.nt, _p(ndim, C.c_int), _p(dims, C.c_int64),
                                               _p(delta, C.c_float), _p(ranks, C.c_int),
                                               _p(np.ascontiguousarray(codes, np.int8), C.c_int8),
                                               _p(np.ascontiguousarray(scales, np.float32),
                                                  C.c_float), C.byref(err)))
        return err.value

    def adamw_step(self, p, g, m, v, step, lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8,
                   weight_decay=0.01, warmup_steps=0):
        """adamw_step (optim.cpp:15-47); returns (p, m, v, step) (inputs untouched)."""
        p = np.array(p, np.float32, copy=True); m = np.array(m, np.float32, copy=True)
        v = np.array(v, np.float32, copy=True); g = np.ascontiguousarray(g, np.float32)
        st = C.c_int64(step)
        self._check(self.lib.orc_adamw_step(C.c_int64(p.size), C.c_float(lr), C.c_float(beta1),
                                            C.c_float(beta2), C.c_float(eps),
                                            C.c_float(weight_decay), C.c_int64(warmup_steps),
                                            C.byref(st), _p(p, C.c_float), _p(g, C.c_float),
                                            _p(m, C.c_float), _p(v, C.c_float)))
        return p, m, v, st.value

    def nesterov(self, anchor, v, delta, gamma=0.7, beta=0.9, classical=False):
        anchor = np.array(anchor, np.float32, copy=True); v = np.array(v, np.float32, copy=True)
        delta = np.ascontiguousarray(delta, np.float32)
        self._check(self.lib.orc_nesterov(C.c_int64(anchor.size), C.c_float(gamma),
                                          C.c_float(beta), int(classical), _p(anchor, C.c_float),
                                          _p(v, C.c_float), _p(delta, C.c_float)))
        return anchor, v

    def effective_rank(self, table: Table, data, tau, r_max):
        ndim, dims = table.arrays()
        n2 = sum(1 for s in table.shapes if len(s) == 2)
        per = np.zeros(max(1, n2), np.int32)
        agg = C.c_int(0); z = C.c_int(0)
        data = np.ascontiguousarray(data, np.float32)
        self._check(self.lib.orc_effective_rank(table.nt, _p(ndim, C.c_int), _p(dims, C.c_int64),
                                                _p(data, C.c_float), C.c_double(tau), r_max,
                                                _p(per, C.c_int), C.byref(agg), C.byref(z)))
        return per[:n2], agg.value, bool(z.value)

    def adapt_compression(self, window, r1, H1, c, h_min):
        w = np.ascontiguousarray(window, np.int32) if len(window) else np.zeros(1, np.int32)
        r = C.c_int(0); h = C.c_int(0)
        self._check(self.lib.orc_adapt_compression(_p(w, C.c_int), len(window), r1, H1, c, h_min,
                                                   C.byref(r), C.byref(h)))
        return r.value, h.value

    def omega_bound(self, r, d, q) -> float:
        return self.lib.orc_omega_bound(r, d, q)

    def payload_bits(self, table: Table, ranks, qbits) -> int:
        ndim, dims = table.arrays()
        ranks = np.ascontiguousarray(ranks, np.int32)
        return self.lib.orc_payload_bits(table.nt, _p(ndim, C.c_int), _p(dims, C.c_int64),
                                         _p(ranks, C.c_int), qbits)

    def serialize(self, table: Table, ranks, rank, qbits, codes, scales) -> bytes:
        ndim, dims = table.arrays()
        ranks = np.ascontiguousarray(ranks, np.int32)
        codes = np.ascontiguousarray(codes, np.int8); scales = np.ascontiguousarray(scales, np.float32)
        args = [table.nt, _p(ndim, C.c_int), _p(dims, C.c_int64), _p(ranks, C.c_int), rank, qbits,
                _p(codes, C.c_int8), _p(scales, C.c_float)]
        n = self.lib.orc_serialize(*args, None, C.c_int64(0))
        if n < 0:
            raise OracleError(-n, self.lib.orc_last_error().decode())
        buf = np.empty(n, np.uint8)
        self.lib.orc_serialize(*args, _p(buf, C.c_uint8), C.c_int64(n))
        return buf.tobytes()

    def outer_round(self, table: Table, D, seed, round_index, rank, qbits, rounding, iters,
                    adaptive, tau, r1, gamma, beta, classical, threads, anchor, velocity,
                    pending, local, warm_rank, warm_q):
        """In-place on anchor/velocity/pending/warm_q (numpy float32, C-contiguous)."""
        ndim, dims = table.arrays()
        wr = C.c_int(warm_rank)
        rp = C.c_int(0); ce = C.c_double(0); bits = C.c_uint64(0)
        en = C.c_double(0); mx = C.c_double(0)
        for arr in (anchor, velocity, pending, local, warm_q):
            assert arr.dtype == np.float32 and arr.flags.c_contiguous
        self._check(self.lib.orc_outer_round(
            D, table.nt, _p(ndim, C.c_int), _p(dims, C.c_int64), C.c_uint64(seed),
            C.c_int64(round_index), rank, qbits, rounding, iters, int(adaptive), C.c_double(tau),
            r1, C.c_float(gamma), C.c_float(beta), int(classical), threads,
            _p(anchor, C.c_float), _p(velocity, C.c_float), _p(pending, C.c_float),
            _p(local, C.c_float), C.byref(wr), _p(warm_q, C.c_float), C.byref(rp), C.byref(ce),
            C.byref(bits), C.byref(en), C.byref(mx)))
        return dict(warm_rank=wr.value, r_prime=rp.value, comp_error=ce.value,
                    payload_bits=bits.value, err_norm0=en.value, max_delta_norm=mx.value)


def ref_mlp_overlapped_run(widths, activation, samples, teacher_hidden, seed, D, H1,
                           total_steps, batch, rank1, qbits, rounding, power_iters, adaptive,
                           eval_fraction=0.05):
    """The reference's own overlapped training run (test_support.hpp:114-218) on the mlp /
    synthetic-regression workload — reference backend only (oracle/_ref). Returns the initial
    model (flat, ParamSet order), final anchor, per-round losses and the train split."""
    if not available("reference"):
        raise OracleError(1, "reference library not built")
    lib = C.CDLL(LIBS["reference"])
    widths = np.ascontiguousarray(widths, np.int32)
    nparams = sum(int(widths[i]) * int(widths[i + 1]) + int(widths[i + 1])
                  for i in range(len(widths) - 1))
    a0 = np.zeros(nparams, np.float32)
    a1 = np.zeros(nparams, np.float32)
    losses = np.zeros(total_steps + 1, np.float64)
    nr = C.c_int(0)
    tx = np.zeros((samples, int(widths[0])), np.float32)
    ty = np.zeros((samples, int(widths[-1])), np.float32)
    nt = C.c_int64(0)
    rc = lib.orc_ref_mlp_overlapped_run(
        _p(widths, C.c_int), len(widths), int(activation == "tanh"), C.c_int64(samples),
        teacher_hidden, C.c_uint64(seed), D, H1, C.c_int64(total_steps), batch, rank1, qbits,
        rounding, power_iters, int(adaptive), C.c_double(eval_fraction), _p(a0, C.c_float),
        _p(a1, C.c_float), _p(losses, C.c_double), C.byref(nr), _p(tx, C.c_float),
        _p(ty, C.c_float), C.byref(nt))
    if rc != 0:
        lib.orc_last_error.restype = C.c_char_p
        raise OracleError(rc, lib.orc_last_error().decode())
    n = nt.value
    return dict(anchor0=a0, anchor=a1, losses=losses[:nr.value], train_x=tx[:n], train_y=ty[:n])


def available(backend: str) -> bool:
    return os.path.exists(LIBS[backend])
