"""Generate golden vectors from the REFERENCE implementation (oracle/_ref/libdlxref.so,
compiled from /root/reference by oracle/Makefile). Run in the build container:

    python tests/golden/gen_golden.py

Writes tests/golden/golden.npz. The CPU tests pin the plain-C restatement
(oracle/dlx_oracle.c) against these vectors; the GPU tests compare the CUDA path with them.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, Table  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")

# Small tensor tables: ragged shapes, a rank-clamped tensor, an all-zero tensor.
TABLES = {
    "mixed": [(24, 18), (18,), (18, 6), (6,), (10, 8)],
    "zero2d": [(16, 12), (12,)],
    "clamp": [(6, 4), (7,), (40, 33)],
}


def main():
    R = Oracle("reference")
    g = {}
    # RNG: stream construction, raw draws, gaussian / uniform fixtures
    for seed, sid in [(1, 0), (7, 3), (0xC0DE, 5)]:
        st = R.stream(seed, sid)
        g[f"rng_state_{seed}_{sid}"] = np.array([st], np.uint64)
        g[f"rng_draws_{seed}_{sid}"] = np.array(R.next_u64(st, 16)[0], np.uint64)
        g[f"rng_gauss_{seed}_{sid}"] = R.gaussian(st, 64)[0]
        g[f"rng_unif_{seed}_{sid}"] = R.uniform(st, 64)[0]
    g["stream_key_c09c_3"] = np.array([R.stream_key(0xC09C, 3)], np.uint64)
    g["stream_key_da7a_1_2"] = np.array([R.stream_key(0xDA7A, 1, 2)], np.uint64)

    # orthonormalisation, including the dependent-column case (tensor_test.cpp:119-131)
    dep = np.array([[1, 2, 0], [0, 0, 0], [0, 0, 1], [0, 0, 0]], np.float32)
    q, rep = R.orthonormalize(dep)
    g["ortho_dep_in"], g["ortho_dep_out"], g["ortho_dep_rep"] = dep, q, np.array([rep])
    m = R.uniform(R.stream(99, 3), 16 * 4)[0].reshape(16, 4)
    g["ortho_in"], g["ortho_out"] = m, R.orthonormalize(m)[0]
    z = np.zeros((10, 3), np.float32)
    g["ortho_zero_out"] = R.orthonormalize(z)[0]

    # compress cases
    for tname, shapes in TABLES.items():
        t = Table(shapes)
        data = R.gaussian(R.stream(3, 0), t.numel())[0]
        if tname == "zero2d":
            data[:] = 0
        if tname == "mixed":
            data[-80:] = 0  # all-zero last tensor
        g[f"c_{tname}_data"] = data
        for q in (2, 4, 5, 8):
            for rnd in (0, 1):
                for rank in (3, 6):
                    st0 = R.stream(12, q * 10 + rnd)
                    cold = R.compress(t, data, rank, q, rnd, 2, st0)
                    key = f"c_{tname}_q{q}_r{rnd}_k{rank}"
                    g[key + "_state0"] = np.array([st0], np.uint64)
                    for k in ("codes", "scales", "q", "ranks"):
                        g[f"{key}_{k}"] = cold[k]
                    g[key + "_bits"] = np.array([cold["bits"]], np.uint64)
                    g[key + "_state1"] = np.array([cold["state"]], np.uint64)
                    # warm restart from the produced Q (compress.cpp:161)
                    warm = R.compress(t, data, rank, q, rnd, 1, st0, warm_rank=rank,
                                      warm_q=cold["q"])
                    for k in ("codes", "scales", "q"):
                        g[f"{key}_warm_{k}"] = warm[k]
                    g[key + "_warm_state1"] = np.array([warm["state"]], np.uint64)
                    g[key + "_wire"] = np.frombuffer(
                        R.serialize(t, cold["ranks"], rank, q, cold["codes"], cold["scales"]),
                        np.uint8)

    # allreduce_avg of D=3 low-rank payloads with a shared stream (collective_test.cpp:62-84)
    t = Table([(16, 12), (12,)])
    codes, scales = [], []
    for i in range(3):
        d = R.gaussian(R.stream(i, 6), t.numel())[0]
        c = R.compress(t, d, 4, 4, 0, 2, R.stream(7, 7))
        codes.append(c["codes"])
        scales.append(c["scales"])
        g[f"ar_codes_{i}"], g[f"ar_scales_{i}"] = c["codes"], c["scales"]
    g["ar_ranks"] = t.ranks(4)
    g["ar_avg"] = R.allreduce_avg(t, t.ranks(4), codes, scales)

    # Nesterov traces (optim_test.cpp:124-155)
    anchor = np.array([1.0], np.float32); v = np.zeros(1, np.float32)
    trace = []
    for dlt in (0.2, -0.1, 0.05):
        anchor, v = R.nesterov(anchor, v, np.array([dlt], np.float32), 0.7, 0.9, False)
        trace.append(anchor[0])
    g["nesterov_trace"] = np.array(trace, np.float32)
    a = R.gaussian(R.stream(5, 1), 257)[0]; vv = R.gaussian(R.stream(5, 2), 257)[0]
    dd = R.gaussian(R.stream(5, 3), 257)[0]
    g["nest_in_a"], g["nest_in_v"], g["nest_in_d"] = a, vv, dd
    for cl in (0, 1):
        oa, ov = R.nesterov(a, vv, dd, 0.7, 0.9, bool(cl))
        g[f"nest_out_a_{cl}"], g[f"nest_out_v_{cl}"] = oa, ov

    # effective rank (compress_test.cpp:323-366)
    t = Table([(64, 64), (16, 12), (8, 8)])
    d = R.gaussian(R.stream(31, 0), t.numel())[0]
    per, agg, allz = R.effective_rank(t, d, 0.5, 64)
    g["er_data"], g["er_per"], g["er_agg"] = d, per, np.array([agg])

    # controller (engine_test.cpp:12-31)
    g["adapt_922_69"] = np.array(R.adapt_compression([2048, 1024, 512, 512, 512], 2048, 125, 5, 13))

    # overlapped rounds (D=2) on a small table: state after 3 rounds
    t = Table(TABLES["mixed"][:4])
    n = t.numel()
    anchor = 0.02 * R.gaussian(R.stream(7, 0), n)[0]
    anchor = anchor.astype(np.float32)
    vel = np.zeros(n, np.float32)
    locs = np.stack([anchor - np.float32(1e-3) * R.gaussian(R.stream(1, 10 + w), n)[0]
                     for w in range(2)]).astype(np.float32)
    pend = np.stack([anchor - locs[w] for w in range(2)]).astype(np.float32)
    warm_q = np.zeros(max(1, sum(s[1] * min(4, *s) for s in t.shapes if len(s) == 2)), np.float32)
    wr = 0
    g["round_anchor0"], g["round_local"] = anchor.copy(), locs.copy()
    for rnd in (2, 3, 4):
        out = R.outer_round(t, 2, 1, rnd, 4, 4, 0, 2, True, 0.5, 4, 0.7, 0.9, False, 1,
                            anchor, vel, pend, locs, wr, warm_q)
        wr = out["warm_rank"]
        g[f"round{rnd}_rprime"] = np.array([out["r_prime"]])
        g[f"round{rnd}_comp_error"] = np.array([out["comp_error"]])
    g["round_anchor"], g["round_vel"], g["round_pend"] = anchor, vel, pend
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
