"""The N>1 path on CPU: two worker processes (gloo, world_size 2) run one overlapped outer
round through the engine's exchange (paper_2506_21263_b200.engine.exchange — the same
function OuterSync uses over NCCL), with the oracle standing in for the device kernels on
each rank. Checks: gathered payloads are in rank order and identical on every rank, worker
0's Q reaches every rank, and every rank ends the round with the anchor / velocity / pending
state of the reference's single-process D=2 round (orc_outer_round, engine.cpp:458-509)."""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHAPES = [(24, 18), (18,), (18, 6), (6,), (10, 8)]
RANK, Q, ITERS, ROUND, SEED = 4, 4, 2, 2, 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _state(R, t, D):
    n = t.numel()
    anchor = (np.float32(0.02) * R.gaussian(R.stream(7, 0), n)[0]).astype(np.float32)
    locs = np.stack([anchor - np.float32(1e-3) * R.gaussian(R.stream(1, 10 + w), n)[0]
                     for w in range(D)]).astype(np.float32)
    pend = np.stack([anchor - locs[w] for w in range(D)]).astype(np.float32)
    return anchor, locs, pend


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from oracle.oracle import Oracle, Table
    from paper_2506_21263_b200.engine import exchange
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    R = Oracle("restatement")
    t = Table(SHAPES)
    ranks = t.ranks(RANK)
    anchor, locs, pend = _state(R, t, world)
    vel = np.zeros_like(anchor)
    st0 = R.stream(SEED, R.stream_key(0xC09C, ROUND))  # shared per-round stream (engine.cpp:226)
    c = R.compress(t, pend[rank], RANK, Q, 0, ITERS, st0)
    # payload = codes then scales (the device payload carries the same two sections)
    codes, scales = c["codes"].view(np.uint8), c["scales"].view(np.uint8)
    pay = torch.from_numpy(np.concatenate([codes, scales]))
    gathered = torch.zeros(world * pay.numel(), dtype=torch.uint8)
    warm_q = torch.from_numpy(c["q"].astype(np.float32).copy())
    g = exchange(pay, gathered, warm_q, world).numpy()
    pb = pay.numel()
    cl = [g[w * pb: w * pb + codes.size].view(np.int8) for w in range(world)]
    sl = [g[w * pb + codes.size: (w + 1) * pb].view(np.float32) for w in range(world)]
    avg = R.allreduce_avg(t, ranks, cl, sl)
    e = (pend[rank] - avg).astype(np.float32)
    new_pend = ((anchor - locs[rank]).astype(np.float32) + e).astype(np.float32)
    a, v = R.nesterov(anchor, vel, avg, 0.7, 0.9, False)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), anchor=a, vel=v, pend=new_pend,
             gathered=g, warm_q=warm_q.numpy(), err=R.measure_error(t, pend[rank], ranks,
                                                                    cl[rank], sl[rank]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_workers_gloo_round(tmp_path, oracle):
    import torch.multiprocessing as mp
    from oracle.oracle import Table
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]
    # every rank holds the same gathered bytes and rank 0's Q
    assert np.array_equal(res[0]["gathered"], res[1]["gathered"])
    assert np.array_equal(res[0]["warm_q"], res[1]["warm_q"])
    # single-process reference round with D = 2 workers
    t = Table(SHAPES)
    anchor, locs, pend = _state(oracle, t, world)
    vel = np.zeros_like(anchor)
    wq = np.zeros(max(1, sum(s[1] * min(RANK, *s) for s in SHAPES if len(s) == 2)), np.float32)
    out = oracle.outer_round(t, world, SEED, ROUND, RANK, Q, 0, ITERS, False, 0.5, RANK, 0.7, 0.9,
                             False, 1, anchor, vel, pend, locs.copy(), 0, wq)
    for r in range(world):
        assert np.array_equal(res[r]["anchor"], anchor), r
        assert np.array_equal(res[r]["vel"], vel), r
        assert np.array_equal(res[r]["pend"], pend[r]), r
    assert res[0]["err"] == pytest.approx(out["comp_error"], rel=0, abs=0)
    assert np.array_equal(res[1]["warm_q"], wq[:res[1]["warm_q"].size])
