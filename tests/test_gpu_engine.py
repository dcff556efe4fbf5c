"""Round orchestration (paper_2506_21263_b200.engine.OuterSync) on the GPU against the oracle's
outer_round (engine.cpp:458-509 collective_average + staging + Nesterov), and the
host-resident pipeline (step_host) against the device-resident step.

Bars: the power iteration runs in fp32 on the device vs fp64 in the reference, so a few
stochastic-rounding codes differ per round (test_compress_* bounds that); the state after
three overlapped rounds must agree to TOL_STATE relative Frobenius distance of the update,
r' within 1 of the reference's and the compression error within 1 %. step_host vs step:
bitwise identical.
"""
import numpy as np
import pytest

from oracle.oracle import Table
from tests._util import rel_fro

pytestmark = pytest.mark.gpu

TOL_STATE = 1e-2
SHAPES = [(64, 48), (48,), (96, 32), (24, 18), (18,), (40, 40)]


def _engine(ctx, shapes, anchor_np, rank, **kw):
    import torch
    from paper_2506_21263_b200 import api
    from paper_2506_21263_b200.engine import OuterConfig, OuterSync
    L = api.Layout(ctx, [(f"t{i}", s) for i, s in enumerate(shapes)])
    cfg = OuterConfig(rank1=rank, qbits=4, power_iters=2, adaptive=True, tau=0.5, seed=1,
                      overlap=True, hold_rank=True, **kw)
    anchor = L.pack(anchor_np)
    return L, OuterSync(L, cfg, anchor)


def test_engine_rounds_match_oracle(ctx, oracle):
    t = Table(SHAPES)
    n = t.numel()
    rank = 4
    anchor0 = (np.float32(0.02) * oracle.gaussian(oracle.stream(7, 0), n)[0]).astype(np.float32)
    local = (anchor0 - np.float32(1e-3) * oracle.gaussian(oracle.stream(1, 10), n)[0]).astype(np.float32)
    L, eng = _engine(ctx, SHAPES, anchor0, rank)
    dlocal = L.pack(local)
    eng.step(dlocal)  # round 1: staging only (engine.cpp:473)
    # oracle: the same state after round 1
    a = anchor0.copy()
    v = np.zeros(n, np.float32)
    pend = (anchor0 - local).astype(np.float32)[None].copy()
    loc = local[None].copy()
    wq = np.zeros(max(1, sum(s[1] * min(rank, *s) for s in SHAPES if len(s) == 2)), np.float32)
    wr = 0
    for rnd in (2, 3, 4):
        rec = eng.step(dlocal)
        out = oracle.outer_round(t, 1, 1, rnd, rank, 4, 0, 2, True, 0.5, rank, 0.7, 0.9, False, 1,
                                 a, v, pend, loc, wr, wq)
        wr = out["warm_rank"]
        assert abs(rec.r_prime - out["r_prime"]) <= 1, (rnd, rec.r_prime, out["r_prime"])
        assert abs(rec.comp_error - out["comp_error"]) <= 1e-2 * out["comp_error"], rnd
    ga = L.unpack(eng.anchor)
    gv = L.unpack(eng.velocity)
    gp = L.unpack(eng.pending)
    assert rel_fro(ga - anchor0, a - anchor0) <= TOL_STATE
    assert rel_fro(gv, v) <= TOL_STATE
    assert rel_fro(gp, pend[0]) <= TOL_STATE


def test_step_host_matches_step(ctx, oracle):
    import torch
    t = Table(SHAPES)
    n = t.numel()
    anchor0 = (np.float32(0.02) * oracle.gaussian(oracle.stream(3, 0), n)[0]).astype(np.float32)
    L1, e1 = _engine(ctx, SHAPES, anchor0, 8)
    L2, e2 = _engine(ctx, SHAPES, anchor0, 8)
    h_anchor = torch.empty(L2.slab_elems, dtype=torch.float32, pin_memory=True)
    for rnd in range(4):
        local = (anchor0 - np.float32(1e-3) * oracle.gaussian(oracle.stream(5, rnd), n)[0]
                 ).astype(np.float32)
        d = L1.pack(local)
        h = torch.empty(L2.slab_elems, dtype=torch.float32, pin_memory=True)
        h.copy_(d)
        r1 = e1.step(d)
        r2 = e2.step_host(h, h_anchor)
        e2.host_wait()
        torch.cuda.synchronize()
        # stats are fp64 atomics (diagnostics; summation order not fixed)
        assert abs(r1.comp_error - r2.comp_error) <= 1e-12 * abs(r1.comp_error)
        assert r1.r_prime == r2.r_prime
        assert torch.equal(e1.anchor, e2.anchor)
        assert torch.equal(e1.velocity, e2.velocity)
        assert torch.equal(e1.pending, e2.pending)
        assert torch.equal(h_anchor, e2.anchor.cpu())


def _lowrank_drift(shapes, rank, seed):
    """Pseudo-gradient with a realistic spectrum (bench-compress's lowrank+noise generator,
    tools/dilocox.cpp:183-192): a decaying rank-`rank` component plus small noise per 2-D
    tensor, small noise on 1-D tensors."""
    rng = np.random.default_rng(seed)
    parts = []
    for s in shapes:
        if len(s) == 2:
            a, b = s
            u = rng.standard_normal((a, rank)).astype(np.float32)
            v = rng.standard_normal((b, rank)).astype(np.float32)
            sv = (1e-3 * 0.7 ** np.arange(rank)).astype(np.float32)
            d = (u * sv) @ v.T + np.float32(1e-6) * rng.standard_normal((a, b)).astype(np.float32)
            parts.append(d.astype(np.float32).reshape(-1))
        else:
            parts.append((np.float32(1e-4) * rng.standard_normal(s)).astype(np.float32))
    return np.concatenate(parts)


def test_engine_mini_opt_c1(ctx, oracle):
    """SURVEY C1 (mini-OPT, 10.76 M params, r = 8, q = 8): three overlapped rounds of the
    engine against the reference round (orc_outer_round) on the full named layout, with a
    low-rank-plus-noise drift (a flat Gaussian spectrum leaves the rank-8 subspace
    ill-determined, which amplifies fp32-vs-fp64 rounding in either implementation)."""
    from paper_2506_21263_b200 import layouts
    shapes = [s for _, s in layouts.mini_opt()]
    t = Table(shapes)
    n = t.numel()
    rank, q = 8, 8
    anchor0 = (np.float32(0.02) * oracle.gaussian(oracle.stream(7, 0), n)[0]).astype(np.float32)
    local = (anchor0 - _lowrank_drift(shapes, rank, 3)).astype(np.float32)
    from paper_2506_21263_b200 import api
    from paper_2506_21263_b200.engine import OuterConfig, OuterSync
    L = api.Layout(ctx, layouts.mini_opt())
    cfg = OuterConfig(rank1=rank, qbits=q, power_iters=2, adaptive=False, seed=1, overlap=True)
    eng = OuterSync(L, cfg, L.pack(anchor0))
    dlocal = L.pack(local)
    eng.step(dlocal)
    a = anchor0.copy()
    v = np.zeros(n, np.float32)
    pend = (anchor0 - local).astype(np.float32)[None].copy()
    loc = local[None].copy()
    wq = np.zeros(max(1, sum(s[1] * min(rank, *s) for s in shapes if len(s) == 2)), np.float32)
    wr = 0
    for rnd in (2, 3, 4):
        rec = eng.step(dlocal)
        out = oracle.outer_round(t, 1, 1, rnd, rank, q, 0, 2, False, 0.5, rank, 0.7, 0.9, False, 1,
                                 a, v, pend, loc, wr, wq)
        wr = out["warm_rank"]
        assert abs(rec.comp_error - out["comp_error"]) <= 1e-2 * out["comp_error"], rnd
        assert rec.payload_bytes == out["payload_bits"] / 8.0
    assert rel_fro(L.unpack(eng.anchor) - anchor0, a - anchor0) <= TOL_STATE
    assert rel_fro(L.unpack(eng.velocity), v) <= TOL_STATE
    assert rel_fro(L.unpack(eng.pending), pend[0]) <= TOL_STATE


@pytest.mark.parametrize("classical", [False, True])
def test_engine_sync_mode_matches_reference(ctx, oracle, classical):
    """run_round_sync (engine.cpp:423-456, dilocox-no-overlap): stage with the carried error
    before compress, then e = delta - Delta and the Nesterov (or classical) step — composed
    here from the oracle's compress / allreduce_avg / nesterov primitives. Each round starts
    the oracle from the engine's own state: a single stochastic-rounding code flip (fp32 vs
    fp64 factors) legitimately sends the error-feedback trajectories of a small tensor apart
    over several rounds, so the per-round map is what is compared."""
    t = Table(SHAPES)
    n = t.numel()
    rank, q = 4, 4
    anchor0 = (np.float32(0.02) * oracle.gaussian(oracle.stream(7, 0), n)[0]).astype(np.float32)
    L, eng = _engine(ctx, SHAPES, anchor0, rank)
    eng.cfg.overlap = False
    eng.cfg.adaptive = False
    eng.cfg.outer_classical = classical
    ranks = t.ranks(rank)
    wr, wq = 0, None
    for rnd in (1, 2, 3):
        a = L.unpack(eng.anchor)
        v = L.unpack(eng.velocity)
        e = L.unpack(eng.pending) if rnd > 1 else np.zeros(n, np.float32)
        local = (a - np.float32(1e-3) * oracle.gaussian(oracle.stream(2, rnd), n)[0]).astype(np.float32)
        rec = eng.step(L.pack(local))
        delta = ((a - local).astype(np.float32) + e).astype(np.float32)       # engine.cpp:434
        st = oracle.stream(1, oracle.stream_key(0xC09C, rnd))                  # engine.cpp:226
        c = oracle.compress(t, delta, rank, q, 0, 2, st, wr, wq)
        avg = oracle.allreduce_avg(t, ranks, [c["codes"]], [c["scales"]])
        e_ref = (delta - avg).astype(np.float32)
        a_ref, v_ref = oracle.nesterov(a, v, avg, 0.7, 0.9, classical)
        wr, wq = rank, c["q"]
        ce = oracle.measure_error(t, delta, ranks, c["codes"], c["scales"])
        assert abs(rec.comp_error - ce) <= 1e-2 * ce
        assert rel_fro(L.unpack(eng.anchor) - a, a_ref - a) <= 2e-2, rnd
        assert rel_fro(L.unpack(eng.velocity), v_ref) <= 2e-2, rnd
        assert rel_fro(L.unpack(eng.pending), e_ref) <= 2e-2, rnd
