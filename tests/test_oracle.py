"""Pin the CPU oracle (plain-C restatement) against the reference: golden vectors generated
from the reference (tests/golden/gen_golden.py) and, where the reference library is built,
direct side-by-side runs. Also the reference's own known-answer tests for the hot path
(compress_test.cpp, tensor_test.cpp, optim_test.cpp, collective_test.cpp, engine_test.cpp).
"""
import numpy as np
import pytest

from oracle.oracle import OracleError, Table

TABLES = {
    "mixed": [(24, 18), (18,), (18, 6), (6,), (10, 8)],
    "zero2d": [(16, 12), (12,)],
    "clamp": [(6, 4), (7,), (40, 33)],
}


def test_rng_matches_golden(oracle, golden):
    for seed, sid in [(1, 0), (7, 3), (0xC0DE, 5)]:
        st = oracle.stream(seed, sid)
        assert st == int(golden[f"rng_state_{seed}_{sid}"][0])
        assert np.array_equal(np.array(oracle.next_u64(st, 16)[0], np.uint64),
                              golden[f"rng_draws_{seed}_{sid}"])
        assert np.array_equal(oracle.gaussian(st, 64)[0], golden[f"rng_gauss_{seed}_{sid}"])
        assert np.array_equal(oracle.uniform(st, 64)[0], golden[f"rng_unif_{seed}_{sid}"])
    assert oracle.stream_key(0xC09C, 3) == int(golden["stream_key_c09c_3"][0])
    assert oracle.stream_key(0xDA7A, 1, 2) == int(golden["stream_key_da7a_1_2"][0])


def test_orthonormalize_matches_golden(oracle, golden):
    q, rep = oracle.orthonormalize(golden["ortho_dep_in"])
    assert rep == int(golden["ortho_dep_rep"][0]) == 1
    assert np.array_equal(q, golden["ortho_dep_out"])
    assert np.array_equal(oracle.orthonormalize(golden["ortho_in"])[0], golden["ortho_out"])
    assert np.array_equal(oracle.orthonormalize(np.zeros((10, 3), np.float32))[0],
                          golden["ortho_zero_out"])


@pytest.mark.parametrize("tname", list(TABLES))
@pytest.mark.parametrize("q", [2, 4, 5, 8])
@pytest.mark.parametrize("rnd", [0, 1])
@pytest.mark.parametrize("rank", [3, 6])
def test_compress_matches_golden(oracle, golden, tname, q, rnd, rank):
    t = Table(TABLES[tname])
    key = f"c_{tname}_q{q}_r{rnd}_k{rank}"
    data = golden[f"c_{tname}_data"]
    st0 = int(golden[key + "_state0"][0])
    c = oracle.compress(t, data, rank, q, rnd, 2, st0)
    for k in ("codes", "scales", "q", "ranks"):
        assert np.array_equal(c[k], golden[f"{key}_{k}"]), k
    assert c["bits"] == int(golden[key + "_bits"][0])
    assert c["state"] == int(golden[key + "_state1"][0])
    w = oracle.compress(t, data, rank, q, rnd, 1, st0, warm_rank=rank, warm_q=c["q"])
    for k in ("codes", "scales", "q"):
        assert np.array_equal(w[k], golden[f"{key}_warm_{k}"]), k
    assert w["state"] == int(golden[key + "_warm_state1"][0])
    wire = oracle.serialize(t, c["ranks"], rank, q, c["codes"], c["scales"])
    assert np.array_equal(np.frombuffer(wire, np.uint8), golden[key + "_wire"])


def test_allreduce_and_nesterov_match_golden(oracle, golden):
    t = Table([(16, 12), (12,)])
    avg = oracle.allreduce_avg(t, golden["ar_ranks"], [golden[f"ar_codes_{i}"] for i in range(3)],
                               [golden[f"ar_scales_{i}"] for i in range(3)])
    assert np.array_equal(avg, golden["ar_avg"])
    a, v = np.array([1.0], np.float32), np.zeros(1, np.float32)
    out = []
    for d in (0.2, -0.1, 0.05):
        a, v = oracle.nesterov(a, v, np.array([d], np.float32), 0.7, 0.9, False)
        out.append(a[0])
    assert np.array_equal(np.array(out, np.float32), golden["nesterov_trace"])
    for cl in (0, 1):
        oa, ov = oracle.nesterov(golden["nest_in_a"], golden["nest_in_v"], golden["nest_in_d"],
                                 0.7, 0.9, bool(cl))
        assert np.array_equal(oa, golden[f"nest_out_a_{cl}"])
        assert np.array_equal(ov, golden[f"nest_out_v_{cl}"])


def test_effective_rank_and_controller_match_golden(oracle, golden):
    t = Table([(64, 64), (16, 12), (8, 8)])
    per, agg, _ = oracle.effective_rank(t, golden["er_data"], 0.5, 64)
    assert np.array_equal(per, golden["er_per"]) and agg == int(golden["er_agg"][0])
    assert tuple(oracle.adapt_compression([2048, 1024, 512, 512, 512], 2048, 125, 5, 13)) == \
        tuple(golden["adapt_922_69"]) == (922, 69)


def test_overlapped_rounds_match_golden(oracle, golden):
    t = Table(TABLES["mixed"][:4])
    anchor = golden["round_anchor0"].copy()
    locs = golden["round_local"].copy()
    vel = np.zeros_like(anchor)
    pend = np.stack([anchor - locs[w] for w in range(2)]).astype(np.float32)
    warm_q = np.zeros(max(1, sum(s[1] * min(4, *s) for s in t.shapes if len(s) == 2)), np.float32)
    wr = 0
    for rnd in (2, 3, 4):
        out = oracle.outer_round(t, 2, 1, rnd, 4, 4, 0, 2, True, 0.5, 4, 0.7, 0.9, False, 1,
                                 anchor, vel, pend, locs, wr, warm_q)
        wr = out["warm_rank"]
        assert out["r_prime"] == int(golden[f"round{rnd}_rprime"][0])
        assert out["comp_error"] == float(golden[f"round{rnd}_comp_error"][0])
    assert np.array_equal(anchor, golden["round_anchor"])
    assert np.array_equal(vel, golden["round_vel"])
    assert np.array_equal(pend, golden["round_pend"])


def test_restatement_equals_reference_random(oracle, reference):
    """Direct side-by-side on fresh random tables (bit-exact)."""
    rng = np.random.default_rng(0)
    for trial in range(6):
        shapes = []
        for _ in range(4):
            if rng.random() < 0.6:
                shapes.append((int(rng.integers(2, 40)), int(rng.integers(2, 40))))
            else:
                shapes.append((int(rng.integers(1, 30)),))
        t = Table(shapes)
        data = reference.gaussian(reference.stream(trial, 1), t.numel())[0]
        rank, q, rnd = int(rng.integers(1, 9)), int(rng.integers(2, 9)), int(rng.integers(0, 2))
        st = reference.stream(trial, 2)
        a = reference.compress(t, data, rank, q, rnd, 2, st)
        b = oracle.compress(t, data, rank, q, rnd, 2, st)
        for k in ("codes", "scales", "q", "ranks", "bits", "state"):
            assert np.array_equal(a[k], b[k]), (trial, k)


def test_singular_values_restated_with_jacobi(oracle, reference):
    m = reference.gaussian(reference.stream(31, 0), 48 * 20)[0].reshape(48, 20)
    s1, s2 = oracle.singular_values(m), reference.singular_values(m)
    assert np.allclose(s1, s2, rtol=1e-10, atol=1e-10 * s2[0])


# ---- reference known-answer tests restated against the oracle -------------------------------

def planted(o, a, b, rank, seed):
    st = o.stream(seed, 0x9A9)
    u, st = o.gaussian(st, a * rank)
    v, _ = o.gaussian(st, b * rank)
    return o.matmul_nt(u.reshape(a, rank), v.reshape(b, rank))


def test_lowrank_exact_capture(oracle):
    m = planted(oracle, 64, 40, 5, 3)  # compress_test.cpp:33-39
    p, q, _ = oracle.lowrank_approx(m, 5, None, 2, oracle.stream(1, 1))
    rec = oracle.matmul_nt(p, q)
    assert np.linalg.norm(rec - m) / np.linalg.norm(m) < 1e-5


def test_lowrank_zero_matrix_is_zero(oracle):
    p, q, _ = oracle.lowrank_approx(np.zeros((10, 8), np.float32), 3, None, 2, oracle.stream(1, 1))
    assert not p.any()  # compress_test.cpp:49-56


def test_validation_errors(oracle):
    with pytest.raises(OracleError) as e:
        oracle.lowrank_approx(np.zeros((10, 8), np.float32), 9, None, 2, 1)
    assert e.value.kind == "ValidationError"
    with pytest.raises(OracleError):
        oracle.quantize(np.ones(4, np.float32), 9, 0, 1)
    with pytest.raises(OracleError):
        oracle.effective_rank(Table([(4, 4)]), np.zeros(16, np.float32), 1.0, 4)


def test_zero_paramset_formula_volume(oracle):
    t = Table([(16, 12), (12,)])  # compress_test.cpp:130-144
    c = oracle.compress(t, np.zeros(t.numel(), np.float32), 4, 4, 0, 2, oracle.stream(1, 2))
    assert not oracle.decompress(t, c["ranks"], c["codes"], c["scales"]).any()
    assert c["bits"] == (16 + 12) * 4 * 4 + 2 * 4 * 32 + 12 * 4 + 32


def test_omega_bound_values(oracle):
    assert oracle.omega_bound(4, 4, 0) == 0.0
    assert oracle.omega_bound(2, 4, 1) == 0.75
    assert abs(oracle.omega_bound(1024, 4096, 4) - 0.984375) < 1e-12


def test_controller_clamps(oracle):
    assert oracle.adapt_compression([2048, 1024], 2048, 125, 5, 13) == (2048, 125)
    assert oracle.adapt_compression([64, 64, 64], 64, 120, 3, 12) == (64, 12)
    assert oracle.adapt_compression([1, 1, 1], 64, 120, 3, 12) == (1, 118)


def test_measure_error_under_omega_bound(oracle):
    t = Table([(64, 64)])  # compress_test.cpp:241-253 (smaller)
    bound = oracle.omega_bound(8, 64, 4)
    for seed in range(5):
        d = oracle.gaussian(oracle.stream(seed, 0x6A), t.numel())[0]
        c = oracle.compress(t, d, 8, 4, 0, 2, oracle.stream(seed, 1))
        assert oracle.measure_error(t, d, c["ranks"], c["codes"], c["scales"]) <= bound


def test_adamw_restatement_matches_reference(oracle, reference):
    """adamw_step (optim.cpp:15-47): the plain-C restatement is bit-identical to the
    reference library over several steps, with and without LR warm-up, and both raise
    NumericError on a non-finite gradient."""
    n = 4097
    p = (np.float32(0.02) * oracle.gaussian(oracle.stream(3, 1), n)[0]).astype(np.float32)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    pr, mr, vr, step, stepr = p.copy(), m.copy(), v.copy(), 0, 0
    for k in range(5):
        g = (np.float32(1e-2) * oracle.gaussian(oracle.stream(4, k), n)[0]).astype(np.float32)
        warm = 3 if k % 2 else 0
        p, m, v, step = oracle.adamw_step(p, g, m, v, step, warmup_steps=warm)
        pr, mr, vr, stepr = reference.adamw_step(pr, g, mr, vr, stepr, warmup_steps=warm)
        assert step == stepr
        assert np.array_equal(p, pr) and np.array_equal(m, mr) and np.array_equal(v, vr)
    from oracle.oracle import OracleError
    g[7] = np.nan
    for backend in (oracle, reference):
        with pytest.raises(OracleError):
            backend.adamw_step(p, g, m, v, step)
