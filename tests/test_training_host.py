"""CPU checks of the inner-training host logic (paper_2506_21263_b200/training.py): the
batch-index RNG reproduces the reference's RngStream draws (golden fixtures generated from
the reference), below() is the reference's rejection rule, the mlp ParamSet table follows
build_model's order, and shard() matches data.cpp's contiguous split."""
import numpy as np
import pytest

from paper_2506_21263_b200 import api
from paper_2506_21263_b200.training import M64, _next_u64, below, mlp_table, shard


@pytest.mark.parametrize("seed,sid", [(1, 0), (7, 3), (49374, 5)])
def test_next_u64_matches_reference_draws(golden, seed, sid):
    st = api.rng_stream(seed, sid)
    assert st == int(golden[f"rng_state_{seed}_{sid}"][0])
    want = golden[f"rng_draws_{seed}_{sid}"]
    got = []
    for _ in range(len(want)):
        st, v = _next_u64(st)
        got.append(v)
    assert np.array_equal(np.array(got, dtype=np.uint64), want.astype(np.uint64))


def test_below_rejection_rule():
    st = api.rng_stream(3, api.stream_key(0xDA7A, 0))
    for n in (1, 2, 3, 7, 1900, 2**63 + 5):
        s2, v = below(st, n)
        if n <= 1:
            assert v == 0 and s2 == st
            continue
        limit = M64 - (M64 % n)
        s, raw = _next_u64(st)
        while raw >= limit:
            s, raw = _next_u64(s)
        assert (s2, v) == (s, raw % n)
        assert 0 <= v < n
        st = s2


def test_mlp_table_and_shard():
    t = mlp_table([16, 64, 8])
    assert t == [("w1", (16, 64)), ("b1", (64,)), ("w2", (64, 8)), ("b2", (8,))]
    x = np.arange(20 * 3, dtype=np.float32).reshape(20, 3)
    y = np.arange(20, dtype=np.float32).reshape(20, 1)
    xs, ys = shard(x, y, 3, 1)
    assert xs.shape == (6, 3) and np.array_equal(xs, x[6:12]) and np.array_equal(ys, y[6:12])
