"""Per-tensor comparison of the sync-mode engine round against the oracle primitives."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle.oracle import Oracle, Table
from paper_2506_21263_b200 import api
from paper_2506_21263_b200.engine import OuterConfig, OuterSync
from tests._util import rel_fro, split_dense
oracle = Oracle("restatement")
SHAPES = [(64, 48), (48,), (96, 32), (24, 18), (18,), (40, 40)]
t = Table(SHAPES); n = t.numel(); rank, q = 4, 4
ctx = api.Context(0)
L = api.Layout(ctx, [(f"t{i}", s) for i, s in enumerate(SHAPES)])
anchor0 = (np.float32(0.02) * oracle.gaussian(oracle.stream(7, 0), n)[0]).astype(np.float32)
eng = OuterSync(L, OuterConfig(rank1=rank, qbits=q, adaptive=False, overlap=False, seed=1), L.pack(anchor0))
ranks = t.ranks(rank)
a = anchor0.copy(); v = np.zeros(n, np.float32); e = np.zeros(n, np.float32); wr, wq = 0, None
for rnd in (1, 2, 3):
    local = (a - np.float32(1e-3) * oracle.gaussian(oracle.stream(2, rnd), n)[0]).astype(np.float32)
    rec = eng.step(L.pack(local))
    delta = ((a - local).astype(np.float32) + e).astype(np.float32)
    st = oracle.stream(1, oracle.stream_key(0xC09C, rnd))
    c = oracle.compress(t, delta, rank, q, 0, 2, st, wr, wq)
    avg = oracle.allreduce_avg(t, ranks, [c["codes"]], [c["scales"]])
    e = (delta - avg).astype(np.float32)
    a, v = oracle.nesterov(a, v, avg, 0.7, 0.9, False)
    wr, wq = rank, c["q"]
    ga, gv, gp = L.unpack(eng.anchor), L.unpack(eng.velocity), L.unpack(eng.pending)
    print("round", rnd, "comp_error", rec.comp_error)
    for i, (x, y, p, pr) in enumerate(zip(split_dense(SHAPES, ga - anchor0), split_dense(SHAPES, a - anchor0),
                                         split_dense(SHAPES, gp), split_dense(SHAPES, e))):
        print(f"  t{i} {SHAPES[i]} anchor-upd rel {rel_fro(x, y):.2e}  e rel {rel_fro(p, pr):.2e}")

# round-1 compress alone: codes agreement per tensor
from tests._util import decode_payload, split_q
delta1 = (anchor0 - (anchor0 - np.float32(1e-3) * oracle.gaussian(oracle.stream(2, 1), n)[0]).astype(np.float32)).astype(np.float32)
st = oracle.stream(1, oracle.stream_key(0xC09C, 1))
res = api.compress(L, L.pack(delta1), rank, api.QuantSpec(q, 0), None, 0, 2, st)
ref = oracle.compress(t, delta1, rank, q, 0, 2, st)
codes, scales = decode_payload(L, res.payload, rank, q)
print("codes equal frac", (codes == ref["codes"]).mean(), "n codes", codes.size)
qg = L.factors_from_device(res.q_factors, rank, 1)
qr = split_q(SHAPES, rank, ref["q"])
for i, (x, y) in enumerate(zip(qg, qr)):
    print("Q", i, x.shape, "max|dQ|", np.abs(x - y).max(), "proj diff", np.abs(x @ x.T - y @ y.T).max())
