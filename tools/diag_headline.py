"""Per-column diagnosis of the headline compress parity (tests/test_gpu_headline.py): the
scales, codes and Q factors of dlx_compress vs the compiled reference on the OPT-1.3B
embedding + position table + decoder layer, worst offenders first
(profiles/r02_headline_compress_diag.log)."""
import sys, numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import torch
from oracle.oracle import Oracle, Table
from tests.test_gpu_headline import _head_table, _lowrank_noise, RANK, Q
from tests._util import decode_payload, split_q
from paper_2506_21263_b200 import api
R = Oracle("reference")
ctx = api.Context(0)
tbl = _head_table(); shapes = [s for _, s in tbl]; t = Table(shapes)
L = api.Layout(ctx, tbl)
flat = _lowrank_noise(shapes, 2026)
st0 = R.stream(1, R.stream_key(0xC09C, 2))
ref = R.compress(t, flat, RANK, Q, 0, 2, st0)
res = api.compress(L, L.pack(flat), RANK, api.QuantSpec(Q, api.STOCHASTIC), None, 0, 2, st0)
codes, scales = decode_payload(L, res.payload, RANK, Q)
rel = np.abs(scales - ref["scales"]) / np.maximum(np.abs(ref["scales"]), 1e-30)
# map scale index -> (tensor, side, col)
idx = []
for i, s in enumerate(shapes):
    if len(s) == 2:
        r = min(RANK, *s)
        idx += [(i, 'P', j) for j in range(r)] + [(i, 'Q', j) for j in range(r)]
    else:
        idx.append((i, '1d', 0))
order = np.argsort(-rel)[:15]
for k in order:
    print(idx[k], shapes[idx[k][0]], rel[k], scales[k], ref["scales"][k])
print("codes equal", (codes == ref["codes"]).mean())
qs = L.factors_from_device(res.q_factors, RANK, 1)
for i,(g, w) in enumerate(zip(qs, split_q(shapes, RANK, ref["q"]))):
    print("Q", i, np.abs(g-w).max(axis=0)[-4:], np.abs(g - w).max())
