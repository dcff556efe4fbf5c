"""Effective rank at D = 1, 2 (OPT-1.3B, r = 32) with the small-K kernel vs the large-K one."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_21263_b200 import api, layouts
ctx = api.Context(0)
L = api.Layout(ctx, layouts.opt_1_3b())
r, q = 32, 4
delta = L.empty()
api.fill_gaussian(L, delta, 1e-3, seed=1, tag=1, worker=0)
pay = api.compress(L, delta, r, api.QuantSpec(q, 0), None, 0, 2, 12345).payload
for bf in (128, 0):
    api.set_option("effrank_big_from", bf)
    for D in (1, 2):
        g = pay.repeat(D)
        for _ in range(2): api.effective_rank_device(L, g, D, r, q, 0.5)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(5): api.effective_rank_device(L, g, D, r, q, 0.5)
        e1.record(); torch.cuda.synchronize()
        per, en = api.effective_rank_device(L, g, D, r, q, 0.5)
        print(f"big_from={bf} D={D}: {e0.elapsed_time(e1) / 5:.3f} ms  sum(per)={int(per.sum())}")
