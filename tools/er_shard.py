"""Effective rank at D workers on one GPU (payload replicated), whole vs one shard of S
(dlx_effective_rank_shard: what each of S ranks runs) — per-rank time of the measurement."""
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
for D in [int(x) for x in os.environ.get("DS", "2,4,8").split(",")]:
    g = pay.repeat(D)
    for S in sorted({1, D}):
        for _ in range(2):
            api.effective_rank_device(L, g, D, r, q, 0.5, shard=0, nshards=S)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        api.effective_rank_device(L, g, D, r, q, 0.5, shard=0, nshards=S)
        e1.record(); torch.cuda.synchronize()
        print(f"D={D} K={D*r} shard 0/{S}: effective_rank {e0.elapsed_time(e1):.3f} ms", flush=True)
