"""Time the fused outer update at D = 1, 2, 4, 8 workers on one GPU (payloads replicated;
experiments only): the tcgen05 path covers K = D*r <= 64, larger K runs the SIMT path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_21263_b200 import api, layouts

ctx = api.Context(0)
L = api.Layout(ctx, layouts.opt_1_3b())
r, q = int(os.environ.get("RANK_R", "32")), 4
delta = L.empty()
api.fill_gaussian(L, delta, 1e-3, seed=1, tag=1, worker=0)
res = api.compress(L, delta, r, api.QuantSpec(q, 0), None, 0, 2, 12345)
pay = res.payload
anchor, local, vel = L.empty(), L.empty(), L.empty()
api.fill_gaussian(L, anchor, 0.02, seed=2, tag=2, worker=0)
api.fill_gaussian(L, local, 0.02, seed=3, tag=3, worker=0)
stats = torch.zeros(8, dtype=torch.float64, device="cuda")
for D in [int(x) for x in os.environ.get("DS", "1,2,4,8").split(",")]:
    g = pay.repeat(D)
    for _ in range(2):
        api.outer_update(L, g, D, r, q, delta, anchor, local, vel, 0.7, 0.9, False,
                         mode=api.OVERLAPPED, self_index=int(os.environ.get('SELF', '0')), stats=stats)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    n = 3
    for _ in range(n):
        api.outer_update(L, g, D, r, q, delta, anchor, local, vel, 0.7, 0.9, False,
                         mode=api.OVERLAPPED, self_index=int(os.environ.get('SELF', '0')), stats=stats)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"r={r} D={D} K={D*r}: outer_update {ms:.3f} ms  {28 * L.total_params / ms / 1e6:.0f} GB/s", flush=True)

# effective rank at the same D
for D in [int(x) for x in os.environ.get("DS", "1,2,4,8").split(",")]:
    g = pay.repeat(D)
    for _ in range(2):
        api.effective_rank_device(L, g, D, r, q, 0.5)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    api.effective_rank_device(L, g, D, r, q, 0.5)
    e1.record(); torch.cuda.synchronize()
    print(f"r={r} D={D} K={D*r}: effective_rank {e0.elapsed_time(e1):.3f} ms", flush=True)
