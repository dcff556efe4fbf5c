"""One rank's share of a D-worker round on one GPU (payload replicated): the fused outer
update at D alone, the effective-rank shard (1/D of the tensors) alone, and both together
with the measurement on a high-priority side stream (what OuterSync does at world = D)."""
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
anchor, local, vel = L.empty(), L.empty(), L.empty()
api.fill_gaussian(L, anchor, 0.02, seed=2, tag=2, worker=0)
api.fill_gaussian(L, local, 0.02, seed=3, tag=3, worker=0)
stats = torch.zeros(8, dtype=torch.float64, device="cuda")
side = torch.cuda.Stream(priority=-1)
for D in [int(x) for x in os.environ.get("DS", "2,4,8").split(",")]:
    g = pay.repeat(D)
    def ou():
        api.outer_update(L, g, D, r, q, delta, anchor, local, vel, 0.7, 0.9, False,
                         mode=api.OVERLAPPED, self_index=0, stats=stats)
    def er(stream=None):
        api.effective_rank_device(L, g, D, r, q, 0.5, stream=stream, shard=0, nshards=D)
    def both():
        cur = torch.cuda.current_stream()
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            er(side)
        ou()
        cur.wait_stream(side)
    for name, fn in (("outer_update", ou), ("effrank shard", er), ("both", both)):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(3):
            fn()
        e1.record(); torch.cuda.synchronize()
        print(f"D={D}: {name} {e0.elapsed_time(e1) / 3:.3f} ms", flush=True)
