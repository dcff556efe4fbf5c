"""Time one K1 / K2 sweep over the OPT-1.3B layout (experiments; run on a GPU box)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_21263_b200 import api, layouts

ctx = api.Context(0)
L = api.Layout(ctx, layouts.opt_1_3b())
r = int(os.environ.get("RANK_R", "32"))
slab = L.empty()
api.fill_gaussian(L, slab, 1e-3, seed=1, tag=1, worker=0)
Q = torch.randn(L.factor_offsets(r, 1)[1], device="cuda")
P = torch.randn(L.factor_offsets(r, 0)[1], device="cuda")
for which, fin in ((0, Q), (1, P)):
    for _ in range(2):
        api.debug_sweep(L, r, which, slab, fin, True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    n = 5
    for _ in range(n):
        api.debug_sweep(L, r, which, slab, fin, True)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"variant={os.environ.get('DLX_SWEEP_VARIANT','0')} r={r} K{which+1}: {ms:.3f} ms  {L.total_params*4/ms/1e6:.0f} GB/s", flush=True)
