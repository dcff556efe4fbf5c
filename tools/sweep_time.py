"""Power-iteration sweeps alone on OPT-1.3B (r = 32): K1 / K2 launch times from the library's
per-launch CUDA events (dlx_kernel_time) over a few compress calls."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_21263_b200 import api, layouts
ctx = api.Context(0)
L = api.Layout(ctx, layouts.opt_1_3b())
r, q = int(os.environ.get("RANK_R", "32")), 4
delta = L.empty()
api.fill_gaussian(L, delta, 1e-3, seed=1, tag=1, worker=0)
for _ in range(2):
    api.compress(L, delta, r, api.QuantSpec(q, 0), None, 0, 2, 12345)
torch.cuda.synchronize()
api.set_option("kernel_events", 1)
n = 5
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(n):
    api.compress(L, delta, r, api.QuantSpec(q, 0), None, 0, 2, 12345)
e1.record(); torch.cuda.synchronize()
for k in ("k_tc_sweep_k1", "k_tc_sweep_k2"):
    ms, by, nl = api.kernel_time(k)
    print(f"{k}: {ms / max(nl, 1):.3f} ms/launch  {by / (ms / 1e3) / 1e9:.0f} GB/s  ({nl} launches)")
print(f"compress: {e0.elapsed_time(e1) / n:.3f} ms")
api.set_option("kernel_events", 0)
