"""SURVEY §8d 'overlap efficiency': inner AdamW steps (the overlap partner, dlx_adamw_step)
on one stream while an outer-synchronisation round runs on another, OPT-1.3B layout, one
GPU. Reports the inner-step time alone and with the outer round active, and the round time
alone / concurrent. Both are HBM-bound on one B200, so the GPU-side overlap mostly shares
bandwidth; what the one-step delay hides in DiLoCoX is the (WAN) exchange."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_21263_b200 import api, layouts
from paper_2506_21263_b200.engine import OuterConfig, OuterSync

ctx = api.Context(0)
L = api.Layout(ctx, layouts.opt_1_3b())
anchor = L.empty(); api.fill_gaussian(L, anchor, 0.02, seed=7, tag=0xA7C4, worker=0)
local = L.empty(); api.fill_gaussian(L, local, -1e-3, seed=1, tag=0xDA7A, worker=0, base=anchor)
eng = OuterSync(L, OuterConfig(rank1=32, qbits=4, hold_rank=True), anchor)
params = local.clone()
grads = L.empty(); api.fill_gaussian(L, grads, 1e-3, seed=3, tag=0x6AD, worker=0)
st = api.AdamWState(params)
inner = torch.cuda.Stream()
for _ in range(3):
    eng.step(local)
    api.adamw_step(ctx, st, params, grads)
torch.cuda.synchronize()
def ev():
    return torch.cuda.Event(enable_timing=True)
H = 4
# alone
e0, e1 = ev(), ev(); e0.record()
for _ in range(H): api.adamw_step(ctx, st, params, grads)
e1.record(); torch.cuda.synchronize(); t_in = e0.elapsed_time(e1) / H
e0, e1 = ev(), ev(); e0.record(); eng.step(local); e1.record(); torch.cuda.synchronize()
t_out = e0.elapsed_time(e1)
# concurrent: H inner steps on the inner stream, one outer round on the main stream
torch.cuda.synchronize()
m0, m1, i0, i1 = ev(), ev(), ev(), ev()
cur = torch.cuda.current_stream()
m0.record(cur)
inner.wait_stream(cur)
with torch.cuda.stream(inner):
    i0.record(inner)
    for _ in range(H): api.adamw_step(ctx, st, params, grads, stream=inner)
    i1.record(inner)
eng.step(local)
m1.record(cur)
cur.wait_stream(inner)
torch.cuda.synchronize()
t_in_c = i0.elapsed_time(i1) / H
t_out_c = m0.elapsed_time(m1)
t_tot = m0.elapsed_time(i1) if i1.query() else None
print(f"inner AdamW step alone {t_in:.3f} ms ({28 * L.slab_elems / t_in / 1e6:.0f} GB/s); "
      f"outer round alone {t_out:.3f} ms")
print(f"concurrent: inner step {t_in_c:.3f} ms (slowdown x{t_in_c / t_in:.2f}), outer round "
      f"{t_out_c:.3f} ms (x{t_out_c / t_out:.2f}); serial sum {H * t_in + t_out:.3f} ms, "
      f"concurrent span {max(H * t_in_c, t_out_c):.3f} ms")
