"""Does the effective-rank kernel hide behind the fused outer update when run on a side
stream (co-resident CTAs)? Experiments only."""
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
stats = torch.zeros(8, dtype=torch.float64, device="cuda")
side = torch.cuda.Stream()
for D in [int(x) for x in os.environ.get("DS", "4,8").split(",")]:
    g = pay.repeat(D)
    def outer():
        api.outer_update(L, g, D, r, q, delta, anchor, local, vel, 0.7, 0.9, False,
                         mode=api.OVERLAPPED, self_index=0, stats=stats)
    def er(stream=None):
        return api.effective_rank_device(L, g, D, r, q, 0.5, stream=stream)
    for _ in range(2):
        outer(); er()
    torch.cuda.synchronize()
    def timeit(fn, n=3):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(n): fn()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n
    t_o = timeit(outer)
    t_e = timeit(lambda: er())
    t_s = timeit(lambda: (outer(), er()))
    def conc():
        cur = torch.cuda.current_stream()
        side.wait_stream(cur)
        outer()
        with torch.cuda.stream(side):
            er(side)
        cur.wait_stream(side)
    t_c = timeit(conc)
    print(f"D={D}: outer {t_o:.3f}  effrank {t_e:.3f}  serial {t_s:.3f}  concurrent {t_c:.3f} ms", flush=True)
