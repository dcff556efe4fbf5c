"""Timeline of OuterSync.step_host (host-resident parameters): per step, when the H2D of the
local parameters, the round's kernels and the D2H of the anchor start/end (experiments)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_21263_b200 import api, layouts
from paper_2506_21263_b200.engine import OuterConfig, OuterSync

ctx = api.Context(0)
L = api.Layout(ctx, layouts.opt_1_3b())
anchor = L.empty("cuda:0")
api.fill_gaussian(L, anchor, 0.02, seed=7, tag=0xA7C4, worker=0)
local = L.empty("cuda:0")
api.fill_gaussian(L, local, -1e-3, seed=1, tag=0xDA7A, worker=0, base=anchor)
eng = OuterSync(L, OuterConfig(rank1=32, qbits=4, hold_rank=True), anchor)
h_local = torch.empty(L.slab_elems, dtype=torch.float32, pin_memory=True)
h_local.copy_(local)
h_anchor = torch.empty(L.slab_elems, dtype=torch.float32, pin_memory=True)
eng.step(local)
for _ in range(3):
    eng.step_host(h_local, h_anchor)
eng.host_wait(); torch.cuda.synchronize()
t0 = time.perf_counter()
marks = []
for i in range(4):
    ta = time.perf_counter()
    eng.step_host(h_local, h_anchor)
    tb = time.perf_counter()
    marks.append((ta - t0, tb - t0))
eng.host_wait(); torch.cuda.synchronize()
t1 = time.perf_counter()
for a, b in marks:
    print(f"step_host call {a*1e3:8.1f} -> {b*1e3:8.1f} ms  ({(b-a)*1e3:.1f})")
print(f"total {(t1-t0)*1e3:.1f} ms for 4 steps")
# copies alone, both directions together and separately
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
dl = torch.empty_like(local)
for name, fn in [("h2d", lambda: dl.copy_(h_local, non_blocking=True)),
                 ("d2h", lambda: h_anchor.copy_(anchor, non_blocking=True))]:
    torch.cuda.synchronize(); t = time.perf_counter(); fn(); torch.cuda.synchronize()
    print(name, f"{(time.perf_counter()-t)*1e3:.1f} ms")
torch.cuda.synchronize(); t = time.perf_counter()
with torch.cuda.stream(s1): dl.copy_(h_local, non_blocking=True)
with torch.cuda.stream(s2): h_anchor.copy_(anchor, non_blocking=True)
torch.cuda.synchronize(); print("duplex", f"{(time.perf_counter()-t)*1e3:.1f} ms")
