import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2506_21263_b200 import api
ctx = api.Context(0)
shapes = [(2600, 96), (96,), (130, 300), (64, 4096), (33, 36)]
rank = int(sys.argv[1]) if len(sys.argv) > 1 else 100
L = api.Layout(ctx, [(f"t{i}", s) for i, s in enumerate(shapes)])
rng = np.random.default_rng(0)
flat = [rng.standard_normal(int(np.prod(s))).astype(np.float32) for s in shapes]
slab = L.to_slab(flat)
for tc in (1, 0):
    api.set_option("tensor_cores", tc)
    r = api.compress(L, slab, rank, api.QuantSpec(8, 1), None, 0, 2, 12345)
    torch.cuda.synchronize()
    print("ok tc", tc, flush=True)
