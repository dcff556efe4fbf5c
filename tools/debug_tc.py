"""Diagnose the tcgen05 sweeps against numpy on small problems (run on a GPU box)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2506_21263_b200 import api

ctx = api.Context(0)
rng = np.random.default_rng(0)
for (a, b), r in [((128, 32), 16), ((256, 64), 16), ((128, 128), 32), ((300, 96), 8), ((2600, 96), 8)]:
    L = api.Layout(ctx, [("w", (a, b))])
    d = rng.standard_normal((a, b)).astype(np.float32)
    q = rng.standard_normal((b, r)).astype(np.float32)
    p = rng.standard_normal((a, r)).astype(np.float32)
    slab = L.to_slab([d])
    Q = L.factors_to_device([q], r, 1)
    P = L.factors_to_device([p], r, 0)
    for which, fin, want in ((0, Q, d.astype(np.float64) @ q), (1, P, d.T.astype(np.float64) @ p)):
        res = {}
        for tc in (1, 0):
            out = api.debug_sweep(L, r, which, slab, fin, tc)
            torch.cuda.synchronize()
            got = L.factors_from_device(out, r, 0 if which == 0 else 1)[0]
            res[tc] = got
        err_tc = np.abs(res[1] - want).max() / np.abs(want).max()
        err_si = np.abs(res[0] - want).max() / np.abs(want).max()
        print(f"shape {(a,b)} r={r} K{which+1}: rel err tc={err_tc:.3e} simt={err_si:.3e}")
        if err_tc > 1e-3:
            g = res[1]
            print("  tc[0:4,0:4]=", np.round(g[:4, :4], 3).tolist())
            print("  want[0:4,0:4]=", np.round(want[:4, :4], 3).tolist())
            bad = np.abs(g - want) > 1e-3 * np.abs(want).max()
            print("  bad rows:", np.where(bad.any(1))[0][:20].tolist(), "bad cols:", np.where(bad.any(0))[0][:20].tolist(), "frac", bad.mean())
            # try to detect permutations / scaling
            for cand_name, cand in (("transposed-k", None),):
                pass
            nz = np.abs(g).max()
            print("  tc max|.|", nz, "want max", np.abs(want).max())
