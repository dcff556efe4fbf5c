"""Effective-rank kernel choice at 64 < K <= 128: time effective_rank_device (code Grams +
eigenproblems) with effrank_big_from = 64 (blocked DMMA k_effrank_big) and = 128 (k_effrank),
per layout / D / r (payload of one compress replicated D times). Prints one JSON line per
case; the two settings must give the same per-tensor k."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_21263_b200 import api, layouts

ctx = api.Context(0)
for cfg, r, Ds in (("opt-1.3b", 32, (3, 4)), ("llama7b-layer", 64, (2,)),
                   ("llama7b-layer", 128, (1,)), ("llama7b-layer", 96, (1,))):
    L = api.Layout(ctx, layouts.CONFIGS[cfg]())
    delta = L.empty()
    api.fill_gaussian(L, delta, 1e-3, seed=1, tag=1, worker=0)
    q = 4
    pay = api.compress(L, delta, r, api.QuantSpec(q, 0), None, 0, 2, 12345).payload
    for D in Ds:
        g = pay.repeat(D)
        res = {}
        for bf in (64, 128):
            api.set_option("effrank_big_from", bf)
            per, _ = api.effective_rank_device(L, g, D, r, q, 0.5)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(5):
                api.effective_rank_device(L, g, D, r, q, 0.5)
            e1.record()
            torch.cuda.synchronize()
            res[bf] = (e0.elapsed_time(e1) / 5, per.cpu())
        api.set_option("effrank_big_from", 96)
        print(json.dumps({"config": cfg, "r": r, "D": D, "K": D * r,
                          "ms_big64": res[64][0], "ms_big128": res[128][0],
                          "same_k": bool(torch.equal(res[64][1], res[128][1]))}), flush=True)
    del L
