"""SURVEY C5 accuracy sweep: compression error of the device compress on the full OPT-1.3B
layout for q in {2, 4, 8} x r in {4, ..., 256} (low-rank + noise drift, the realistic-spectrum
generator), with the CPU oracle's error on one decoder-layer tensor subset beside it.
Writes profiles/c5_accuracy.md. Run on a GPU box."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from oracle.oracle import Oracle, Table
from paper_2506_21263_b200 import api, layouts

oracle = Oracle("restatement")
ctx = api.Context(0)
table = layouts.opt_1_3b()
L = api.Layout(ctx, table)
shapes = [s for _, s in table]
# device drift: per 2-D tensor a rank-16 decaying component + noise (deterministic seeds)
gen = torch.Generator(device="cuda").manual_seed(5)
delta = L.empty()
host_parts = []
off = L.offsets
for i, s in enumerate(shapes):
    o = int(off[i])
    if len(s) == 2:
        a, b = s
        u = torch.randn(a, 16, device="cuda", generator=gen)
        v = torch.randn(b, 16, device="cuda", generator=gen)
        sv = 1e-3 * 0.8 ** torch.arange(16, device="cuda", dtype=torch.float32)
        d = (u * sv) @ v.T + 1e-5 * torch.randn(a, b, device="cuda", generator=gen)
        delta[o:o + a * b] = d.reshape(-1)
    else:
        delta[o:o + s[0]] = 1e-4 * torch.randn(s[0], device="cuda", generator=gen)
torch.cuda.synchronize()
# oracle subset: the first decoder layer's attention projections + biases
sub_idx = [i for i, (nm, s) in enumerate(table) if nm.startswith("layers.0.") and ("proj" in nm)]
sub_shapes = [shapes[i] for i in sub_idx]
sub_data = np.concatenate([delta[int(off[i]):int(off[i]) + int(np.prod(shapes[i]))].cpu().numpy()
                           for i in sub_idx])
sub_t = Table(sub_shapes)
Ls = api.Layout(ctx, [(f"s{i}", s) for i, s in enumerate(sub_shapes)])
rows = []
stats = torch.zeros(8, dtype=torch.float64, device="cuda")
z = L.empty(); za = L.empty(); zv = L.empty()
for q in (2, 4, 8):
    for r in (4, 8, 16, 32, 64, 128, 256):
        st = 12345
        t0 = time.time()
        res = api.compress(L, delta, r, api.QuantSpec(q, api.STOCHASTIC), None, 0, 2, st)
        # full-model measure_error through the fused update (self_index = 0, D = 1)
        pend = delta.clone()
        api.outer_update(L, res.payload, 1, r, q, pend, za, None, zv, 0.7, 0.9, False,
                         mode=api.SYNC, self_index=0, stats=stats)
        s_ = stats.cpu().numpy()
        err_gpu = s_[0] / s_[1]
        # oracle vs device on the subset
        rs = api.compress(Ls, Ls.pack(sub_data), r, api.QuantSpec(q, api.STOCHASTIC), None, 0, 2, st)
        s2 = torch.zeros(8, dtype=torch.float64, device="cuda")
        api.outer_update(Ls, rs.payload, 1, r, q, Ls.pack(sub_data), Ls.empty(), None, Ls.empty(),
                         0.7, 0.9, False, mode=api.SYNC, self_index=0, stats=s2)
        s2 = s2.cpu().numpy()
        ref = oracle.compress(sub_t, sub_data, r, q, 0, 2, st)
        err_ref = oracle.measure_error(sub_t, sub_data, sub_t.ranks(r), ref["codes"], ref["scales"])
        rows.append((q, r, err_gpu, s2[0] / s2[1], err_ref, L.payload_bits(r, q) / 8 / 1e6,
                     time.time() - t0))
        print(rows[-1], flush=True)
out = ["# C5 accuracy sweep (SURVEY §8d)", "",
       "OPT-1.3B layout, low-rank (16, decaying) + noise drift, stochastic rounding, "
       "power_iters = 2. `measure_error` = ||dec(payload) - delta||^2 / ||delta||^2 "
       "(compress.cpp:246-262): full model on the GPU; on the layer-0 attention projections "
       "for the GPU and the CPU oracle (fp64 reference restatement) side by side.", "",
       "| q | r | full model (GPU) | layer-0 subset (GPU) | layer-0 subset (oracle) | payload MB |",
       "|---|---|---|---|---|---|"]
for q, r, eg, es, er, mb, _ in rows:
    out.append(f"| {q} | {r} | {eg:.4e} | {es:.4e} | {er:.4e} | {mb:.3f} |")
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
open(os.path.join(ROOT, "profiles", "c5_accuracy.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out))
