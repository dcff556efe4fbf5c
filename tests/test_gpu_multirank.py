"""N>1 on real GPUs (skipped with fewer than 2 devices): two ranks (torchrun, NCCL over
NVLink) run overlapped rounds through OuterSync; every rank must end with bitwise-identical
anchors and velocities (SPEC anchor consistency: the all-gathered payloads are reconstructed
with a self_index-independent summation order), and the result must match a single-process
D=2 reference round (orc_outer_round) within the state tolerance."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r'''
import json, os, sys
sys.path.insert(0, os.environ["DLX_ROOT"])
import numpy as np, torch, torch.distributed as dist
from oracle.oracle import Oracle, Table
from paper_2506_21263_b200 import api
from paper_2506_21263_b200.engine import OuterConfig, OuterSync
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{rank}"))
shapes = [(96, 64), (64,), (64, 200), (200,), (130, 48)]
R = Oracle("restatement")
t = Table(shapes)
n = t.numel()
anchor0 = (np.float32(0.02) * R.gaussian(R.stream(7, 0), n)[0]).astype(np.float32)
locs = [(anchor0 - np.float32(1e-3) * R.gaussian(R.stream(1, 10 + w), n)[0]).astype(np.float32)
        for w in range(world)]
ctx = api.Context(rank)
L = api.Layout(ctx, [(f"t{i}", s) for i, s in enumerate(shapes)])
cfg = OuterConfig(rank1=8, qbits=4, power_iters=2, adaptive=True, seed=1, overlap=True,
                  hold_rank=True)
eng = OuterSync(L, cfg, L.pack(anchor0), world=world, rank=rank)
dl = L.pack(locs[rank])
recs = [eng.step(dl) for _ in range(4)]
torch.cuda.synchronize()
out = {"anchor": L.unpack(eng.anchor).tolist(), "vel": L.unpack(eng.velocity).tolist(),
       "pend": L.unpack(eng.pending).tolist(), "rprime": [r.r_prime for r in recs]}
json.dump(out, open(os.path.join(os.environ["DLX_OUT"], f"rank{rank}.json"), "w"))
dist.barrier()
dist.destroy_process_group()
'''


@pytest.mark.parametrize("lib_nccl", ["1", "0"])
def test_two_ranks_nccl_identical_state(tmp_path, oracle, lib_nccl):
    """lib_nccl = 1: the exchange through the C-ABI (dlx_exchange, the library's own NCCL
    communicator); 0: through torch.distributed."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    env = dict(os.environ, DLX_ROOT=ROOT, DLX_OUT=str(tmp_path), DLX_LIB_NCCL=lib_nccl)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(29531 + int(lib_nccl)),
           str(script)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = [json.load(open(tmp_path / f"rank{k}.json")) for k in range(2)]
    a0, a1 = np.array(res[0]["anchor"], np.float32), np.array(res[1]["anchor"], np.float32)
    assert np.array_equal(a0, a1), "anchors differ across ranks"
    assert np.array_equal(np.array(res[0]["vel"]), np.array(res[1]["vel"]))
    assert res[0]["rprime"] == res[1]["rprime"]
    # single-process D=2 reference rounds (rounds 2..4; round 1 stages only)
    from oracle.oracle import Table
    shapes = [(96, 64), (64,), (64, 200), (200,), (130, 48)]
    t = Table(shapes)
    n = t.numel()
    anchor0 = (np.float32(0.02) * oracle.gaussian(oracle.stream(7, 0), n)[0]).astype(np.float32)
    locs = np.stack([(anchor0 - np.float32(1e-3) * oracle.gaussian(oracle.stream(1, 10 + w), n)[0])
                     for w in range(2)]).astype(np.float32)
    a = anchor0.copy()
    v = np.zeros(n, np.float32)
    pend = np.stack([anchor0 - locs[w] for w in range(2)]).astype(np.float32)
    wq = np.zeros(max(1, sum(s[1] * min(8, *s) for s in shapes if len(s) == 2)), np.float32)
    wr = 0
    for rnd in (2, 3, 4):
        out = oracle.outer_round(t, 2, 1, rnd, 8, 4, 0, 2, False, 0.5, 8, 0.7, 0.9, False, 1,
                                 a, v, pend, locs.copy(), wr, wq)
        wr = out["warm_rank"]
    from tests._util import rel_fro
    assert rel_fro(a0 - anchor0, a - anchor0) <= 1e-2
    for k in range(2):
        assert rel_fro(np.array(res[k]["pend"], np.float32), pend[k]) <= 1e-2


PY_WORKER = r'''
import json, os, sys
sys.path.insert(0, os.environ["DLX_ROOT"])
import numpy as np, torch, torch.distributed as dist
from paper_2506_21263_b200 import api, layouts
from paper_2506_21263_b200.engine import OuterConfig, OuterSync
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{rank}"))
ctx = api.Context(rank)
L = api.Layout(ctx, layouts.mini_opt())
anchor = L.empty()
api.fill_gaussian(L, anchor, 0.02, seed=7, tag=0xA7C4, worker=0)
local = L.empty()
api.fill_gaussian(L, local, -1e-3, seed=1, tag=0xDA7A, worker=rank, base=anchor)
cfg = OuterConfig(rank1=8, qbits=4, power_iters=2, adaptive=True, window_c=5, H1=125, seed=1,
                  overlap=True, hold_rank=False)
eng = OuterSync(L, cfg, anchor, world=world, rank=rank)
recs = [eng.step(local) for _ in range(4)]
torch.cuda.synchronize()
L.unpack(eng.anchor).tofile(os.path.join(os.environ["DLX_OUT"], f"py{rank}.bin"))
json.dump([r.r_prime for r in recs], open(os.path.join(os.environ["DLX_OUT"], f"py{rank}.json"), "w"))
dist.barrier()
dist.destroy_process_group()
'''


def test_cpp_worker_processes_match_python_engine(tmp_path):
    """A pure C++ host (cpp/worker_main: one process per GPU, NCCL bootstrapped from a file,
    everything through the C-ABI — dlx_ctx_create_dist, dlx_compress, dlx_exchange,
    dlx_effective_rank, dlx_outer_update, dlx_adapt_compression) on the SURVEY C1 layout:
    both ranks end with bitwise-identical anchors, and the result is bitwise identical to the
    Python engine (OuterSync over torchrun) on the same inputs — the same kernels in the
    same order, whichever host drives them (the Python engine is checked against the
    reference in test_gpu_engine / test_gpu_headline)."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    exe = os.path.join(ROOT, "cpp", "_build", "worker_main")
    if not os.path.exists(exe):
        pytest.skip("cpp/_build/worker_main not built")
    uid = tmp_path / "uid"
    procs = [subprocess.Popen([exe, str(r), "2", str(r), str(uid), str(tmp_path / f"cpp{r}"),
                               "4", "8", "4", "1"], stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True) for r in range(2)]
    for p in procs:
        out, err = p.communicate(timeout=600)
        assert p.returncode == 0, err[-3000:]
    c0 = np.fromfile(tmp_path / "cpp0.bin", dtype=np.float32)
    c1 = np.fromfile(tmp_path / "cpp1.bin", dtype=np.float32)
    assert np.array_equal(c0, c1), "C++ workers disagree"
    script = tmp_path / "pyworker.py"
    script.write_text(PY_WORKER)
    env = dict(os.environ, DLX_ROOT=ROOT, DLX_OUT=str(tmp_path))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29541", str(script)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    p0 = np.fromfile(tmp_path / "py0.bin", dtype=np.float32)
    assert np.array_equal(p0, c0), "C++ host and Python host disagree"
    rp_cpp = [int(line.split()[2]) for line in open(tmp_path / "cpp0.txt")]
    assert rp_cpp == json.load(open(tmp_path / "py0.json"))


XCHG_WORKER = r'''
import os, sys
sys.path.insert(0, os.environ["DLX_ROOT"])
import torch, torch.distributed as dist
from paper_2506_21263_b200 import api
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{rank}"))
ctx = api.Context(rank)
api.ensure_comm(ctx, rank, world)
pb = 1000003
pay = torch.full((pb,), rank + 1, dtype=torch.uint8, device="cuda")
gat = torch.zeros(world * pb, dtype=torch.uint8, device="cuda")
wq = torch.full((77777,), float(rank + 10), device="cuda")
side = torch.cuda.Stream()
with torch.cuda.stream(side):
    api.exchange(ctx, pay, gat, wq, defer_warm=True)   # broadcast joined later
    ctx.wait_warm()
    out = torch.zeros(1, dtype=torch.int32, device="cuda")
torch.cuda.current_stream().wait_stream(side)
ok = all(bool((gat[w * pb:(w + 1) * pb] == w + 1).all()) for w in range(world))
ok = ok and bool((wq == 10.0).all())
# the all-gather helper and the exact f64 sum used by the effective-rank shards
x = torch.full((5,), float(rank + 1), dtype=torch.float64, device="cuda")
api.comm_allreduce_sum_f64(ctx, x)
ok = ok and bool((x == world * (world + 1) / 2).all())
ctx.comm_check()
torch.cuda.synchronize()
open(os.path.join(os.environ["DLX_OUT"], f"x{rank}"), "w").write("ok" if ok else "bad")
dist.barrier()
dist.destroy_process_group()
'''


def test_library_exchange_primitives(tmp_path):
    """dlx_exchange (all-gather in worker order + worker-0 broadcast, deferred and joined with
    dlx_exchange_wait_warm), dlx_comm_allreduce_sum_f64 and dlx_comm_check over two ranks."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    script = tmp_path / "xworker.py"
    script.write_text(XCHG_WORKER)
    env = dict(os.environ, DLX_ROOT=ROOT, DLX_OUT=str(tmp_path))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29551", str(script)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert [open(tmp_path / f"x{k}").read() for k in range(2)] == ["ok", "ok"]
