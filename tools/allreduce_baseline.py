"""the per-step all-reduce baseline DiLoCoX replaces, at OPT-1.3B scale:
every inner step the workers average the full fp32 gradient slab (5.26 GB), vs the compressed
round's exchange (all-gather of the 15.4 MB payloads + the worker-0 warm-Q broadcast, through
the library's communicator: dlx_exchange). Two averaging variants of the baseline:
  nccl_avg  — ncclAllReduce(AVG) (what a DDP baseline runs; summation order is NCCL's)
  exact     — all-gather of the D slabs + the worker-order fp64 mean (dlx_mean_slabs), the
              reference's canonical mean (engine.cpp:559-570) as training.train_allreduce_per_step
              does it; bit-identical on every rank
Run under torchrun (N >= 2)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

from paper_2506_21263_b200 import api, layouts

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{rank}"))
ctx = api.Context(rank)
api.ensure_comm(ctx, rank, world)
n = layouts.numel(layouts.opt_1_3b())
g = torch.randn(n, device="cuda")
mean = torch.empty_like(g)
slabs = torch.empty(world * n, device="cuda") if world * n * 4 < 60e9 else None
pay = torch.zeros(15418344, dtype=torch.uint8, device="cuda")
gat = torch.zeros(world * pay.numel(), dtype=torch.uint8, device="cuda")
q = torch.zeros(14285312, device="cuda")  # worker-0 warm Q (57.1 MB, r = 32)


def timed(fn, k=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / k], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def exact():
    api.comm_allgather(ctx, g, slabs)
    api.mean_slabs(ctx, slabs, world, n, out=mean)


t_ar = timed(lambda: dist.all_reduce(g, op=dist.ReduceOp.AVG))
t_exact = timed(exact) if slabs is not None else None
t_ex = timed(lambda: api.exchange(ctx, pay, gat, q))
if rank == 0:
    print(json.dumps({"n_gpus": world, "per_step_nccl_avg_ms": t_ar,
                      "per_step_exact_mean_ms": t_exact,
                      "allreduce_bus_GBps": 2 * (world - 1) / world * 4 * n / t_ar / 1e6,
                      "dilocox_round_exchange_ms": t_ex,
                      "bytes_per_step_allreduce": 4 * n, "bytes_per_round_payload": pay.numel()}))
dist.destroy_process_group()
