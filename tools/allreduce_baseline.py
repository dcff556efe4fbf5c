"""the per-step all-reduce baseline DiLoCoX replaces: an NCCL all-reduce
(average) of the full fp32 gradient slab of OPT-1.3B every inner step, vs the compressed
round's exchange (all-gather of 15.4 MB payloads + warm-Q broadcast). Run under torchrun."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_2506_21263_b200 import layouts
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{rank}"))
n = layouts.numel(layouts.opt_1_3b())
g = torch.randn(n, device="cuda")
pay = torch.zeros(15418344, dtype=torch.uint8, device="cuda")
gat = torch.zeros(world * pay.numel(), dtype=torch.uint8, device="cuda")
q = torch.zeros(14285312, device="cuda")  # worker-0 warm Q (57.1 MB)
def timed(fn, k=5):
    for _ in range(2): fn()
    torch.cuda.synchronize(); dist.barrier()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(k): fn()
    e1.record(); torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / k], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
t_ar = timed(lambda: dist.all_reduce(g, op=dist.ReduceOp.AVG))
t_ex = timed(lambda: (dist.all_gather_into_tensor(gat, pay), dist.broadcast(q, src=0)))
if rank == 0:
    print(json.dumps({"n_gpus": world, "per_step_allreduce_ms": t_ar,
                      "allreduce_bus_GBps": 2 * (world - 1) / world * 4 * n / t_ar / 1e6,
                      "dilocox_round_exchange_ms": t_ex,
                      "bytes_per_step_allreduce": 4 * n, "bytes_per_round_payload": pay.numel()}))
dist.destroy_process_group()
