"""Host<->device copy bandwidth probe (pinned, pageable, chunked, both directions at once).
Experiments only."""
import time
import torch

dev = torch.device("cuda:0")
for gb in (0.25, 1.0, 5.0):
    n = int(gb * 2**30) // 4
    h = torch.empty(n, dtype=torch.float32, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
    d = torch.empty(n, dtype=torch.float32, device=dev)
    d2 = torch.empty(n, dtype=torch.float32, device=dev)
    h.fill_(1.0)
    s1 = torch.cuda.Stream()
    s2 = torch.cuda.Stream()
    for name, fn in [
        ("h2d", lambda: d.copy_(h, non_blocking=True)),
        ("d2h", lambda: h2.copy_(d, non_blocking=True)),
    ]:
        fn(); torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        print(f"{gb:5.2f} GB {name}: {n*4/e0.elapsed_time(e1)/1e6:7.1f} GB/s", flush=True)
    # both directions concurrently
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{gb:5.2f} GB duplex: {2*n*4/dt/1e9:7.1f} GB/s aggregate", flush=True)
    del h, h2, d, d2
print(torch.cuda.get_device_name(), flush=True)
