"""Host<->device copy bandwidth from pinned memory (the e2e ceiling)."""
import json
import torch

for mb in (12.6, 16.8, 25.2):
    n = int(mb * 1e6)
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        d.copy_(h); h.copy_(d)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    for _ in range(10):
        d.copy_(h, non_blocking=True)
    e[1].record()
    for _ in range(10):
        h.copy_(d, non_blocking=True)
    e[2].record()
    torch.cuda.synchronize()
    print(json.dumps({"MB": mb, "h2d_GBs": n * 10 / e[0].elapsed_time(e[1]) / 1e6,
                      "d2h_GBs": n * 10 / e[1].elapsed_time(e[2]) / 1e6}))
