"""Host<->device copy bandwidth on this box (pinned buffers), alone and concurrently."""
import json

import torch

n = 805306368 // 2
h = torch.empty(n, dtype=torch.bfloat16).pin_memory()
d = torch.empty(n, dtype=torch.bfloat16, device="cuda")
hd = torch.empty(n // 6, dtype=torch.bfloat16).pin_memory()
dd = torch.empty(n // 6, dtype=torch.bfloat16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        hd.copy_(dd, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


h2d = t(lambda: d.copy_(h, non_blocking=True))
d2h = t(lambda: hd.copy_(dd, non_blocking=True))
bb = t(both)
print(json.dumps({"h2d_GBps": 2 * n / h2d / 1e6, "d2h_GBps": 2 * (n // 6) / d2h / 1e6, "h2d_ms": h2d,
                  "d2h_ms": d2h, "both_ms": bb}))
