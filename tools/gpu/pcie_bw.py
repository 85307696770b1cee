"""Host<->device link bandwidth on the box: pinned H2D, D2H, and both at once
on two streams (the ceiling of the e2e host-buffer path)."""
import json
import torch

n = 1 << 30
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


h2d = timed(lambda: d1.copy_(h1, non_blocking=True))
d2h = timed(lambda: h2.copy_(d2, non_blocking=True))
bi = timed(both)
print(json.dumps({"h2d_gbs": n / h2d / 1e6, "d2h_gbs": n / d2h / 1e6, "bidir_each_gbs": n / bi / 1e6,
                  "bytes": n}))
