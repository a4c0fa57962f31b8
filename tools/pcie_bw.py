"""Diagnostic: pinned H2D / D2H bandwidth, alone and concurrently (the bound
of the pipelined e2e figure), for a C2-sized state (18.9 MB)."""
import torch

n = 131072 * 18
h1 = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=50):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d1.copy_(h1, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return 8 * n * (h2d + d2h) / ms / 1e6, ms


run(True, True, 5)
for name, a, b in (("H2D", True, False), ("D2H", False, True), ("both", True, True)):
    gbs, ms = run(a, b)
    print(f"{name}: {gbs:.1f} GB/s total, {ms:.3f} ms per 18.9 MB pair")
