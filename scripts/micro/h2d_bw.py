"""Pinned H2D bandwidth on the box: one copy of the C2 population's bytes, and the same split over two streams."""
import torch
n = 107_560_960
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for mode in ("one", "two", "one", "two"):
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        if mode == "one":
            d.copy_(h, non_blocking=True)
        else:
            s1.wait_stream(torch.cuda.current_stream()); s2.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s1):
                d[: n // 2].copy_(h[: n // 2], non_blocking=True)
            with torch.cuda.stream(s2):
                d[n // 2:].copy_(h[n // 2:], non_blocking=True)
            torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    print(mode, "median ms", round(ts[5], 3), "GB/s", round(n / ts[5] / 1e6, 1))
