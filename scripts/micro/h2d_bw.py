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
# the evaluate pipeline's copy pattern: 12 chunks x (nodes 2.1 MB + conns 6.7 MB)
nb, cb = 10_000 * 64 * 40, 10_000 * 256 * 32
hn, hc = h[:nb], h[nb:nb + cb]
dn_, dc_ = d[:nb], d[nb:nb + cb]
for chunks in (1, 6, 12, 24):
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for k in range(chunks):
            n0, n1 = nb * k // chunks, nb * (k + 1) // chunks
            c0, c1 = cb * k // chunks, cb * (k + 1) // chunks
            dn_[n0:n1].copy_(hn[n0:n1], non_blocking=True)
            dc_[c0:c1].copy_(hc[c0:c1], non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    print("chunks", chunks, "median ms", round(ts[5], 3), "GB/s", round(n / ts[5] / 1e6, 1))
