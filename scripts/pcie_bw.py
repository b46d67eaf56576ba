"""H2D / D2H bandwidth of pinned copies on one GPU with 1, 2 and 4 streams, alone and with a
concurrent D2H (why buffer_copy splits large copies over two copy streams)."""
import torch, time
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True); h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h2 = torch.empty(n // 2, dtype=torch.uint8, pin_memory=True)
d2 = torch.empty(n // 2, dtype=torch.uint8, device="cuda")
def run(ns, d2h=False):
    ss = [torch.cuda.Stream() for _ in range(ns)]
    torch.cuda.synchronize(); t = time.perf_counter()
    for r in range(3):
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                a, b = i * n // ns, (i + 1) * n // ns
                d[a:b].copy_(h[a:b], non_blocking=True)
        if d2h:
            s2 = torch.cuda.Stream()
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 3
    return n / dt / 1e9
for ns in (1, 2, 4):
    print(f"H2D 1 GiB, {ns} streams: {run(ns):.1f} GB/s; with a concurrent 0.5 GiB D2H: {run(ns, True):.1f} GB/s (H2D bytes / time)")
