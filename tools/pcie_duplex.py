"""PCIe copy-engine probe: H2D and D2H alone, back to back, and concurrently on two streams
(pinned host memory, CUDA events, best of 20)."""
import torch

s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for mb in (0.64, 1.28, 2.56, 10.24):
    n = int(mb * 1e6)
    hi = torch.empty(n, dtype=torch.uint8).pin_memory()
    ho = torch.empty(n, dtype=torch.uint8).pin_memory()
    di = torch.empty(n, dtype=torch.uint8, device="cuda")
    do = torch.empty(n, dtype=torch.uint8, device="cuda")

    def timed(fn):
        best = 1e9
        for _ in range(20):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            cur = torch.cuda.current_stream()
            e0.record(cur)
            fn(cur)
            e1.record(cur)
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3)
        return best

    def h2d(cur):
        di.copy_(hi, non_blocking=True)

    def d2h(cur):
        ho.copy_(do, non_blocking=True)

    def serial(cur):
        di.copy_(hi, non_blocking=True)
        ho.copy_(do, non_blocking=True)

    def duplex(cur):
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            di.copy_(hi, non_blocking=True)
        with torch.cuda.stream(s2):
            ho.copy_(do, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    r = {k: timed(f) for k, f in (("h2d", h2d), ("d2h", d2h), ("serial", serial), ("duplex", duplex))}
    print(f"{mb:6.2f} MB: " + "  ".join(f"{k} {v:7.1f} us ({n / v / 1e3:5.1f} GB/s)" for k, v in r.items()))
