"""Raw PCIe copy rates on this box (pinned host memory, CUDA events), the
floor under bench.py's e2e leg: H2D of 0.8 GB (configs[1] weights) and D2H of
4 GB (1e9 draws), alone and concurrently.
    python scripts/pcie_probe.py"""
import torch

h_w = torch.empty(10**8, dtype=torch.float64, pin_memory=True)
h_o = torch.empty(10**9, dtype=torch.int32, pin_memory=True)
d_w = torch.empty_like(h_w, device="cuda")
d_o = torch.empty_like(h_o, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def both():
    cur = torch.cuda.current_stream()
    e = torch.cuda.Event()
    e.record(cur)
    s1.wait_event(e)
    s2.wait_event(e)
    with torch.cuda.stream(s1):
        d_w.copy_(h_w, non_blocking=True)
    with torch.cuda.stream(s2):
        h_o.copy_(d_o, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


h2d = timed(lambda: d_w.copy_(h_w, non_blocking=True))
d2h = timed(lambda: h_o.copy_(d_o, non_blocking=True))
bo = timed(both)
print(f"H2D 0.8 GB: {h2d:.2f} ms ({0.8e9 / h2d / 1e6:.1f} GB/s); D2H 4 GB: {d2h:.2f} ms "
      f"({4e9 / d2h / 1e6:.1f} GB/s); sum {h2d + d2h:.2f} ms; both concurrently {bo:.2f} ms")
