"""PCIe copy-engine rates on this box (not a benchmark): pinned H2D alone,
D2H alone, and both directions at once, 320 MB each way, CUDA events."""
import torch

n = 320 * 2**20 // 4
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n // 2, dtype=torch.float32).pin_memory()
d_in = torch.empty(n, dtype=torch.float32, device="cuda")
d_out = torch.ones(n // 2, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    fn()
    for s in (s1, s2):
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


for name, fn in (("h2d 320MB", h2d), ("d2h 160MB", d2h), ("both", lambda: (h2d(), d2h()))):
    ts = sorted(timed(fn) for _ in range(7))
    ms = ts[3]
    print(f"{name}: {ms:.3f} ms  h2d-equivalent {320 * 2**20 / 1e6 / ms:.1f} GB/s", flush=True)
