"""PCIe probe: H2D-only, D2H-only and concurrent H2D + D2H throughput with pinned
buffers of the A3 b8 step's sizes (3 x 4.84 MB in, 4.84 MB out)."""
import torch

n = 96 * 197 * 64
h_in = [torch.randn(n).pin_memory() for _ in range(3)]
h_out = torch.empty(n).pin_memory()
d_in = [torch.empty(n, device="cuda") for _ in range(3)]
d_out = torch.randn(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=50):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    with torch.cuda.stream(s1):
        for d, h in zip(d_in, h_in):
            d.copy_(h, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


def both():
    with torch.cuda.stream(s1):
        for d, h in zip(d_in, h_in):
            d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


for name, fn, nbytes in [("h2d", h2d, 3 * 4 * n), ("d2h", d2h, 4 * n), ("both", both, 4 * 4 * n)]:
    ms = timeit(fn)
    print(f"{name}: {ms * 1e3:.1f} us per step, {nbytes / ms / 1e6:.1f} GB/s")
