"""Pinned host <-> device copy bandwidth on the box (context for bench.py's e2e number): H2D
alone, D2H alone, and both at once on two streams; 537 MB each (config 5's X / Y at nrhs 32)."""
import torch

n = 537 * 1024 * 1024 // 16
h_in = torch.empty(n, dtype=torch.complex128).pin_memory()
h_out = torch.empty(n, dtype=torch.complex128).pin_memory()
d_in = torch.empty(n, dtype=torch.complex128, device="cuda")
d_out = torch.empty(n, dtype=torch.complex128, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
nb = n * 16


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t1 = timed(lambda: d_in.copy_(h_in, non_blocking=True))
t2 = timed(lambda: h_out.copy_(d_out, non_blocking=True))
t3 = timed(both)
print(f"H2D {nb / t1 / 1e6:.1f} GB/s ({t1:.2f} ms)  D2H {nb / t2 / 1e6:.1f} GB/s ({t2:.2f} ms)  "
      f"both {t3:.2f} ms ({2 * nb / t3 / 1e6:.1f} GB/s total)")
