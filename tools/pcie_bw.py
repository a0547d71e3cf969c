"""Host<->device copy bandwidth on the box: H2D, D2H, and both at once on
two streams (pinned host memory), for the e2e step's per-step volume."""
import torch

n = 26 * 1024 * 1024
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def both():
    e = torch.cuda.current_stream()
    s1.wait_stream(e)
    s2.wait_stream(e)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    e.wait_stream(s1)
    e.wait_stream(s2)


for name, fn in (("h2d", lambda: d_in.copy_(h_in, non_blocking=True)),
                 ("d2h", lambda: h_out.copy_(d_out, non_blocking=True)),
                 ("both", both)):
    ms = timed(fn)
    print(f"{name:5s} {ms:.3f} ms  {n / ms / 1e6:.1f} GB/s per direction")
