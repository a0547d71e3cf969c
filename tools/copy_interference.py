"""Does a concurrent host<->device DMA slow the step kernels?  Times pass 1
and pass 2 of the device-resident step (repeated on the same state) alone and
while a large H2D or D2H copy runs on another stream."""
import sys

sys.path.insert(0, ".")
import torch

from oracle import oracle as orc
from paper_2406_09654_b200 import physics
from tests.test_gpu_parity import make_dev

H = W = 1024
p0 = orc.synth_planes(H, W, 64, seed=1)
dev = make_dev(p0, 64, orc.synth_net(64, 0, seed=2))
sc = physics.step_scalars(0, physics.PhysicsParams())
big_h = torch.empty(512 << 20, dtype=torch.uint8, pin_memory=True)
big_d = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
cs = torch.cuda.Stream()
ks = torch.cuda.Stream()
n = 30


def timed(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(ks):
        a.record()
        for _ in range(n):
            fn()
        b.record()
    return a, b


kernels = {
    "pass1": lambda: dev.pass1(sc, 0, stream=ks.cuda_stream),
    "pass2": lambda: dev.pass2(0, stream=ks.cuda_stream),
}
dev.pass1(sc, 0)
for name, fn in kernels.items():
    for mode in ("alone", "h2d", "d2h", "alone"):
        torch.cuda.synchronize()
        if mode != "alone":
            with torch.cuda.stream(cs):
                if mode == "h2d":
                    big_d.copy_(big_h, non_blocking=True)
                else:
                    big_h.copy_(big_d, non_blocking=True)
        a, b = timed(fn)
        torch.cuda.synchronize()
        print(f"{name} {mode:6s}: {a.elapsed_time(b) / n * 1e3:.1f} us")
