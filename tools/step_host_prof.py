"""Wall time of evo_step_host (host planes in, host planes out) on config 2
for several band counts, pinned vs pageable host planes."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from oracle import oracle as orc
from paper_2406_09654_b200 import physics
from paper_2406_09654_b200.substrate import STANDARD_CHANNELS, PlaneSet
from tests.test_gpu_parity import make_dev
import os

H = W = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
p0 = orc.synth_planes(H, W, 64, seed=1)
dev = make_dev(p0, 64, orc.synth_net(64, 0, seed=2))


def planes():
    if os.environ.get("EVO_SEPARATE_PLANES"):
        return orc.Planes(np.empty((H, W), np.float32), np.empty((H, W), np.float32),
                          np.empty((3, H, W), np.float32), np.empty((H, W), np.int32), np.empty((H, W), np.uint8))
    ps = PlaneSet(STANDARD_CHANNELS, H, W)  # one host block (the engine's layout)
    return orc.Planes(ps.channels["energy"][0], ps.channels["infrastructure"][0], ps.channels["communication"],
                      ps.genome_index, ps.rotation)


a, b = planes(), planes()
for x, y in zip((a.E, a.I, a.C, a.gi, a.rot), (p0.E, p0.I, p0.C, p0.gi, p0.rot)):
    x[...] = y
sc = physics.step_scalars(0, physics.PhysicsParams())
import os
import threading


def sample_clocks(fn, seconds=1.0):
    """Run fn repeatedly for ~seconds while sampling the SM clock (NVML)."""
    import pynvml

    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    clocks, stop = [], threading.Event()

    def poll():
        while not stop.is_set():
            clocks.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            time.sleep(0.002)

    th = threading.Thread(target=poll)
    th.start()
    t0, n = time.perf_counter(), 0
    while time.perf_counter() - t0 < seconds:
        fn()
        n += 1
    stop.set()
    th.join()
    return (time.perf_counter() - t0) / n * 1e3, sorted(clocks)[len(clocks) // 2], min(clocks), max(clocks)


if os.environ.get("EVO_CLOCKS"):
    dev.pin(a)
    dev.pin(b)
    for bands in (1, 4):
        ms, med, lo, hi = sample_clocks(lambda: dev.step_host(a, b, sc, 0, bands=bands))
        print(f"step_host bands={bands}: {ms:.3f} ms, SM clock median {med} min {lo} max {hi} MHz")

    def resident():
        dev.step_raw(sc, 0)
        dev.sync()
    ms, med, lo, hi = sample_clocks(resident)
    print(f"device-resident step: {ms:.3f} ms, SM clock median {med} min {lo} max {hi} MHz")
    sys.exit(0)
if os.environ.get("EVO_PIPE_TRACE"):
    dev.pin(a)
    dev.pin(b)
    for bands in (3, 4, 6):
        for _ in range(3):
            dev.step_host(a, b, sc, 0, bands=bands)
    sys.exit(0)
for pinned in (False, True):
    if pinned:
        dev.pin(a)
        dev.pin(b)
    for bands in (1, 2, 3, 4, 6, 8, 12, 0):
        for _ in range(3):
            dev.step_host(a, b, sc, 0, bands=bands)
        n = 20
        t0 = time.perf_counter()
        for _ in range(n):
            dev.step_host(a, b, sc, 0, bands=bands)
        ms = (time.perf_counter() - t0) / n * 1e3
        print(f"pinned={pinned} bands={bands:2d}: {ms:.3f} ms/step  {H * W / ms / 1e6:.2f} G cell-updates/s")
