"""Time config-3 field-radiation events (host NEAT + device selection / CPPN
expression / remap) on a device-resident C3 state, with a phase breakdown."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2406_09654_b200 import engine, neat, radiation  # noqa: E402

st = engine.baseline_state("c3")
dev = engine.device_of(st)
st._evo_binding.sync_params(st.pool)
dev.upload(st.substrate.front)
dev.sync()
orig = {n: getattr(obj, n) for obj, n in ((neat, "mutate_batch"),)}
timers = {}


def timed(name, fn):
    def w(*a, **k):
        t0 = time.perf_counter()
        r = fn(*a, **k)
        timers[name] = timers.get(name, 0.0) + time.perf_counter() - t0
        return r
    return w


neat.mutate_batch = timed("mutate_batch", neat.mutate_batch)
neat.mutate_batch_deferred = timed("plan_mutate", neat.mutate_batch_deferred)
neat.number_deferred = timed("number", neat.number_deferred)
dev.select_cells = timed("select_cells", dev.select_cells)
dev.remap_selected = timed("remap", dev.remap_selected)
dev.express_cppn = timed("express_cppn", dev.express_cppn)
st.pool.admit_batch = timed("admit_batch", st.pool.admit_batch)
neat.compile_programs = timed("compile", neat.compile_programs)
for k in range(4):
    t = 50 * (k + 1)
    st.substrate.step_counter = t
    timers.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = radiation.field_radiation(st, t, 0.01)
    dev.sync()
    tot = 1e3 * (time.perf_counter() - t0)
    print(f"radiation event {k}: {tot:.1f} ms {r} " + ", ".join(f"{n} {1e3 * v:.2f}" for n, v in timers.items()),
          flush=True)

if "--profile" in sys.argv:
    import cProfile
    import pstats

    st.substrate.step_counter = 300
    pr = cProfile.Profile()
    pr.enable()
    for k in range(3):
        radiation.field_radiation(st, 300 + 50 * k, 0.01)
        dev.sync()
    pr.disable()
    pstats.Stats(pr).sort_stats("cumtime").print_stats(40)
