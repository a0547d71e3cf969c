import time, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2406_09654_b200 import engine, physics
st = engine.baseline_state('c2')
engine.step(st); torch.cuda.synchronize()
b = engine._binding(st); dev = b.dev; sub = st.substrate
def t(f, n=20):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
print("engine.step      %.3f ms" % t(lambda: engine.step(st)))
print("upload           %.3f ms" % t(lambda: dev.upload(sub.front)))
print("download         %.3f ms" % t(lambda: dev.download(sub.back)))
sc = physics.step_scalars(0, st.config.physics)
print("step_raw         %.3f ms" % t(lambda: (dev.step_raw(sc, 0), dev.sync())))
print("read_census      %.3f ms" % t(lambda: dev.read_census()))
print("read_stats       %.3f ms" % t(lambda: dev.read_stats()))
counts = dev.read_census()[0]
print("update_census    %.3f ms" % t(lambda: st.pool.update_census(counts, 5)))
print("sync_params      %.3f ms" % t(lambda: b.sync_params(st.pool)))
