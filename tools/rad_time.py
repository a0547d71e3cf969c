"""Time one config-3 field-radiation event (host mutate + admission + device
selection / CPPN expression / remap) on a device-resident C3 state."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2406_09654_b200 import engine, radiation  # noqa: E402

st = engine.baseline_state("c3")
dev = engine.device_of(st)
st._evo_binding.sync_params(st.pool)
dev.upload(st.substrate.front)
dev.sync()
for k in range(3):
    t = 50 * (k + 1)
    st.substrate.step_counter = t
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prof = {}
    r = radiation.field_radiation(st, t, 0.01)
    dev.sync()
    print(f"radiation event {k}: {1e3 * (time.perf_counter() - t0):.1f} ms {r}", flush=True)
import cProfile, pstats  # noqa: E402,E401
st.substrate.step_counter = 200
pr = cProfile.Profile()
pr.enable()
radiation.field_radiation(st, 200, 0.01)
dev.sync()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
