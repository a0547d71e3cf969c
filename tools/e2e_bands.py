"""e2e (evo_step_host) wall time of a BASELINE config for several row-band
counts: python tools/e2e_bands.py c3 4 8 16"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2406_09654_b200 import engine, physics  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
st = engine.baseline_state(cfg)
dev = engine.device_of(st)
st._evo_binding.sync_params(st.pool)
f, b = st.substrate.front, st.substrate.back
dev.pin(f)
dev.pin(b)
sc = physics.step_scalars(0, st.config.physics)
for nb in [int(x) for x in sys.argv[2:]] or [4, 8, 16]:
    for _ in range(2):
        dev.step_host(f, b, sc, 0, bands=nb)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        dev.step_host(f, b, sc, 0, bands=nb)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / 5 * 1e3
    print(f"{cfg} bands {nb}: {ms:.2f} ms/step, {st.substrate.width * st.substrate.height / ms / 1e6:.3f} G cell-updates/s",
          flush=True)
