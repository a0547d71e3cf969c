"""Per-band timeline of evo_step_host on a config (EVO_PIPE_TRACE=1 must be
set in the environment): python tools/e2e_trace.py [c3]"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2406_09654_b200 import engine  # noqa: E402

st = engine.baseline_state(sys.argv[1] if len(sys.argv) > 1 else "c3")
for _ in range(3):
    engine.step(st)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    engine.step(st)
torch.cuda.synchronize()
print(f"engine.step {1e3 * (time.perf_counter() - t0) / 5:.2f} ms", file=sys.stderr)
