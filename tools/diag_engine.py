"""Diagnostics for tests/test_radiation.py::test_engine_step_with_radiation_equals_its_components."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2406_09654_b200 import _lib, engine, physics, radiation  # noqa: E402
from paper_2406_09654_b200.device import DeviceSubstrate  # noqa: E402
from paper_2406_09654_b200.substrate import create_substrate  # noqa: E402
from tests.test_radiation import _front, _golden, _pool  # noqa: E402

z, g = _golden()
case = "dense"
seed = int(z[case + "_seed"])
cfg = engine.ExperimentConfig(grid=engine.GridConfig(64, 64), seed=seed)
pool_a = _pool(z, g, case, net_factory=radiation.device_net_factory(16))
pool_b = _pool(z, g, case)
sub_a, sub_b = create_substrate(64, 64), create_substrate(64, 64)
_front(sub_a, z, case + "_pre_")
_front(sub_b, z, case + "_pre_")
state = engine.SimState(substrate=sub_a, pool=pool_a, config=cfg, master_seed=seed)
dev = DeviceSubstrate(64, 64, pool_b.capacity, hidden=0)
af = engine.build_action_field(state)
af2 = engine.build_action_field(state)
print("af repeat equal:", np.array_equal(af.block(), af2.block()))
engine.step(state)
dev.set_slots(pool_b.slot_states())
dev.upload(sub_b.front)
dev.set_actions(af.cells, af.block())
dev.step_raw(physics.step_scalars(0, cfg.physics), 0, flags=_lib.F_INJECT_ACTIONS | _lib.F_RECORD_EVENTS | _lib.F_NO_CENSUS)
dev.download(sub_b.back)
Ea = sub_a.front.channels["energy"][0]
Eb = sub_b.back.channels["energy"][0]
d = np.argwhere(Ea.view(np.uint32) != Eb.view(np.uint32))
print("E differs at", len(d), "cells; first", d[:6].tolist())
for (y, x) in d[:6]:
    c = y * 64 + x
    k = np.searchsorted(af.cells, c)
    print(" cell", c, "Ea", Ea[y, x], "Eb", Eb[y, x], "pre E", z[case + "_pre_E"][y, x], "gi", z[case + "_pre_gi"][y, x],
          "act", af.block()[k] if k < len(af.cells) and af.cells[k] == c else None)
# the same step without radiation through engine.step (host planes)
cfg2 = engine.ExperimentConfig(grid=engine.GridConfig(64, 64), seed=seed,
                               evolution=engine.EvolutionRates(p_radiation=0.0, p_merge=0.0))
pool_c = _pool(z, g, case, net_factory=radiation.device_net_factory(16))
sub_c = create_substrate(64, 64)
_front(sub_c, z, case + "_pre_")
st_c = engine.SimState(substrate=sub_c, pool=pool_c, config=cfg2, master_seed=seed)
engine.step(st_c)
Ec = sub_c.front.channels["energy"][0]
print("no-radiation engine.step vs radiation engine.step E differ:", int((Ec.view(np.uint32) != Ea.view(np.uint32)).sum()),
      "vs injected:", int((Ec.view(np.uint32) != Eb.view(np.uint32)).sum()))
