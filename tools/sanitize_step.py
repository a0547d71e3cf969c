"""Exercise every device kernel of the library on small worlds, for
compute-sanitizer (memcheck / racecheck / synccheck, one tool per run):

    compute-sanitizer --tool racecheck python tools/sanitize_step.py

Paths: the per-tile direct kernel (export and not), the gather path (FFMA2
and tcgen05 nets) and genome-sorted rows for a large direct pool, the cluster-sharded tile kernel, the hidden-layer net on
the tensor cores and on the CUDA cores, injected actions, pass 2 with events,
strips with halo exchange, the CPPN expression kernel, field-radiation
selection / remap, render, MSC and plane sums; 64x64 and 256x256."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import oracle as orc  # noqa: E402
from paper_2406_09654_b200 import _lib, engine, neat, physics, radiation  # noqa: E402
from paper_2406_09654_b200.device import DeviceSubstrate  # noqa: E402
from paper_2406_09654_b200.hypernet import DenseParams, DirectParams  # noqa: E402


def params(net):
    if net.hidden == 0:
        return [DirectParams(net.w2[i], net.b2[i]) for i in range(net.capacity)]
    return [DenseParams(net.w1[i], net.b1[i], net.w2[i], net.b2[i]) for i in range(net.capacity)]


def world(n, g, hidden, flags_list, steps=2):
    p = orc.synth_planes(n, n, g, seed=n + g)
    net = orc.synth_net(g, hidden, seed=g)
    ph = physics.PhysicsParams(cycle_period=20)
    for flags in flags_list:
        dev = DeviceSubstrate(n, n, g, hidden=hidden)
        dev.set_params(params(net))
        dev.set_slots(np.ones(g, np.int8))
        dev.upload(p)
        for t in range(steps):
            dev.step_raw(physics.step_scalars(t, ph), t, flags=flags)
        if flags & _lib.F_EXPORT_ACTIONS:
            cells, acts = dev.get_actions()
            dev.set_actions(cells, acts)
            dev.step_raw(physics.step_scalars(steps, ph), steps, flags=_lib.F_INJECT_ACTIONS | _lib.F_RECORD_EVENTS)
            dev.read_events()
        dev.render_rgb()
        dev.read_census()
        dev.close()


def main():
    ex, rec = _lib.F_EXPORT_ACTIONS, _lib.F_RECORD_EVENTS
    for n in (64, 256):
        world(n, 8, 0, [0, ex | rec, _lib.F_MMA_NET])                           # per-tile direct kernel
        world(n, 300, 0, [0, rec, _lib.F_UNFUSED], steps=4)                      # gather: fused + lazy steps, unfused
        world(n, 300, 0, [ex, _lib.F_TC_DIRECT, _lib.F_TC_DIRECT | ex,         # gather (export / tcgen05)
                          _lib.F_ROWS_NET, _lib.F_SHARD_NET, _lib.F_TILE_NET])   # rows / sharded / tile
        world(n, 20, 128, [0, ex, _lib.F_CUDA_CORE_NET])                        # tcgen05 hidden net
        world(n, 6, 16, [0, _lib.F_TC_NET])                                     # narrow hidden layer
    # strips (halo pack / unpack, census finish)
    from paper_2406_09654_b200.strips import DeviceStrip, StripPlan, step_local

    p = orc.synth_planes(64, 48, 5, seed=3)
    net = orc.synth_net(5, 0, seed=3)
    plan = StripPlan(64, 48, 2)
    strips = []
    for r in range(2):
        s = DeviceStrip(plan, r, 5)
        s.dev.set_params(params(net))
        s.dev.set_slots(np.ones(5, np.int8))
        r0, h = plan.rows(r)
        s.dev.upload_arrays(p.E[r0:r0 + h], p.I[r0:r0 + h], p.C[:, r0:r0 + h], p.gi[r0:r0 + h], p.rot[r0:r0 + h])
        strips.append(s)
    for t in range(2):
        step_local(strips, physics.step_scalars(t, physics.PhysicsParams()), t)
    # strips on the gather path: fused / lazy steps, record and texture rows through the halo calls
    p = orc.synth_planes(64, 48, 300, seed=4)
    net = orc.synth_net(300, 0, seed=4)
    big = []
    for r in range(2):
        s = DeviceStrip(plan, r, 300)
        s.dev.set_params(params(net))
        s.dev.set_slots(np.ones(300, np.int8))
        r0, h = plan.rows(r)
        s.dev.upload_arrays(p.E[r0:r0 + h], p.I[r0:r0 + h], p.C[:, r0:r0 + h], p.gi[r0:r0 + h], p.rot[r0:r0 + h])
        big.append(s)
    for t in range(4):
        step_local(big, physics.step_scalars(t, physics.PhysicsParams()), t)
    for s in big:
        s.dev.render_rgb()
    # engine with adoption radiation (device CPPN expression, host NEAT, patches),
    # field radiation (selection / remap), observables
    cfg = engine.ExperimentConfig(grid=engine.GridConfig(64, 64), seed=2, initial_population=30)
    st = engine.new_state(cfg)
    engine.run(st, 3)
    engine.step(st)
    radiation.field_radiation(st, st.t, 0.05)
    engine.run(st, 2)
    from paper_2406_09654_b200 import metrics

    metrics.msc_device(engine.device_of(st))
    metrics.census(st)
    neat.compile_programs([st.pool.genome(int(s)) for s in st.pool.live_slots()[:4]])
    print("sanitize workload done")


if __name__ == "__main__":
    main()
