"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container only (it imports the read-only reference from
/root/reference/pkg/src, which does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_ref \
        python tests/golden/make_golden.py

Outputs (committed, small, npz-compressed) are consumed by
tests/test_oracle_golden.py (pins the oracle to the reference) and by the
GPU parity tests (tests/test_gpu_parity.py).  Nothing here is a copy of a
reference test: the reference is only *called* to produce outputs.

Files:
  physics_cases.npz  random 16x16/13x11 pre-states + full 13-wide action
                     blocks + physics params + t -> reference post-state,
                     events, census counts (phases energy_cycle ->
                     apply_invest_liquidate -> write_communication ->
                     resolve_exploration -> census bincount).
  explore_cases.npz  the reference's own randomized exploration case
                     generator (test_physics.py:311-331) -> reference
                     resolve_exploration output.
  forward_cases.npz  reference forward_batched (hidden 16) outputs.
  step_hidden.npz    64x64, 8 genomes, hidden 16: reference engine.step for
                     6 consecutive steps (pre, actions, post, events).
  step_direct.npz    BASELINE config 1 (64x64, 8 genomes, 45->13 direct,
                     period 20, seed 0) run 100 steps through reference
                     engine.step with forward_batched replaced by the
                     direct restatement (sgemm -> +b -> same sigmoid/clip,
                     SURVEY.md §8d): per-step digests + actions/states at
                     a few steps.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import evoca  # noqa: E402
from evoca import engine, physics, hypernet  # noqa: E402
from evoca.config import ExperimentConfig, GridConfig, HypernetConfig  # noqa: E402
from evoca.neuroevo import EvolutionRates, GenomePool, InnovationCounter, init_genome  # noqa: E402
from evoca.physics import ActionField, PhysicsParams  # noqa: E402
from evoca.rng import stream  # noqa: E402
from evoca.substrate import create_substrate  # noqa: E402

from oracle import oracle as orc  # noqa: E402


def _planes_to_arrays(p):
    return (
        p.plane("energy").copy(),
        p.plane("infrastructure").copy(),
        p.channels["communication"].copy(),
        p.genome_index.copy(),
        p.rotation.copy(),
    )


def _load(p, E, I, C, gi, rot):
    p.plane("energy")[:] = E
    p.plane("infrastructure")[:] = I
    p.channels["communication"][:] = C
    p.genome_index[:] = gi
    p.rotation[:] = rot


def _events_arr(ev):
    return np.stack(
        [
            ev.target.astype(np.float64),
            ev.source.astype(np.float64),
            ev.winner_slot.astype(np.float64),
            ev.defender_slot.astype(np.float64),
            ev.direction.astype(np.float64),
            ev.quantity.astype(np.float64),
        ],
        axis=1,
    ) if len(ev) else np.zeros((0, 6))


PHYS_FIELDS = (
    "cycle_amplitude", "cycle_period", "drain_fraction", "invest_rate", "liquidate_rate",
    "invest_efficiency", "liquidate_efficiency", "explore_fraction", "upkeep",
    "decay_on_starvation", "death_threshold",
)


def physics_cases(n_cases=40):
    out = {}
    for c in range(n_cases):
        g = stream(2406, c, "golden_physics")
        h, w = (16, 16) if c % 3 else (11, 13)
        sub = create_substrate(w, h)
        p = sub.front
        occ = g.random((h, w)) < (0.3 + 0.6 * g.random())
        gi = np.where(occ, g.integers(0, 12, (h, w)), -1).astype(np.int32)
        E = g.uniform(0, 2, (h, w)).astype(np.float32)
        I = g.uniform(0, 2, (h, w)).astype(np.float32)
        # sprinkle exact zeros / tiny stocks to exercise starvation and death
        I[g.random((h, w)) < 0.1] = 0
        I[g.random((h, w)) < 0.05] = np.float32(5e-4)
        C = g.uniform(0, 1, (3, h, w)).astype(np.float32)
        rot = g.integers(0, 8, (h, w)).astype(np.uint8)
        _load(p, E, I, C, gi, rot)
        cells = np.flatnonzero(gi.ravel() >= 0).astype(np.int64)
        # a few listed cells vacate before the phases (like a mid-step death)
        if len(cells) > 4:
            vic = cells[g.random(len(cells)) < 0.05]
            p.genome_index.ravel()[vic] = -1
        n = len(cells)
        acts = g.uniform(0, 1, (n, 13)).astype(np.float32)
        # exact actuator ties and saturation values
        tie = g.random(n) < 0.25
        acts[tie, 5 + 3] = acts[tie, 5 + 6]
        sat = g.random(n) < 0.05
        acts[sat, 5:] = np.nextafter(np.float32(1.0), np.float32(0.0))
        params = PhysicsParams(
            cycle_amplitude=float(g.choice([0.0, 0.1, 0.4, 1.0])),
            cycle_period=int(g.choice([2, 4, 20, 100])),
            drain_fraction=float(g.uniform(0, 1)),
            invest_rate=float(g.uniform(0.2, 2)),
            liquidate_rate=float(g.uniform(0.2, 2)),
            invest_efficiency=float(g.uniform(0.5, 1)),
            liquidate_efficiency=float(g.uniform(0.5, 1)),
            explore_fraction=float(g.uniform(0.1, 0.9)),
            upkeep=float(g.uniform(0, 0.2)),
            decay_on_starvation=float(g.uniform(0, 0.5)),
            death_threshold=float(g.choice([1e-3, 0.05])),
        )
        t = int(g.choice([0, 1, 5, 20, 25, 40, 75, 99, 100]))
        pre = _planes_to_arrays(p)
        af = ActionField(
            cells=cells, invest=acts[:, 0], liquidate=acts[:, 1],
            comm=acts[:, 2:5], explore=acts[:, 5:13],
        )
        physics.energy_cycle(p, t, params)
        physics.apply_invest_liquidate(p, af, params)
        physics.write_communication(p, af)
        ev = physics.resolve_exploration(p, af, params)
        gi_post = p.genome_index
        counts = np.bincount(gi_post[gi_post >= 0], minlength=12)
        post = _planes_to_arrays(p)
        key = f"c{c:02d}_"
        for name, arr in zip(("E", "I", "C", "gi", "rot"), pre):
            out[key + "pre_" + name] = arr
        for name, arr in zip(("E", "I", "C", "gi", "rot"), post):
            out[key + "post_" + name] = arr
        out[key + "cells"] = cells
        out[key + "acts"] = acts
        out[key + "t"] = np.int64(t)
        out[key + "phys"] = np.array([getattr(params, f) for f in PHYS_FIELDS], np.float64)
        out[key + "events"] = _events_arr(ev)
        out[key + "counts"] = counts
    out["n_cases"] = np.int64(n_cases)
    out["phys_fields"] = np.array(PHYS_FIELDS)
    return out


def explore_cases(n_cases=50):
    from test_physics import _random_exploration_case

    out = {}
    for c in range(n_cases):
        g = stream(1234, c, "exploration_case")
        planes, actions, alpha = _random_exploration_case(g)
        pre = _planes_to_arrays(planes)
        ev = physics.resolve_exploration(planes, actions, PhysicsParams(explore_fraction=alpha))
        post = _planes_to_arrays(planes)
        key = f"c{c:02d}_"
        for name, arr in zip(("E", "I", "C", "gi", "rot"), pre):
            out[key + "pre_" + name] = arr
        for name, arr in zip(("I", "gi", "rot"), (post[1], post[3], post[4])):
            out[key + "post_" + name] = arr
        out[key + "cells"] = actions.cells
        out[key + "explore"] = actions.explore
        out[key + "alpha"] = np.float64(alpha)
        out[key + "events"] = _events_arr(ev)
    out["n_cases"] = np.int64(n_cases)
    return out


def forward_cases():
    out = {}
    g = np.random.default_rng(77)
    for c, hidden in enumerate((16, 16, 4, 32)):
        w1 = (g.standard_normal((hidden, 45)) * 0.5).astype(np.float32)
        b1 = (g.standard_normal(hidden) * 0.1).astype(np.float32)
        w2 = (g.standard_normal((13, hidden)) * 0.5).astype(np.float32)
        b2 = (g.standard_normal(13) * 0.1).astype(np.float32)
        s = g.uniform(-1, 2, (257, 45)).astype(np.float32)
        if c == 1:
            s[:8] *= np.float32(1e4)  # saturation rows
        y = hypernet.forward_batched(hypernet.DenseParams(w1, b1, w2, b2), s)
        key = f"c{c}_"
        out.update({key + "w1": w1, key + "b1": b1, key + "w2": w2, key + "b2": b2, key + "s": s, key + "y": y})
    out["n_cases"] = np.int64(4)
    return out


class _Direct:
    """Direct 45->13 params for the BASELINE extension."""

    def __init__(self, w, b):
        self.w = w
        self.b = b


def _direct_forward(params, sensors):
    # sgemm, + bias, then the reference sigmoid sequence and clip
    # (hypernet.py:245-251 with the hidden layer removed).
    z = np.asarray(sensors, np.float32) @ params.w.T
    z += params.b
    np.negative(z, out=z)
    np.exp(z, out=z)
    z += np.float32(1.0)
    np.reciprocal(z, out=z)
    np.clip(z, hypernet._SIG_LO, hypernet._SIG_HI, out=z)
    return z


def _make_state(p0: orc.Planes, params_list, period, seed=0):
    h, w = p0.shape
    cfg = ExperimentConfig(grid=GridConfig(w, h), seed=seed, initial_population=0)
    cfg.physics.cycle_period = period
    cfg.evolution = EvolutionRates(p_radiation=0.0, p_merge=0.0)
    cfg.hypernet = HypernetConfig(hidden_size=16)
    sub = create_substrate(w, h)
    pool = GenomePool(capacity=len(params_list))
    for i, prm in enumerate(params_list):
        slot = pool.admit(init_genome(stream(seed, 0, "golden_genome", i), pool.innovations), (), 0)
        pool.slots[slot].params = prm
    _load(sub.front, p0.E, p0.I, p0.C, p0.gi, p0.rot)
    return engine.SimState(substrate=sub, pool=pool, config=cfg, master_seed=seed)


def _run_recording(state, steps, keep):
    out = {"digest": []}
    t_keep = set(keep)
    captured = {}
    orig = engine.build_action_field

    def spy(st):
        af = orig(st)
        captured["af"] = af
        return af

    engine.build_action_field = spy
    try:
        for k in range(steps):
            pre = _planes_to_arrays(state.substrate.front)
            engine.step(state)
            if k in t_keep:
                af = captured["af"]
                acts = np.concatenate(
                    [af.invest[:, None], af.liquidate[:, None], af.comm, af.explore], axis=1
                )
                key = f"s{k:03d}_"
                for name, arr in zip(("E", "I", "C", "gi", "rot"), pre):
                    out[key + "pre_" + name] = arr
                for name, arr in zip(("E", "I", "C", "gi", "rot"), _planes_to_arrays(state.substrate.front)):
                    out[key + "post_" + name] = arr
                out[key + "cells"] = af.cells
                out[key + "acts"] = acts
                out[key + "adoptions"] = np.int64(state.last_adoptions)
                counts = np.bincount(state.substrate.front.genome_index[state.substrate.front.genome_index >= 0],
                                     minlength=state.pool.capacity)
                out[key + "counts"] = counts
            out["digest"].append(engine.digest(state))
    finally:
        engine.build_action_field = orig
    out["digest"] = np.array(out["digest"], dtype=np.uint64)
    out["keep"] = np.array(sorted(t_keep), np.int64)
    return out


def step_hidden():
    p0 = orc.synth_planes(64, 64, 8, seed=5)
    g = np.random.default_rng(6)
    params = []
    for _ in range(8):
        params.append(hypernet.DenseParams(
            (g.standard_normal((16, 45)) * 0.5).astype(np.float32),
            (g.standard_normal(16) * 0.1).astype(np.float32),
            (g.standard_normal((13, 16)) * 0.5).astype(np.float32),
            (g.standard_normal(13) * 0.1).astype(np.float32),
        ))
    state = _make_state(p0, params, period=20, seed=5)
    out = _run_recording(state, 6, keep=range(6))
    for i, prm in enumerate(params):
        out[f"w1_{i}"], out[f"b1_{i}"], out[f"w2_{i}"], out[f"b2_{i}"] = prm.w1, prm.b1, prm.w2, prm.b2
    return out


def step_direct():
    p0 = orc.synth_planes(64, 64, 8, seed=0)
    net = orc.synth_net(8, hidden=0, seed=0)
    params = [_Direct(net.w2[i], net.b2[i]) for i in range(8)]
    state = _make_state(p0, params, period=20, seed=0)
    orig = engine.forward_batched
    engine.forward_batched = _direct_forward
    try:
        out = _run_recording(state, 100, keep=(0, 1, 2, 19, 20, 21, 99))
    finally:
        engine.forward_batched = orig
    return out


def main():
    np.savez_compressed(os.path.join(HERE, "physics_cases.npz"), **physics_cases())
    np.savez_compressed(os.path.join(HERE, "explore_cases.npz"), **explore_cases())
    np.savez_compressed(os.path.join(HERE, "forward_cases.npz"), **forward_cases())
    np.savez_compressed(os.path.join(HERE, "step_hidden.npz"), **step_hidden())
    np.savez_compressed(os.path.join(HERE, "step_direct.npz"), **step_direct())
    with open(os.path.join(HERE, "PROVENANCE.txt"), "w") as f:
        import numba

        f.write(
            "generated by tests/golden/make_golden.py from /root/reference/pkg/src (evoca "
            f"{evoca.__version__}); numpy {np.__version__}, numba {numba.__version__}\n"
        )
    print("ok")


if __name__ == "__main__":
    main()
