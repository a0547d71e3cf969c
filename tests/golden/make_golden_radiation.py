"""Golden steps of the reference with adoption-driven radiation ON.

Runs the REFERENCE ``evoca.engine.step`` (/root/reference/pkg/src, read-only)
with its default evolution rates (p_radiation 0.02, p_merge 0.2,
neuroevo.py:170-185) on 64x64 worlds with the default 45->16->13 net, and
records per step what is needed to replay the step on the device with the
reference's actions injected and this package's host radiation
(paper_2406_09654_b200.radiation.apply_radiation):

  * the front planes before step 0 and after every step;
  * the reference's ActionField of every step (cells + 13 columns);
  * the genome plane right before apply_radiation (after exploration) and the
    adoption events handed to it;
  * the pool after every step: slot state / lineage / death step, phylogeny
    records, the innovation counter, and every genome admitted that step.

Two cases: "sparse" is the reference's own seeding (new_state: 64 organisms
on an empty world, so adoptions land on empty cells and only mutations
fire); "dense" overwrites the seeded world with every cell occupied by one of
the 64 seed genomes, in a GenomePool of capacity 160 (live defenders:
merges; the pool fills in the first step, later admissions evict dead slots).

Build container only (imports the reference):
    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_ref \\
        python tests/golden/make_golden_radiation.py
-> tests/golden/radiation_steps.npz + radiation_genomes.json
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from evoca import engine, physics  # noqa: E402
from evoca.config import ExperimentConfig, GridConfig  # noqa: E402

STEPS = {"sparse": 14, "dense": 12}
DENSE_CAPACITY = 160


def _genome_json(g):
    return {"nodes": [[n.id, n.role, n.activation] for n in g.nodes],
            "connections": [[c.innovation, c.src, c.dst, c.weight, bool(c.enabled)] for c in g.connections]}


def _planes(p):
    return (p.plane("energy").copy(), p.plane("infrastructure").copy(), p.channels["communication"].copy(),
            p.genome_index.copy(), p.rotation.copy())


def _pool_arrays(pool):
    code = {"free": 0, "live": 1, "dead": 2}
    st = np.array([code[s.state] for s in pool.slots], np.int8)
    lin = np.array([s.lineage_id for s in pool.slots], np.int64)
    death = np.array([s.death_step for s in pool.slots], np.int64)
    recs = sorted(pool.records.values(), key=lambda r: r.lineage_id)
    rec = np.array([[r.lineage_id, r.slot, r.birth_step, -1 if r.death_step is None else r.death_step,
                     r.peak_population, r.parents[0] if len(r.parents) > 0 else -1,
                     r.parents[1] if len(r.parents) > 1 else -1, len(r.parents)] for r in recs], np.int64)
    return st, lin, death, rec


def run_case(name: str, steps: int, out: dict, genomes: dict) -> None:
    cfg = ExperimentConfig(grid=GridConfig(64, 64), seed=11)
    cfg.validate()
    if name == "dense":
        from evoca.neuroevo import GenomePool

        st = engine.new_state(cfg, seed_population=False)
        st.pool = GenomePool(capacity=DENSE_CAPACITY, net_factory=st.pool.net_factory)
        engine.seed_initial_population(st, cfg.initial_population)
    else:
        st = engine.new_state(cfg)
    sub = st.substrate
    key = name + "_"
    out[key + "capacity"] = np.int64(st.pool.capacity)
    if name == "dense":
        g = np.random.default_rng(5)
        f = sub.front
        f.plane("energy")[:] = g.random((64, 64), dtype=np.float32)
        f.plane("infrastructure")[:] = g.random((64, 64), dtype=np.float32)
        f.channels["communication"][:] = g.standard_normal((3, 64, 64)).astype(np.float32)
        f.rotation[:] = g.integers(0, 8, (64, 64)).astype(np.uint8)
        f.genome_index[:] = g.integers(0, 64, (64, 64)).astype(np.int32)
    E, I, C, gi, rot = _planes(sub.front)
    out[key + "pre_E"], out[key + "pre_I"], out[key + "pre_C"] = E, I, C
    out[key + "pre_gi"], out[key + "pre_rot"] = gi, rot
    genomes[name] = {"initial": [_genome_json(st.pool.genome(s)) for s in range(64)],
                     "innovation": [st.pool.innovations.next_innovation, st.pool.innovations.next_node_id],
                     "admitted": []}
    out[key + "steps"] = np.int64(steps)
    captured = {}
    orig_baf = engine.build_action_field
    orig_rad = engine.apply_radiation

    def baf(state):
        a = orig_baf(state)
        captured["actions"] = a
        return a

    def rad(events, pool, rates, planes, seed, t):
        captured["gi_pre_rad"] = planes.genome_index.copy()
        captured["events"] = events
        captured["lineage_before"] = pool.next_lineage_id
        return orig_rad(events, pool, rates, planes, seed, t)

    engine.build_action_field = baf
    engine.apply_radiation = rad
    try:
        for k in range(steps):
            engine.step(st)
            a = captured["actions"]
            sk = f"{key}s{k:02d}_"
            out[sk + "cells"] = a.cells.astype(np.int64)
            out[sk + "acts"] = np.concatenate([a.invest[:, None], a.liquidate[:, None], a.comm, a.explore],
                                              axis=1).astype(np.float32)
            ev = captured["events"]
            out[sk + "events"] = np.stack([ev.target.astype(np.float64), ev.source.astype(np.float64),
                                           ev.winner_slot.astype(np.float64), ev.defender_slot.astype(np.float64),
                                           ev.direction.astype(np.float64), ev.quantity.astype(np.float64)],
                                          axis=1) if len(ev) else np.zeros((0, 6))
            out[sk + "gi_pre_rad"] = captured["gi_pre_rad"]
            E, I, C, gi, rot = _planes(sub.front)
            out[sk + "post_E"], out[sk + "post_I"], out[sk + "post_C"] = E, I, C
            out[sk + "post_gi"], out[sk + "post_rot"] = gi, rot
            pst, lin, death, rec = _pool_arrays(st.pool)
            out[sk + "pool_state"], out[sk + "pool_lineage"], out[sk + "pool_death"] = pst, lin, death
            out[sk + "records"] = rec
            out[sk + "innovation"] = np.array([st.pool.innovations.next_innovation,
                                               st.pool.innovations.next_node_id], np.int64)
            new = [r for r in st.pool.records.values() if r.lineage_id >= captured["lineage_before"]]
            genomes[name]["admitted"].append([[r.lineage_id, r.slot, _genome_json(st.pool.genome(r.slot))]
                                              for r in sorted(new, key=lambda r: r.lineage_id)])
            out[sk + "stats"] = np.array([st.last_adoptions, st.last_extinctions], np.int64)
            print(f"{name} step {k}: events {len(ev)}, admitted {len(new)}, live {st.pool.live_count()}, "
                  f"extinct {st.last_extinctions}")
    finally:
        engine.build_action_field = orig_baf
        engine.apply_radiation = orig_rad
    out[key + "rates"] = np.array([cfg.evolution.p_radiation, cfg.evolution.p_merge], np.float64)
    out[key + "seed"] = np.int64(cfg.seed)


def main():
    out, genomes = {}, {}
    for name, steps in STEPS.items():
        run_case(name, steps, out, genomes)
    np.savez_compressed(os.path.join(HERE, "radiation_steps.npz"), **out)
    with open(os.path.join(HERE, "radiation_genomes.json"), "w") as f:
        json.dump(genomes, f)
    prov = os.path.join(HERE, "PROVENANCE.txt")
    if "make_golden_radiation" not in open(prov).read():
        with open(prov, "a") as f:
            f.write("radiation_steps.npz, radiation_genomes.json: tests/golden/make_golden_radiation.py "
                    "(reference engine.step with p_radiation 0.02, p_merge 0.2)\n")


if __name__ == "__main__":
    main()
