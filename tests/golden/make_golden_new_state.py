"""Golden vectors for state construction, produced by the REFERENCE.

Run in the build container only (imports /root/reference/pkg/src):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden_new_state.py

Writes new_state_cases.npz: for a few configs, the reference new_state()
front planes (seed_initial_population placement, headings, stocks), the
innovation counter after seeding, and every seeded slot's expressed
DenseParams (reference generate_network via the pool's net factory); plus
reference gather_sensors vectors for a few cells of a random state; reference
render_rgb frames (substrate.py:147-165) of a random state at three norms.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from evoca import config as rcfg  # noqa: E402
from evoca import engine as reng  # noqa: E402

CASES = [  # (width, height, seed, initial_population, hidden)
    (24, 20, 3, 10, 16),
    (16, 16, 0, 64, 16),
    (40, 8, 11, 5, 32),
]


def main():
    out = {}
    for k, (w, h, seed, pop, hidden) in enumerate(CASES):
        cfg = rcfg.ExperimentConfig(grid=rcfg.GridConfig(w, h), seed=seed, initial_population=pop,
                                    hypernet=rcfg.HypernetConfig(hidden_size=hidden))
        cfg.validate()
        st = reng.new_state(cfg)
        f = st.substrate.front
        out[f"c{k}_meta"] = np.array([w, h, seed, pop, hidden], np.int64)
        out[f"c{k}_E"] = f.plane("energy").copy()
        out[f"c{k}_I"] = f.plane("infrastructure").copy()
        out[f"c{k}_C"] = f.channels["communication"].copy()
        out[f"c{k}_gi"] = f.genome_index.copy()
        out[f"c{k}_rot"] = f.rotation.copy()
        inn = st.pool.innovations
        out[f"c{k}_counter"] = np.array([inn.next_innovation, inn.next_node_id], np.int64)
        for s in range(pop):
            p = st.pool.params(s)
            out[f"c{k}_s{s}_w1"], out[f"c{k}_s{s}_b1"] = p.w1, p.b1
            out[f"c{k}_s{s}_w2"], out[f"c{k}_s{s}_b2"] = p.w2, p.b2
    # gather_sensors on a random state
    g = np.random.default_rng(5)
    cfg = rcfg.ExperimentConfig(grid=rcfg.GridConfig(9, 7), seed=1, initial_population=0)
    st = reng.new_state(cfg)
    f = st.substrate.front
    f.channels["energy"][0] = g.random((7, 9), dtype=np.float32)
    f.channels["infrastructure"][0] = g.random((7, 9), dtype=np.float32)
    f.channels["communication"][:] = g.standard_normal((3, 7, 9)).astype(np.float32)
    f.rotation[:] = g.integers(0, 8, (7, 9)).astype(np.uint8)
    out["gs_E"], out["gs_I"] = f.plane("energy").copy(), f.plane("infrastructure").copy()
    out["gs_C"], out["gs_rot"] = f.channels["communication"].copy(), f.rotation.copy()
    cells = [(0, 0), (8, 6), (4, 3), (8, 0), (0, 6)]
    out["gs_cells"] = np.array(cells, np.int64)
    out["gs_out"] = np.stack([reng.gather_sensors(st.substrate, x, y) for x, y in cells])
    # render_rgb on a state with out-of-range stocks, empty cells and large slots
    from evoca.substrate import render_rgb

    f.channels["energy"][0] = (g.standard_normal((7, 9)) * 2).astype(np.float32)
    f.channels["energy"][0][0, :3] = [np.float32(0.5 / 255), np.float32(1.5 / 255), np.float32(2.5 / 255)]
    f.channels["infrastructure"][0] = g.random((7, 9), dtype=np.float32) * 3
    f.genome_index[:] = g.integers(-1, 4096, (7, 9)).astype(np.int32)
    out["rgb_E"], out["rgb_I"], out["rgb_gi"] = f.plane("energy").copy(), f.plane("infrastructure").copy(), f.genome_index.copy()
    out["rgb_norms"] = np.array([[1.0, 1.0], [2.5, 0.7], [0.3, 3.0]])
    out["rgb_px"] = np.stack([render_rgb(st.substrate, a, b).pixels for a, b in out["rgb_norms"]])
    # multi-scale complexity (metrics.py:57-103) and census plane totals
    from evoca import metrics as rmet
    from evoca.substrate import create_substrate

    for k, (w, h) in enumerate([(37, 50), (64, 64), (130, 70)]):
        sub = create_substrate(w, h)
        f = sub.front
        f.channels["energy"][0] = np.exp(g.standard_normal((h, w)) * 2).astype(np.float32)
        inf = g.random((h, w), dtype=np.float32)
        inf[g.random((h, w)) < 0.9] = 0
        f.channels["infrastructure"][0] = inf
        f.channels["communication"][:] = g.standard_normal((3, h, w)).astype(np.float32)
        out[f"msc{k}_E"], out[f"msc{k}_I"] = f.plane("energy").copy(), f.plane("infrastructure").copy()
        out[f"msc{k}_C"] = f.channels["communication"].copy()
        for name, sb in (("energy", 0), ("infrastructure", 0), ("communication", 1)):
            rep = rmet.msc_of_substrate(sub, name, sb)
            out[f"msc{k}_{name}{sb}"] = np.array(list(rep.contributions) + [rep.total, rep.side])
        out[f"msc{k}_sums"] = np.array([float(f.plane("energy").sum(dtype=np.float64)),
                                        float(f.plane("infrastructure").sum(dtype=np.float64))])
        side = 1 << min(h.bit_length() - 1, w.bit_length() - 1)
        rep = rmet.msc(f.plane("energy")[:side, :side], n_scales=2)
        out[f"msc{k}_E_n2"] = np.array(list(rep.contributions) + [rep.total, rep.side])
    np.savez_compressed(os.path.join(HERE, "new_state_cases.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
