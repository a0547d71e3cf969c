"""State construction and the steering API of the engine mirror against the
reference's own outputs (tests/golden/new_state_cases.npz, produced by
tests/golden/make_golden_new_state.py from the reference new_state /
gather_sensors): placement, headings, stocks and innovation counter on the
CPU; the device-expressed seed networks on the GPU (bit-exact with the
reference generate_network)."""

import os

import numpy as np
import pytest

from paper_2406_09654_b200 import engine
from paper_2406_09654_b200.radiation import DeviceExpressed
from paper_2406_09654_b200.substrate import create_substrate

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "new_state_cases.npz"))
CASES = sorted({k.split("_")[0] for k in GOLD.files if k.startswith("c") and k.endswith("_meta")})


def _config(k):
    w, h, seed, pop, hidden = (int(v) for v in GOLD[f"{k}_meta"])
    cfg = engine.ExperimentConfig(grid=engine.GridConfig(w, h), seed=seed, initial_population=pop,
                                  hypernet=engine.HypernetConfig(hidden_size=hidden))
    cfg.validate()
    return cfg, pop


@pytest.mark.parametrize("k", CASES)
def test_new_state_matches_reference_placement(k):
    cfg, pop = _config(k)
    st = engine.new_state(cfg)
    f = st.substrate.front
    assert np.array_equal(f.channels["energy"][0], GOLD[f"{k}_E"])
    assert np.array_equal(f.channels["infrastructure"][0], GOLD[f"{k}_I"])
    assert np.array_equal(f.channels["communication"], GOLD[f"{k}_C"])
    assert np.array_equal(f.genome_index, GOLD[f"{k}_gi"])
    assert np.array_equal(f.rotation, GOLD[f"{k}_rot"])
    inn = st.pool.innovations
    assert [inn.next_innovation, inn.next_node_id] == list(GOLD[f"{k}_counter"])
    assert st.pool.live_count() == pop
    for s in range(pop):
        assert isinstance(st.pool.params(s), DeviceExpressed)
    assert st.master_seed == cfg.seed and st.t == 0


def test_new_state_without_population():
    cfg = engine.ExperimentConfig(grid=engine.GridConfig(8, 8), initial_population=5)
    st = engine.new_state(cfg, seed_population=False)
    assert (st.substrate.front.genome_index == -1).all() and st.pool.live_count() == 0


def test_seed_population_limits():
    cfg = engine.ExperimentConfig(grid=engine.GridConfig(4, 4), initial_population=0)
    st = engine.new_state(cfg)
    with pytest.raises(ValueError, match="cell count"):
        engine.seed_initial_population(st, 17)
    with pytest.raises(ValueError, match="capacity"):
        engine.seed_initial_population(st, engine.DEFAULT_POOL_CAPACITY + 1)


def test_config_validation_errors():
    bad = [
        (lambda c: setattr(c.grid, "width", 3), "grid.width"),
        (lambda c: setattr(c, "seed", -1), "seed"),
        (lambda c: setattr(c, "initial_population", 513), "initial_population"),
        (lambda c: setattr(c, "initial_population", 17), "fit on the grid"),
        (lambda c: setattr(c.hypernet, "tau", 1.0), "tau"),
        (lambda c: setattr(c.evolution, "p_merge", 1.5), "p_merge"),
        (lambda c: setattr(c.physics, "cycle_period", 1), "cycle_period"),
    ]
    for mutate, msg in bad:
        cfg = engine.ExperimentConfig(grid=engine.GridConfig(4, 4), initial_population=0)
        mutate(cfg)
        with pytest.raises(ValueError, match=msg):
            cfg.validate()


def test_gather_sensors_matches_reference():
    sub = create_substrate(9, 7)
    f = sub.front
    f.channels["energy"][0] = GOLD["gs_E"]
    f.channels["infrastructure"][0] = GOLD["gs_I"]
    f.channels["communication"][:] = GOLD["gs_C"]
    f.rotation[:] = GOLD["gs_rot"]
    for (x, y), want in zip(GOLD["gs_cells"], GOLD["gs_out"]):
        got = engine.gather_sensors(sub, int(x), int(y))
        assert got.dtype == np.float32 and np.array_equal(got, want)


def test_steering_api():
    cfg = engine.ExperimentConfig(grid=engine.GridConfig(8, 8), initial_population=2)
    st = engine.new_state(cfg)
    items = {d["path"]: d for d in engine.describe_params(st)}
    assert len(items) == 24
    assert items["physics.explore_fraction"]["value"] == st.config.physics.explore_fraction
    engine.apply_param(st, "physics.explore_fraction", 0.25)
    assert st.config.physics.explore_fraction == 0.25
    engine.apply_param(st, "physics.cycle_period", 40.0)
    assert st.config.physics.cycle_period == 40 and isinstance(st.config.physics.cycle_period, int)
    for path, value, msg in [("physics.nope", 1.0, "unknown"), ("physics.upkeep", True, "number"),
                             ("physics.cycle_period", 2.5, "integer"), ("physics.upkeep", 2.0, r"\[0.0, 1.0\]"),
                             ("hypernet.w_max", 0.0, "w_max")]:
        with pytest.raises(ValueError, match=msg):
            engine.apply_param(st, path, value)
    assert st.config.physics.upkeep == engine.PhysicsParams().upkeep
    engine.apply_param(st, "hypernet.tau", 0.3)
    child = st.pool.net_factory(st.pool.genome(0))
    assert isinstance(child, DeviceExpressed) and child.tau == 0.3


@pytest.mark.gpu
@pytest.mark.parametrize("k", CASES)
def test_new_state_device_expression_matches_reference(k):
    """The seed networks, expressed on the device in one batched launch at the
    first step, equal the reference generate_network bit for bit; the state
    then steps."""
    cfg, pop = _config(k)
    st = engine.new_state(cfg)
    engine.device_of(st)
    engine._binding(st).sync_params(st.pool)
    for s in range(pop):
        p = st.pool.params(s)
        for name in ("w1", "b1", "w2", "b2"):
            assert np.array_equal(getattr(p, name), GOLD[f"{k}_s{s}_{name}"]), (s, name)
    engine.step(st)
    engine.run(st, 3)
    assert st.t == 4
