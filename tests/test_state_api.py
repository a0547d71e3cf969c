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


def _rgb_substrate():
    sub = create_substrate(9, 7)
    sub.front.channels["energy"][0] = GOLD["rgb_E"]
    sub.front.channels["infrastructure"][0] = GOLD["rgb_I"]
    sub.front.genome_index[:] = GOLD["rgb_gi"]
    return sub


def test_render_rgb_host_matches_reference():
    from paper_2406_09654_b200.substrate import render_rgb

    sub = _rgb_substrate()
    for (ne, ni), want in zip(GOLD["rgb_norms"], GOLD["rgb_px"]):
        assert np.array_equal(render_rgb(sub, ne, ni).pixels, want)


@pytest.mark.gpu
def test_render_rgb_device_matches_reference():
    from oracle import oracle as orc
    from paper_2406_09654_b200.device import DeviceSubstrate
    from paper_2406_09654_b200.substrate import render_rgb

    sub = _rgb_substrate()
    dev = DeviceSubstrate(9, 7, 4096)
    dev.upload(sub.front)
    for (ne, ni), want in zip(GOLD["rgb_norms"], GOLD["rgb_px"]):
        assert np.array_equal(dev.render_rgb(ne, ni), want)
    dev.close()
    # a larger random state (rounding ties, empty cells, big slots), device vs host
    H, W = 300, 257
    p = orc.synth_planes(H, W, 500, seed=3)
    p.E[:] = (np.random.default_rng(1).standard_normal((H, W)) * 1.5).astype(np.float32)
    p.E[0, :256] = (np.arange(256, dtype=np.float32) + np.float32(0.5)) / np.float32(255)
    p.gi[np.random.default_rng(2).random((H, W)) < 0.2] = -1
    big = create_substrate(W, H)
    big.front.channels["energy"][0], big.front.channels["infrastructure"][0] = p.E, p.I
    big.front.genome_index[:] = p.gi
    dev = DeviceSubstrate(W, H, 500)
    dev.upload(p)
    for ne, ni in ((1.0, 1.0), (0.37, 5.0)):
        assert np.array_equal(dev.render_rgb(ne, ni), render_rgb(big, ne, ni).pixels)
    dev.close()


@pytest.mark.gpu
def test_device_hook_renders_without_download():
    cfg = engine.ExperimentConfig(grid=engine.GridConfig(64, 48), initial_population=40, seed=4)
    st = engine.new_state(cfg)
    frames = []

    def grab(s):
        assert engine._binding(s).device_ahead  # no download happened for this hook
        frames.append((s.t, engine.render_rgb(s).pixels.copy()))

    engine.run(st, 6, hooks=[engine.Hook(3, grab, device=True)])
    assert [t for t, _ in frames] == [3, 6]
    # the last frame equals the host render of the final (downloaded) state
    from paper_2406_09654_b200.substrate import render_rgb

    assert np.array_equal(frames[-1][1], render_rgb(st.substrate).pixels)


def test_slot_pool_admit_batch_equals_sequential_admit():
    from paper_2406_09654_b200.pool import SlotPool

    def fresh():
        p = SlotPool(12)
        for i in range(12):
            p.install(i, None, birth_step=0)
        p._state[[1, 4, 5, 9]] = 2
        p._death[[1, 4, 5, 9]] = [7, 3, 7, 1]
        p._state[[2, 10]] = 0
        return p

    a, b = fresh(), fresh()
    genomes = [object() for _ in range(8)]
    got = a.admit_batch(genomes, [(i,) for i in range(8)], birth_step=5)
    want = []
    for i, gnm in enumerate(genomes):
        s = b.admit(gnm, parents=(i,), birth_step=5)
        if s is None:
            break
        want.append(s)
    assert got == want == [2, 10, 9, 4, 1, 5]
    assert np.array_equal(a.slot_states(), b.slot_states()) and np.array_equal(a._death, b._death)
    assert [(r.slot, r.parents, r.birth_step) for r in a.records.values()] == \
        [(r.slot, r.parents, r.birth_step) for r in b.records.values()]
