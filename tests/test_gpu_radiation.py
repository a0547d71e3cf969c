"""Device field radiation (BASELINE config 3 extension) and the device
expression of admitted children, against host restatements:
  * evo_select_cells == occupied[Generator(Philox(key)).random(n_occ) < p]
    (the host stream rng.stream(seed, t, "field_radiation"), bit-exact);
  * evo_remap_selected moves exactly the selected cells;
  * radiation.field_radiation == host NEAT on a pool copy (same streams) +
    oracle generate_direct for the children's weights;
  * engine.run (device-resident) == engine.step loop with radiation due."""

import copy

import numpy as np
import pytest

from oracle import cppn as ocppn
from paper_2406_09654_b200 import engine, neat, radiation
from paper_2406_09654_b200.device import DeviceSubstrate
from tests.test_gpu_cppn import assert_tables_equal

pytestmark = pytest.mark.gpu


def _planes(h, w, cap, seed, empty=0.3):
    g = np.random.default_rng(seed)
    E = g.random((h, w), dtype=np.float32)
    I = g.random((h, w), dtype=np.float32)
    C = g.standard_normal((3, h, w)).astype(np.float32)
    gi = g.integers(0, cap, (h, w), dtype=np.int32)
    gi[g.random((h, w)) < empty] = -1
    rot = g.integers(0, 8, (h, w), dtype=np.uint8)
    return E, I, C, gi, rot


@pytest.mark.parametrize("p", [0.0, 0.01, 0.3, 1.0])
@pytest.mark.parametrize("shape", [(100, 77), (64, 64), (3, 5000)])
def test_select_matches_host_stream(p, shape):
    h, w = shape
    cap = 9
    E, I, C, gi, rot = _planes(h, w, cap, seed=h * w)
    dev = DeviceSubstrate(w, h, cap)
    dev.upload_arrays(E, I, C, gi, rot)
    key = neat.stream_key(7, 50, "field_radiation")
    counts, n = dev.select_cells(key, p)
    occ = np.flatnonzero(gi.ravel() >= 0)
    want = occ[np.random.Generator(np.random.Philox(key=key)).random(len(occ)) < p]
    assert n == len(want)
    np.testing.assert_array_equal(dev.read_selected(), want)
    np.testing.assert_array_equal(counts, np.bincount(gi.ravel()[want], minlength=cap))
    # remap parents 0..3 to 5..8, others stay
    smap = np.full(cap, -1, np.int32)
    smap[:4] = np.arange(5, 9)
    dev.remap_selected(smap)
    out = [np.empty_like(a) for a in (E, I, C, gi, rot)]
    dev.download_arrays(*out)
    exp = gi.ravel().copy()
    moved = want[exp[want] < 4]
    exp[moved] = smap[exp[moved]]
    np.testing.assert_array_equal(out[3].ravel(), exp)
    dev.close()


@pytest.mark.parametrize("p", [0.02, 0.002])  # 0.002: some live slots get no child (the plan's subset path)
def test_field_radiation_vs_host_neat(p):
    st = engine.baseline_state("c3", width=96, height=80, genomes=12)
    engine.run(st, 3)
    t = st.substrate.step_counter
    gi0 = st.substrate.front.genome_index.ravel().copy()
    pool_copy = copy.deepcopy(st.pool)
    pool_copy.net_factory = None
    info = radiation.field_radiation(st, t, p)
    # host restatement of the same event
    occ = np.flatnonzero(gi0 >= 0)
    sel = occ[neat.stream(st.master_seed, t, "field_radiation").random(len(occ)) < p]
    parents = np.unique(gi0[sel])
    exp_gi = gi0.copy()
    children = {}
    for par in parents:
        child = neat.mutate(pool_copy.genome(int(par)), neat.EvolutionRates(),
                            neat.stream(st.master_seed, t, "mutate", int(par)), pool_copy.innovations)
        slot = pool_copy.admit(child, parents=(pool_copy.lineage(int(par)),), birth_step=t)
        children[slot] = child
        exp_gi[sel[gi0[sel] == par]] = slot
    assert info["selected"] == len(sel) and info["children"] == len(children) > 0
    engine.sync_to_host(st)
    np.testing.assert_array_equal(st.substrate.front.genome_index.ravel(), exp_gi)
    dev = engine.device_of(st)
    for slot, child in children.items():
        assert st.pool.genome(slot) == child
        w, b = ocppn.generate_direct(child)
        _, _, w2, b2 = dev.get_params_arrays(slot, 1)
        assert_tables_equal(w2[0], w, f"child slot {slot}")
        assert_tables_equal(b2[0], b, f"child slot {slot} bias")
        p = st.pool.params(slot)
        assert isinstance(p, radiation.DeviceExpressed) and np.array_equal(p.w, w2[0])


def test_run_equals_step_loop_with_radiation():
    a = engine.baseline_state("c3", width=64, height=48, genomes=8)
    b = engine.baseline_state("c3", width=64, height=48, genomes=8)
    a.config.field_radiation.every = b.config.field_radiation.every = 4
    a.config.field_radiation.p = b.config.field_radiation.p = 0.05
    engine.run(a, 13)
    for _ in range(13):
        engine.step(b)
    assert engine.digest(a) == engine.digest(b)
    assert a.pool.live_count() == b.pool.live_count()
    assert a.pool.next_lineage_id == b.pool.next_lineage_id > 8


@pytest.mark.parametrize("world", [1, 2, 3])
def test_field_radiation_over_strips(world):
    """Config-3 field radiation on 1-3 row strips (one identical pool per
    strip, the strips' occupied cells drawing after those above them,
    parent counts summed): the genome plane and the children equal the
    host restatement of the one-context event."""
    from paper_2406_09654_b200.strips import DeviceStrip, StripPlan, field_radiation_local

    H, W = 80, 96
    st = engine.baseline_state("c3", width=W, height=H, genomes=12)
    t = 7
    f = st.substrate.front
    gi0 = f.genome_index.ravel().copy()
    pools = [copy.deepcopy(st.pool) for _ in range(world)]
    ref = copy.deepcopy(st.pool)
    ref.net_factory = None
    occ = np.flatnonzero(gi0 >= 0)
    sel = occ[neat.stream(st.master_seed, t, "field_radiation").random(len(occ)) < 0.02]
    exp_gi = gi0.copy()
    children = {}
    for par in np.unique(gi0[sel]):
        child = neat.mutate(ref.genome(int(par)), neat.EvolutionRates(),
                            neat.stream(st.master_seed, t, "mutate", int(par)), ref.innovations)
        slot = ref.admit(child, parents=(ref.lineage(int(par)),), birth_step=t)
        children[slot] = child
        exp_gi[sel[gi0[sel] == par]] = slot
    plan = StripPlan(H, W, world)
    strips = []
    for r, pool in zip(range(world), pools):
        s = DeviceStrip(plan, r, pool.capacity, hidden=0)
        s.dev.set_params([pool.params(k) for k in range(pool.capacity)])  # as bench.py's strip setup
        s.dev.set_slots(np.asarray(pool.slot_states(), np.int8))
        row0, h = plan.rows(r)
        Cm = f.channels["communication"]
        s.dev.upload_arrays(f.channels["energy"][0][row0:row0 + h], f.channels["infrastructure"][0][row0:row0 + h],
                            Cm[:, row0:row0 + h], f.genome_index[row0:row0 + h], f.rotation[row0:row0 + h])
        strips.append(s)
    info = field_radiation_local(strips, pools, st.master_seed, t, 0.02)
    assert info["selected"] == len(sel) and info["children"] == len(children) > 0
    got = np.empty((H, W), np.int32)
    for r, s in enumerate(strips):
        row0, h = plan.rows(r)
        E = np.empty((h, W), np.float32)
        Cm = np.empty((3, h, W), np.float32)
        gi = np.empty((h, W), np.int32)
        s.dev.download_arrays(E, E.copy(), Cm, gi, np.empty((h, W), np.uint8))
        got[row0:row0 + h] = gi
        s.dev.close()
    np.testing.assert_array_equal(got.ravel(), exp_gi)
    for pool in pools:
        for slot, child in children.items():
            assert pool.genome(slot) == child
