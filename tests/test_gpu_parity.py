"""Parity of the CUDA path (through the C ABI) against the oracle and the
reference's golden vectors.  Tiers:
  A  given identical actions, post-state / events / census bit-exact;
  B  device actions vs reference (or oracle) actions within 1e-5 relative;
  D  free-running: integer state bit-exact, continuous within tolerance.
Continuous tolerance: |a-b| <= 1e-5 * max(|b|, 1)."""

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2406_09654_b200 import _lib, engine, physics
from paper_2406_09654_b200.device import DeviceSubstrate
from paper_2406_09654_b200.hypernet import DenseParams, DirectParams
from tests import _cases as CS

pytestmark = pytest.mark.gpu

TOL = 1e-5


def close(a, b, tol=TOL):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return bool(np.all(np.abs(a - b) <= tol * np.maximum(np.abs(b), 1.0)))


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-30))) if a.size else 0.0


def oracle_phys_to_params(ph: orc.Phys) -> physics.PhysicsParams:
    return physics.PhysicsParams(**{k: getattr(ph, k) for k in physics.PhysicsParams.__dataclass_fields__})


def net_params(net: orc.Net):
    if net.hidden == 0:
        return [DirectParams(net.w2[i], net.b2[i]) for i in range(net.capacity)]
    return [DenseParams(net.w1[i], net.b1[i], net.w2[i], net.b2[i]) for i in range(net.capacity)]


def make_dev(p: orc.Planes, capacity: int, net: orc.Net | None = None, live=None):
    h, w = p.shape
    dev = DeviceSubstrate(w, h, capacity, hidden=0 if net is None else net.hidden)
    if net is not None:
        dev.set_params(net_params(net))
    st = np.zeros(capacity, np.int8)
    st[: capacity if live is None else live] = 1
    dev.set_slots(st)
    dev.upload(p)
    return dev


def download(dev) -> orc.Planes:
    h, w = dev.height, dev.width
    p = orc.Planes(np.empty((h, w), np.float32), np.empty((h, w), np.float32), np.empty((3, h, w), np.float32),
                   np.empty((h, w), np.int32), np.empty((h, w), np.uint8))
    dev.download(p)
    return p


def events_rows(ev):
    return [(float(t), float(s), float(w), float(d), float(r), float(q))
            for t, s, w, d, r, q in zip(ev.target, ev.source, ev.winner_slot, ev.defender_slot, ev.direction,
                                        ev.quantity)]


# -- tier A: physics given the reference's actions ---------------------------------


@pytest.mark.parametrize("c", range(40))
def test_physics_cases_bit_exact(c):
    z = CS.load("physics_cases.npz")
    case = CS.physics_case(z, c)
    dev = make_dev(case["pre"], 12)
    dev.set_actions(case["acts"].cells, case["acts"].a)
    params = oracle_phys_to_params(case["phys"])
    dev.step_raw(physics.step_scalars(case["t"], params), case["t"],
                 flags=_lib.F_INJECT_ACTIONS | _lib.F_RECORD_EVENTS)
    post = download(dev)
    assert post.equal(case["post"])
    assert events_rows(dev.read_events()) == case["events"]
    counts, _, _, _ = dev.read_census()
    assert np.array_equal(counts, case["counts"])
    dev.close()


def test_explore_cases_bit_exact():
    z = CS.load("explore_cases.npz")
    for c in range(int(z["n_cases"])):
        key = f"c{c:02d}_"
        p = CS.planes(z, key, "pre")
        cells = z[key + "cells"]
        a = np.zeros((len(cells), 13), np.float32)
        a[:, 5:] = z[key + "explore"]
        af = physics.ActionField.from_block(cells, a)
        planes = _planeset(p)
        ev = physics.resolve_exploration(planes, af, physics.PhysicsParams(explore_fraction=float(z[key + "alpha"])))
        assert np.array_equal(planes.channels["infrastructure"][0].view(np.uint32), z[key + "post_I"].view(np.uint32))
        assert np.array_equal(planes.genome_index, z[key + "post_gi"])
        assert np.array_equal(planes.rotation, z[key + "post_rot"])
        assert events_rows(ev) == [tuple(r) for r in z[key + "events"].tolist()]


def _planeset(p: orc.Planes):
    from paper_2406_09654_b200.substrate import create_substrate

    h, w = p.shape
    ps = create_substrate(w, h).front
    ps.channels["energy"][0] = p.E
    ps.channels["infrastructure"][0] = p.I
    ps.channels["communication"][:] = p.C
    ps.genome_index[:] = p.gi
    ps.rotation[:] = p.rot
    return ps


# -- reference known-answer cases (test_physics.py values), through the shims -------


def _ps(w=4, h=4):
    from paper_2406_09654_b200.substrate import create_substrate

    return create_substrate(w, h).front


def _acts(cells, **kw):
    n = len(cells)
    a = np.zeros((n, 13), np.float32)
    if "invest" in kw:
        a[:, 0] = kw["invest"]
    if "liquidate" in kw:
        a[:, 1] = kw["liquidate"]
    if "comm" in kw:
        a[:, 2:5] = kw["comm"]
    if "explore" in kw:
        a[:, 5:13] = kw["explore"]
    return physics.ActionField.from_block(np.asarray(cells, np.int64), a)


def test_energy_cycle_values():
    p = _ps()
    physics.energy_cycle(p, 25, physics.PhysicsParams(cycle_amplitude=0.4, cycle_period=100))
    assert np.allclose(p.plane("energy"), 0.4, atol=1e-7)
    p = _ps()
    p.plane("energy")[:] = 2.0
    physics.energy_cycle(p, 75, physics.PhysicsParams(cycle_amplitude=0.4, cycle_period=100, drain_fraction=0.5))
    assert np.allclose(p.plane("energy"), 1.6, rtol=1e-6)
    p = _ps()
    src = np.zeros((4, 4), np.float32)
    src[0, 0] = 2.0
    physics.energy_cycle(p, 1, physics.PhysicsParams(cycle_amplitude=0.5, cycle_period=4, energy_source_map=src))
    assert p.plane("energy")[0, 0] == pytest.approx(1.0, rel=1e-6)
    assert p.plane("energy")[1, 1] == 0.0
    p = _ps()
    p.plane("energy")[:] = 3.0
    physics.energy_cycle(p, 7, physics.PhysicsParams(cycle_amplitude=0.0))
    assert (p.plane("energy") == 3.0).all()


def test_invest_liquidate_values():
    p = _ps()
    p.genome_index[0, 0] = 0
    p.plane("energy")[0, 0] = 1.0
    physics.apply_invest_liquidate(p, _acts([0], invest=[0.5]),
                                   physics.PhysicsParams(invest_rate=1.0, invest_efficiency=0.9, upkeep=0.0))
    assert p.plane("energy")[0, 0] == pytest.approx(0.5, rel=1e-6)
    assert p.plane("infrastructure")[0, 0] == pytest.approx(0.45, rel=1e-6)
    p = _ps()
    p.genome_index[0, 0] = 0
    p.plane("energy")[0, 0] = 0.05
    p.plane("infrastructure")[0, 0] = 10.0
    physics.apply_invest_liquidate(p, _acts([0]), physics.PhysicsParams(upkeep=0.1, decay_on_starvation=0.1))
    assert p.plane("energy")[0, 0] == 0.0
    assert p.plane("infrastructure")[0, 0] == pytest.approx(9.0, rel=1e-6)
    assert p.genome_index[0, 0] == 0
    p = _ps()
    p.genome_index[0, 0] = 3
    p.plane("infrastructure")[0, 0] = 5e-4
    physics.apply_invest_liquidate(p, _acts([0]), physics.PhysicsParams(upkeep=0.0, death_threshold=1e-3))
    assert p.genome_index[0, 0] == -1
    assert p.plane("infrastructure")[0, 0] == pytest.approx(5e-4)
    p = _ps()
    p.plane("energy")[0, 0] = 1.0
    physics.apply_invest_liquidate(p, _acts([0], invest=[0.9]), physics.PhysicsParams())
    assert p.plane("energy")[0, 0] == 1.0 and p.plane("infrastructure")[0, 0] == 0.0


def test_communication_values():
    p = _ps()
    p.genome_index[0, 0] = 0
    physics.write_communication(p, _acts([0], comm=[[0.2, 0.5, 0.8]]))
    assert p.channels["communication"][:, 0, 0].tolist() == pytest.approx([0.2, 0.5, 0.8])
    p = _ps()
    p.channels["communication"][:, 1, 1] = 1.0
    physics.write_communication(p, physics.ActionField.empty())
    assert p.channels["communication"][:, 1, 1] == pytest.approx(0.9)
    physics.write_communication(p, physics.ActionField.empty())
    assert p.channels["communication"][0, 1, 1] == pytest.approx(0.81)


def test_exploration_hand_examples():
    p = _ps()
    p.genome_index[1, 1] = 3
    p.rotation[1, 1] = 2
    p.plane("infrastructure")[1, 1] = 2.0
    p.plane("infrastructure")[2, 1] = 0.3
    ex = np.zeros((1, 8), np.float32)
    ex[0, 0] = 0.8
    ex[0, 5] = 0.1
    ev = physics.resolve_exploration(p, _acts([5], explore=ex), physics.PhysicsParams(explore_fraction=0.5))
    assert p.plane("infrastructure")[1, 1] == pytest.approx(1.2, rel=1e-6)
    assert p.plane("infrastructure")[2, 1] == pytest.approx(1.1, rel=1e-6)
    assert p.genome_index[2, 1] == 3 and p.rotation[2, 1] == 2
    e = ev.aslist()[0]
    assert (e.target, e.source, e.winner_slot, e.defender_slot, e.direction) == (9, 5, 3, -1, 2)
    # tie on quantity: lower source index wins
    p = _ps()
    for (x, y), rot in (((0, 1), 0), ((2, 1), 4)):
        p.genome_index[y, x] = x
        p.rotation[y, x] = rot
        p.plane("infrastructure")[y, x] = 1.0
    ex = np.zeros((2, 8), np.float32)
    ex[:, 0] = 0.5
    ev = physics.resolve_exploration(p, _acts([4, 6], explore=ex), physics.PhysicsParams(explore_fraction=1.0))
    assert len(ev) == 1 and ev.aslist()[0].source == 4 and p.genome_index[1, 1] == 0
    # actuator tie: slot 0
    p = _ps()
    p.genome_index[0, 0] = 1
    p.plane("infrastructure")[0, 0] = 1.0
    ev = physics.resolve_exploration(p, _acts([0], explore=np.full((1, 8), 0.5, np.float32)),
                                     physics.PhysicsParams(explore_fraction=1.0))
    assert ev.aslist()[0].direction == 0


# -- full steps from the reference's golden runs ---------------------------------------


def _golden_net(name):
    z = CS.load(name)
    return z, (CS.step_net(z, 16) if name == "step_hidden.npz" else orc.synth_net(8, 0, seed=0))


@pytest.mark.parametrize("name", ["step_hidden.npz", "step_direct.npz"])
def test_full_step_reference_actions_bit_exact(name):
    z, net = _golden_net(name)
    params = physics.PhysicsParams(cycle_period=20)
    for k in z["keep"].tolist():
        key = f"s{k:03d}_"
        pre = CS.planes(z, key, "pre")
        dev = make_dev(pre, 8, net)
        dev.set_actions(z[key + "cells"], z[key + "acts"])
        dev.step_raw(physics.step_scalars(k, params), k, flags=_lib.F_INJECT_ACTIONS)
        assert download(dev).equal(CS.planes(z, key, "post")), k
        assert dev.read_stats()[0] == int(z[key + "adoptions"])
        assert np.array_equal(dev.read_census()[0], z[key + "counts"])
        dev.close()


@pytest.mark.parametrize("name", ["step_hidden.npz", "step_direct.npz"])
def test_device_actions_vs_reference(name):
    z, net = _golden_net(name)
    params = physics.PhysicsParams(cycle_period=20)
    for k in z["keep"].tolist():
        key = f"s{k:03d}_"
        pre = CS.planes(z, key, "pre")
        dev = make_dev(pre, 8, net)
        dev.step_raw(physics.step_scalars(k, params), k, flags=_lib.F_EXPORT_ACTIONS)
        cells, acts = dev.get_actions()
        assert np.array_equal(cells, z[key + "cells"])
        assert rel_err(acts, z[key + "acts"]) <= TOL
        # and against the oracle's float64-dot restatement
        oa = orc.act(pre, net)
        assert rel_err(acts, oa.a) <= TOL
        dev.close()


def test_config1_free_running_100_steps():
    """BASELINE config 1 from the reference's initial state, 100 steps
    device-resident: genome/rotation planes bit-identical to the reference
    at every recorded step, continuous channels within tolerance."""
    z, net = _golden_net("step_direct.npz")
    pre = CS.planes(z, "s000_", "pre")
    dev = make_dev(pre, 8, net)
    params = physics.PhysicsParams(cycle_period=20)
    keep = set(z["keep"].tolist())
    for t in range(100):
        dev.step_raw(physics.step_scalars(t, params), t)
        if t in keep:
            got = download(dev)
            ref = CS.planes(z, f"s{t:03d}_", "post")
            assert np.array_equal(got.gi, ref.gi), t
            assert np.array_equal(got.rot, ref.rot), t
            assert close(got.E, ref.E) and close(got.I, ref.I) and close(got.C, ref.C), t
    dev.close()


# -- device vs oracle on assorted shapes --------------------------------------------------


def _step_vs_oracle(p0, net, phys, steps, capacity=None, t0=0, flags=0):
    cap = capacity or net.capacity
    dev = make_dev(p0, cap, net)
    params = oracle_phys_to_params(phys)
    p = p0
    for t in range(t0, t0 + steps):
        dev.step_raw(physics.step_scalars(t, params), t, flags=_lib.F_EXPORT_ACTIONS | _lib.F_RECORD_EVENTS | flags)
        cells, acts = dev.get_actions()
        ref = orc.step(p, t, net, phys, acts=orc.Actions(cells, acts))
        got = download(dev)
        assert got.equal(ref.planes), f"t={t}"
        assert events_rows(dev.read_events()) == [tuple(map(float, r)) for r in ref.events.rows()], f"t={t}"
        assert np.array_equal(dev.read_census()[0], ref.counts[:cap]), f"t={t}"
        oa = orc.act(p, net)
        assert np.array_equal(oa.cells, cells)
        assert rel_err(acts, oa.a) <= TOL, f"t={t}"
        p = got
    dev.close()
    return p


@pytest.mark.parametrize("h,w,g", [(1, 1, 1), (2, 3, 2), (3, 3, 3), (5, 7, 4), (31, 33, 5), (40, 65, 9),
                                   (129, 100, 64), (64, 64, 8)])
def test_shapes_vs_oracle(h, w, g):
    p0 = orc.synth_planes(h, w, g, seed=h * 1000 + w)
    # leave some cells empty
    rng = np.random.default_rng(h + w)
    p0.gi[rng.random((h, w)) < 0.2] = -1
    net = orc.synth_net(g, 0, seed=7)
    _step_vs_oracle(p0, net, orc.Phys(cycle_period=4), steps=6)


def test_hidden_nets_vs_oracle():
    for hidden, g in ((16, 6), (1, 3), (13, 4), (128, 5)):
        p0 = orc.synth_planes(48, 40, g, seed=hidden)
        net = orc.synth_net(g, hidden, seed=hidden)
        _step_vs_oracle(p0, net, orc.Phys(cycle_period=20), steps=3)


def test_sparse_infrastructure_contention():
    p0 = orc.synth_planes(96, 96, 16, seed=5, sparse_infra=True)
    net = orc.synth_net(16, 0, seed=5)
    _step_vs_oracle(p0, net, orc.Phys(cycle_period=20, explore_fraction=0.9), steps=5)


def test_empty_world():
    p0 = orc.synth_planes(40, 40, 4, seed=1)
    p0.gi[:] = -1
    net = orc.synth_net(4, 0, seed=1)
    _step_vs_oracle(p0, net, orc.Phys(cycle_period=20), steps=3)


def test_config2_full_size_tier_a():
    """BASELINE config 2 at full size (1024x1024, 64 genomes): two steps,
    device actions injected into the oracle physics -> bit-exact state,
    events and census; device actions within tolerance of the oracle's."""
    p0 = orc.synth_planes(1024, 1024, 64, seed=0)
    net = orc.synth_net(64, 0, seed=0)
    _step_vs_oracle(p0, net, orc.Phys(cycle_period=20), steps=2)


# -- engine-level properties ------------------------------------------------------------


def test_engine_step_equals_run_and_is_deterministic():
    a = engine.baseline_state("c1")
    b = engine.baseline_state("c1")
    c = engine.baseline_state("c1")
    for _ in range(7):
        engine.step(a)
    engine.run(b, 7)
    engine.run(c, 3)
    engine.run(c, 4)
    assert engine.digest(a) == engine.digest(b) == engine.digest(c)
    assert a.t == b.t == c.t == 7
    assert a.pool.live_count() == b.pool.live_count()


def test_engine_matches_oracle_c1():
    st = engine.baseline_state("c1")
    p = orc.synth_planes(64, 64, 8, seed=0)
    net = orc.synth_net(8, 0, seed=0)
    for t in range(5):
        af = engine.build_action_field(st)
        res = orc.step(p, t, net, orc.Phys(cycle_period=20), acts=orc.Actions(af.cells, af.block()))
        engine.step(st)
        f = st.substrate.front
        assert np.array_equal(f.genome_index, res.planes.gi)
        assert np.array_equal(f.channels["energy"][0], res.planes.E)
        assert st.last_adoptions == len(res.events)
        p = res.planes
    assert engine.digest(st) == orc.digest(p)


def _rot_plane(p):
    n = p.shape[-1]
    ys, xs = np.mgrid[0:n, 0:n]
    out = np.empty_like(p)
    out[..., xs, (n - ys) % n] = p[..., ys, xs]
    return out


def test_rotation_equivariance_bit_exact():
    """Quarter-turning the world commutes with stepping it (the reference's
    acceptance property, test_acceptance.py:225-264), bit-exactly."""
    p0 = orc.synth_planes(64, 64, 8, seed=3)
    net = orc.synth_net(8, 0, seed=3)
    pr = orc.Planes(_rot_plane(p0.E), _rot_plane(p0.I), _rot_plane(p0.C), _rot_plane(p0.gi),
                    _rot_plane(((p0.rot + 2) % 8).astype(np.uint8)))
    params = physics.PhysicsParams(cycle_period=20)
    da, db = make_dev(p0, 8, net), make_dev(pr, 8, net)
    for t in range(30):
        da.step_raw(physics.step_scalars(t, params), t)
        db.step_raw(physics.step_scalars(t, params), t)
    a, b = download(da), download(db)
    assert np.array_equal(_rot_plane(a.gi), b.gi)
    assert np.array_equal(_rot_plane(((a.rot + 2) % 8).astype(np.uint8)), b.rot)
    for x, y in ((a.E, b.E), (a.I, b.I), (a.C, b.C)):
        assert np.array_equal(_rot_plane(x), y)


def test_conservation_lossless():
    p0 = orc.synth_planes(128, 128, 16, seed=9)
    p0.C[:] = 0.5
    net = orc.synth_net(16, 0, seed=9)
    params = physics.PhysicsParams(cycle_amplitude=0.0, drain_fraction=0.0, invest_efficiency=1.0,
                                   liquidate_efficiency=1.0, upkeep=0.0, decay_on_starvation=0.0)
    dev = make_dev(p0, 16, net)
    tot0 = float(p0.E.astype(np.float64).sum() + p0.I.astype(np.float64).sum())
    for t in range(100):
        dev.step_raw(physics.step_scalars(t, params), t)
    p = download(dev)
    tot = float(p.E.astype(np.float64).sum() + p.I.astype(np.float64).sum())
    assert abs(tot - tot0) / tot0 < 1e-4
    assert (p.E >= 0).all() and (p.I >= 0).all()
    assert ((p.gi >= -1) & (p.gi < 16)).all() and (p.rot < 8).all()


def test_census_deaths_tracked_on_device():
    p0 = orc.synth_planes(32, 32, 6, seed=2)
    p0.gi[p0.gi == 5] = 4  # slot 5 live in the pool but owns no cell -> dies at t+1
    net = orc.synth_net(6, 0, seed=2)
    dev = make_dev(p0, 6, net)
    dev.step_raw(physics.step_scalars(0, physics.PhysicsParams()), 0)
    counts, state, death, peak = dev.read_census()
    assert counts[5] == 0 and state[5] == 2 and death[5] == 1
    assert dev.read_stats()[1] >= 1
    assert (peak[:5] == counts[:5]).all()


# -- hidden-layer controller on the tensor cores (tcgen05 3xTF32) ----------------------------


def _actions(dev, t, params, flags=0):
    dev.step_raw(physics.step_scalars(t, params), t, flags=_lib.F_EXPORT_ACTIONS | flags)
    return dev.get_actions()


@pytest.mark.parametrize("hidden,genomes,shape", [(128, 300, (96, 80)), (16, 7, (33, 70)), (64, 1, (40, 40)),
                                                  (128, 2, (1, 300))])
def test_tensor_core_net_vs_oracle_and_cuda_core(hidden, genomes, shape):
    """BASELINE config-5 net shape (45->128 tanh->13, N(0,0.3), sparse infra)
    and odd shapes: many genomes with 1-cell groups, a single genome spanning
    several 128-row tiles with a partial last tile, a 1-row torus.  Device
    actions vs the oracle's float64 forward within 1e-5 relative, and the
    physics bit-exact given them; the CUDA-core FP32 path as a cross-check."""
    h, w = shape
    p0 = orc.synth_planes(h, w, genomes, seed=hidden + genomes, sparse_infra=True)
    net = orc.synth_net(genomes, hidden, seed=3)
    phys = orc.Phys(cycle_period=20)
    params = oracle_phys_to_params(phys)
    oa = orc.act(p0, net)
    dev = make_dev(p0, genomes, net)
    cells, acts = _actions(dev, 0, params, _lib.F_TC_NET)  # tensor cores at every hidden width (both layers)
    assert np.array_equal(cells, oa.cells)
    err_tc = rel_err(acts, oa.a)
    assert err_tc <= TOL
    ref = orc.step(p0, 0, net, phys, acts=orc.Actions(cells, acts))
    assert download(dev).equal(ref.planes)
    dev.close()
    dev = make_dev(p0, genomes, net)  # layer 2 on the CUDA cores (the round-2 kernel)
    cells3, acts3 = _actions(dev, 0, params, _lib.F_TC_NET | _lib.F_L2_CUDA_CORE)
    assert np.array_equal(cells3, cells) and rel_err(acts3, oa.a) <= TOL
    dev.close()
    dev = make_dev(p0, genomes, net)  # the same tcgen05 net over the gather sort instead of sensor rows
    cells4, acts4 = _actions(dev, 0, params, _lib.F_TC_NET | _lib.F_GATHER_NET)
    assert np.array_equal(cells4, cells) and np.array_equal(acts4, acts)
    ref4 = orc.step(p0, 0, net, phys, acts=orc.Actions(cells4, acts4))
    assert download(dev).equal(ref4.planes)
    dev.close()
    dev = make_dev(p0, genomes, net)
    cells2, acts2 = _actions(dev, 0, params, _lib.F_CUDA_CORE_NET)
    assert np.array_equal(cells2, cells) and rel_err(acts2, oa.a) <= TOL
    print(f"H={hidden}: tcgen05 x2 {err_tc:.3g}, layer 2 FFMA {rel_err(acts3, oa.a):.3g}, FP32 {rel_err(acts2, oa.a):.3g}")
    dev.close()


def test_tensor_core_net_free_running_matches_oracle():
    """A few device-resident steps of a hidden-128 world against the oracle
    (tier A per step with the device's own actions)."""
    p0 = orc.synth_planes(64, 64, 40, seed=11, sparse_infra=True)
    net = orc.synth_net(40, 128, seed=11)
    _step_vs_oracle(p0, net, orc.Phys(cycle_period=20), steps=4)


@pytest.mark.parametrize("genomes,shape", [(300, (96, 80)), (1024, (64, 64)), (90, (1, 500)), (2048, (37, 129)),
                                           (70, (2, 3)), (512, (300, 257))])
def test_genome_sorted_direct_path_matches_tile_path(genomes, shape):
    """Pools larger than the tile kernel's shared-memory weight table (68
    slots) run the direct net on cells sorted by (band, slot, rotation),
    gathering their Moore neighbourhoods from the sense texture
    (evoca_gather.cu; EVO_F_ROWS_NET: the earlier sensor rows through HBM);
    per-cell arithmetic (FFMA2 pairing, k order, bias, sigmoid) is the tile
    kernel's, so every path gives bit-identical states, and tier A holds vs
    the oracle.  Shapes: a 1-row and a 2-row torus (ghost rows = the strip's
    own rows), odd widths (x seam), the largest gather pool (2048 slots)."""
    h, w = shape
    p0 = orc.synth_planes(h, w, genomes, seed=genomes)
    net = orc.synth_net(genomes, 0, seed=5)
    phys = orc.Phys(cycle_period=20)
    params = oracle_phys_to_params(phys)
    a = make_dev(p0, genomes, net)  # gather, 8-float decided records
    b = make_dev(p0, genomes, net)  # per-tile kernel
    c = make_dev(p0, genomes, net)  # gather, full 13-actuator rows (export)
    d = make_dev(p0, genomes, net)  # genome-sorted sensor rows
    e = make_dev(p0, genomes, net)  # genome-sorted sensor rows, export
    for t in range(3):
        sc = physics.step_scalars(t, params)
        a.step_raw(sc, t)
        b.step_raw(sc, t, flags=_lib.F_TILE_NET)
        c.step_raw(sc, t, flags=_lib.F_EXPORT_ACTIONS)
        d.step_raw(sc, t, flags=_lib.F_ROWS_NET)
        e.step_raw(sc, t, flags=_lib.F_ROWS_NET | _lib.F_EXPORT_ACTIONS)
        want = download(b)
        for x, name in ((a, "gather"), (c, "gather export"), (d, "rows"), (e, "rows export")):
            assert download(x).equal(want), f"{name} t={t}"
        ca, aa = c.get_actions()
        ce, ae = e.get_actions()
        assert np.array_equal(ca, ce) and np.array_equal(aa, ae), f"t={t}"
    # the decided records of a non-export step are not actuator rows
    with pytest.raises(ValueError):
        a.get_actions()
    for x in (a, b, c, d, e):
        x.close()
    _step_vs_oracle(p0, net, phys, steps=2)


@pytest.mark.parametrize("genomes,shape", [(300, (96, 80)), (1024, (64, 64)), (90, (1, 500)), (2048, (70, 260)),
                                           (512, (2, 36)), (128, (131, 516)), (8192, (64, 128))])
@pytest.mark.parametrize("phases", [_lib.PH_ALL, _lib.PH_ENERGY | _lib.PH_INVEST | _lib.PH_EXPLORE,
                                    _lib.PH_COMM | _lib.PH_EXPLORE])
def test_fused_gather_step_matches_unfused(genomes, shape, phases):
    """evo_step on the gather path runs the physics in the net's epilogue and
    hands pass 2 one 32-byte record per cell (no k_physics_rows, no mid
    planes; FusedPhysics in evoca_internal.h).  EVO_F_UNFUSED keeps the
    round-2d kernels: planes, census counts, adoption events and stats are
    bit-identical, with unoccupied cells (their records come from the texture
    build), starving cells (communication decay re-reads the cell's record),
    phase subsets, a 1- and a 2-row torus, widths off the 32-cell warp
    tile and the 256-cell TMA box, and the largest pool (8192 slots: 70 KB of
    shared memory per pass-2 CTA)."""
    h, w = shape
    p0 = orc.synth_planes(h, w, genomes, seed=genomes + 1)
    rng = np.random.default_rng(7)
    p0.gi[rng.random((h, w)) < 0.3] = -1  # unoccupied cells
    p0.I[rng.random((h, w)) < 0.2] *= np.float32(0.002)  # cells that starve below the death threshold
    net = orc.synth_net(genomes, 0, seed=9)
    phys = orc.Phys(cycle_period=4)
    params = oracle_phys_to_params(phys)
    a = make_dev(p0, genomes, net)
    b = make_dev(p0, genomes, net)
    for t in range(4):
        sc = physics.step_scalars(t, params)
        a.step_raw(sc, t, phases=phases, flags=_lib.F_RECORD_EVENTS)
        b.step_raw(sc, t, phases=phases, flags=_lib.F_RECORD_EVENTS | _lib.F_UNFUSED)
        assert download(a).equal(download(b)), f"t={t}"
        for ca, cb in zip(a.read_census(), b.read_census()):
            assert np.array_equal(ca, cb)
        assert a.read_stats() == b.read_stats()
        assert events_rows(a.read_events()) == events_rows(b.read_events())
    # a step without event records, then a bare pass 1 / pass 2 pair (mid planes again)
    sc = physics.step_scalars(4, params)
    a.step_raw(sc, 4, phases=phases)
    b.step_raw(sc, 4, phases=phases, flags=_lib.F_UNFUSED)
    assert download(a).equal(download(b))
    sc = physics.step_scalars(5, params)
    a.pass1(sc, 5, phases=phases)
    a.pass2(5)
    a.swap()
    b.step_raw(sc, 5, phases=phases)
    assert download(a).equal(download(b))
    sc = physics.step_scalars(6, params)  # the pair evo_step itself issues
    a.pass1(sc, 6, phases=phases, flags=_lib.F_FUSE_MID)
    a.pass2(6)
    a.swap()
    b.step_raw(sc, 6, phases=phases, flags=_lib.F_UNFUSED)
    assert download(a).equal(download(b))
    # consecutive evo_steps are lazy: pass 2 leaves E', C' and the final I in
    # the sense texture only (the next step ranks the genome plane and builds
    # no texture) until something reads the planes; census, stats, events and
    # genome patches do not
    rng2 = np.random.default_rng(11)
    for t in range(7, 12):
        sc = physics.step_scalars(t, params)
        a.step_raw(sc, t, phases=phases, flags=_lib.F_RECORD_EVENTS)
        b.step_raw(sc, t, phases=phases, flags=_lib.F_RECORD_EVENTS | _lib.F_UNFUSED)
        assert a.read_stats() == b.read_stats()
        assert events_rows(a.read_events()) == events_rows(b.read_events())
        if t == 9:  # a genome patch between lazy steps (field radiation's device half)
            cells = rng2.choice(h * w, size=max(1, h * w // 50), replace=False).astype(np.int64)
            slots = rng2.integers(0, genomes, size=len(cells)).astype(np.int32)
            a.patch_genomes(cells, slots)
            b.patch_genomes(cells, slots)
        if t == 10:  # an observable straight from the lazy state
            assert np.array_equal(a.render_rgb(), b.render_rgb())
    for ca, cb in zip(a.read_census(), b.read_census()):
        assert np.array_equal(ca, cb)
    assert download(a).equal(download(b))
    k = 4  # evo_run, then a plain download
    scs = [physics.step_scalars(12 + i, params) for i in range(k)]
    a.run(scs, 12)
    for i in range(k):
        b.step_raw(scs[i], 12 + i, flags=_lib.F_UNFUSED)
    assert download(a).equal(download(b))
    a.close()
    b.close()


def test_sigmoid_reciprocal_is_correctly_rounded():
    """squash (hypernet.py:246-251) divides through an inline MUFU.RCP +
    residual step instead of __frcp_rn's branchy form: identical bits for
    every float in [1, 2^125) - 1 + exp(-z) for z > -86.6 (below that the
    output is clamped to 2^-126 either way)."""
    import ctypes as C

    n = C.c_uint64(1)
    _lib.check(_lib.load().evo_debug_rcp_check(C.byref(n)))
    assert n.value == 0


@pytest.mark.parametrize("genomes,hidden,shape", [(8, 0, (64, 64)), (300, 0, (96, 80)), (20, 128, (64, 96)),
                                                  (6, 16, (33, 70))])
def test_evo_run_graphs_equal_step_loop(genomes, hidden, shape):
    """evo_run captures its steps (all but the first) into CUDA graphs of up to
    128 steps; the planes, census, stats and the device's step state afterwards
    equal a loop of evo_step - per-tile kernel, gather path (lazy fused
    steps inside the graph), tensor-core and CUDA-core hidden nets; two runs
    back to back, a run of 3 (eager: below the graph threshold), then single
    steps again."""
    h, w = shape
    p0 = orc.synth_planes(h, w, genomes, seed=genomes + 3)
    net = orc.synth_net(genomes, hidden, seed=2)
    params = oracle_phys_to_params(orc.Phys(cycle_period=7))
    a = make_dev(p0, genomes, net)
    b = make_dev(p0, genomes, net)
    t = 0
    for k in (9, 140, 3, 5):
        scs = [physics.step_scalars(t + i, params) for i in range(k)]
        a.run(scs, t)
        for i in range(k):
            b.step_raw(scs[i], t + i)
        t += k
        assert a.read_stats() == b.read_stats()
        for ca, cb in zip(a.read_census(), b.read_census()):
            assert np.array_equal(ca, cb)
        assert download(a).equal(download(b)), f"k={k}"
    sc = physics.step_scalars(t, params)
    a.step_raw(sc, t)
    b.step_raw(sc, t)
    assert download(a).equal(download(b))
    a.close()
    b.close()


@pytest.mark.parametrize("shape", [(96, 80), (70, 258), (1, 512)])
def test_tma_texture_build_matches_lsu_build(shape, monkeypatch):
    """The gather path's texture build through TMA (k_gs_count_tma, the
    default for whole-strip steps) and the LSU kernel it replaced
    (EVO_NO_TMA) give bit-identical steps, including widths that are not a
    multiple of the 256-cell TMA box and a 1-row torus."""
    h, w = shape
    p0 = orc.synth_planes(h, w, 300, seed=w)
    net = orc.synth_net(300, 0, seed=7)
    params = oracle_phys_to_params(orc.Phys(cycle_period=20))
    states = []
    for no_tma in (False, True):  # the maps are made at a context's first gather step
        if no_tma:
            monkeypatch.setenv("EVO_NO_TMA", "1")
        d = make_dev(p0, 300, net)
        got = []
        for t in range(3):
            d.step_raw(physics.step_scalars(t, params), t)
            got.append(download(d))
        d.close()
        states.append(got)
    for t in range(3):
        assert states[0][t].equal(states[1][t]), f"t={t}"


@pytest.mark.parametrize("genomes,shape", [(8, (64, 64)), (64, (128, 96)), (1, (33, 40))])
def test_gather_path_on_small_pools_matches_tile_path(genomes, shape):
    """EVO_F_GATHER_NET forces the large-pool gather path on a pool the tile
    kernel holds in shared memory: bit-identical states and actions."""
    h, w = shape
    p0 = orc.synth_planes(h, w, genomes, seed=genomes + 3)
    net = orc.synth_net(genomes, 0, seed=genomes)
    params = oracle_phys_to_params(orc.Phys(cycle_period=20))
    a, b = make_dev(p0, genomes, net), make_dev(p0, genomes, net)
    for t in range(3):
        sc = physics.step_scalars(t, params)
        a.step_raw(sc, t, flags=_lib.F_GATHER_NET | _lib.F_EXPORT_ACTIONS)
        b.step_raw(sc, t, flags=_lib.F_EXPORT_ACTIONS)
        assert download(a).equal(download(b)), f"t={t}"
        ca, aa = a.get_actions()
        cb, ab = b.get_actions()
        assert np.array_equal(ca, cb) and np.array_equal(aa, ab), f"t={t}"
    a.close()
    b.close()


@pytest.mark.parametrize("genomes,shape,sigma", [(300, (96, 80), 0.5), (1024, (64, 64), 0.5), (90, (1, 500), 0.5),
                                                 (2048, (37, 129), 0.5), (256, (128, 128), 1.5), (80, (200, 3), 3.0)])
def test_tc_direct_net_vs_oracle(genomes, shape, sigma):
    """The large-pool direct net on tcgen05 (EVO_F_TC_DIRECT: 128-cell tiles
    of one (slot, rotation) group, A = [hi | lo] split over TMEM and shared
    memory, B = the rotation-permuted [W_hi | W_lo], two accumulators):
    actions vs the oracle's float64 forward within 1e-5 relative or - where
    an FP32 forward itself misses that (large weights: CPPN-expressed weights
    reach |w| = 3, logits beyond 50 whose float32 ulp alone is ~4e-6) -
    within twice the FP32 fixed-order tile kernel's error (the rule the
    radiation tests apply to the reference's own OpenBLAS forward);
    physics tier A given them; the decided (non-export) variant identical;
    three free-running steps tier A against the oracle."""
    h, w = shape
    p0 = orc.synth_planes(h, w, genomes, seed=genomes + 17)
    net = orc.synth_net(genomes, 0, seed=genomes, sigma=sigma)
    phys = orc.Phys(cycle_period=20)
    params = oracle_phys_to_params(phys)
    oa = orc.act(p0, net)
    dev = make_dev(p0, genomes, net)
    cells_f, acts_f = _actions(dev, 0, params, _lib.F_TILE_NET)
    dev.close()
    err_fp32 = rel_err(acts_f, oa.a)
    dev = make_dev(p0, genomes, net)
    cells, acts = _actions(dev, 0, params, _lib.F_TC_DIRECT)
    assert np.array_equal(cells, oa.cells) and np.array_equal(cells_f, cells)
    err = rel_err(acts, oa.a)
    print(f"tcgen05 {err:.3g}, FP32 tile kernel {err_fp32:.3g}")
    assert err <= max(TOL, 2.0 * err_fp32)
    ref = orc.step(p0, 0, net, phys, acts=orc.Actions(cells, acts))
    got = download(dev)
    assert got.equal(ref.planes)
    dev.close()
    dev = make_dev(p0, genomes, net)
    dev.step_raw(physics.step_scalars(0, params), 0, flags=_lib.F_TC_DIRECT)
    assert download(dev).equal(got)
    dev.close()
    if sigma <= 0.5:
        _step_vs_oracle(p0, net, phys, steps=3, flags=_lib.F_TC_DIRECT)


# -- direct net on the tensor cores (k_pass1_mma, mma.sync 3xTF32) ---------------------------


@pytest.mark.parametrize("genomes,shape,hole", [(64, (96, 80), False), (8, (64, 64), False), (1, (40, 33), False),
                                                 (64, (1, 300), False), (13, (70, 35), True), (64, (128, 128), True)])
def test_mma_direct_net_vs_oracle_and_ffma(genomes, shape, hole):
    """EVO_F_MMA_NET runs the direct 45->13 net of pools <= 64 slots as
    mma.sync m16n8k8 TF32 (3xTF32 split, 8-cell genome blocks; a measured
    alternative to the default FFMA2 tile kernel): device actions vs the
    oracle within 1e-5 relative, explore argmax and physics tier A given them,
    the export and decided variants bit-identical, the default path within
    the same tolerance.  Shapes: full pools, a single genome, a 1-row torus,
    partial tiles, unoccupied slots."""
    h, w = shape
    p0 = orc.synth_planes(h, w, genomes, seed=genomes * 7 + h)
    if hole:  # a live slot without cells
        p0.gi[p0.gi == 3] = 4
    live = None
    net = orc.synth_net(genomes, 0, seed=genomes + 1)
    phys = orc.Phys(cycle_period=20)
    params = oracle_phys_to_params(phys)
    oa = orc.act(p0, net)
    dev = make_dev(p0, genomes, net, live=live)
    cells, acts = _actions(dev, 0, params, _lib.F_MMA_NET)
    assert np.array_equal(cells, oa.cells)
    assert rel_err(acts, oa.a) <= TOL
    ref = orc.step(p0, 0, net, phys, acts=orc.Actions(cells, acts))
    got = download(dev)
    assert got.equal(ref.planes)
    dev.close()
    dev = make_dev(p0, genomes, net, live=live)  # decided (non-export) variant
    dev.step_raw(physics.step_scalars(0, params), 0, flags=_lib.F_MMA_NET)
    assert download(dev).equal(got)
    dev.close()
    dev = make_dev(p0, genomes, net, live=live)
    cells2, acts2 = _actions(dev, 0, params)
    assert np.array_equal(cells2, cells) and rel_err(acts2, oa.a) <= TOL
    dev.close()


def test_mma_direct_net_follows_parameter_updates():
    """The fragment-order weight copy is rebuilt after evo_set_params: a step
    after replacing the nets uses the new weights."""
    p0 = orc.synth_planes(48, 48, 16, seed=21)
    net_a = orc.synth_net(16, 0, seed=1)
    net_b = orc.synth_net(16, 0, seed=2)
    params = oracle_phys_to_params(orc.Phys(cycle_period=20))
    dev = make_dev(p0, 16, net_a)
    _actions(dev, 0, params, _lib.F_MMA_NET)
    dev.set_params(net_params(net_b))
    dev.upload(p0)
    cells, acts = _actions(dev, 0, params, _lib.F_MMA_NET)
    oa = orc.act(p0, net_b)
    assert np.array_equal(cells, oa.cells) and rel_err(acts, oa.a) <= TOL
    dev.close()


@pytest.mark.parametrize("genomes,live,shape", [(100, 100, (64, 64)), (200, 200, (96, 80)), (300, 300, (70, 35)),
                                                (700, 400, (128, 96)), (90, 90, (1, 500))])
def test_cluster_sharded_path_matches_rows_and_tile(genomes, live, shape):
    """The cluster-sharded tile kernel for large direct pools (k_pass1_shard,
    EVO_F_SHARD_NET: 64 resident genomes per CTA, records through DSMEM,
    stragglers beyond 64 x 4 resident slots from global weights) must be
    bit-identical to the genome-sorted rows path and the per-tile kernel,
    including slots marked free or dead in the pool (stragglers) and partial
    tiles."""
    h, w = shape
    p0 = orc.synth_planes(h, w, genomes, seed=genomes + h)
    net = orc.synth_net(genomes, 0, seed=genomes)
    st = np.zeros(genomes, np.int8)
    st[:live] = 1
    st[live:] = 2  # cells of "dead" slots: evaluated as stragglers
    phys = orc.Phys(cycle_period=20)
    params = oracle_phys_to_params(phys)
    devs = []
    for _ in range(3):
        d = make_dev(p0, genomes, net)
        d.set_slots(st)
        devs.append(d)
    a, b, c = devs
    for t in range(3):
        sc = physics.step_scalars(t, params)
        a.step_raw(sc, t, flags=_lib.F_SHARD_NET)   # cluster-sharded tile kernel (A/B)
        b.step_raw(sc, t)                           # genome-sorted rows (default for large pools)
        c.step_raw(sc, t, flags=_lib.F_TILE_NET)    # per-tile kernel, weights from global
        want = download(b)
        assert download(a).equal(want), f"t={t}"
        assert download(c).equal(want), f"t={t}"
        assert a.read_stats()[0] == b.read_stats()[0]
    for d in devs:
        d.close()
