"""Host-side logic of the package, checked against the oracle on CPU."""

import math

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2406_09654_b200 import physics, synth
from paper_2406_09654_b200.hypernet import DenseParams, DirectParams, pack_params
from paper_2406_09654_b200.pool import SlotPool


@pytest.mark.parametrize("period", [2, 3, 4, 20, 100, 7919])
@pytest.mark.parametrize("amp", [0.0, 0.1, 1.0])
def test_step_scalars_match_reference_rho(period, amp):
    phys = physics.PhysicsParams(cycle_amplitude=amp, cycle_period=period, drain_fraction=0.37)
    for t in list(range(0, 3 * period + 2)) + [10**6 + 17]:
        s = physics.step_scalars(t, phys)
        mode, r32, d32 = orc.rho_terms(t, orc.Phys(cycle_amplitude=amp, cycle_period=period, drain_fraction=0.37))
        assert s.rho_mode == mode
        assert np.float32(s.rho_f32) == r32
        assert np.float32(s.drain_f32) == d32


def test_step_scalars_casts():
    s = physics.step_scalars(0, physics.PhysicsParams(explore_fraction=0.1, death_threshold=1e-3))
    assert np.float32(s.explore_fraction) == np.float32(0.1)
    assert np.float32(s.death_threshold) == np.float32(1e-3)


def test_synth_matches_oracle_generator():
    for sparse in (False, True):
        E, I, C, gi, rot = synth.synth_arrays(33, 17, 7, seed=4, sparse_infra=sparse)
        p = orc.synth_planes(33, 17, 7, seed=4, sparse_infra=sparse)
        for a, b in zip((E, I, C, gi, rot), p.arrays()):
            assert a.dtype == b.dtype and np.array_equal(a, b)
    direct = synth.synth_params(5, 0, seed=2)
    net = orc.synth_net(5, 0, seed=2)
    for i, d in enumerate(direct):
        assert np.array_equal(d.w, net.w2[i]) and np.array_equal(d.b, net.b2[i])
    hid = synth.synth_params(3, 128, seed=2)
    net = orc.synth_net(3, 128, seed=2)
    for i, d in enumerate(hid):
        assert np.array_equal(d.w1, net.w1[i]) and np.array_equal(d.w2, net.w2[i])


def test_rotation_tables_match_reference_kats():
    # test_physics.py:46-76 known answers
    assert physics.KERNEL_OFFSETS.tolist() == [[1, 0], [1, 1], [0, 1], [-1, 1], [-1, 0], [-1, -1], [0, -1], [1, -1]]
    assert physics.rotation_permutation(0).tolist() == [0, 1, 7, 2, 6, 3, 5, 4]
    assert physics.rotation_permutation(2).tolist() == [2, 3, 1, 4, 0, 5, 7, 6]
    assert np.array_equal(physics.PERM_TABLE, orc.PERM)
    with pytest.raises(ValueError):
        physics.rotation_permutation(8)


def test_pack_params_layout():
    d = [DirectParams(np.arange(13 * 45, dtype=np.float32).reshape(13, 45), np.arange(13, dtype=np.float32)), None]
    w1, b1, w2, b2 = pack_params(d, 0)
    assert w1 is None and w2.shape == (2, 13, 45) and not w2[1].any()
    h = [DenseParams(np.ones((4, 45), np.float32), np.ones(4, np.float32), np.ones((13, 4), np.float32),
                     np.ones(13, np.float32))]
    w1, b1, w2, b2 = pack_params(h, 4)
    assert w1.shape == (1, 4, 45) and w2.shape == (1, 13, 4)
    with pytest.raises(ValueError):
        pack_params(h, 5)


def test_slot_pool_census_contract():
    pool = SlotPool(4)
    for s in range(3):
        pool.install(s, None)
    dead = pool.update_census(np.array([2, 0, 1, 0]), step=10)
    assert dead == [1]
    assert pool.record_for_slot(0).peak_population == 2
    assert pool.records[pool.lineage(1)].death_step == 10
    # deferred device census folds to the same records
    p2 = SlotPool(4)
    for s in range(3):
        p2.install(s, None)
    dead2 = p2.apply_device_census(np.array([1, 2, 1, 0], np.int8), np.array([-1, 10, -1, -1]),
                                   np.array([2, 0, 1, 0], np.int32))
    assert dead2 == [1]
    assert p2.records[p2.lineage(1)].death_step == 10
    assert p2.record_for_slot(0).peak_population == 2


# -- pool admission, device-expression placeholders, program linearisation --------------


def test_slot_pool_admission_matches_reference_rules():
    """GenomePool.admit (neuroevo.py:451-487): lowest free slot, else the dead
    slot with the oldest death step (lowest index on ties), else None."""
    from paper_2406_09654_b200 import neat

    pool = SlotPool(4, net_factory=lambda g: ("params", g))
    g = neat.init_genome(np.random.default_rng(0), pool.innovations)
    assert [pool.admit(g, birth_step=0) for _ in range(4)] == [0, 1, 2, 3]
    assert pool.admit(g) is None and not pool.can_admit()
    # slots 2 and 1 die at steps 5 and 7, slot 3 at step 5 too
    counts = np.array([9, 9, 0, 0])
    pool.update_census(counts, 5)
    pool.update_census(np.array([9, 0, 0, 0]), 7)
    assert pool.can_admit()
    assert pool.admit(g, parents=(0,), birth_step=8) == 2  # oldest death (5), lowest index of the tie
    assert pool.admit(g, birth_step=8) == 3
    assert pool.admit(g, birth_step=8) == 1
    assert pool.admit(g) is None
    assert pool.params(2) == ("params", g) and pool.genome(2) is g
    assert pool.record_for_slot(2).parents == (0,)


def test_device_expressed_placeholder_surface():
    from paper_2406_09654_b200 import neat
    from paper_2406_09654_b200.radiation import DeviceExpressed

    g = neat.init_genome(np.random.default_rng(1), neat.InnovationCounter())
    direct = DeviceExpressed(g, 0)
    dense = DeviceExpressed(g, 16)
    assert not hasattr(direct, "w1") and not hasattr(dense, "w")
    with pytest.raises(RuntimeError):
        _ = direct.w  # not generated yet: no silent host fallback
    with pytest.raises(RuntimeError):
        _ = dense.w1

    class FakeDev:
        def get_params_arrays(self, slot, n):
            assert (slot, n) == (3, 1)
            return None, None, np.full((1, 13, 45), 2.0, np.float32), np.zeros((1, 13), np.float32)

    direct.bind(FakeDev(), 3)
    assert direct.expressed and direct.w.shape == (13, 45) and float(direct.w[0, 0]) == 2.0


def test_compile_programs_rejects_malformed_genomes():
    from paper_2406_09654_b200 import neat

    rng = np.random.default_rng(2)
    g = neat.init_genome(rng, neat.InnovationCounter())
    # a cycle in the full gene graph
    h = neat.NodeGene(7, "hidden", "sine")
    cyc = neat.CppnGenome(g.nodes + (h,), g.connections + (neat.ConnGene(99, 5, 7, 1.0, True),
                                                            neat.ConnGene(100, 7, 5, 1.0, True)))
    with pytest.raises(ValueError):
        neat.compile_programs([cyc])
    bad = neat.CppnGenome(tuple(n for n in g.nodes if n.id != 6), tuple(c for c in g.connections if c.dst != 6))
    with pytest.raises(ValueError):
        neat.compile_programs([bad])
    node_off, nodes, esrc, ew, outs = neat.compile_programs([g, g])
    assert node_off.tolist() == [0, 7, 14] and outs.tolist() == [[5, 6], [5, 6]]
    assert len(esrc) == 20 and np.all(esrc < 7)


def test_layout_coords_match_reference_layout():
    from oracle import cppn as ocppn
    from paper_2406_09654_b200 import neat

    for hidden in (0, 16, 128):
        inp, hid, out = ocppn.make_layout(hidden)
        np.testing.assert_array_equal(neat.layout_coords(hidden), np.vstack([inp, hid, out]))


def test_apply_device_census_incremental_fold():
    """SlotPool.apply_device_census visits only the live slots whose occupant
    or device peak changed since the last fold (a config-3 radiation event
    folds ~1000 slots); records, states and deaths equal the plain per-slot
    loop over random census sequences with deaths, re-installs into dead
    slots and peaks written to the records behind its back."""
    rng = np.random.default_rng(0)
    cap = 64

    def plain(pool, state, death, peak):
        dead = []
        for i in np.flatnonzero(pool._state == 1):
            rec = pool.records[int(pool._lineage[i])]
            if peak[i] > rec.peak_population:
                rec.peak_population = int(peak[i])
            if state[i] == 2:
                pool._state[i] = 2
                pool._death[i] = int(death[i])
                rec.death_step = int(death[i])
                dead.append(int(i))
        return dead

    a, b = SlotPool(cap), SlotPool(cap)
    for pool in (a, b):
        for s in range(40):
            pool.install(s, object())
    dev_peak = np.zeros(cap, np.int32)
    for step in range(1, 60):
        live = a._state == 1
        dev_peak = np.where(live, np.maximum(dev_peak, rng.integers(0, 50, cap)), dev_peak).astype(np.int32)
        if step % 3:
            dev_peak = dev_peak.copy()  # many folds see unchanged peaks
        st = a._state.copy()
        dying = live & (rng.random(cap) < 0.05)
        st[dying] = 2
        death = np.where(dying, step, -1).astype(np.int64)
        assert a.apply_device_census(st, death, dev_peak) == plain(b, st, death, dev_peak)
        if step % 7 == 0:  # a dead slot gets a new occupant: the device peak starts over
            for s in np.flatnonzero(a._state == 2)[:2]:
                a.install(int(s), object(), birth_step=step)
                b.install(int(s), object(), birth_step=step)
                dev_peak[s] = 0
        if step % 11 == 0:  # a snapshot load writes record peaks directly
            s = int(np.flatnonzero(a._state == 1)[0])
            for pool in (a, b):
                pool.record_for_slot(s).peak_population = 1000
        assert np.array_equal(a._state, b._state) and np.array_equal(a._death, b._death)
        assert {k: (r.peak_population, r.death_step) for k, r in a.records.items()} == \
               {k: (r.peak_population, r.death_step) for k, r in b.records.items()}
