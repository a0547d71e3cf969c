"""evo_step_host: one step of host-resident planes pipelined over row bands
(upload band b+1 while pass 1 runs on band b, download each band once its
pass 2 is done).  Every band count must reproduce the whole-grid device step
(upload + evo_step + download) bit for bit: planes, census, statistics and
adoption events, for the tile kernel, the genome-sorted rows path and the
tensor-core hidden net, on torus heights that do and do not divide into
32-row tiles."""

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2406_09654_b200 import _lib, physics
from tests.test_gpu_parity import download, make_dev

pytestmark = pytest.mark.gpu


def _empty(h, w):
    return orc.Planes(np.empty((h, w), np.float32), np.empty((h, w), np.float32), np.empty((3, h, w), np.float32),
                      np.empty((h, w), np.int32), np.empty((h, w), np.uint8))


def _run_pair(p0, cap, net, bands, steps, flags=0, source_map=None, live=None):
    ref = make_dev(p0, cap, net, live=live)
    dev = make_dev(p0, cap, net, live=live)
    params = physics.PhysicsParams(cycle_period=20, explore_fraction=0.8)
    cur = p0
    for t in range(steps):
        sc = physics.step_scalars(t, params)
        ref.step_raw(sc, t, flags=flags, source_map=source_map)
        out = _empty(*p0.shape)
        counts, adopt, ext = dev.step_host(cur, out, sc, t, flags=flags, bands=bands, source_map=source_map)
        want = download(ref)
        assert out.equal(want), f"bands={bands} t={t}"
        a_ref, e_ref = ref.read_stats()
        assert (adopt, ext) == (a_ref, e_ref), f"bands={bands} t={t}"
        if flags & _lib.F_NO_CENSUS:
            assert counts is None
            ev_ref, ev = ref.read_events(), dev.read_events()
            for f in ("target", "source", "winner_slot", "defender_slot", "direction", "quantity"):
                assert np.array_equal(getattr(ev, f), getattr(ev_ref, f)), f
            ref.census_finish(t)
            dev.census_finish(t)
        else:
            c_ref, s_ref, d_ref, pk_ref = ref.read_census()
            assert np.array_equal(counts, c_ref)
            c2, s2, d2, pk2 = dev.read_census()
            assert np.array_equal(s2, s_ref) and np.array_equal(d2, d_ref) and np.array_equal(pk2, pk_ref)
        # the device copy of the new state is current too
        assert download(dev).equal(want)
        cur = out
    ref.close()
    dev.close()


@pytest.mark.parametrize("bands", [1, 2, 3, 5, 8, 0])
@pytest.mark.parametrize("shape", [(64, 64), (100, 70), (257, 96)])
def test_step_host_direct_tile_kernel(shape, bands):
    H, W = shape
    p0 = orc.synth_planes(H, W, 8, seed=H + bands)
    p0.I[np.random.default_rng(3).random((H, W)) < 0.3] = 0
    _run_pair(p0, 8, orc.synth_net(8, 0, seed=5), bands, steps=4)


@pytest.mark.parametrize("bands", [1, 4, 0])
def test_step_host_c2_size(bands):
    p0 = orc.synth_planes(1024, 1024, 64, seed=11)
    _run_pair(p0, 64, orc.synth_net(64, 0, seed=12), bands, steps=2)


@pytest.mark.parametrize("bands", [2, 3])
def test_step_host_genome_sorted_rows(bands):
    """cap > 68: the direct net through the genome-sorted rows path per band."""
    H, W = 160, 96
    p0 = orc.synth_planes(H, W, 100, seed=bands)
    _run_pair(p0, 100, orc.synth_net(100, 0, seed=6), bands, steps=3)


@pytest.mark.parametrize("bands", [2, 4])
def test_step_host_tensor_core_hidden(bands):
    H, W = 128, 64
    p0 = orc.synth_planes(H, W, 24, seed=bands, sparse_infra=True)
    _run_pair(p0, 24, orc.synth_net(24, 128, seed=4), bands, steps=2)


def test_step_host_events_and_source_map():
    """Host-radiation flags (events recorded, census deferred) and an energy
    source map, band-offset like the planes."""
    H, W = 130, 64
    p0 = orc.synth_planes(H, W, 8, seed=21)
    src = np.random.default_rng(2).random((H, W)).astype(np.float32)
    _run_pair(p0, 8, orc.synth_net(8, 0, seed=7), 3, steps=3,
              flags=_lib.F_RECORD_EVENTS | _lib.F_NO_CENSUS, source_map=src)


def test_step_host_dead_slots_census():
    H, W = 96, 96
    p0 = orc.synth_planes(H, W, 8, seed=8)
    _run_pair(p0, 8, orc.synth_net(8, 0, seed=9), 3, steps=3, live=5)


def test_step_host_rejects_out_of_range_planes():
    H, W = 64, 64
    p0 = orc.synth_planes(H, W, 8, seed=1)
    dev = make_dev(p0, 8, orc.synth_net(8, 0, seed=2))
    sc = physics.step_scalars(0, physics.PhysicsParams())
    bad = orc.Planes(p0.E, p0.I, p0.C, p0.gi.copy(), p0.rot)
    bad.gi[40, 3] = 8
    with pytest.raises(ValueError, match="genome_index"):
        dev.step_host(bad, _empty(H, W), sc, 0, bands=2)
    bad = orc.Planes(p0.E, p0.I, p0.C, p0.gi, p0.rot.copy())
    bad.rot[0, 0] = 9
    with pytest.raises(ValueError, match="rotation"):
        dev.step_host(bad, _empty(H, W), sc, 0, bands=2)
    # the context is still usable and matches a fresh step
    out = _empty(H, W)
    dev.step_host(p0, out, sc, 0, bands=2)
    ref = make_dev(p0, 8, orc.synth_net(8, 0, seed=2))
    ref.step_raw(sc, 0)
    assert out.equal(download(ref))
    ref.close()
    dev.close()


def _planeset(p):
    from paper_2406_09654_b200.substrate import STANDARD_CHANNELS, PlaneSet

    h, w = p.shape
    ps = PlaneSet(STANDARD_CHANNELS, h, w)
    ps.channels["energy"][0] = p.E
    ps.channels["infrastructure"][0] = p.I
    ps.channels["communication"][...] = p.C
    ps.genome_index[...] = p.gi
    ps.rotation[...] = p.rot
    return ps


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("bands", [1, 3, 4])
def test_step_host_block_layout(bands, pinned):
    """This package's PlaneSet (one host block, equally spaced 4-byte planes):
    one 2-D copy per band each way; pinned or pageable."""
    H, W = 200, 128
    p0 = orc.synth_planes(H, W, 8, seed=30 + bands)
    net = orc.synth_net(8, 0, seed=31)
    ref = make_dev(p0, 8, net)
    dev = make_dev(p0, 8, net)
    a, b = _planeset(p0), _planeset(p0)
    if pinned:
        dev.pin(a)
        dev.pin(b)
    params = physics.PhysicsParams(cycle_period=20)
    for t in range(3):
        sc = physics.step_scalars(t, params)
        ref.step_raw(sc, t)
        dev.step_host(a, b, sc, t, bands=bands)
        want = download(ref)
        got = orc.Planes(b.channels["energy"][0], b.channels["infrastructure"][0], b.channels["communication"],
                         b.genome_index, b.rotation)
        assert got.equal(want), f"t={t}"
        a, b = b, a
    ref.close()
    dev.close()
