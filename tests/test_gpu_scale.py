"""Parity at the BASELINE sizes the benchmark runs (SURVEY.md §8c, §0 hazard 5).

* Config 3 at full size (4096x4096, 256 genomes, pool capacity 2048: the
  genome-sorted large-pool path): two steps in tier A against the oracle
  with the device's exported actions; the benchmark's non-export variant
  bit-identical to the export variant.
* Config 2 at full size: the non-export tile kernel (the benchmarked
  ``k_pass1_direct<0,1>``) bit-identical to the export variant, three steps.
* Windowed oracle for grids the CPU oracle cannot step whole: the step's
  dependency radius is 2, so a window with a 2-cell apron stepped toroidally
  by the oracle reproduces the full grid's interior bit for bit, given the
  actions of the window's cells.  Those actions come from a second, small
  device context holding the window with a 3-cell apron (per-cell forward
  arithmetic does not depend on the rest of the grid; cells 1+ away from its
  border see their true neighbourhoods).  Config 4 at full size (16384x16384,
  1024 genomes) and a config-5 slice (4096x32768 torus, 45->128->13,
  4096 genomes, 90 % of cells without infrastructure), windows in the middle
  and across both torus seams."""

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2406_09654_b200 import _lib, physics
from paper_2406_09654_b200.device import DeviceSubstrate
from tests.test_gpu_parity import download, events_rows, make_dev, net_params, oracle_phys_to_params, rel_err

pytestmark = pytest.mark.gpu

TOL = 1e-5


def test_config3_full_size_tier_a():
    h = w = 4096
    genomes, cap = 256, 2048
    p0 = orc.synth_planes(h, w, genomes, seed=0)
    net = orc.synth_net(genomes, 0, seed=0)
    phys = orc.Phys(cycle_period=20)
    params = oracle_phys_to_params(phys)
    dev = make_dev(p0, cap, net, live=genomes)
    fast = make_dev(p0, cap, net, live=genomes)  # the benchmark's variant (decided rows, no export)
    rows = make_dev(p0, cap, net, live=genomes)  # sensor rows through HBM (EVO_F_ROWS_NET)
    p = p0
    for t in range(2):
        sc = physics.step_scalars(t, params)
        dev.step_raw(sc, t, flags=_lib.F_EXPORT_ACTIONS | _lib.F_RECORD_EVENTS)
        fast.step_raw(sc, t)
        rows.step_raw(sc, t, flags=_lib.F_ROWS_NET)
        cells, acts = dev.get_actions()
        ref = orc.step(p, t, net, phys, acts=orc.Actions(cells, acts))
        got = download(dev)
        assert got.equal(ref.planes), f"t={t}"
        assert download(fast).equal(got), f"t={t}"
        assert download(rows).equal(got), f"t={t}"
        assert events_rows(dev.read_events()) == [tuple(map(float, r)) for r in ref.events.rows()], f"t={t}"
        counts = dev.read_census()[0]
        assert np.array_equal(counts[:genomes], ref.counts[:genomes]) and not counts[genomes:].any()
        oa = orc.act(p, net)
        assert np.array_equal(oa.cells, cells)
        assert rel_err(acts, oa.a) <= TOL, f"t={t}"
        p = got
    # the steady state of a run: six steps as one evo_run (CUDA graph; the E, I,
    # C state stays in the sense texture between the steps) against six
    # unfused steps, at full size
    scs = [physics.step_scalars(2 + i, params) for i in range(6)]
    fast.run(scs, 2)
    for i in range(6):
        rows.step_raw(scs[i], 2 + i, flags=_lib.F_UNFUSED)
    assert fast.read_stats() == rows.read_stats()
    assert np.array_equal(fast.read_census()[0], rows.read_census()[0])
    assert download(fast).equal(download(rows))
    dev.close()
    fast.close()
    rows.close()


def test_config2_nonexport_kernel_equals_export():
    p0 = orc.synth_planes(1024, 1024, 64, seed=0)
    net = orc.synth_net(64, 0, seed=0)
    params = physics.PhysicsParams(cycle_period=20)
    a, b = make_dev(p0, 64, net), make_dev(p0, 64, net)
    for t in range(3):
        sc = physics.step_scalars(t, params)
        a.step_raw(sc, t)  # k_pass1_direct<0,1>: the benchmarked kernel
        b.step_raw(sc, t, flags=_lib.F_EXPORT_ACTIONS)  # k_pass1_direct<1,1>
        assert download(a).equal(download(b)), f"t={t}"
        assert a.read_stats() == b.read_stats()
    a.close()
    b.close()


# -- windowed oracle ----------------------------------------------------------------------------


def _window(p: orc.Planes, y0: int, x0: int, n: int, apron: int) -> orc.Planes:
    h, w = p.shape
    ys = (np.arange(y0 - apron, y0 + n + apron) % h)[:, None]
    xs = (np.arange(x0 - apron, x0 + n + apron) % w)[None, :]
    c = np.ascontiguousarray
    return orc.Planes(c(p.E[ys, xs]), c(p.I[ys, xs]), c(p.C[:, ys, xs]), c(p.gi[ys, xs]), c(p.rot[ys, xs]))


def _window_actions(pre: orc.Planes, y0, x0, n, net, capacity, params, t):
    """Actions of the window + 2-cell apron from a small device context that
    holds the window + 3-cell apron (cells in oracle-window coordinates)."""
    wp = _window(pre, y0, x0, n, 3)
    m = n + 6
    dev = DeviceSubstrate(m, m, capacity, hidden=net.hidden)
    dev.set_params(net_params(net))
    dev.set_slots(np.ones(capacity, np.int8))
    dev.upload(wp)
    dev.step_raw(physics.step_scalars(t, params), t, flags=_lib.F_EXPORT_ACTIONS)
    cells, acts = dev.get_actions()
    dev.close()
    y, x = cells // m, cells % m
    keep = (y >= 1) & (y < m - 1) & (x >= 1) & (x < m - 1)
    return ((y[keep] - 1) * (n + 4) + (x[keep] - 1)).astype(np.int64), acts[keep]


def _windowed_check(h, w, genomes, hidden, sparse, windows, n=256, seed=0):
    pre = orc.synth_planes(h, w, genomes, seed=seed, sparse_infra=sparse)
    net = orc.synth_net(genomes, hidden, seed=seed)
    phys = orc.Phys(cycle_period=20)
    params = oracle_phys_to_params(phys)
    t = 1  # night step of a period-20 cycle starts at t = 11; t = 1 is a day step
    dev = make_dev(pre, genomes, net)
    dev.step_raw(physics.step_scalars(t, params), t)
    expected = []
    for (y0, x0) in windows:
        cells, acts = _window_actions(pre, y0, x0, n, net, genomes, params, t)
        win = _window(pre, y0, x0, n, 2)
        oa = orc.act(win, net)  # tier B where the toroidal window sees true neighbourhoods
        m = n + 4
        ok = lambda c: (c // m >= 1) & (c // m < m - 1) & (c % m >= 1) & (c % m < m - 1)  # noqa: E731
        assert np.array_equal(oa.cells[ok(oa.cells)], cells[ok(cells)])
        assert rel_err(acts[ok(cells)], oa.a[ok(oa.cells)]) <= TOL
        res = orc.step(win, t, net, phys, acts=orc.Actions(cells, acts))
        expected.append(_window(res.planes, 2, 2, n, 0))
    del pre
    post = orc.Planes(np.empty((h, w), np.float32), np.empty((h, w), np.float32), np.empty((3, h, w), np.float32),
                      np.empty((h, w), np.int32), np.empty((h, w), np.uint8))
    dev.download(post)
    dev.close()
    for (y0, x0), want in zip(windows, expected):
        got = _window(post, y0, x0, n, 0)
        assert got.equal(want), f"window at ({y0}, {x0})"


def test_config4_full_size_windowed_oracle():
    h = w = 16384
    _windowed_check(h, w, 1024, 0, False, [(8000, 8100), (h - 128, w - 100), (100, w - 128), (h - 100, 50)])


def test_config5_net_slice_windowed_oracle():
    h, w = 4096, 32768
    _windowed_check(h, w, 4096, 128, True, [(2000, 16000), (h - 128, w - 128), (10, 30000)])
