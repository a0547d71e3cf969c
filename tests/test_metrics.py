"""Observables (metrics.py): multi-scale complexity and census totals, on the
host and on the device, against the reference's own values
(tests/golden/new_state_cases.npz, tests/golden/make_golden_new_state.py)."""

import os

import numpy as np
import pytest

from paper_2406_09654_b200 import metrics
from paper_2406_09654_b200.substrate import create_substrate

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "new_state_cases.npz"))
KS = sorted({k.split("_")[0] for k in GOLD.files if k.startswith("msc") and k.endswith("_sums")})
PLANES = [("energy", 0), ("infrastructure", 0), ("communication", 1)]


def _sub(k):
    E = GOLD[f"{k}_E"]
    h, w = E.shape
    sub = create_substrate(w, h)
    sub.front.channels["energy"][0] = E
    sub.front.channels["infrastructure"][0] = GOLD[f"{k}_I"]
    sub.front.channels["communication"][:] = GOLD[f"{k}_C"]
    return sub


def _check(rep, want):
    got = np.array(list(rep.contributions) + [rep.total, rep.side])
    assert got.shape == want.shape and np.array_equal(got, want), (got, want)


@pytest.mark.parametrize("k", KS)
def test_msc_host_matches_reference(k):
    sub = _sub(k)
    for name, sb in PLANES:
        _check(metrics.msc_of_substrate(sub, name, sb), GOLD[f"{k}_{name}{sb}"])
    E = GOLD[f"{k}_E"]
    side = GOLD[f"{k}_energy0"][-1].astype(int)
    _check(metrics.msc(E[:side, :side], n_scales=2), GOLD[f"{k}_E_n2"])


@pytest.mark.parametrize("k", KS)
def test_census_host_matches_reference(k):
    from paper_2406_09654_b200.pool import SlotPool

    row = metrics.census(_sub(k), SlotPool(4))
    assert [row.total_energy, row.total_infrastructure] == list(GOLD[f"{k}_sums"])


def test_msc_errors():
    with pytest.raises(ValueError, match="square"):
        metrics.msc(np.zeros((4, 8)))
    with pytest.raises(ValueError, match="power of two"):
        metrics.msc(np.zeros((6, 6)))
    with pytest.raises(ValueError, match="n_scales"):
        metrics.msc(np.zeros((4, 4)), n_scales=0)


@pytest.mark.gpu
@pytest.mark.parametrize("k", KS)
def test_msc_and_sums_device_match_reference(k):
    import ctypes as C

    from paper_2406_09654_b200.device import DeviceSubstrate

    sub = _sub(k)
    dev = DeviceSubstrate(sub.width, sub.height, 4)
    dev.upload(sub.front)
    for name, sb in PLANES:
        _check(metrics.msc_device(dev, name, sb), GOLD[f"{k}_{name}{sb}"])
    e, i = C.c_double(), C.c_double()
    dev.lib.evo_plane_sums(dev.ctx, C.byref(e), C.byref(i))
    assert [e.value, i.value] == list(GOLD[f"{k}_sums"])
    dev.close()


@pytest.mark.gpu
def test_msc_and_sums_device_match_host_large():
    """Device exact sums vs the host fsum restatement on a 256^2 crop of a
    non-square grid with mixed-sign, wide-range values; numpy-order totals
    on a 1000 x 1100 grid (chunk tails, pairwise splits)."""
    import ctypes as C

    from paper_2406_09654_b200.device import DeviceSubstrate

    g = np.random.default_rng(9)
    sub = create_substrate(300, 260)
    sub.front.channels["energy"][0] = (np.exp(g.standard_normal((260, 300)) * 8) *
                                       np.sign(g.standard_normal((260, 300)))).astype(np.float32)
    sub.front.channels["communication"][:] = g.standard_normal((3, 260, 300)).astype(np.float32)
    dev = DeviceSubstrate(300, 260, 4)
    dev.upload(sub.front)
    for name, sb in (("energy", 0), ("communication", 2)):
        a, b = metrics.msc_device(dev, name, sb), metrics.msc_of_substrate(sub, name, sb)
        assert a == b
    a = metrics.msc_device(dev, "energy", 0, n_scales=3)
    b = metrics.msc(sub.front.channels["energy"][0][2:258, 22:278], n_scales=3)
    assert (a.contributions, a.total, a.side) == (b.contributions, b.total, b.side)
    dev.close()
    big = create_substrate(1100, 1000)
    big.front.channels["energy"][0] = np.exp(g.standard_normal((1000, 1100)) * 6).astype(np.float32)
    big.front.channels["infrastructure"][0] = g.random((1000, 1100), dtype=np.float32)
    dev = DeviceSubstrate(1100, 1000, 4)
    dev.upload(big.front)
    e, i = C.c_double(), C.c_double()
    dev.lib.evo_plane_sums(dev.ctx, C.byref(e), C.byref(i))
    assert e.value == float(big.front.channels["energy"][0].sum(dtype=np.float64))
    assert i.value == float(big.front.channels["infrastructure"][0].sum(dtype=np.float64))
    dev.close()


@pytest.mark.gpu
def test_device_hook_observables_match_host():
    from paper_2406_09654_b200 import engine

    cfg = engine.ExperimentConfig(grid=engine.GridConfig(96, 80), initial_population=60, seed=2)
    st = engine.new_state(cfg)
    seen = {}

    def probe(s):
        seen["msc"] = metrics.msc_of_substrate(s)
        seen["census"] = metrics.census(s)

    engine.run(st, 5, hooks=[engine.Hook(5, probe, device=True)])
    assert seen["msc"] == metrics.msc_of_substrate(st.substrate)
    assert seen["census"] == metrics.census(st.substrate, st.pool)
