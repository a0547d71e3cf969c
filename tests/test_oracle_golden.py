"""Pin the CPU oracle to the reference: every golden vector produced by
running the reference (tests/golden/make_golden.py) must be reproduced
bit-exactly (integer/physics) or within the reference's own 1e-6
forward-pass band."""

import numpy as np
import pytest

from oracle import oracle as orc
from tests import _cases as C


def _physics(case):
    p = case["pre"].copy()
    ev = orc.physics(p, case["acts"], case["t"], case["phys"])
    return p, ev


@pytest.mark.parametrize("c", range(40))
def test_physics_cases_bit_exact(c):
    z = C.load("physics_cases.npz")
    case = C.physics_case(z, c)
    p, ev = _physics(case)
    assert p.equal(case["post"])
    assert C.events_rows(ev) == case["events"]
    assert np.array_equal(orc.census(p.gi, 12), case["counts"])


def test_explore_cases_bit_exact():
    z = C.load("explore_cases.npz")
    for c in range(int(z["n_cases"])):
        key = f"c{c:02d}_"
        p = C.planes(z, key, "pre")
        cells = z[key + "cells"]
        a = np.zeros((len(cells), 13), np.float32)
        a[:, 5:] = z[key + "explore"]
        ev = orc.explore(p, orc.Actions(cells, a), orc.Phys(explore_fraction=float(z[key + "alpha"])))
        assert np.array_equal(p.I.view(np.uint32), z[key + "post_I"].view(np.uint32))
        assert np.array_equal(p.gi, z[key + "post_gi"])
        assert np.array_equal(p.rot, z[key + "post_rot"])
        assert C.events_rows(ev) == [tuple(r) for r in z[key + "events"].tolist()]


def test_forward_within_reference_band():
    z = C.load("forward_cases.npz")
    for c in range(int(z["n_cases"])):
        k = f"c{c}_"
        net = orc.Net(z[k + "w1"].shape[0], z[k + "w2"][None], z[k + "b2"][None], z[k + "w1"][None], z[k + "b1"][None])
        y = orc.forward(net, 0, z[k + "s"])
        ref = z[k + "y"]
        assert np.abs(y - ref).max() < 1e-6
        assert ((y > 0) & (y < 1)).all()


@pytest.mark.parametrize("name,hidden", [("step_hidden.npz", 16), ("step_direct.npz", 0)])
def test_full_step_tiers(name, hidden):
    """Tier A: reference actions injected -> bit-exact post-state.
    Tier B: oracle actions vs reference actions <= 1e-5 relative.
    Sensing is a pure copy and is checked via the actions."""
    z = C.load(name)
    if hidden:
        net = C.step_net(z, hidden)
    else:
        net = orc.synth_net(8, hidden=0, seed=0)
    phys = orc.Phys(cycle_period=20)
    for k in z["keep"].tolist():
        key = f"s{k:03d}_"
        pre = C.planes(z, key, "pre")
        post = C.planes(z, key, "post")
        ref_acts = orc.Actions(z[key + "cells"], z[key + "acts"])
        res = orc.step(pre, k, net, phys, acts=ref_acts)
        assert res.planes.equal(post), f"step {k}"
        assert len(res.events) == int(z[key + "adoptions"])
        assert np.array_equal(res.counts, z[key + "counts"])
        mine = orc.act(pre, net)
        assert np.array_equal(mine.cells, ref_acts.cells)
        rel = np.abs(mine.a - ref_acts.a) / np.maximum(np.abs(ref_acts.a), 1e-30)
        assert rel.max() <= 1e-5


def close(a, b, tol=1e-5):
    """Continuous-channel tolerance used throughout: |a-b| <= tol*max(|b|,1)
    (1e-5 relative, with a unit floor so that cancellation near zero in
    E - cost does not turn an ulp into a large relative error)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return bool(np.all(np.abs(a - b) <= tol * np.maximum(np.abs(b), 1.0)))


def test_direct_run_free_running():
    """Tier D on config 1 (64x64, 8 genomes, direct net, 100 steps): the
    oracle free-running from the reference's initial state keeps the
    integer state (genome, rotation) bit-identical to the reference at
    every recorded step and the continuous channels within tolerance.
    (Digests cannot agree: the reference's sgemm bits are unpinned.)"""
    z = C.load("step_direct.npz")
    p = C.planes(z, "s000_", "pre")
    net = orc.synth_net(8, hidden=0, seed=0)
    phys = orc.Phys(cycle_period=20)
    keep = set(z["keep"].tolist())
    for t in range(100):
        p = orc.step(p, t, net, phys).planes
        if t in keep:
            post = C.planes(z, f"s{t:03d}_", "post")
            assert np.array_equal(p.gi, post.gi), t
            assert np.array_equal(p.rot, post.rot), t
            for a, b in ((p.E, post.E), (p.I, post.I), (p.C, post.C)):
                assert close(a, b), t


def test_digest_matches_reference_definition():
    z = C.load("step_direct.npz")
    p = C.planes(z, "s000_", "post")
    assert orc.digest(p) == int(z["digest"][0])


def test_rho_night_at_full_period():
    # physics.py:186: rho computed in float64; sin(2*pi) is -2.4e-16 -> night.
    mode, _, drain = orc.rho_terms(20, orc.Phys(cycle_period=20))
    assert mode == 2 and drain > 0
    assert orc.rho_terms(0, orc.Phys(cycle_period=20))[0] == 0
