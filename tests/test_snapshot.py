"""Snapshots in the reference's file format: a snapshot written by the
reference (tests/golden/snapshot_ref.crls, tests/golden/make_golden_snapshot.py)
loads here and saves back byte for byte; device-resident states save the
parameter bytes they ran on and resume on them."""

import os

import numpy as np
import pytest

from paper_2406_09654_b200 import engine, snapshot

REF = os.path.join(os.path.dirname(__file__), "golden", "snapshot_ref.crls")


def test_reference_snapshot_round_trips_bytewise(tmp_path):
    st = snapshot.load_snapshot(REF)
    assert st.t == 25 and st.substrate.width == 16 and st.substrate.height == 12
    assert st.config.evolution.p_radiation == 0.05 and st.master_seed == 7
    out = tmp_path / "again.crls"
    snapshot.save_snapshot(st, out)
    assert out.read_bytes() == open(REF, "rb").read()


def test_snapshot_errors(tmp_path):
    data = open(REF, "rb").read()
    bad = tmp_path / "bad.crls"
    bad.write_bytes(b"XXXX" + data[4:])
    with pytest.raises(snapshot.SnapshotError, match="magic"):
        snapshot.load_snapshot(bad)
    bad.write_bytes(data[:-10])
    with pytest.raises(snapshot.SnapshotError, match="truncated"):
        snapshot.load_snapshot(bad)
    bad.write_bytes(data[:4] + b"\x02\x00" + data[6:])
    with pytest.raises(snapshot.SnapshotError, match="version"):
        snapshot.load_snapshot(bad)


def test_config_round_trip():
    cfg = engine.ExperimentConfig(grid=engine.GridConfig(8, 8))
    assert engine.parse_config(engine.config_to_dict(cfg)) == cfg
    assert "field_radiation" not in engine.config_to_dict(cfg)
    cfg.field_radiation.every = 50
    assert engine.parse_config(engine.config_to_dict(cfg)).field_radiation.every == 50
    with pytest.raises(ValueError, match="unknown key"):
        engine.parse_config({"nope": 1})
    with pytest.raises(ValueError, match="integer"):
        engine.parse_config({"seed": 1.5})


@pytest.mark.gpu
def test_device_state_snapshot_resumes_exactly(tmp_path):
    """A device-resident world (seed networks expressed on the device, direct
    and hidden nets) saves its device parameter bytes; the loaded copy steps
    bit-identically to the original."""
    for hidden in (16, 0):
        cfg = engine.ExperimentConfig(grid=engine.GridConfig(48, 40), seed=3, initial_population=30,
                                      hypernet=engine.HypernetConfig(hidden_size=hidden))
        a = engine.new_state(cfg)
        engine.run(a, 4)
        path = tmp_path / f"w{hidden}.crls"
        snapshot.save_snapshot(a, path)
        b = snapshot.load_snapshot(path)
        assert engine.digest(b) == engine.digest(a)
        for s in range(30):
            pa, pb = a.pool.params(s), b.pool.params(s)
            for name in (("w1", "b1", "w2", "b2") if hidden else ("w", "b")):
                assert np.array_equal(getattr(pa, name), getattr(pb, name))
        engine.run(a, 3)
        engine.run(b, 3)
        assert engine.digest(a) == engine.digest(b) and a.t == b.t == 7
        snapshot.save_snapshot(b, tmp_path / "b2.crls")
        snapshot.save_snapshot(a, tmp_path / "a2.crls")
        assert (tmp_path / "b2.crls").read_bytes() == (tmp_path / "a2.crls").read_bytes()


@pytest.mark.gpu
def test_fresh_state_snapshot_at_step_zero(tmp_path):
    """A fresh new_state saves before its first step (the reference saves at
    step 0): the deferred seed networks are expressed on the device for the
    snapshot, and the loaded copy steps identically."""
    cfg = engine.ExperimentConfig(grid=engine.GridConfig(32, 24), seed=5, initial_population=12)
    a = engine.new_state(cfg)
    path = tmp_path / "fresh.crls"
    snapshot.save_snapshot(a, path)
    b = snapshot.load_snapshot(path)
    assert b.t == 0 and engine.digest(a) == engine.digest(b)
    for s in range(12):
        assert np.array_equal(a.pool.params(s).w1, b.pool.params(s).w1)
    engine.run(a, 3)
    engine.run(b, 3)
    assert engine.digest(a) == engine.digest(b)
