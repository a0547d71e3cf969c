"""Reference snapshot fixture, produced by the REFERENCE.

Run in the build container only (imports /root/reference/pkg/src):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden_snapshot.py

Builds a small world with the reference new_state (hidden 16, default
radiation probabilities so the pool holds live, dead and re-admitted slots),
runs 25 reference steps and writes the reference save_snapshot bytes to
snapshot_ref.crls.
"""

import os
import sys

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from evoca import config as rcfg  # noqa: E402
from evoca import engine as reng  # noqa: E402
from evoca.snapshot import save_snapshot  # noqa: E402


def main():
    cfg = rcfg.ExperimentConfig(grid=rcfg.GridConfig(16, 12), seed=7, initial_population=8)
    cfg.evolution.p_radiation = 0.05
    cfg.validate()
    st = reng.new_state(cfg)
    reng.run(st, 25)
    save_snapshot(st, os.path.join(HERE, "snapshot_ref.crls"))
    states = [s.state for s in st.pool.slots if s.state != "free"]
    print("t", st.t, "slots", {k: states.count(k) for k in set(states)}, "records", len(st.pool.records))


if __name__ == "__main__":
    main()
