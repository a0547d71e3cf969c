"""Loaders for the committed golden fixtures (tests/golden/*.npz)."""

import os

import numpy as np

from oracle import oracle as orc

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def planes(z, key, which):
    return orc.Planes(
        z[f"{key}{which}_E"].copy(), z[f"{key}{which}_I"].copy(), z[f"{key}{which}_C"].copy(),
        z[f"{key}{which}_gi"].copy(), z[f"{key}{which}_rot"].copy(),
    )


def phys_from(z, key):
    vals = z[key + "phys"]
    names = [str(s) for s in z["phys_fields"]]
    kw = dict(zip(names, vals.tolist()))
    kw["cycle_period"] = int(kw["cycle_period"])
    return orc.Phys(**kw)


def physics_case(z, c):
    key = f"c{c:02d}_"
    return dict(
        pre=planes(z, key, "pre"),
        post=planes(z, key, "post"),
        acts=orc.Actions(z[key + "cells"], z[key + "acts"]),
        t=int(z[key + "t"]),
        phys=phys_from(z, key),
        events=[tuple(r) for r in z[key + "events"].tolist()],
        counts=z[key + "counts"],
    )


def events_rows(ev):
    return [(float(t), float(s), float(w), float(d), float(r), float(q)) for t, s, w, d, r, q in ev.rows()]


def step_net(z, hidden, genomes=8):
    if hidden == 0:
        return None
    w1 = np.stack([z[f"w1_{i}"] for i in range(genomes)])
    b1 = np.stack([z[f"b1_{i}"] for i in range(genomes)])
    w2 = np.stack([z[f"w2_{i}"] for i in range(genomes)])
    b2 = np.stack([z[f"b2_{i}"] for i in range(genomes)])
    return orc.Net(hidden, w2, b2, w1, b1)
