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


# -- CPPN fixtures (tests/golden/make_golden_cppn.py) ----------------------------------


def cppn_doc():
    import json

    with open(os.path.join(GOLDEN, "cppn_genomes.json")) as f:
        return json.load(f)


def genome_from_json(d):
    from paper_2406_09654_b200 import neat

    nodes = tuple(neat.NodeGene(int(n["id"]), n["role"], n["act"]) for n in d["nodes"])
    conns = tuple(neat.ConnGene(int(c["innov"]), int(c["from"]), int(c["to"]), float(c["w"]), bool(c["on"]))
                  for c in d["conns"])
    return neat.CppnGenome(nodes, conns)


def cppn_genomes():
    doc = cppn_doc()
    return [genome_from_json(g) for g in doc["genomes"]], doc


def run_program(prog, gi, queries):
    """Evaluate genome ``gi`` of a compile_programs() batch exactly as the
    device kernel does (node records in order, edges summed as
    total = total + w * v starting from 0.0, float64 activations)."""
    node_off, nodes, esrc, ew, outs = prog
    acts = [np.sin, lambda x: np.exp(-np.square(x)), lambda x: 1.0 / (1.0 + np.exp(-x)), np.tanh,
            lambda x: x, np.abs]
    q = np.asarray(queries, np.float64)
    vals = []
    for r in nodes[node_off[gi]:node_off[gi + 1]]:
        act, ipos, b, e = (int(v) for v in r)
        if act < 0:
            vals.append(q[:, ipos])
            continue
        total = np.zeros(len(q))
        for k in range(b, e):
            total = total + ew[k] * vals[esrc[k]]
        vals.append(acts[act](total))
    return np.stack([vals[outs[gi, 0]], vals[outs[gi, 1]]], axis=1)
