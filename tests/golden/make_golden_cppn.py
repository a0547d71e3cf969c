"""Golden vectors for the CPPN expression path, produced by the REFERENCE.

Run in the build container only (imports /root/reference/pkg/src):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_cppn.py

Writes
  cppn_genomes.json  genome structures (reference genome_to_json format plus
                     the reference topological order) and mutate cases
                     (parent, rates, stream key, counter before -> the
                     reference child and counter after);
  cppn_cases.npz     per genome: reference generate_network outputs at
                     hidden 16 (w1, b1, w2, b2) and, for the direct 45->13
                     block, reference evaluate_cppn_batch + _express on the
                     input->actuator queries (w, b); hidden-128 outputs for
                     a few genomes.
Genomes: reference init_genome, the BASELINE config-3 topology (built with
paper_2406_09654_b200.neat.init_c3_genome, converted to reference types),
and lineages grown with the reference mutate at high structural rates (all
six activations appear).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from evoca import hypernet, neuroevo  # noqa: E402
from evoca.rng import stream  # noqa: E402

from paper_2406_09654_b200 import neat  # noqa: E402


def to_ref(g):
    return neuroevo.CppnGenome(
        tuple(neuroevo.NodeGene(n.id, n.role, n.activation) for n in g.nodes),
        tuple(neuroevo.ConnGene(c.innovation, c.src, c.dst, float(c.weight), bool(c.enabled)) for c in g.connections))


def direct_block(g, tau=hypernet.DEFAULT_TAU, w_max=hypernet.DEFAULT_W_MAX):
    lay = hypernet.make_layout(1)
    inp, out = lay.input_coords, lay.output_coords
    d = np.repeat(out, len(inp), axis=0)
    s = np.tile(inp, (len(out), 1))
    q = np.vstack([np.column_stack([s, d, np.ones(len(d))]),
                   np.column_stack([np.zeros((13, 2)), out, np.ones(13)])])
    sig = hypernet.evaluate_cppn_batch(g, q)
    n = 13 * 45
    return (hypernet._express(sig[:n, 0], tau, w_max).reshape(13, 45), hypernet._express(sig[n:, 1], tau, w_max))


def main():
    rng = np.random.default_rng(2406)
    counter = neuroevo.InnovationCounter()
    genomes = []
    for _ in range(6):
        genomes.append(neuroevo.init_genome(rng, counter))
    c3c = neat.InnovationCounter(counter.next_innovation, counter.next_node_id)
    for _ in range(6):
        genomes.append(to_ref(neat.init_c3_genome(rng, c3c)))
    counter = neuroevo.InnovationCounter(c3c.next_innovation, c3c.next_node_id)
    wild = neuroevo.EvolutionRates(weight_perturb_prob=0.8, weight_perturb_sigma=0.7, weight_reset_prob=0.1,
                                   add_connection_prob=0.6, add_node_prob=0.5, toggle_enable_prob=0.08)
    for lin in range(4):
        g = genomes[lin * 2]
        for gen in range(24):
            g = neuroevo.mutate(g, wild, stream(7, gen, "golden-lineage", lin), counter)
            if gen % 4 == 3:
                genomes.append(g)
    # mutate cases: parents x rates x stream keys, reference children recorded
    cases = []
    rate_sets = {"default": neuroevo.EvolutionRates(), "wild": wild}
    for i, parent in enumerate(genomes[::3]):
        for rname, rates in rate_sets.items():
            before = (counter.next_innovation, counter.next_node_id)
            child = neuroevo.mutate(parent, rates, stream(11, i, "mutate", 50 + i), counter)
            cases.append({"parent": genomes.index(parent), "rates": rname, "key": [11, i, "mutate", 50 + i],
                          "counter_before": before, "counter_after": (counter.next_innovation, counter.next_node_id),
                          "child": neuroevo.genome_to_json(child)})
    acts = sorted({n.activation for g in genomes for n in g.nodes if n.role == "hidden"})
    print("genomes", len(genomes), "hidden activations present:", acts,
          "max nodes", max(len(g.nodes) for g in genomes))
    arrays = {}
    for i, g in enumerate(genomes):
        p = hypernet.generate_network(g, hypernet.make_layout(16))
        arrays[f"h16_w1_{i}"], arrays[f"h16_b1_{i}"] = p.w1, p.b1
        arrays[f"h16_w2_{i}"], arrays[f"h16_b2_{i}"] = p.w2, p.b2
        arrays[f"direct_w_{i}"], arrays[f"direct_b_{i}"] = direct_block(g)
        if i % 5 == 0:
            p = hypernet.generate_network(g, hypernet.make_layout(128))
            arrays[f"h128_w1_{i}"], arrays[f"h128_b1_{i}"] = p.w1, p.b1
            arrays[f"h128_w2_{i}"], arrays[f"h128_b2_{i}"] = p.w2, p.b2
    doc = {"genomes": [dict(neuroevo.genome_to_json(g), topo=hypernet._topo_order(g)) for g in genomes],
           "rates": {k: vars(v) for k, v in rate_sets.items()}, "mutate_cases": cases,
           "tau": hypernet.DEFAULT_TAU, "w_max": hypernet.DEFAULT_W_MAX}
    with open(os.path.join(HERE, "cppn_genomes.json"), "w") as f:
        json.dump(doc, f, indent=0)
    np.savez_compressed(os.path.join(HERE, "cppn_cases.npz"), **arrays)
    print("wrote cppn_genomes.json, cppn_cases.npz")


if __name__ == "__main__":
    main()
