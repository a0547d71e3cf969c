"""CPU checks of the CPPN path: the oracle and the host NEAT restatement
against reference-produced golden vectors (tests/golden/make_golden_cppn.py),
and the program linearisation that feeds evo_express_cppn."""

import numpy as np
import pytest

from oracle import cppn as ocppn
from paper_2406_09654_b200 import neat
from tests import _cases


@pytest.fixture(scope="module")
def golden():
    genomes, doc = _cases.cppn_genomes()
    return genomes, doc, _cases.load("cppn_cases.npz")


def test_oracle_dense_h16_bit_exact(golden):
    genomes, doc, z = golden
    for i, g in enumerate(genomes):
        w1, b1, w2, b2 = ocppn.generate_dense(g, 16, doc["tau"], doc["w_max"])
        for name, v in (("w1", w1), ("b1", b1), ("w2", w2), ("b2", b2)):
            np.testing.assert_array_equal(v.view(np.uint32), z[f"h16_{name}_{i}"].view(np.uint32), err_msg=f"{name} {i}")


def test_oracle_dense_h128_bit_exact(golden):
    genomes, doc, z = golden
    n = 0
    for i, g in enumerate(genomes):
        if f"h128_w1_{i}" not in z:
            continue
        w1, b1, w2, b2 = ocppn.generate_dense(g, 128, doc["tau"], doc["w_max"])
        for name, v in (("w1", w1), ("b1", b1), ("w2", w2), ("b2", b2)):
            np.testing.assert_array_equal(v.view(np.uint32), z[f"h128_{name}_{i}"].view(np.uint32))
        n += 1
    assert n >= 5


def test_oracle_direct_block_bit_exact(golden):
    genomes, doc, z = golden
    nonzero = 0
    for i, g in enumerate(genomes):
        w, b = ocppn.generate_direct(g, doc["tau"], doc["w_max"])
        np.testing.assert_array_equal(w.view(np.uint32), z[f"direct_w_{i}"].view(np.uint32))
        np.testing.assert_array_equal(b.view(np.uint32), z[f"direct_b_{i}"].view(np.uint32))
        nonzero += int(np.count_nonzero(w))
    assert nonzero > 1000  # the fixtures express real weights, not just thresholded zeros


def test_topo_order_matches_reference(golden):
    genomes, doc, _ = golden
    for g, d in zip(genomes, doc["genomes"]):
        assert neat.topo_order(g) == d["topo"]


def test_mutate_matches_reference(golden):
    genomes, doc, _ = golden
    rates = {k: neat.EvolutionRates(**{f: v[f] for f in neat.EvolutionRates.__dataclass_fields__})
             for k, v in doc["rates"].items()}
    assert len(doc["mutate_cases"]) >= 20
    for case in doc["mutate_cases"]:
        counter = neat.InnovationCounter(*case["counter_before"])
        seed, step, purpose, index = case["key"]
        child = neat.mutate(genomes[case["parent"]], rates[case["rates"]], neat.stream(seed, step, purpose, index),
                            counter)
        want = _cases.genome_from_json(case["child"])
        assert child == want
        assert (counter.next_innovation, counter.next_node_id) == tuple(case["counter_after"])


def test_program_linearisation_reproduces_oracle(golden):
    genomes, doc, _ = golden
    prog = neat.compile_programs(genomes)
    inp, _, out = ocppn.make_layout(0)
    rng = np.random.default_rng(5)
    q = np.column_stack([rng.uniform(-1, 1, (64, 4)), np.ones(64)])
    for i, g in enumerate(genomes):
        np.testing.assert_array_equal(_cases.run_program(prog, i, q), ocppn.evaluate_batch(g, q))


def test_stream_matches_reference_derivation():
    # rng.py:19-33 pins the derivation; two equal tuples give equal streams,
    # distinct purposes differ
    a = neat.stream(3, 9, "mutate", 4).random(4)
    b = neat.stream(3, 9, "mutate", 4).random(4)
    c = neat.stream(3, 9, "merge", 4).random(4)
    np.testing.assert_array_equal(a, b)
    assert not np.array_equal(a, c)


def test_c3_genome_topology():
    g = neat.init_c3_genome(np.random.default_rng(0), neat.InnovationCounter())
    hidden = [n for n in g.nodes if n.role == "hidden"]
    assert len(hidden) == 8 and {n.activation for n in hidden} == {"sine", "gaussian", "tanh"}
    assert all(c.src in (0, 1, 2, 3) for c in g.connections if c.dst in {n.id for n in hidden})
    w, b = ocppn.generate_direct(g)
    assert np.all(b == 0)  # bias output unconnected: tanh(0) = 0
    assert np.count_nonzero(w) > 0
