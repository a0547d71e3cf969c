"""The native host NEAT of the radiation feed (csrc/evoca_neat.cpp) against
this package's Python restatement of the reference's ``mutate``
(neuroevo.py:233-299; itself pinned to reference-generated children in
tests/test_cppn_cpu.py) and program linearisation (compile_programs_py,
pinned to the CPPN oracle).  Host-only functions of the library: no GPU."""

import numpy as np
import pytest

from paper_2406_09654_b200 import neat, synth


def _lineage(n_parents, rounds, rates, seed=3):
    """Parents plus a few generations of children (sequential Python mutate),
    so structural mutations (added nodes / connections) appear."""
    gs, ctr = synth.synth_genomes(n_parents, seed)
    pool = list(gs)
    for r in range(rounds):
        pool += [neat.mutate(g, rates, neat.stream(seed, 100 + r, "mutate", i), ctr) for i, g in enumerate(pool)]
    return pool, ctr


@pytest.mark.parametrize("rates", [neat.EvolutionRates(),
                                   neat.EvolutionRates(add_connection_prob=0.6, add_node_prob=0.5,
                                                       toggle_enable_prob=0.2, weight_reset_prob=0.3)])
def test_mutate_batch_equals_python_mutate(rates):
    wild = neat.EvolutionRates(add_connection_prob=0.5, add_node_prob=0.4, toggle_enable_prob=0.1)
    parents, ctr = _lineage(24, 3, wild)
    c_py = neat.InnovationCounter(ctr.next_innovation, ctr.next_node_id)
    c_nat = neat.InnovationCounter(ctr.next_innovation, ctr.next_node_id)
    keys = [neat.stream_key(7, 50, "mutate", i) for i in range(len(parents))]
    want = [neat.mutate(g, rates, neat.stream(7, 50, "mutate", i), c_py) for i, g in enumerate(parents)]
    got = neat.mutate_batch(parents, rates, keys, c_nat)
    assert (c_nat.next_innovation, c_nat.next_node_id) == (c_py.next_innovation, c_py.next_node_id)
    assert len(got) == len(want)
    for a, b in zip(got, want):
        assert a == b and b == a
        assert hash(a) == hash(b)
    # children of packed children (the next radiation event mutates them)
    want2 = [neat.mutate(g, rates, neat.stream(7, 100, "mutate", i), c_py) for i, g in enumerate(want)]
    got2 = neat.mutate_batch(got, rates, [neat.stream_key(7, 100, "mutate", i) for i in range(len(got))], c_nat)
    assert all(a == b for a, b in zip(got2, want2))


def test_native_compile_equals_python_layout():
    wild = neat.EvolutionRates(add_connection_prob=0.5, add_node_prob=0.4, toggle_enable_prob=0.1)
    genomes, _ = _lineage(16, 3, wild)
    genomes.append(neat.init_genome(np.random.default_rng(4), neat.InnovationCounter()))
    got = neat.compile_programs(genomes)
    want = neat.compile_programs_py(genomes)
    for a, b in zip(got, want):
        assert a.dtype == b.dtype and np.array_equal(a, b)


def test_native_normal_draws_match_numpy():
    """mutate's perturbations are numpy normal draws: with reset off and
    perturb always on, every weight moves by exactly normal(0, sigma) of the
    genome's stream (slow ziggurat paths included over ~60k draws)."""
    rates = neat.EvolutionRates(weight_perturb_prob=1.0, weight_reset_prob=0.0, add_connection_prob=0.0,
                                add_node_prob=0.0, toggle_enable_prob=0.0, weight_perturb_sigma=0.7)
    g = neat.CppnGenome(tuple(neat.NodeGene(i, "input", "identity") for i in range(5))
                        + (neat.NodeGene(5, "output", "tanh"), neat.NodeGene(6, "output", "tanh")),
                        tuple(neat.ConnGene(i, i % 5, 5 + (i // 5) % 2, 0.0, True) for i in range(10)))
    n = 3000
    kids = neat.mutate_batch([g] * n, rates, [neat.stream_key(1, 2, "mutate", i) for i in range(n)],
                             neat.InnovationCounter(10, 7))
    for i in range(0, n, 7):
        rng = neat.stream(1, 2, "mutate", i)
        want = []
        for _ in range(10):
            rng.random()
            rng.random()
            want.append(0.0 + rng.normal(0.0, 0.7))
        assert [c.weight for c in kids[i].connections] == want


def test_deferred_numbering_equals_mutate_batch_on_subsets():
    """A radiation event's host draws are made for every live slot before
    the selection is known (evo_neat_mutate_deferred) and numbered for the
    admitted ones afterwards: equal to mutate_batch over those parents
    alone, children and compiled programs alike."""
    wild = neat.EvolutionRates(add_connection_prob=0.5, add_node_prob=0.4, toggle_enable_prob=0.1)
    parents, ctr = _lineage(20, 3, wild)
    keys = [neat.stream_key(9, 150, "mutate", i) for i in range(len(parents))]
    deferred = neat.mutate_batch_deferred(parents, wild, keys)
    progs = neat.compile_programs(deferred)
    rng = np.random.default_rng(5)
    for take in (np.arange(len(parents)), np.sort(rng.choice(len(parents), 37, replace=False)), np.array([3]),
                 np.array([], np.int64)):
        c_ref = neat.InnovationCounter(ctr.next_innovation, ctr.next_node_id)
        c_def = neat.InnovationCounter(ctr.next_innovation, ctr.next_node_id)
        want = neat.mutate_batch([parents[i] for i in take], wild, [keys[i] for i in take], c_ref)
        got = neat.number_deferred([deferred[i] for i in take], c_def)
        assert (c_def.next_innovation, c_def.next_node_id) == (c_ref.next_innovation, c_ref.next_node_id)
        assert len(got) == len(want) and all(a == b for a, b in zip(got, want))
        if len(take):
            for a, b in zip(neat.subset_programs(progs, take), neat.compile_programs(want)):
                assert a.dtype == b.dtype and np.array_equal(a, b)
