"""Batched CPPN expression on the device (evo_express_cppn) against the
reference's generate_network outputs (tests/golden/cppn_cases.npz) and the
oracle (oracle/cppn.py).

Bar: the float32 weight tables equal the reference's bit for bit.  The only
admitted exception is a float64 transcendental (sin/exp/tanh) differing by an
ulp between CUDA's libdevice and NumPy, which can move a signal across a
float32 rounding boundary: such cells must be within 1 float32 ulp and rare
(<= 1e-4 of the table)."""

import numpy as np
import pytest

from oracle import cppn as ocppn
from paper_2406_09654_b200 import neat
from paper_2406_09654_b200.device import DeviceSubstrate
from tests import _cases as CS

pytestmark = pytest.mark.gpu


def assert_tables_equal(got, want, what):
    got = np.ascontiguousarray(got, np.float32)
    want = np.ascontiguousarray(want, np.float32)
    assert got.shape == want.shape, what
    gi, wi = got.view(np.int32).astype(np.int64), want.view(np.int32).astype(np.int64)
    bad = gi != wi
    n = int(bad.sum())
    if n:
        assert np.all(np.abs(gi[bad] - wi[bad]) <= 1), f"{what}: mismatch beyond 1 ulp"
        assert n <= max(1, 1e-4 * got.size), f"{what}: {n} one-ulp mismatches"


@pytest.fixture(scope="module")
def golden():
    genomes, doc = CS.cppn_genomes()
    return genomes, doc, CS.load("cppn_cases.npz")


def test_direct_block_vs_reference(golden):
    genomes, doc, z = golden
    n = len(genomes)
    dev = DeviceSubstrate(8, 8, n + 3, hidden=0)
    slots = np.arange(3, 3 + n, dtype=np.int32)[::-1].copy()  # non-trivial slot order
    dev.express_cppn(slots, genomes, doc["tau"], doc["w_max"])
    _, _, w2, b2 = dev.get_params_arrays(0, n + 3)
    for i, s in enumerate(slots):
        assert_tables_equal(w2[s], z[f"direct_w_{i}"], f"direct w genome {i}")
        assert_tables_equal(b2[s], z[f"direct_b_{i}"], f"direct b genome {i}")
    assert np.all(w2[:3] == 0) and np.all(b2[:3] == 0)  # untouched slots
    dev.close()


@pytest.mark.parametrize("hidden", [16, 128])
def test_dense_vs_reference(golden, hidden):
    genomes, doc, z = golden
    idx = [i for i in range(len(genomes)) if f"h{hidden}_w1_{i}" in z]
    dev = DeviceSubstrate(8, 8, len(idx), hidden=hidden)
    dev.express_cppn(np.arange(len(idx), dtype=np.int32), [genomes[i] for i in idx], doc["tau"], doc["w_max"])
    w1, b1, w2, b2 = dev.get_params_arrays(0, len(idx))
    for k, i in enumerate(idx):
        for name, v in (("w1", w1[k]), ("b1", b1[k]), ("w2", w2[k]), ("b2", b2[k])):
            assert_tables_equal(v, z[f"h{hidden}_{name}_{i}"], f"h{hidden} {name} genome {i}")
    dev.close()


def test_random_lineages_vs_oracle():
    """Many mutated pattern networks (host NEAT) expressed in one launch."""
    rng = np.random.default_rng(9)
    counter = neat.InnovationCounter()
    wild = neat.EvolutionRates(add_connection_prob=0.5, add_node_prob=0.4, toggle_enable_prob=0.05)
    genomes = []
    for lin in range(12):
        g = neat.init_c3_genome(rng, counter) if lin % 2 else neat.init_genome(rng, counter)
        for gen in range(lin * 2):
            g = neat.mutate(g, wild, neat.stream(1, gen, "lineage", lin), counter)
        genomes.append(g)
    dev = DeviceSubstrate(8, 8, 16, hidden=0)
    slots = np.array([15, 2, 7, 0, 9, 11, 4, 13, 1, 6, 10, 3], np.int32)
    dev.express_cppn(slots, genomes)
    _, _, w2, b2 = dev.get_params_arrays(0, 16)
    for g, s in zip(genomes, slots):
        w, b = ocppn.generate_direct(g)
        assert_tables_equal(w2[s], w, f"slot {s}")
        assert_tables_equal(b2[s], b, f"slot {s} bias")
    dev.close()


def test_express_rejects_bad_arguments(golden):
    genomes, doc, _ = golden
    dev = DeviceSubstrate(8, 8, 4, hidden=0)
    with pytest.raises(ValueError):
        dev.express_cppn([0], genomes[:1], tau=1.0)
    with pytest.raises(ValueError):
        dev.express_cppn([0], genomes[:1], w_max=0.0)
    with pytest.raises(ValueError):
        dev.express_cppn([4], genomes[:1])
    dev.close()
