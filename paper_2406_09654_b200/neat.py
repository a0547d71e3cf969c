"""Host-side NEAT genome types, mutation and CPPN program linearisation.

NEAT genetics stay on the host (north_star (6)); this module is the part of
the reference's ``neuroevo`` the device path needs to feed the batched CPPN
kernel:

* ``NodeGene`` / ``ConnGene`` / ``CppnGenome`` with the reference's field
  names (/root/reference/pkg/src/evoca/neuroevo.py:54-85), so reference
  genomes are accepted unchanged;
* ``mutate`` - the reference's variation operator restated step for step
  (neuroevo.py:233-299: weight reset/perturb, toggles, add-connection,
  add-node, in that fixed order and draw order), so a given Philox stream
  yields the same child (pinned by tests/golden/cppn_cases.npz);
* ``crossover`` - recombination of two parents (neuroevo.py:329-351) in the
  reference's draw order (pinned by tests/golden/radiation_steps.npz);
* ``init_genome`` (neuroevo.py:212-230) and ``init_c3_genome``, the
  BASELINE config-3 pattern network (4 coordinate inputs -> 8 hidden
  sin/gauss/tanh nodes -> weight output, weights N(0,1));
* ``topo_order`` (hypernet.py:100-125: Kahn with an id-sorted frontier over
  the full gene graph) and ``compile_programs``, which lays a batch of
  genomes out as the flat program arrays of ``evo_express_cppn``.
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass, replace

import numpy as np

__all__ = [
    "ACTIVATIONS",
    "NodeGene",
    "ConnGene",
    "CppnGenome",
    "InnovationCounter",
    "EvolutionRates",
    "init_genome",
    "init_c3_genome",
    "mutate",
    "crossover",
    "topo_order",
    "compile_programs",
    "compile_programs_py",
    "PackedGenome",
    "pack",
    "mutate_batch",
    "mutate_batch_deferred",
    "number_deferred",
    "subset_programs",
    "layout_coords",
    "stream",
    "stream_key",
]

ACTIVATIONS = ("sine", "gaussian", "sigmoid", "tanh", "identity", "abs")  # neuroevo.py:43
ACT_CODE = {a: i for i, a in enumerate(ACTIVATIONS)}  # device activation codes (evoca_b200.h)
N_INPUTS = 5
INPUT_IDS = (0, 1, 2, 3, 4)
OUTPUT_IDS = (5, 6)
FIRST_FREE_NODE_ID = 7


@dataclass(frozen=True)
class NodeGene:
    id: int
    role: str  # "input" | "hidden" | "output"
    activation: str


@dataclass(frozen=True)
class ConnGene:
    innovation: int
    src: int
    dst: int
    weight: float
    enabled: bool


@dataclass(frozen=True)
class CppnGenome:
    nodes: tuple
    connections: tuple


class InnovationCounter:
    """Shared innovation / node-id source (neuroevo.py:151-171)."""

    def __init__(self, next_innovation: int = 0, next_node_id: int = FIRST_FREE_NODE_ID):
        self.next_innovation = next_innovation
        self.next_node_id = next_node_id

    def new_innovation(self) -> int:
        n = self.next_innovation
        self.next_innovation += 1
        return n

    def new_node_id(self) -> int:
        n = self.next_node_id
        self.next_node_id += 1
        return n


@dataclass
class EvolutionRates:
    """Variation probabilities (neuroevo.py:174-208 defaults)."""

    weight_perturb_prob: float = 0.8
    weight_perturb_sigma: float = 0.5
    weight_reset_prob: float = 0.05
    add_connection_prob: float = 0.05
    add_node_prob: float = 0.03
    toggle_enable_prob: float = 0.01


def stream_key(master_seed: int, step: int, purpose: str, index: int = 0) -> int:
    """128-bit Philox key of the derivation tuple: blake2b-128 of
    (seed, step, len(purpose), purpose, index) (the reference's rng.stream,
    rng.py:19-33)."""
    import hashlib
    import struct

    m = 0xFFFFFFFFFFFFFFFF
    tag = purpose.encode("utf-8")
    packed = (struct.pack("<QQ", master_seed & m, step & m) + struct.pack("<H", len(tag)) + tag
              + struct.pack("<Q", index & m))
    return int.from_bytes(hashlib.blake2b(packed, digest_size=16).digest(), "little")


def stream(master_seed: int, step: int, purpose: str, index: int = 0) -> np.random.Generator:
    """Counter-based Philox stream of the derivation tuple (rng.py:19-33)."""
    return np.random.Generator(np.random.Philox(key=stream_key(master_seed, step, purpose, index)))


def _base_nodes():
    return tuple([NodeGene(i, "input", "identity") for i in INPUT_IDS]
                 + [NodeGene(i, "output", "tanh") for i in OUTPUT_IDS])


def init_genome(rng: np.random.Generator, counter: InnovationCounter) -> CppnGenome:
    """Every input wired to both outputs, weights U[-1, 1) (neuroevo.py:212-230)."""
    conns = []
    for src in INPUT_IDS:
        for dst in OUTPUT_IDS:
            conns.append(ConnGene(counter.new_innovation(), src, dst, float(rng.uniform(-1.0, 1.0)), True))
    return CppnGenome(_base_nodes(), tuple(conns))


def init_c3_genome(rng: np.random.Generator, counter: InnovationCounter, hidden: int = 8) -> CppnGenome:
    """BASELINE config 3 pattern network: the four
    coordinate inputs feed ``hidden`` nodes whose activations cycle through
    sine/gaussian/tanh, which feed the weight output; weights N(0, 1).  The
    constant input and the bias output stay unconnected (bias signal
    tanh(0) = 0 => biases 0) until mutation wires them."""
    acts = ("sine", "gaussian", "tanh")
    nodes = list(_base_nodes())
    hid = []
    for h in range(hidden):
        nid = counter.new_node_id()
        nodes.append(NodeGene(nid, "hidden", acts[h % 3]))
        hid.append(nid)
    conns = []
    for nid in hid:
        for src in INPUT_IDS[:4]:
            conns.append(ConnGene(counter.new_innovation(), src, nid, float(rng.standard_normal()), True))
    for nid in hid:
        conns.append(ConnGene(counter.new_innovation(), nid, OUTPUT_IDS[0], float(rng.standard_normal()), True))
    return CppnGenome(tuple(nodes), tuple(conns))


def _creates_cycle(conns, src: int, dst: int) -> bool:
    """Is ``src`` reachable from ``dst`` in the full gene graph (neuroevo.py:121-143)."""
    if src == dst:
        return True
    out: dict = {}
    for c in conns:
        out.setdefault(c.src, []).append(c.dst)
    stack, seen = [dst], {dst}
    while stack:
        n = stack.pop()
        if n == src:
            return True
        for m in out.get(n, ()):
            if m not in seen:
                seen.add(m)
                stack.append(m)
    return False


def _descendants(conns) -> dict:
    """Nodes reachable from each node over the full gene graph (disabled
    edges included; the graph is acyclic, mutate never closes a cycle)."""
    out: dict = {}
    for c in conns:
        out.setdefault(c.src, []).append(c.dst)
    memo: dict = {}
    for root in list(out):
        if root in memo:
            continue
        stack = [(root, iter(out.get(root, ())))]
        onpath = {root}
        while stack:
            n, it = stack[-1]
            m = next(it, None)
            if m is None:
                acc = set()
                for k in out.get(n, ()):
                    acc.add(k)
                    acc |= memo[k]
                memo[n] = acc
                onpath.discard(n)
                stack.pop()
            elif m not in memo:
                if m in onpath:  # not a DAG: the caller falls back to per-pair search
                    return {}
                onpath.add(m)
                stack.append((m, iter(out.get(m, ()))))
    return memo


def mutate(genome, rates: EvolutionRates, rng: np.random.Generator, counter: InnovationCounter) -> CppnGenome:
    """Mutated copy of ``genome`` (neuroevo.py:233-299), same operation and
    draw order as the reference (the add-connection candidates are the
    reference's list, cycle-checked against precomputed descendant sets)."""
    conns = list(genome.connections)
    nodes = list(genome.nodes)
    rnd = rng.random
    p_reset, p_perturb, sigma = rates.weight_reset_prob, rates.weight_perturb_prob, rates.weight_perturb_sigma
    for i, c in enumerate(conns):
        if rnd() < p_reset:
            conns[i] = ConnGene(c.innovation, c.src, c.dst, float(rng.uniform(-1.0, 1.0)), c.enabled)
        elif rnd() < p_perturb:
            conns[i] = ConnGene(c.innovation, c.src, c.dst, c.weight + float(rng.normal(0.0, sigma)), c.enabled)
    p_toggle = rates.toggle_enable_prob
    for i, c in enumerate(conns):
        if rnd() < p_toggle:
            conns[i] = ConnGene(c.innovation, c.src, c.dst, c.weight, not c.enabled)
    if rnd() < rates.add_connection_prob:
        roles = {n.id: n.role for n in nodes}
        taken = {(c.src, c.dst) for c in conns}
        ordered = sorted(roles)
        desc = _descendants(conns)
        if desc or not conns:
            empty: set = set()
            cands = [(s, d) for s in ordered if roles[s] != "output" for d in ordered
                     if roles[d] != "input" and d != s and (s, d) not in taken and s not in desc.get(d, empty)]
        else:
            cands = [(s, d) for s in ordered if roles[s] != "output" for d in ordered
                     if roles[d] != "input" and (s, d) not in taken and not _creates_cycle(conns, s, d)]
        if cands:
            s, d = cands[int(rng.integers(len(cands)))]
            conns.append(ConnGene(counter.new_innovation(), s, d, float(rng.uniform(-1.0, 1.0)), True))
    if rnd() < rates.add_node_prob:
        enabled = [i for i, c in enumerate(conns) if c.enabled]
        if enabled:
            pick = enabled[int(rng.integers(len(enabled)))]
            old = conns[pick]
            nid = counter.new_node_id()
            act = ACTIVATIONS[int(rng.integers(len(ACTIVATIONS)))]
            conns[pick] = ConnGene(old.innovation, old.src, old.dst, old.weight, False)
            nodes.append(NodeGene(nid, "hidden", act))
            conns.append(ConnGene(counter.new_innovation(), old.src, nid, 1.0, True))
            conns.append(ConnGene(counter.new_innovation(), nid, old.dst, old.weight, True))
    return CppnGenome(tuple(nodes), tuple(conns))


def _paired_genes(a, b):
    """Innovation-ordered walk over two connection lists (both are kept in
    ascending innovation order by mutate): yields (gene of a | None, gene of
    b | None), both set for a matching innovation (neuroevo.py:304-326)."""
    ca, cb = a.connections, b.connections
    i = j = 0
    while i < len(ca) or j < len(cb):
        ka = ca[i].innovation if i < len(ca) else None
        kb = cb[j].innovation if j < len(cb) else None
        if kb is None or (ka is not None and ka < kb):
            yield ca[i], None
            i += 1
        elif ka is None or kb < ka:
            yield None, cb[j]
            j += 1
        else:
            yield ca[i], cb[j]
            i += 1
            j += 1


def crossover(fitter, other, rng: np.random.Generator) -> CppnGenome:
    """Child of two genomes, ``fitter`` first (neuroevo.py:329-351), with the
    reference's draw order: for every gene of the fitter parent, a matching
    gene first draws which parent's weight to take (< 0.5: the fitter's);
    then any gene disabled in a parent draws once more and stays disabled
    unless that draw is >= 0.75.  Genes only the other parent has are
    dropped, so the child keeps the fitter's node and edge sets."""
    genes = []
    for mine, theirs in _paired_genes(fitter, other):
        if mine is None:
            continue
        if theirs is None:
            weight, was_off = mine.weight, not mine.enabled
        else:
            weight = mine.weight if rng.random() < 0.5 else theirs.weight
            was_off = not (mine.enabled and theirs.enabled)
        enabled = True if not was_off else bool(rng.random() >= 0.75)
        genes.append(replace(mine, weight=weight, enabled=enabled))
    return CppnGenome(fitter.nodes, tuple(genes))


def topo_order(genome) -> list:
    """Kahn's algorithm over the full gene graph (disabled edges included),
    id-sorted frontier (hypernet.py:100-125)."""
    indeg = {n.id: 0 for n in genome.nodes}
    out: dict = {n.id: [] for n in genome.nodes}
    for c in genome.connections:
        indeg[c.dst] += 1
        out[c.src].append(c.dst)
    frontier = [n for n, d in indeg.items() if d == 0]
    heapq.heapify(frontier)
    order = []
    while frontier:
        n = heapq.heappop(frontier)
        order.append(n)
        for m in out[n]:
            indeg[m] -= 1
            if indeg[m] == 0:
                heapq.heappush(frontier, m)
    if len(order) != len(indeg):
        raise ValueError("gene graph contains a cycle")
    return order


def layout_coords(hidden: int) -> np.ndarray:
    """Neuron coordinates (45 sensors, ``hidden`` hidden, 13 actuators) x
    (u, v) as the reference's make_layout builds them (hypernet.py:64-74),
    float64, flattened for evo_express_cppn."""
    slots = np.linspace(-1.0, 1.0, 9)
    subs = np.linspace(-1.0, 1.0, 5)
    inputs = np.array([(u, v) for u in slots for v in subs], dtype=np.float64)
    parts = [inputs]
    if hidden > 0:
        parts.append(np.stack([np.linspace(-1.0, 1.0, hidden), np.zeros(hidden)], axis=1))
    parts.append(np.stack([np.linspace(-1.0, 1.0, 13), np.zeros(13)], axis=1))
    return np.ascontiguousarray(np.vstack(parts), np.float64)


def compile_programs_py(genomes):
    """Flatten a batch of genomes into ``evo_express_cppn`` programs (the
    Python statement of the layout; ``compile_programs`` runs the native
    equivalent, tests/test_neat_native.py pins the two together).

    Per genome, nodes in ``topo_order``; node record (int32 x4):
    ``[act_code | -1 for inputs, input_position | -1, edge_begin, edge_end]``
    (edges are global indices into ``edge_src`` / ``edge_w``); incoming
    edges of a node are its ENABLED connections in connection-list order
    (the reference's summation order, hypernet.py:140-153), ``edge_src`` is
    the source node's position in the genome's own node list.  ``outs``
    holds the positions of the two output nodes in ascending id order
    (weight signal, bias signal; hypernet.py:154-155).
    Returns (node_off int32 [n+1], nodes int32 [N,4], edge_src int32 [E],
    edge_w float64 [E], outs int32 [n,2]).
    """
    node_off = [0]
    nodes, edge_src, edge_w, outs = [], [], [], []
    for gnm in genomes:
        order = topo_order(gnm)
        pos = {nid: i for i, nid in enumerate(order)}
        role = {n.id: n for n in gnm.nodes}
        input_pos = {nid: i for i, nid in enumerate(sorted(n.id for n in gnm.nodes if n.role == "input"))}
        if len(input_pos) != N_INPUTS:
            raise ValueError("a pattern network needs exactly five inputs")
        incoming: dict = {}
        for c in gnm.connections:
            if c.enabled:
                incoming.setdefault(c.dst, []).append(c)
        for nid in order:
            nd = role[nid]
            if nd.role == "input":
                nodes.append((-1, input_pos[nid], len(edge_src), len(edge_src)))
                continue
            if nd.activation not in ACT_CODE:
                raise ValueError(f"unknown activation {nd.activation!r}")
            b = len(edge_src)
            for c in incoming.get(nid, ()):
                edge_src.append(pos[c.src])
                edge_w.append(float(c.weight))
            nodes.append((ACT_CODE[nd.activation], -1, b, len(edge_src)))
        out_ids = sorted(n.id for n in gnm.nodes if n.role == "output")
        if len(out_ids) != 2:
            raise ValueError("a pattern network needs exactly two outputs")
        outs.append((pos[out_ids[0]], pos[out_ids[1]]))
        node_off.append(len(nodes))
    return (np.asarray(node_off, np.int32), np.asarray(nodes, np.int32).reshape(-1, 4),
            np.asarray(edge_src, np.int32), np.asarray(edge_w, np.float64), np.asarray(outs, np.int32).reshape(-1, 2))


# -- native host NEAT (csrc/evoca_neat.cpp) -------------------------------------------------

ROLE_CODE = {"input": 0, "hidden": 1, "output": 2}
ROLE_NAME = ("input", "hidden", "output")


class Flat:
    """A genome as flat arrays (node id / role / activation code;
    connection innovation / src / dst / weight / enabled)."""

    __slots__ = ("nid", "nrole", "nact", "inn", "src", "dst", "w", "en")

    def __init__(self, nid, nrole, nact, inn, src, dst, w, en):
        self.nid, self.nrole, self.nact = nid, nrole, nact
        self.inn, self.src, self.dst, self.w, self.en = inn, src, dst, w, en


class PackedGenome(CppnGenome):
    """A pattern network held as flat arrays - the children of the native
    mutation.  ``nodes`` / ``connections`` (the reference's gene tuples) are
    built on first access; the radiation feed itself (mutation of children
    in later events, program compilation) works on the arrays."""

    def __init__(self, flat: Flat | None, batch=None, index: int = 0):  # noqa: D107 - bypasses the dataclass init
        object.__setattr__(self, "_flat", flat)
        object.__setattr__(self, "_batch", batch)  # (GenomeBatch, index) when flat is still unsliced
        object.__setattr__(self, "_index", index)
        object.__setattr__(self, "_genes", None)

    def _materialise(self):
        genes = object.__getattribute__(self, "_genes")
        if genes is None:
            f = pack(self)
            nodes = tuple(NodeGene(int(i), ROLE_NAME[int(r)], ACTIVATIONS[int(a)])
                          for i, r, a in zip(f.nid.tolist(), f.nrole.tolist(), f.nact.tolist()))
            conns = tuple(ConnGene(n, s_, d, w, bool(e)) for n, s_, d, w, e in
                          zip(f.inn.tolist(), f.src.tolist(), f.dst.tolist(), f.w.tolist(), f.en.tolist()))
            genes = (nodes, conns)
            object.__setattr__(self, "_genes", genes)
        return genes

    @property
    def nodes(self):
        return self._materialise()[0]

    @property
    def connections(self):
        return self._materialise()[1]

    def __eq__(self, other):
        if not hasattr(other, "nodes") or not hasattr(other, "connections"):
            return NotImplemented
        return self.nodes == tuple(other.nodes) and self.connections == tuple(other.connections)

    def __hash__(self):
        return hash((self.nodes, self.connections))

    def __repr__(self):
        f = pack(self)
        return f"PackedGenome({len(f.nid)} nodes, {len(f.inn)} connections)"


class GenomeBatch:
    """The concatenated arrays of one native mutation's children (node /
    connection offsets per genome); its PackedGenome members slice it on
    demand, and consecutive members are handed to the next native call as
    one slice instead of being re-concatenated."""

    __slots__ = ("node_off", "conn_off", "arrays")

    def __init__(self, node_off, conn_off, arrays):
        self.node_off, self.conn_off, self.arrays = node_off, conn_off, arrays  # arrays: Flat order

    def flat(self, i: int) -> Flat:
        a, b = int(self.node_off[i]), int(self.node_off[i + 1])
        c, d = int(self.conn_off[i]), int(self.conn_off[i + 1])
        nid, nrole, nact, inn, src, dst, w, en = self.arrays
        return Flat(nid[a:b], nrole[a:b], nact[a:b], inn[c:d], src[c:d], dst[c:d], w[c:d], en[c:d])


def pack(genome) -> Flat:
    """Flat arrays of a genome (cached on this package's genome objects)."""
    f = genome.__dict__.get("_flat") if hasattr(genome, "__dict__") else None
    if f is not None:
        return f
    b = genome.__dict__.get("_batch") if hasattr(genome, "__dict__") else None
    if b is not None:
        f = b.flat(genome.__dict__["_index"])
        object.__setattr__(genome, "_flat", f)
        return f
    nodes, conns = genome.nodes, genome.connections
    f = Flat(np.fromiter((n.id for n in nodes), np.int64, len(nodes)),
             np.fromiter((ROLE_CODE[n.role] for n in nodes), np.int8, len(nodes)),
             np.fromiter((ACT_CODE[n.activation] for n in nodes), np.int8, len(nodes)),
             np.fromiter((c.innovation for c in conns), np.int64, len(conns)),
             np.fromiter((c.src for c in conns), np.int64, len(conns)),
             np.fromiter((c.dst for c in conns), np.int64, len(conns)),
             np.fromiter((c.weight for c in conns), np.float64, len(conns)),
             np.fromiter((c.enabled for c in conns), np.uint8, len(conns)))
    if isinstance(genome, CppnGenome):
        object.__setattr__(genome, "_flat", f)
    return f


_FLAT_FIELDS = (("nid", np.int64), ("nrole", np.int8), ("nact", np.int8), ("inn", np.int64), ("src", np.int64),
                ("dst", np.int64), ("w", np.float64), ("en", np.uint8))


def _concat(genomes):
    """(node_off, nid, nrole, nact, conn_off, inn, src, dst, w, en) of a list
    of genomes; runs of consecutive members of one GenomeBatch are taken as
    single slices of its arrays.  A list with no such run becomes a batch
    itself (the genomes are immutable), so the next call over the same
    genomes - the seed population's first mutation after its expression -
    skips the per-genome concatenation."""
    n = len(genomes)
    fresh = True
    parts = [[] for _ in _FLAT_FIELDS]
    node_off = np.zeros(n + 1, np.int32)
    conn_off = np.zeros(n + 1, np.int32)
    i = 0
    while i < n:
        g = genomes[i]
        d = g.__dict__ if hasattr(g, "__dict__") else {}
        b = d.get("_batch")
        if b is not None:
            fresh = False
            i0 = d["_index"]
            j = i + 1
            while j < n and getattr(genomes[j], "__dict__", {}).get("_batch") is b and \
                    genomes[j].__dict__["_index"] == i0 + (j - i):
                j += 1
            i1 = i0 + (j - i)
            na, nb = int(b.node_off[i0]), int(b.node_off[i1])
            ca, cb = int(b.conn_off[i0]), int(b.conn_off[i1])
            for k, arr in enumerate(b.arrays):
                parts[k].append(arr[na:nb] if k < 3 else arr[ca:cb])
            node_off[i + 1:j + 1] = node_off[i] + (b.node_off[i0 + 1:i1 + 1] - na)
            conn_off[i + 1:j + 1] = conn_off[i] + (b.conn_off[i0 + 1:i1 + 1] - ca)
            i = j
            continue
        f = pack(g)
        for k, (name, _) in enumerate(_FLAT_FIELDS):
            parts[k].append(getattr(f, name))
        node_off[i + 1] = node_off[i] + len(f.nid)
        conn_off[i + 1] = conn_off[i] + len(f.inn)
        i += 1
    cat = [np.ascontiguousarray(np.concatenate(p) if len(p) > 1 else (p[0] if p else np.empty(0, dt)), dt)
           for p, (_, dt) in zip(parts, _FLAT_FIELDS)]
    if fresh and n > 1 and all(isinstance(g, CppnGenome) for g in genomes):
        batch = GenomeBatch(node_off, conn_off, tuple(cat))
        for i, g in enumerate(genomes):
            object.__setattr__(g, "_batch", batch)
            object.__setattr__(g, "_index", i)
    return (node_off, cat[0], cat[1], cat[2], conn_off, cat[3], cat[4], cat[5], cat[6], cat[7])


def _native():
    from . import _lib

    return _lib.load()


def _neat_check(rc):
    if rc != 0:
        raise ValueError(_native().evo_neat_last_error().decode("utf-8", "replace"))


def mutate_batch(genomes, rates, keys, counter: InnovationCounter) -> list:
    """``mutate`` of each genome on its own stream (128-bit Philox keys, e.g.
    ``stream_key(seed, t, "mutate", index)``), in list order, consuming the
    shared innovation counter as sequential ``mutate`` calls would; native
    (evo_neat_mutate).  Returns PackedGenome children."""
    return _mutate_native(genomes, rates, keys, counter)


DEFERRED_NODE = np.iinfo(np.int64).max  # EVO_NEAT_DEFERRED_NODE


def mutate_batch_deferred(genomes, rates, keys) -> list:
    """``mutate_batch`` with the numbering left open (evo_neat_mutate_deferred):
    the k-th new connection of a child has innovation -1 - k, its new node
    the id DEFERRED_NODE.  ``number_deferred`` over any ordered subset then
    equals ``mutate_batch`` over the parents of that subset alone."""
    return _mutate_native(genomes, rates, keys, None)


def _excl_cumsum(x):
    out = np.zeros(len(x), np.int64)
    if len(x) > 1:
        np.cumsum(x[:-1], out=out[1:])
    return out


def number_deferred(children, counter: InnovationCounter) -> list:
    """Final innovation numbers / node ids for deferred children, taken from
    ``counter`` in list order (per child: its new connections in creation
    order, then its new node) - exactly what evo_neat_mutate draws."""
    n = len(children)
    if n == 0:
        return []
    node_off, nid, nrole, nact, conn_off, inn, src, dst, w, en = _concat(children)
    gc = np.repeat(np.arange(n), np.diff(conn_off))
    gn = np.repeat(np.arange(n), np.diff(node_off))
    newc = inn < 0
    cnt = np.bincount(gc[newc], minlength=n)
    inn = inn.copy()
    inn[newc] = (counter.next_innovation + _excl_cumsum(cnt))[gc[newc]] + (-1 - inn[newc])
    newn = nid == DEFERRED_NODE
    has = np.bincount(gn[newn], minlength=n)
    nbase = counter.next_node_id + _excl_cumsum(has)
    nid = np.where(newn, nbase[gn], nid)
    src = np.where(src == DEFERRED_NODE, nbase[gc], src)
    dst = np.where(dst == DEFERRED_NODE, nbase[gc], dst)
    counter.next_innovation += int(cnt.sum())
    counter.next_node_id += int(has.sum())
    batch = GenomeBatch(node_off, conn_off, (nid, nrole, nact, inn, src, dst, w, en))
    return [PackedGenome(None, batch, g) for g in range(n)]


def _mutate_native(genomes, rates, keys, counter):
    from ._lib import ptr

    n = len(genomes)
    if n == 0:
        return []
    lib = _native()
    node_off, nid, nrole, nact, conn_off, inn, src, dst, w, en = _concat(genomes)
    m = (1 << 64) - 1
    kw = np.array([h for k in keys for h in (int(k) & m, (int(k) >> 64) & m)], np.uint64)
    r = np.array([rates.weight_reset_prob, rates.weight_perturb_prob, rates.weight_perturb_sigma,
                  rates.add_connection_prob, rates.add_node_prob, rates.toggle_enable_prob], np.float64)
    NN, NC = len(nid) + n, len(inn) + 3 * n
    o_node_off, o_conn_off = np.empty(n + 1, np.int32), np.empty(n + 1, np.int32)
    o_nid, o_nrole, o_nact = np.empty(NN, np.int64), np.empty(NN, np.int8), np.empty(NN, np.int8)
    o_inn, o_src, o_dst = np.empty(NC, np.int64), np.empty(NC, np.int64), np.empty(NC, np.int64)
    o_w, o_en = np.empty(NC, np.float64), np.empty(NC, np.uint8)
    io = [ptr(node_off), ptr(nid), ptr(nrole), ptr(nact), ptr(conn_off), ptr(inn), ptr(src), ptr(dst), ptr(w),
          ptr(en), ptr(o_node_off), ptr(o_nid), ptr(o_nrole), ptr(o_nact), ptr(o_conn_off), ptr(o_inn), ptr(o_src),
          ptr(o_dst), ptr(o_w), ptr(o_en)]
    if counter is None:
        _neat_check(lib.evo_neat_mutate_deferred(n, ptr(kw), ptr(r), *io))
    else:
        ctr = np.array([counter.next_innovation, counter.next_node_id], np.int64)
        _neat_check(lib.evo_neat_mutate(n, ptr(kw), ptr(r), ptr(ctr), *io))
        counter.next_innovation, counter.next_node_id = int(ctr[0]), int(ctr[1])
    batch = GenomeBatch(o_node_off, o_conn_off, (o_nid, o_nrole, o_nact, o_inn, o_src, o_dst, o_w, o_en))
    return [PackedGenome(None, batch, g) for g in range(n)]


def _ranges(starts, ends):
    """Concatenated aranges [starts[i], ends[i])."""
    lens = np.asarray(ends, np.int64) - np.asarray(starts, np.int64)
    tot = int(lens.sum())
    return np.repeat(np.asarray(starts, np.int64) - _excl_cumsum(lens), lens) + np.arange(tot)


def subset_programs(programs, idx):
    """The ``compile_programs`` arrays of the genomes ``idx`` (in that order)
    cut out of the arrays of a larger batch (edge ranges rebased)."""
    prog_off, nodes, esrc, ew, outs = programs
    idx = np.asarray(idx, np.int64)
    ns, nd = prog_off[idx].astype(np.int64), prog_off[idx + 1].astype(np.int64)
    eb, ee = nodes[ns, 2].astype(np.int64), nodes[nd - 1, 3].astype(np.int64)
    sub = nodes[_ranges(ns, nd)].copy()
    shift = (_excl_cumsum(ee - eb) - eb).astype(np.int32)
    sub[:, 2:4] += np.repeat(shift, nd - ns)[:, None]
    eidx = _ranges(eb, ee)
    off = np.zeros(len(idx) + 1, np.int32)
    np.cumsum(nd - ns, out=off[1:])
    return off, sub, np.ascontiguousarray(esrc[eidx]), np.ascontiguousarray(ew[eidx]), np.ascontiguousarray(outs[idx])


def compile_programs(genomes):
    """``evo_express_cppn`` programs of a batch of genomes (the layout of
    ``compile_programs_py``), linearised natively (evo_neat_compile)."""
    from ._lib import ptr

    n = len(genomes)
    node_off, nid, nrole, nact, conn_off, inn, src, dst, w, en = _concat(genomes)
    prog_off = np.empty(n + 1, np.int32)
    nodes = np.empty((max(len(nid), 1), 4), np.int32)
    esrc = np.empty(max(len(inn), 1), np.int32)
    ew = np.empty(max(len(inn), 1), np.float64)
    outs = np.empty((max(n, 1), 2), np.int32)
    _neat_check(_native().evo_neat_compile(n, ptr(node_off), ptr(nid), ptr(nrole), ptr(nact), ptr(conn_off),
                                           ptr(src), ptr(dst), ptr(w), ptr(en), ptr(prog_off), ptr(nodes),
                                           ptr(esrc), ptr(ew), ptr(outs)))
    ne = int(en.sum()) if n else 0
    return (prog_off, np.ascontiguousarray(nodes[:len(nid)]), np.ascontiguousarray(esrc[:ne]),
            np.ascontiguousarray(ew[:ne]), np.ascontiguousarray(outs[:n]))
