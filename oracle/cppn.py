"""CPU oracle for the batched CPPN expression kernel (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline may import
this module; the product never does.

Restates, in float64 NumPy, the reference's pattern-network evaluation and
weight expression (/root/reference/pkg/src/evoca/hypernet.py):
  make_layout          hypernet.py:64-74
  evaluate_cppn_batch  hypernet.py:128-156 (Kahn order :100-125; incoming
                       sums in connection-list order, ``total + w * v``)
  _express             hypernet.py:168-180
  generate_network     hypernet.py:183-220 (dst-major query blocks)
plus ``generate_direct``: the same expression restricted to the BASELINE
45->13 direct block (queries input coord -> actuator coord; biases from the
bias signal of ((0, 0), actuator coord) queries).
Pinned to the reference by tests/golden/cppn_cases.npz.
"""

from __future__ import annotations

import heapq

import numpy as np

N_SENSORS = 45
N_ACTUATORS = 13

_ACT = {
    "sine": np.sin,
    "gaussian": lambda x: np.exp(-np.square(x)),
    "sigmoid": lambda x: 1.0 / (1.0 + np.exp(-x)),
    "tanh": np.tanh,
    "identity": lambda x: x,
    "abs": np.abs,
}


def make_layout(hidden: int):
    slots = np.linspace(-1.0, 1.0, 9)
    subs = np.linspace(-1.0, 1.0, 5)
    inputs = np.array([(u, v) for u in slots for v in subs], dtype=np.float64)
    hid = (np.stack([np.linspace(-1.0, 1.0, hidden), np.zeros(hidden)], axis=1) if hidden > 0
           else np.zeros((0, 2)))
    outs = np.stack([np.linspace(-1.0, 1.0, N_ACTUATORS), np.zeros(N_ACTUATORS)], axis=1)
    return inputs, hid, outs


def topo_order(genome):
    indeg = {n.id: 0 for n in genome.nodes}
    out = {n.id: [] for n in genome.nodes}
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
    return order


def evaluate_batch(genome, queries):
    q = np.asarray(queries, dtype=np.float64)
    roles = {n.id: n for n in genome.nodes}
    input_pos = {nid: i for i, nid in enumerate(sorted(n.id for n in genome.nodes if n.role == "input"))}
    incoming = {}
    for c in genome.connections:
        if c.enabled:
            incoming.setdefault(c.dst, []).append(c)
    vals = {}
    for nid in topo_order(genome):
        node = roles[nid]
        if node.role == "input":
            vals[nid] = q[:, input_pos[nid]]
            continue
        total = np.zeros(len(q))
        for c in incoming.get(nid, ()):
            total = total + c.weight * vals[c.src]
        vals[nid] = _ACT[node.activation](total)
    out_ids = sorted(n.id for n in genome.nodes if n.role == "output")
    return np.stack([vals[i] for i in out_ids], axis=1)


def express(signals, tau: float, w_max: float):
    s = np.asarray(signals, dtype=np.float64)
    mag = np.abs(s)
    scaled = np.sign(s) * np.minimum((mag - tau) / (1.0 - tau), 1.0) * w_max
    out = np.where(mag > tau, scaled, 0.0)
    out = np.where(np.isfinite(s), out, 0.0)
    return out.astype(np.float32)


def _queries(dst, src):
    d = np.repeat(dst, len(src), axis=0)
    s = np.tile(src, (len(dst), 1))
    return np.column_stack([s, d, np.ones(len(d))])


def generate_dense(genome, hidden: int, tau: float = 0.2, w_max: float = 3.0):
    """(w1 (H,45), b1 (H,), w2 (13,H), b2 (13,)) float32, reference layout."""
    inp, hid, out = make_layout(hidden)
    nh, ni, no = len(hid), len(inp), len(out)
    blocks = [_queries(hid, inp), _queries(out, hid),
              np.column_stack([np.zeros((nh + no, 2)), np.vstack([hid, out]), np.ones(nh + no)])]
    sig = evaluate_batch(genome, np.vstack(blocks))
    n1, n2 = nh * ni, no * nh
    w1 = express(sig[:n1, 0], tau, w_max).reshape(nh, ni)
    w2 = express(sig[n1:n1 + n2, 0], tau, w_max).reshape(no, nh)
    b = express(sig[n1 + n2:, 1], tau, w_max)
    return w1, b[:nh].copy(), w2, b[nh:].copy()


def generate_direct(genome, tau: float = 0.2, w_max: float = 3.0):
    """(w (13,45), b (13,)) float32 for the 45->13 direct controller."""
    inp, _, out = make_layout(0)
    q = np.vstack([_queries(out, inp), np.column_stack([np.zeros((N_ACTUATORS, 2)), out, np.ones(N_ACTUATORS)])])
    sig = evaluate_batch(genome, q)
    n = N_ACTUATORS * N_SENSORS
    return express(sig[:n, 0], tau, w_max).reshape(N_ACTUATORS, N_SENSORS), express(sig[n:, 1], tau, w_max)
