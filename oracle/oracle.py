"""CPU oracle for the evoca per-step substrate update.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2406_09654_b200`` imports,
links or executes this module; only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg use it, and
only as the checker (or as the timed CPU baseline arm).

This is an independent restatement of the reference algorithm
(``/root/reference/pkg/src/evoca``, cited per function) written against
numpy (+ numba for the two scalar loops the reference also compiles with
numba, so the CPU baseline is timed on the same kind of code).  It is
pinned against vectors produced by the reference itself
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``;
``tests/test_oracle_golden.py``).

Float32 semantics: every physics operation is a separately rounded
float32 operation in the reference's order (numpy never contracts into
FMA).  The controller forward pass is the one place where the reference
is not bit-reproducible (OpenBLAS sgemm, batch-composition dependent, see
SURVEY.md §8c); the oracle evaluates the dot products in float64 and
rounds once, which is within the reference's own 1e-6 self-consistency
band, and the GPU is compared against it with a stated tolerance.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

try:  # the reference compiles these two loops with numba too
    import numba

    _njit = numba.njit(cache=False)
except Exception:  # pragma: no cover - numba is in the image
    numba = None

    def _njit(f):
        return f


# -- geometry (physics.py:40-62) ---------------------------------------------

# Direction j is the Moore offset at angle j*45 deg counterclockwise from
# east, stored as (dx, dy).  physics.py:40-43
OFFSETS = np.array(
    [(1, 0), (1, 1), (0, 1), (-1, 1), (-1, 0), (-1, -1), (0, -1), (1, -1)], dtype=np.int64
)
_DX = np.ascontiguousarray(OFFSETS[:, 0])
_DY = np.ascontiguousarray(OFFSETS[:, 1])
# Visit order for heading r is r+{0,+1,-1,+2,-2,+3,-3,+4} mod 8.  physics.py:48-58
_DELTAS = (0, 1, -1, 2, -2, 3, -3, 4)
PERM = np.array([[(r + d) % 8 for d in _DELTAS] for r in range(8)], dtype=np.int64)

N_SENSORS = 45
N_ACTUATORS = 13
SIG_HI = np.nextafter(np.float32(1.0), np.float32(0.0))  # hypernet.py:45
SIG_LO = np.float32(2.0 ** -126)  # hypernet.py:46


# -- state -------------------------------------------------------------------


@dataclass
class Planes:
    """One buffer of SoA state (substrate.py:52-75): E, I (H,W) f32,
    C (3,H,W) f32, gi (H,W) i32 (-1 empty), rot (H,W) u8 in 0..7."""

    E: np.ndarray
    I: np.ndarray
    C: np.ndarray
    gi: np.ndarray
    rot: np.ndarray

    @property
    def shape(self):
        return self.gi.shape

    def copy(self) -> "Planes":
        return Planes(self.E.copy(), self.I.copy(), self.C.copy(), self.gi.copy(), self.rot.copy())

    def equal(self, other: "Planes") -> bool:
        return all(
            np.array_equal(a.view(np.uint8), b.view(np.uint8))
            for a, b in zip(self.arrays(), other.arrays())
        )

    def arrays(self):
        return (self.E, self.I, self.C, self.gi, self.rot)


@dataclass
class Phys:
    """PhysicsParams defaults (physics.py:65-80)."""

    cycle_amplitude: float = 0.1
    cycle_period: int = 100
    energy_source_map: np.ndarray | None = None
    drain_fraction: float = 0.05
    invest_rate: float = 1.0
    liquidate_rate: float = 1.0
    invest_efficiency: float = 0.9
    liquidate_efficiency: float = 0.9
    explore_fraction: float = 0.5
    upkeep: float = 0.02
    decay_on_starvation: float = 0.1
    death_threshold: float = 1e-3


@dataclass
class Net:
    """Per-slot controller weights.  hidden == 0 is the BASELINE direct
    45->13 extension (w2 (cap,13,45), b2 (cap,13)); hidden > 0 is the
    reference DenseParams stack (hypernet.py:77-84)."""

    hidden: int
    w2: np.ndarray
    b2: np.ndarray
    w1: np.ndarray | None = None
    b1: np.ndarray | None = None

    @property
    def capacity(self) -> int:
        return self.w2.shape[0]


@dataclass
class Events:
    """AdoptionEvents columns (physics.py:134-175), ascending target."""

    target: np.ndarray
    source: np.ndarray
    winner_slot: np.ndarray
    defender_slot: np.ndarray
    direction: np.ndarray
    quantity: np.ndarray

    def __len__(self):
        return len(self.target)

    def rows(self):
        return [
            (int(t), int(s), int(w), int(d), int(r), float(q))
            for t, s, w, d, r, q in zip(
                self.target, self.source, self.winner_slot, self.defender_slot,
                self.direction, self.quantity,
            )
        ]


def empty_events() -> Events:
    return Events(
        np.empty(0, np.int64), np.empty(0, np.int64), np.empty(0, np.int32),
        np.empty(0, np.int32), np.empty(0, np.int64), np.empty(0, np.float32),
    )


# -- synthetic BASELINE inputs (SURVEY.md §8d generator draw order) -----------


def synth_planes(height: int, width: int, genomes: int, seed: int = 0, sparse_infra: bool = False) -> Planes:
    g = np.random.default_rng(seed)
    E = g.random((height, width), dtype=np.float32)
    I = g.random((height, width), dtype=np.float32)
    if sparse_infra:
        I[g.random((height, width)) < 0.9] = 0
    C = g.standard_normal((3, height, width)).astype(np.float32)
    theta = g.random((height, width)) * (2.0 * np.pi)
    rot = (np.floor(theta / (np.pi / 4)) % 8).astype(np.uint8)
    gi = g.integers(0, genomes, (height, width), dtype=np.int32)
    return Planes(E, I, C, gi, rot)


def synth_net(genomes: int, hidden: int = 0, seed: int = 0, sigma: float | None = None) -> Net:
    g = np.random.default_rng(seed + 1)
    if hidden == 0:
        s = 0.5 if sigma is None else sigma
        w2 = np.stack([(g.standard_normal((13, 45)) * s).astype(np.float32) for _ in range(genomes)])
        return Net(0, w2, np.zeros((genomes, 13), np.float32))
    s = 0.3 if sigma is None else sigma
    w1s, w2s = [], []
    for _ in range(genomes):
        w1s.append((g.standard_normal((hidden, 45)) * s).astype(np.float32))
        w2s.append((g.standard_normal((13, hidden)) * s).astype(np.float32))
    return Net(hidden, np.stack(w2s), np.zeros((genomes, 13), np.float32),
               np.stack(w1s), np.zeros((genomes, hidden), np.float32))


# -- sensing (engine.py:57-58, 142-190) ----------------------------------------


@_njit
def _sense_loop(stack, cells, rot, perm, dx, dy, width, height, out):  # pragma: no cover
    for n in range(cells.shape[0]):
        c = cells[n]
        x = c % width
        y = c // width
        for ch in range(5):
            out[n, ch] = stack[ch, c]
        r = rot[c]
        for s in range(8):
            j = perm[r, s]
            nb = ((y + dy[j]) % height) * width + (x + dx[j]) % width
            for ch in range(5):
                out[n, 5 * (s + 1) + ch] = stack[ch, nb]


def sense(p: Planes, cells: np.ndarray) -> np.ndarray:
    """45 sensors per listed cell: slot 0 self, slots 1..8 the Moore
    neighbours in PERM[rot] order, channels E, I, C0, C1, C2."""
    h, w = p.shape
    stack = np.empty((5, h * w), np.float32)
    stack[0] = p.E.ravel()
    stack[1] = p.I.ravel()
    stack[2:5] = p.C.reshape(3, -1)
    out = np.empty((len(cells), N_SENSORS), np.float32)
    _sense_loop(stack, np.asarray(cells, np.int64), p.rot.ravel().astype(np.int64), PERM, _DX, _DY, w, h, out)
    return out


# -- controller (hypernet.py:233-252) ------------------------------------------


def squash(z: np.ndarray) -> np.ndarray:
    """Output nonlinearity, op for op: negate, exp, +1, reciprocal, clip
    (each a float32 numpy ufunc, hypernet.py:246-251)."""
    z = np.negative(z.astype(np.float32))
    z = np.exp(z)
    z = z + np.float32(1.0)
    z = np.reciprocal(z)
    return np.clip(z, SIG_LO, SIG_HI)


def _dot(a: np.ndarray, b_t: np.ndarray) -> np.ndarray:
    return (a.astype(np.float64) @ b_t.astype(np.float64)).astype(np.float32)


def forward(net: Net, slot: int, sensors: np.ndarray) -> np.ndarray:
    """(n,45) -> (n,13).  Pre-activations: float64 dot rounded to f32,
    then + bias in f32 (the reference adds the bias after the sgemm)."""
    s = np.asarray(sensors, np.float32)
    if net.hidden == 0:
        z = _dot(s, net.w2[slot].T) + net.b2[slot]
        return squash(z)
    z1 = _dot(s, net.w1[slot].T) + net.b1[slot]
    h = np.tanh(z1.astype(np.float32))
    z2 = _dot(h, net.w2[slot].T) + net.b2[slot]
    return squash(z2)


@dataclass
class Actions:
    """ActionField (physics.py:97-119) as one (n,13) block in column order
    invest, liquidate, comm x3, explore x8 (engine.py:224-230)."""

    cells: np.ndarray
    a: np.ndarray

    @property
    def invest(self):
        return self.a[:, 0]

    @property
    def liquidate(self):
        return self.a[:, 1]

    @property
    def comm(self):
        return self.a[:, 2:5]

    @property
    def explore(self):
        return self.a[:, 5:13]


def act(p: Planes, net: Net) -> Actions:
    """Sense every occupied cell (ascending index) and run its genome's
    controller (engine.py:193-230).  Grouping by slot does not change
    per-row results in the oracle (per-row float64 dots)."""
    gi = p.gi.ravel()
    cells = np.flatnonzero(gi >= 0).astype(np.int64)
    out = np.empty((len(cells), N_ACTUATORS), np.float32)
    if len(cells) == 0:
        return Actions(cells, out)
    s = sense(p, cells)
    slots = gi[cells]
    order = np.argsort(slots, kind="stable")
    bounds = np.flatnonzero(np.r_[True, slots[order][1:] != slots[order][:-1], True])
    for a, b in zip(bounds[:-1], bounds[1:]):
        rows = order[a:b]
        out[rows] = forward(net, int(slots[rows[0]]), s[rows])
    return Actions(cells, out)


# -- physics phases (physics.py:178-404) ----------------------------------------


def rho_terms(t: int, phys: Phys):
    """Host-side day/night scalars exactly as physics.py:186-194 computes
    them: rho in float64 via math.sin, then the float32 casts.  Returns
    (mode, rho_f32, drain_f32) with mode 1 = day, 2 = night, 0 = neither."""
    rho = phys.cycle_amplitude * math.sin(2.0 * math.pi * t / phys.cycle_period)
    if rho > 0.0:
        return 1, np.float32(rho), np.float32(0.0)
    if rho < 0.0:
        return 2, np.float32(0.0), np.float32(phys.drain_fraction * -rho)
    return 0, np.float32(0.0), np.float32(0.0)


def energy(p: Planes, t: int, phys: Phys) -> None:
    mode, r32, d32 = rho_terms(t, phys)
    if mode == 1:
        add = r32 if phys.energy_source_map is None else r32 * phys.energy_source_map
        p.E[...] = p.E + add
    elif mode == 2:
        p.E[...] = p.E - d32 * p.E


def invest_liquidate(p: Planes, acts: Actions, phys: Phys) -> None:
    """physics.py:197-233, every op a float32 op in the reference order."""
    gi = p.gi.ravel()
    live = gi[acts.cells] >= 0
    idx = acts.cells[live]
    if len(idx) == 0:
        return
    E = p.E.ravel()
    I = p.I.ravel()
    f = np.float32
    e = E[idx]
    i = I[idx]
    de = acts.invest[live] * np.minimum(e, f(phys.invest_rate))
    e = e - de
    i = i + f(phys.invest_efficiency) * de
    di = acts.liquidate[live] * np.minimum(i, f(phys.liquidate_rate))
    i = i - di
    e = e + f(phys.liquidate_efficiency) * di
    cost = f(phys.upkeep) * i
    fed = e >= cost
    e = np.where(fed, e - cost, f(0.0))
    i = np.where(fed, i, i - f(phys.decay_on_starvation) * i)
    E[idx] = e
    I[idx] = i
    gi[idx[i < f(phys.death_threshold)]] = -1


def communication(p: Planes, acts: Actions) -> None:
    """physics.py:236-247: live actors publish, every empty cell decays."""
    gi = p.gi.ravel()
    C = p.C.reshape(3, -1)
    live = gi[acts.cells] >= 0
    idx = acts.cells[live]
    if len(idx):
        C[:, idx] = acts.comm[live].T
    empty = np.flatnonzero(gi < 0)
    if len(empty):
        C[:, empty] = C[:, empty] * np.float32(0.9)


@_njit
def _settle(tgt, q, src, dirn, infra, gi, rot, ev_t, ev_s, ev_w, ev_d, ev_dir, ev_q):  # pragma: no cover
    # Walk target runs (sorted by target, then q desc, then source asc):
    # sequential f32 sums, first arrival is the candidate winner.
    n = tgt.shape[0]
    m = 0
    a = 0
    while a < n:
        t = tgt[a]
        base = infra[t]
        b = a
        acc = base
        while b < n and tgt[b] == t:
            acc = np.float32(acc + q[b])
            b += 1
        infra[t] = acc
        if q[a] > base:
            ev_t[m] = t
            ev_s[m] = src[a]
            ev_w[m] = gi[src[a]]
            ev_d[m] = gi[t]
            ev_dir[m] = dirn[a]
            ev_q[m] = q[a]
            m += 1
        a = b
    for k in range(m):  # genome writes only after every read
        gi[ev_t[k]] = ev_w[k]
        rot[ev_t[k]] = np.uint8(ev_dir[k])
    return m


def explore(p: Planes, acts: Actions, phys: Phys) -> Events:
    """physics.py:250-343.  Sources: listed cells still alive.  Slot k* =
    first maximal explore actuator; direction PERM[rot, k*];
    q = (f32(alpha) * a[k*]) * I; withdraw all, then per target add
    arrivals in (q desc, source asc) order; first arrival adopts the
    target iff q > infrastructure standing there after withdrawals."""
    h, w = p.shape
    gi = p.gi.ravel()
    live = gi[acts.cells] >= 0
    cells = acts.cells[live]
    if len(cells) == 0:
        return empty_events()
    ex = acts.explore[live]
    n = len(cells)
    k = np.argmax(ex, axis=1)
    rot = p.rot.ravel()
    dirn = PERM[rot[cells].astype(np.int64), k]
    I = p.I.ravel()
    q = (np.float32(phys.explore_fraction) * ex[np.arange(n), k]) * I[cells]
    tx = (cells % w + _DX[dirn]) % w
    ty = (cells // w + _DY[dirn]) % h
    tgt = ty * w + tx
    I[cells] = I[cells] - q
    order = np.lexsort((cells, -q.astype(np.float64), tgt))
    ev = [np.empty(n, np.int64), np.empty(n, np.int64), np.empty(n, np.int32),
          np.empty(n, np.int32), np.empty(n, np.int64), np.empty(n, np.float32)]
    m = _settle(tgt[order], q[order], cells[order], dirn[order], I, gi, rot, *ev)
    return Events(*(a[:m] for a in ev))


def census(gi: np.ndarray, capacity: int) -> np.ndarray:
    """physics.py:395-404: per-slot cell counts of the post-step genome plane."""
    g = gi.ravel()
    return np.bincount(g[g >= 0], minlength=capacity).astype(np.int64)


def physics(p: Planes, acts: Actions, t: int, phys: Phys) -> Events:
    """Phases 5-8 of engine.step (engine.py:240-243) on planes ``p`` in place."""
    energy(p, t, phys)
    invest_liquidate(p, acts, phys)
    communication(p, acts)
    return explore(p, acts, phys)


@dataclass
class StepResult:
    planes: Planes
    actions: Actions
    events: Events
    counts: np.ndarray


def step(front: Planes, t: int, net: Net, phys: Phys, acts: Actions | None = None) -> StepResult:
    """engine.step (engine.py:233-248) without radiation (p_radiation =
    p_merge = 0): sense/act on front, phases on a copy,
    census.  ``acts`` injects an ActionField (parity tier A)."""
    if acts is None:
        acts = act(front, net)
    back = front.copy()
    ev = physics(back, acts, t, phys)
    return StepResult(back, acts, ev, census(back.gi, net.capacity))


# -- digest (engine.py:283-315) ---------------------------------------------------

_FNV_OFFSET = 0xCBF29CE484222325


@_njit
def _fnv(h, data):  # pragma: no cover
    prime = np.uint64(0x100000001B3)
    for k in range(data.size):
        h = (h ^ np.uint64(data[k])) * prime
    return h


def digest(p: Planes) -> int:
    """64-bit FNV-1a over energy, infrastructure, communication x3, genome, rotation bytes."""
    h = np.uint64(_FNV_OFFSET)
    for arr in (p.E, p.I, p.C[0], p.C[1], p.C[2], p.gi, p.rot):
        h = _fnv(h, np.ascontiguousarray(arr).view(np.uint8).reshape(-1))
    return int(h)
