"""Physics API of the reference (physics.py), executed on the device.

Same names and contracts as /root/reference/pkg/src/evoca/physics.py:
``KERNEL_OFFSETS``, ``rotation_permutation``, ``PERM_TABLE``,
``PhysicsParams``, ``ActionField``, ``AdoptionEvent(s)`` and the phase
functions ``energy_cycle``, ``apply_invest_liquidate``,
``write_communication``, ``resolve_exploration``, ``census_deaths``, each
mutating a caller-owned ``PlaneSet`` in place.  The phase functions are thin
shims: upload the planes, run the fused pass-1/pass-2 kernels restricted to
the requested phase (EVO_PH_* mask) with the caller's ActionField injected,
download.  The engine's hot path never goes through them; it runs whole
steps device-resident.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib

__all__ = [
    "KERNEL_OFFSETS",
    "PERM_TABLE",
    "PhysicsParams",
    "ActionField",
    "AdoptionEvent",
    "AdoptionEvents",
    "rotation_permutation",
    "step_scalars",
    "energy_cycle",
    "apply_invest_liquidate",
    "write_communication",
    "resolve_exploration",
    "census_deaths",
]

# Moore neighbourhood counterclockwise from east, (dx, dy) (physics.py:40-43).
KERNEL_OFFSETS = np.array(
    [(1, 0), (1, 1), (0, 1), (-1, 1), (-1, 0), (-1, -1), (0, -1), (1, -1)], dtype=np.int64
)


def rotation_permutation(r: int) -> np.ndarray:
    """[r, r+1, r-1, r+2, r-2, r+3, r-3, r+4] mod 8 (physics.py:48-58)."""
    if not 0 <= r < 8:
        raise ValueError("rotation must be in 0..7")
    return np.array([(r + d) % 8 for d in (0, 1, -1, 2, -2, 3, -3, 4)], dtype=np.int64)


PERM_TABLE = np.stack([rotation_permutation(r) for r in range(8)])


@dataclass
class PhysicsParams:
    """Environmental constants (physics.py:65-94); steerable between steps."""

    cycle_amplitude: float = 0.1
    cycle_period: int = 100
    energy_source_map: Optional[np.ndarray] = None
    drain_fraction: float = 0.05
    invest_rate: float = 1.0
    liquidate_rate: float = 1.0
    invest_efficiency: float = 0.9
    liquidate_efficiency: float = 0.9
    explore_fraction: float = 0.5
    upkeep: float = 0.02
    decay_on_starvation: float = 0.1
    death_threshold: float = 1e-3

    def validate(self) -> None:
        if self.cycle_period < 2:
            raise ValueError("cycle_period must be >= 2")
        if self.cycle_amplitude < 0:
            raise ValueError("cycle_amplitude must be non-negative")
        for name in ("drain_fraction", "invest_efficiency", "liquidate_efficiency",
                     "explore_fraction", "decay_on_starvation"):
            v = getattr(self, name)
            if not 0.0 <= v <= 1.0:
                raise ValueError(f"{name} must be in [0, 1], got {v}")
        for name in ("invest_rate", "liquidate_rate", "upkeep", "death_threshold"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be non-negative")


def step_scalars(t: int, params) -> _lib.EvoScalars:
    """Per-step scalars for the kernels, computed exactly as the reference
    does on the host: rho = A*sin(2*pi*t/P) in float64 (physics.py:186), its
    sign picks day/night, then the np.float32 casts (physics.py:187-194,
    218-233, 286)."""
    rho = params.cycle_amplitude * math.sin(2.0 * math.pi * t / params.cycle_period)
    s = _lib.EvoScalars()
    if rho > 0.0:
        s.rho_mode, s.rho_f32, s.drain_f32 = 1, float(np.float32(rho)), 0.0
    elif rho < 0.0:
        s.rho_mode, s.rho_f32, s.drain_f32 = 2, 0.0, float(np.float32(params.drain_fraction * -rho))
    else:
        s.rho_mode, s.rho_f32, s.drain_f32 = 0, 0.0, 0.0
    f = lambda v: float(np.float32(v))  # noqa: E731
    s.invest_rate = f(params.invest_rate)
    s.liquidate_rate = f(params.liquidate_rate)
    s.invest_efficiency = f(params.invest_efficiency)
    s.liquidate_efficiency = f(params.liquidate_efficiency)
    s.explore_fraction = f(params.explore_fraction)
    s.upkeep = f(params.upkeep)
    s.decay_on_starvation = f(params.decay_on_starvation)
    s.death_threshold = f(params.death_threshold)
    return s


@dataclass
class ActionField:
    """Controller outputs for cells occupied at sensing time, ascending
    (physics.py:97-119)."""

    cells: np.ndarray
    invest: np.ndarray
    liquidate: np.ndarray
    comm: np.ndarray
    explore: np.ndarray

    @staticmethod
    def empty() -> "ActionField":
        return ActionField(
            cells=np.empty(0, np.int64), invest=np.empty(0, np.float32),
            liquidate=np.empty(0, np.float32), comm=np.empty((0, 3), np.float32),
            explore=np.empty((0, 8), np.float32),
        )

    def block(self) -> np.ndarray:
        """(n,13) f32 in the reference column order (engine.py:224-230)."""
        n = len(self.cells)
        out = np.empty((n, 13), np.float32)
        out[:, 0] = self.invest
        out[:, 1] = self.liquidate
        out[:, 2:5] = self.comm
        out[:, 5:13] = self.explore
        return out

    @staticmethod
    def from_block(cells: np.ndarray, a: np.ndarray) -> "ActionField":
        a = np.asarray(a, np.float32)
        return ActionField(np.asarray(cells, np.int64), a[:, 0].copy(), a[:, 1].copy(),
                           a[:, 2:5].copy(), a[:, 5:13].copy())


@dataclass(frozen=True)
class AdoptionEvent:
    target: int
    source: int
    winner_slot: int
    defender_slot: int
    direction: int
    quantity: float


@dataclass
class AdoptionEvents:
    """Takeovers of one step, ascending target (physics.py:134-175)."""

    target: np.ndarray
    source: np.ndarray
    winner_slot: np.ndarray
    defender_slot: np.ndarray
    direction: np.ndarray
    quantity: np.ndarray

    def __len__(self) -> int:
        return len(self.target)

    @staticmethod
    def empty() -> "AdoptionEvents":
        return AdoptionEvents(
            np.empty(0, np.int64), np.empty(0, np.int64), np.empty(0, np.int32),
            np.empty(0, np.int32), np.empty(0, np.int64), np.empty(0, np.float32),
        )

    def aslist(self) -> list[AdoptionEvent]:
        return [
            AdoptionEvent(int(t), int(s), int(w), int(d), int(r), float(q))
            for t, s, w, d, r, q in zip(self.target, self.source, self.winner_slot,
                                        self.defender_slot, self.direction, self.quantity)
        ]


# -- phase shims: operate on a host PlaneSet through the device ---------------


def _run_phases(planes, actions: ActionField, params, t: int, phases: int, record: bool):
    from .device import DeviceSubstrate  # local import: device needs the library

    h, w = planes.genome_index.shape
    cap = max(1, int(planes.genome_index.max()) + 1)
    dev = DeviceSubstrate(w, h, capacity=cap, hidden=0)
    try:
        dev.upload(planes)
        dev.set_actions(actions.cells, actions.block())
        dev.step_raw(step_scalars(t, params), t, phases=phases,
                     flags=_lib.F_INJECT_ACTIONS | (_lib.F_RECORD_EVENTS if record else 0),
                     source_map=params.energy_source_map)
        ev = dev.read_events() if record else None
        dev.download(planes)
        return ev
    finally:
        dev.close()


def energy_cycle(planes, t: int, params: PhysicsParams) -> None:
    """Day/night source term on every cell (physics.py:178-194)."""
    _run_phases(planes, ActionField.empty(), params, t, _lib.PH_ENERGY, False)


def apply_invest_liquidate(planes, actions: ActionField, params: PhysicsParams) -> None:
    """Invest, liquidate, upkeep, starvation, death (physics.py:197-233)."""
    _run_phases(planes, actions, params, 0, _lib.PH_INVEST, False)


def write_communication(planes, actions: ActionField) -> None:
    """Publish comm actuators; decay empty cells by 0.9 (physics.py:236-247)."""
    _run_phases(planes, actions, PhysicsParams(), 0, _lib.PH_COMM, False)


def resolve_exploration(planes, actions: ActionField, params: PhysicsParams) -> AdoptionEvents:
    """Ship, resolve contested targets, adopt (physics.py:250-343)."""
    return _run_phases(planes, actions, params, 0, _lib.PH_EXPLORE, True)


def census_deaths(planes, pool, step: int) -> list[int]:
    """Count cells per slot and retire slots that lost every cell
    (physics.py:395-404).  Host bincount: a census needs the plane on host
    anyway when called through this per-phase API."""
    gi = planes.genome_index
    counts = np.bincount(gi[gi >= 0], minlength=pool.capacity)
    return pool.update_census(counts, step)
