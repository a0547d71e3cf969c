"""Observables of the substrate (metrics.py of the reference): multi-scale
complexity and census rows, computed on the device when the state's newest
planes live there.

* ``msc(field, n_scales)`` / ``msc_of_substrate(sub, channel, sub_plane)``
  restate metrics.py:57-103 on the host (f64 block means with sorted
  members, overlaps by math.fsum).
* ``msc_of_substrate(state, ...)`` for a state bound to a device context
  whose front is newer than the host mirror runs ``evo_msc``: the block-mean
  pyramid and the overlaps' exact sums on the device (4^k-fold repetition of
  the distinct products folded in exactly), bit-identical to the host
  result, with 32 + 31 doubles instead of the planes crossing PCIe.
* ``census(sub_or_state, pool, step)`` (metrics.py:200-213): float64 plane
  totals in numpy's summation order, on the device via ``evo_plane_sums``.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib

__all__ = ["MscReport", "msc", "msc_of_substrate", "CensusRow", "census"]

_PLANE_INDEX = {("energy", 0): 0, ("infrastructure", 0): 1, ("communication", 0): 2, ("communication", 1): 3,
                ("communication", 2): 4}


@dataclass(frozen=True)
class MscReport:
    """Per-scale complexity contributions and their sum (metrics.py:40-47)."""

    contributions: tuple
    total: float
    side: int
    channel: Optional[str] = None


def _block_means(f: np.ndarray) -> np.ndarray:
    q = np.sort(np.stack([f[0::2, 0::2], f[0::2, 1::2], f[1::2, 0::2], f[1::2, 1::2]]), axis=0)
    return ((q[0] + q[1]) + (q[2] + q[3])) * 0.25


def _overlap(a: np.ndarray, b: np.ndarray, side: int) -> float:
    fa = np.repeat(np.repeat(a, side // a.shape[0], axis=0), side // a.shape[1], axis=1)
    fb = np.repeat(np.repeat(b, side // b.shape[0], axis=0), side // b.shape[1], axis=1)
    return math.fsum((fa * fb).ravel().tolist()) / (side * side)


def _report(o_diag, cross, side, channel=None) -> MscReport:
    contribs = [abs(c - 0.5 * (o_diag[k] + o_diag[k + 1])) for k, c in enumerate(cross)]
    return MscReport(tuple(contribs), math.fsum(contribs), side, channel)


def msc(field: np.ndarray, n_scales: Optional[int] = None) -> MscReport:
    """Multi-scale complexity of a square power-of-two field (metrics.py:65-90)."""
    f = np.asarray(field, dtype=np.float64)
    if f.ndim != 2 or f.shape[0] != f.shape[1]:
        raise ValueError("field must be square")
    side = f.shape[0]
    if side < 2 or side & (side - 1):
        raise ValueError("field side must be a power of two >= 2")
    max_scales = side.bit_length() - 1
    k_max = max_scales if n_scales is None else min(n_scales, max_scales)
    if k_max < 1:
        raise ValueError("n_scales must be >= 1")
    fields = [f]
    for _ in range(k_max):
        fields.append(_block_means(fields[-1]))
    o_diag = [_overlap(g, g, side) for g in fields]
    cross = [_overlap(fields[k], fields[k + 1], side) for k in range(k_max)]
    return _report(o_diag, cross, side)


def _device_ahead(obj):
    b = getattr(obj, "_evo_binding", None)
    return b if b is not None and b.device_ahead and not b.dev.strip else None


def msc_device(dev, channel: str = "infrastructure", sub_plane: int = 0, n_scales: Optional[int] = None) -> MscReport:
    """MSC of one plane of a DeviceSubstrate's front (evo_msc)."""
    key = (channel, sub_plane)
    if key not in _PLANE_INDEX:
        raise ValueError(f"unknown plane {channel}[{sub_plane}]")
    if n_scales is not None and n_scales < 1:
        raise ValueError("n_scales must be >= 1")
    sq = np.zeros(32, np.float64)
    cr = np.zeros(31, np.float64)
    side, k_max = C.c_int(), C.c_int()
    _lib.check(dev.lib.evo_msc(dev.ctx, _PLANE_INDEX[key], 0 if n_scales is None else int(n_scales), _lib.ptr(sq),
                               _lib.ptr(cr), C.byref(side), C.byref(k_max)))
    s, km = side.value, k_max.value
    o_diag = [math.ldexp(float(sq[k]), 2 * k) / (s * s) for k in range(km + 1)]
    cross = [math.ldexp(float(cr[k]), 2 * k) / (s * s) for k in range(km)]
    return _report(o_diag, cross, s, channel)


def msc_of_substrate(sub, channel: str = "infrastructure", sub_plane: int = 0) -> MscReport:
    """MSC of one front plane, centre-cropped to a power-of-two square
    (metrics.py:93-103).  ``sub`` may be a Substrate or a SimState; a state
    whose newest planes are on the device is measured there."""
    b = _device_ahead(sub)
    if b is not None:
        return msc_device(b.dev, channel, sub_plane)
    sub = getattr(sub, "substrate", sub)
    plane = sub.front.channels[channel][sub_plane]
    h, w = plane.shape
    side = 1 << min(h.bit_length() - 1, w.bit_length() - 1)
    y0, x0 = (h - side) // 2, (w - side) // 2
    r = msc(plane[y0:y0 + side, x0:x0 + side])
    return MscReport(r.contributions, r.total, side, channel)


@dataclass(frozen=True)
class CensusRow:
    step: int
    live_genomes: int
    total_energy: float
    total_infrastructure: float
    extinctions: int


def census(sub, pool=None, step: Optional[int] = None) -> CensusRow:
    """Population and stock totals (metrics.py:200-213).  ``sub`` may be a
    Substrate (with ``pool``) or a SimState; plane totals of a state whose
    newest planes are on the device are summed there in numpy's order."""
    b = _device_ahead(sub)
    if pool is None:
        pool = sub.pool
    if b is not None:
        from .engine import _fold_census

        _fold_census(sub)  # pool liveness / deaths up to date without downloading planes
        e, i = C.c_double(), C.c_double()
        _lib.check(b.dev.lib.evo_plane_sums(b.dev.ctx, C.byref(e), C.byref(i)))
        s = sub.substrate
        t = s.step_counter if step is None else step
        return CensusRow(t, pool.live_count(), e.value, i.value, len(pool.deaths_at(t)))
    s = getattr(sub, "substrate", sub)
    t = s.step_counter if step is None else step
    front = s.front
    return CensusRow(
        step=t,
        live_genomes=pool.live_count(),
        total_energy=float(front.channels["energy"][0].sum(dtype=np.float64)),
        total_infrastructure=float(front.channels["infrastructure"][0].sum(dtype=np.float64)),
        extinctions=len(pool.deaths_at(t)),
    )
