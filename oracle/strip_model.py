"""CPU model of the strip-decomposed two-pass step (TEST INFRASTRUCTURE ONLY).

Restates, in numpy, exactly the decomposition the device uses
(paper_2406_09654_b200/strips.py, csrc/evoca_kernels.cu): pass 1 on a row
strip whose sensed planes carry exchanged ghost rows, then the pull-form
exploration resolve (each target gathers the shipments aimed at it from its
eight neighbours, ordered by the 64-bit key (bits(q) << 32) | ~global_src,
summed sequentially) on a strip whose pass-1 outputs carry exchanged ghost
rows.  Used by the multi-process gloo tests to check, on CPU, that strips +
halo exchange + global tie-break indices + census reduction reproduce the
full-grid oracle (oracle.step, physics.py:250-343) bit for bit.
"""

from __future__ import annotations

import numpy as np

from . import oracle as orc


def pass1(ext_E, ext_I, ext_C, gi, rot, net, phys, t, W):
    """Strip with ghost rows in ext_* ((h+2, W) / (3, h+2, W)); gi, rot (h, W).
    Returns the pass-1 outputs: back E, C (final), and mid I, gi, proposal
    byte, q for the strip interior."""
    h = gi.shape[0]
    # sense / act: the oracle's sensing on the extended planes, rows 1..h
    ext = orc.Planes(ext_E, ext_I, ext_C, np.full((h + 2, W), -1, np.int32), np.zeros((h + 2, W), np.uint8))
    ext.gi[1:h + 1] = gi
    ext.rot[1:h + 1] = rot
    cells_local = np.flatnonzero(gi.ravel() >= 0)
    cells_ext = cells_local + W  # row offset by the ghost row
    acts = np.empty((len(cells_local), 13), np.float32)
    if len(cells_local):
        # row-independent forward: group by slot like the oracle
        s = _sense_ext(ext, cells_ext, W)
        slots = gi.ravel()[cells_local]
        for g in np.unique(slots):
            m = slots == g
            acts[m] = orc.forward(net, int(g), s[m])
    inner = orc.Planes(ext_E[1:h + 1].copy(), ext_I[1:h + 1].copy(), ext_C[:, 1:h + 1].copy(), gi.copy(), rot.copy())
    a = orc.Actions(cells_local.astype(np.int64), acts)
    orc.energy(inner, t, phys)
    orc.invest_liquidate(inner, a, phys)
    orc.communication(inner, a)
    # proposal + withdrawal (physics.py:276-290)
    rp = rot.astype(np.uint8).copy().ravel()
    q = np.zeros(h * W, np.float32)
    giv = inner.gi.ravel()
    live = giv[a.cells] >= 0
    src = a.cells[live]
    if len(src):
        ex = a.explore[live]
        k = np.argmax(ex, axis=1)
        d = orc.PERM[rot.ravel()[src].astype(np.int64), k]
        Iv = inner.I.ravel()
        qq = (np.float32(phys.explore_fraction) * ex[np.arange(len(src)), k]) * Iv[src]
        Iv[src] = Iv[src] - qq
        q[src] = qq
        rp[src] = (rot.ravel()[src] | (d << 3) | 0x40).astype(np.uint8)
    return inner.E, inner.C, inner.I, inner.gi, rp.reshape(h, W), q.reshape(h, W)


def _sense_ext(ext: orc.Planes, cells_ext, W):
    H2 = ext.gi.shape[0]
    stack = np.empty((5, H2 * W), np.float32)
    stack[0] = ext.E.ravel()
    stack[1] = ext.I.ravel()
    stack[2:5] = ext.C.reshape(3, -1)
    out = np.empty((len(cells_ext), 45), np.float32)
    x = cells_ext % W
    y = cells_ext // W
    out[:, 0:5] = stack[:, cells_ext].T
    rot = ext.rot.ravel()[cells_ext].astype(np.int64)
    for s in range(8):
        j = orc.PERM[rot, s]
        ny = y + orc._DY[j]  # ghost rows make the vertical wrap unnecessary
        nx = (x + orc._DX[j]) % W
        out[:, 5 * (s + 1):5 * (s + 2)] = stack[:, ny * W + nx].T
    return out


def pass2(ext_gi, ext_rp, ext_q, mid_I, row0, Hg, W):
    """Pull resolve on a strip.  ext_* (h+2, W) carry ghost rows of the
    pass-1 outputs; mid_I (h, W).  Returns final I, gi, rot and the local
    census-ready genome plane."""
    h = mid_I.shape[0]
    ys, xs = np.mgrid[0:h, 0:W]
    keys = np.zeros((8, h, W), np.uint64)
    qs = np.zeros((8, h, W), np.float32)
    gis = np.zeros((8, h, W), np.int32)
    for d in range(8):
        sy = ys - orc._DY[d] + 1  # extended row index
        sx = (xs - orc._DX[d]) % W
        rpv = ext_rp[sy, sx]
        hit = (rpv & 0x78) == (0x40 | (d << 3))
        qv = (ext_q[sy, sx] + np.float32(0.0)).astype(np.float32)
        grow = (row0 + sy - 1) % Hg
        gsrc = (grow.astype(np.uint64) * np.uint64(W) + sx.astype(np.uint64))
        k = (qv.view(np.uint32).astype(np.uint64) << np.uint64(32)) | (np.uint64(0xFFFFFFFF) - gsrc)
        keys[d] = np.where(hit, k, np.uint64(0))
        qs[d] = qv
        gis[d] = ext_gi[sy, sx]
    before = mid_I
    acc = before.copy()
    order = np.argsort(keys, axis=0)[::-1]  # descending keys; zeros (absent) last
    sk = np.take_along_axis(keys, order, axis=0)
    sq = np.take_along_axis(qs, order, axis=0)
    for i in range(8):
        acc = np.where(sk[i] != 0, (acc + sq[i]).astype(np.float32), acc)
    wq = (sk[0] >> np.uint64(32)).astype(np.uint32).view(np.float32)
    adopt = (sk[0] != 0) & (wq > before)
    wd = order[0]
    wgi = np.take_along_axis(gis, wd[None], axis=0)[0]
    own_gi = ext_gi[1:h + 1]
    own_rot = (ext_rp[1:h + 1] & 7).astype(np.uint8)
    gi = np.where(adopt, wgi, own_gi).astype(np.int32)
    rot = np.where(adopt, wd, own_rot).astype(np.uint8)
    return acc.astype(np.float32), gi, rot, int(adopt.sum())
