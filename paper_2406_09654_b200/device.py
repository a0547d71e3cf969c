"""Device-resident substrate: a Python handle on one ``evo_ctx``.

Everything here is a thin wrapper over the C ABI (include/evoca_b200.h); the
arrays passed in are host numpy arrays (pinned ones make the transfers
asynchronous when a stream is given).  Streams are raw ``cudaStream_t``
handles as integers (e.g. ``torch.cuda.current_stream().cuda_stream``);
``None`` uses the context's own stream and makes transfers synchronous.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check, ptr
from .hypernet import N_ACTUATORS, N_SENSORS, pack_params
from .physics import AdoptionEvents

__all__ = ["DeviceSubstrate"]

PLANES = {"energy": 0, "infra": 1, "comm": 2, "genome": 3, "rotation": 4,
          "mid_infra": 5, "mid_genome": 6, "mid_proposal": 7, "mid_quantity": 8,
          "census_counts": 9, "stats": 10}


def _stream(s):
    """None -> the context's own stream (NULL); 0 (a framework's handle for
    the legacy default stream) -> cudaStreamLegacy; else the raw handle."""
    if s is None:
        return None
    s = int(s)
    return C.c_void_p(1 if s == 0 else s)


def _arrays_of(planes):
    """(E, I, C, gi, rot) views of a PlaneSet-like object (reference
    PlaneSet, this package's mirror, or anything with E/I/C/gi/rot)."""
    if hasattr(planes, "channels"):
        return (planes.channels["energy"][0], planes.channels["infrastructure"][0],
                planes.channels["communication"], planes.genome_index, planes.rotation)
    return planes.E, planes.I, planes.C, planes.gi, planes.rot


class DeviceSubstrate:
    def __init__(self, width: int, height: int, capacity: int, hidden: int = 0, device: int = 0,
                 row0: int | None = None, height_global: int | None = None):
        self.lib = _lib.load()
        self.width, self.height, self.capacity, self.hidden = width, height, capacity, hidden
        self.row0 = 0 if row0 is None else int(row0)
        self.height_global = height if height_global is None else int(height_global)
        self.strip = row0 is not None
        ctx = C.c_void_p()
        if self.strip:
            check(self.lib.evo_create_strip(C.byref(ctx), width, height, self.row0, self.height_global,
                                            capacity, hidden, device))
        else:
            check(self.lib.evo_create(C.byref(ctx), width, height, capacity, hidden, device))
        self.ctx = ctx
        self._src_map_id = None
        self._pinned = {}

    # -- lifetime -------------------------------------------------------------
    def close(self) -> None:
        for key in list(getattr(self, "_pinned", {})):
            self.lib.evo_host_unregister(C.c_void_p(key))
        self._pinned = {}
        if self.ctx:
            self.lib.evo_destroy(self.ctx)
            self.ctx = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    # -- state transfer -------------------------------------------------------
    def _check_shapes(self, E, I, Cm, gi, rot):
        h, w = self.height, self.width
        if E.shape != (h, w) or I.shape != (h, w) or Cm.shape != (3, h, w) or gi.shape != (h, w) or rot.shape != (h, w):
            raise ValueError("plane shapes do not match the device substrate")
        if E.dtype != np.float32 or I.dtype != np.float32 or Cm.dtype != np.float32:
            raise ValueError("channel planes must be float32")
        if gi.dtype != np.int32 or rot.dtype != np.uint8:
            raise ValueError("genome_index must be int32 and rotation uint8")

    def upload_arrays(self, E, I, Cm, gi, rot, stream=None) -> None:
        E, I, Cm, gi, rot = (np.ascontiguousarray(a) for a in (E, I, Cm, gi, rot))
        self._check_shapes(E, I, Cm, gi, rot)
        if rot.size and rot.max() > 7:
            raise ValueError("rotation must be in 0..7")
        if gi.size and gi.max() >= self.capacity:
            raise ValueError("genome_index refers to a slot outside the pool capacity")
        self._keep = (E, I, Cm, gi, rot)  # keep alive across async copies
        check(self.lib.evo_upload_planes(self.ctx, ptr(E), ptr(I), ptr(Cm), ptr(gi), ptr(rot), _stream(stream)))

    def step_host(self, front, back, scalars, t: int, flags: int = 0, bands: int = 0, source_map=None,
                  stream=None):
        """One step of host-resident planes (evo_step_host): uploads `front`,
        steps, writes the new planes into `back`, pipelined over row bands.
        Returns (census counts or None, adoptions, extinctions)."""
        if self.strip:
            raise ValueError("step_host steps a single-strip context")
        src = [np.ascontiguousarray(a) for a in _arrays_of(front)]
        self._check_shapes(*src)
        dst = list(_arrays_of(back))
        self._check_shapes(*dst)
        for a in dst:
            if not a.flags["C_CONTIGUOUS"] or not a.flags["WRITEABLE"]:
                raise ValueError("step_host targets must be writeable C-contiguous arrays")
        if source_map is not None or self._src_map_id is not None:
            if source_map is None or id(source_map) != self._src_map_id:
                self.set_source_map(source_map)
        census = not (flags & _lib.F_NO_CENSUS)
        counts = np.empty(self.capacity, np.int32) if census else None
        st = np.zeros(2, np.int64)
        check(self.lib.evo_step_host(self.ctx, C.byref(scalars), int(t), int(flags), *(ptr(a) for a in src),
                                     *(ptr(a) for a in dst), ptr(counts), ptr(st), int(bands), _stream(stream)))
        return counts, int(st[0]), int(st[1])

    def render_rgb(self, norm_energy: float = 1.0, norm_infrastructure: float = 1.0) -> np.ndarray:
        """(H, W, 4) uint8 RGBA frame of the device front (evo_render_rgb)."""
        px = np.empty((self.height, self.width, 4), np.uint8)
        check(self.lib.evo_render_rgb(self.ctx, float(norm_energy), float(norm_infrastructure), ptr(px), None))
        return px

    def download_arrays(self, E, I, Cm, gi, rot, stream=None) -> None:
        for a in (E, I, Cm, gi, rot):
            if a is not None and not a.flags["C_CONTIGUOUS"]:
                raise ValueError("download targets must be C-contiguous")
        check(self.lib.evo_download_planes(self.ctx, ptr(E), ptr(I), ptr(Cm), ptr(gi), ptr(rot), _stream(stream)))

    def pin(self, planes) -> None:
        """Page-lock a PlaneSet's arrays (evo_host_register) so that uploads
        and downloads are direct DMA; the arrays are kept alive and unpinned
        by close()."""
        for a in _arrays_of(planes):
            base = a
            while isinstance(base, np.ndarray) and base.base is not None and isinstance(base.base, np.ndarray):
                base = base.base
            key = base.ctypes.data
            if key in self._pinned:
                continue
            check(self.lib.evo_host_register(C.c_void_p(key), base.nbytes))
            self._pinned[key] = base

    def upload(self, planes, stream=None) -> None:
        self.upload_arrays(*_arrays_of(planes), stream=stream)

    def download(self, planes, stream=None) -> None:
        E, I, Cm, gi, rot = _arrays_of(planes)
        self.download_arrays(E, I, Cm, gi, rot, stream=stream)

    # -- parameters -----------------------------------------------------------
    def set_params_arrays(self, slot0: int, w1, b1, w2, b2) -> None:
        n = w2.shape[0]
        arrs = [None if a is None else np.ascontiguousarray(a, np.float32) for a in (w1, b1, w2, b2)]
        check(self.lib.evo_set_params(self.ctx, slot0, n, *(ptr(a) for a in arrs)))

    def set_params(self, params_list, slot0: int = 0) -> None:
        self.set_params_arrays(slot0, *pack_params(params_list, self.hidden))

    def set_slots(self, state: np.ndarray, peak: np.ndarray | None = None) -> None:
        st = np.ascontiguousarray(state, np.int8)
        pk = None if peak is None else np.ascontiguousarray(peak, np.int32)
        if st.shape != (self.capacity,):
            raise ValueError("slot state must have one entry per slot")
        check(self.lib.evo_set_slots(self.ctx, ptr(st), ptr(pk)))

    def set_source_map(self, m) -> None:
        if m is None:
            if self._src_map_id is not None:
                check(self.lib.evo_set_source_map(self.ctx, None))
            self._src_map_id = None
            return
        a = np.ascontiguousarray(m, np.float32)
        if a.shape != (self.height, self.width):
            raise ValueError("energy_source_map must be (H, W)")
        check(self.lib.evo_set_source_map(self.ctx, ptr(a)))
        self._src_map_id = id(m)

    # -- stepping -------------------------------------------------------------
    def step_raw(self, scalars, t: int, phases: int = _lib.PH_ALL, flags: int = 0, stream=None,
                 source_map=None) -> None:
        if source_map is not None or self._src_map_id is not None:
            if source_map is None or id(source_map) != self._src_map_id:
                self.set_source_map(source_map)
        check(self.lib.evo_step(self.ctx, C.byref(scalars), int(t), phases, flags, _stream(stream)))

    def profile(self, enable: bool = True) -> None:
        """Per-step device timing of ``evo_step`` / ``evo_run`` (start, between the passes, end)."""
        check(self.lib.evo_profile(self.ctx, 1 if enable else 0))

    def profile_read(self):
        """(pass-1 ms, pass-2 ms, steps) summed over the steps recorded since the last read."""
        a, b, n = C.c_double(), C.c_double(), C.c_int()
        check(self.lib.evo_profile_read(self.ctx, C.byref(a), C.byref(b), C.byref(n)))
        return a.value, b.value, n.value

    def pass1(self, scalars, t: int, phases: int = _lib.PH_ALL, flags: int = 0, stream=None) -> None:
        check(self.lib.evo_pass1(self.ctx, C.byref(scalars), int(t), phases, flags, _stream(stream)))

    def pass2(self, t: int, flags: int = 0, stream=None) -> None:
        check(self.lib.evo_pass2(self.ctx, int(t), flags, _stream(stream)))

    def census_finish(self, t: int, stream=None) -> None:
        check(self.lib.evo_census_finish(self.ctx, int(t), _stream(stream)))

    def swap(self) -> None:
        check(self.lib.evo_swap(self.ctx))

    def run(self, scalars_list, t0: int, stream=None, source_map=None) -> None:
        k = len(scalars_list)
        if k == 0:
            return
        if source_map is not None or self._src_map_id is not None:
            if source_map is None or id(source_map) != self._src_map_id:
                self.set_source_map(source_map)
        arr = (_lib.EvoScalars * k)(*scalars_list)
        check(self.lib.evo_run(self.ctx, arr, int(t0), k, _stream(stream)))

    def refresh_ghosts(self, stream=None) -> None:
        check(self.lib.evo_refresh_ghosts(self.ctx, _stream(stream)))

    def sync(self) -> None:
        check(self.lib.evo_sync(self.ctx))

    # -- parity-mode action transfer -------------------------------------------
    def set_actions(self, cells, block) -> None:
        cells = np.ascontiguousarray(cells, np.int64)
        block = np.ascontiguousarray(block, np.float32).reshape(len(cells), N_ACTUATORS)
        check(self.lib.evo_set_actions(self.ctx, ptr(cells), len(cells), ptr(block)))

    def get_actions(self):
        n = C.c_int64()
        cap = self.width * self.height
        cells = np.empty(cap, np.int64)
        acts = np.empty((cap, N_ACTUATORS), np.float32)
        check(self.lib.evo_get_actions(self.ctx, cap, ptr(cells), ptr(acts), C.byref(n)))
        return cells[: n.value].copy(), acts[: n.value].copy()

    # -- results --------------------------------------------------------------
    def read_census(self):
        counts = np.empty(self.capacity, np.int32)
        state = np.empty(self.capacity, np.int8)
        death = np.empty(self.capacity, np.int64)
        peak = np.empty(self.capacity, np.int32)
        check(self.lib.evo_read_census(self.ctx, ptr(counts), ptr(state), ptr(death), ptr(peak)))
        return counts, state, death, peak

    def census_take(self) -> np.ndarray:
        """Counts accumulated by an EVO_F_NO_CENSUS step, cleared on the device."""
        counts = np.empty(self.capacity, np.int32)
        check(self.lib.evo_census_take(self.ctx, ptr(counts)))
        return counts

    def read_stats(self):
        a, e = C.c_int64(), C.c_int64()
        check(self.lib.evo_read_stats(self.ctx, C.byref(a), C.byref(e)))
        return a.value, e.value

    def read_events(self) -> AdoptionEvents:
        cap = self.width * self.height
        t = np.empty(cap, np.int64)
        s = np.empty(cap, np.int64)
        w = np.empty(cap, np.int32)
        d = np.empty(cap, np.int32)
        r = np.empty(cap, np.int64)
        q = np.empty(cap, np.float32)
        m = C.c_int64()
        check(self.lib.evo_read_events(self.ctx, cap, ptr(t), ptr(s), ptr(w), ptr(d), ptr(r), ptr(q), C.byref(m)))
        k = m.value
        return AdoptionEvents(t[:k].copy(), s[:k].copy(), w[:k].copy(), d[:k].copy(), r[:k].copy(), q[:k].copy())

    def patch_genomes(self, cells, slots) -> None:
        cells = np.ascontiguousarray(cells, np.int64)
        slots = np.ascontiguousarray(slots, np.int32)
        check(self.lib.evo_patch_genomes(self.ctx, ptr(cells), ptr(slots), len(cells)))

    def get_params_arrays(self, slot0: int, n: int):
        """Read slots [slot0, slot0+n) back (evo_get_params): (w1, b1, w2, b2)
        in the reference layouts; w1/b1 are None for a direct substrate."""
        H = self.hidden
        w1 = np.zeros((n, H, N_SENSORS), np.float32) if H else None
        b1 = np.zeros((n, H), np.float32) if H else None
        w2 = np.zeros((n, N_ACTUATORS, H if H else N_SENSORS), np.float32)
        b2 = np.zeros((n, N_ACTUATORS), np.float32)
        check(self.lib.evo_get_params(self.ctx, slot0, n, ptr(w1), ptr(b1), ptr(w2), ptr(b2)))
        return w1, b1, w2, b2

    def express_cppn(self, slots, genomes, tau: float = 0.2, w_max: float = 3.0, stream=None,
                     programs=None) -> None:
        """Generate the dense tables of ``slots`` from their pattern networks
        on the device (evo_express_cppn; reference generate_network,
        hypernet.py:183-220).  ``genomes`` are reference or neat.CppnGenome
        objects (``programs``: their neat.compile_programs arrays, if already
        compiled); returns once the tables are written."""
        from . import neat

        slots = np.ascontiguousarray(slots, np.int32)
        if len(slots) != len(genomes):
            raise ValueError("one genome per slot")
        if len(slots) == 0:
            return
        node_off, nodes, esrc, ew, outs = programs if programs is not None else neat.compile_programs(genomes)
        if len(node_off) != len(slots) + 1:
            raise ValueError("programs do not match the genomes")
        coords = neat.layout_coords(self.hidden)
        check(self.lib.evo_express_cppn(self.ctx, len(slots), ptr(slots), ptr(node_off), ptr(nodes), ptr(esrc),
                                        ptr(ew), ptr(outs), ptr(coords), float(tau), float(w_max), _stream(stream)))

    def select_cells(self, key: int, p: float):
        """Field-radiation selection on the front genome plane
        (evo_select_cells): returns (per-slot selected counts, n selected)."""
        counts = np.zeros(self.capacity, np.int32)
        n = C.c_int64()
        lo, hi = int(key) & 0xFFFFFFFFFFFFFFFF, (int(key) >> 64) & 0xFFFFFFFFFFFFFFFF
        check(self.lib.evo_select_cells(self.ctx, lo, hi, float(p), ptr(counts), C.byref(n)))
        return counts, n.value

    def count_occupied(self) -> int:
        """Occupied cells of the front genome plane (evo_count_occupied)."""
        n = C.c_int64()
        check(self.lib.evo_count_occupied(self.ctx, C.byref(n)))
        return n.value

    def select_cells_at(self, key: int, p: float, first_draw: int):
        """evo_select_cells_at: the selection of a row strip whose occupied
        cells take draws first_draw, first_draw + 1, ... of the stream."""
        counts = np.zeros(self.capacity, np.int32)
        n = C.c_int64()
        lo, hi = int(key) & 0xFFFFFFFFFFFFFFFF, (int(key) >> 64) & 0xFFFFFFFFFFFFFFFF
        check(self.lib.evo_select_cells_at(self.ctx, lo, hi, float(p), int(first_draw), ptr(counts), C.byref(n)))
        return counts, n.value

    def read_selected(self) -> np.ndarray:
        n = C.c_int64()
        check(self.lib.evo_read_selected(self.ctx, 0, None, C.byref(n)))
        cells = np.zeros(max(n.value, 1), np.int64)
        check(self.lib.evo_read_selected(self.ctx, len(cells), ptr(cells), C.byref(n)))
        return cells[:n.value]

    def remap_selected(self, slot_map) -> None:
        slot_map = np.ascontiguousarray(slot_map, np.int32)
        if slot_map.shape != (self.capacity,):
            raise ValueError("slot map needs one entry per pool slot")
        check(self.lib.evo_remap_selected(self.ctx, ptr(slot_map)))

    def plane_ptr(self, which: str, buffer: int = 0):
        p = C.c_void_p()
        stride = C.c_int64()
        check(self.lib.evo_plane_ptr(self.ctx, PLANES[which], buffer, C.byref(p), C.byref(stride)))
        return p.value, stride.value
