"""Row-strip sharding of the torus over GPUs.

Each rank owns rows [row0, row0 + h) of the global H x W torus (x wraps
locally, y wraps across rank world-1 <-> 0) as a strip context
(evo_create_strip) whose planes carry one ghost row above and below.  The
step's dependency radius is 2, split over the two passes:

  1. before pass 1 the sensed front planes (E, I, C0..C2) exchange their
     boundary rows with the neighbours (ghost rows -1 and h);
  2. pass 1 (sense, controller, physics tail, shipment proposal);
  3. the pass-1 outputs a neighbour's pass 2 needs - proposal byte,
     shipped quantity, post-death genome - exchange boundary rows;
  4. pass 2 (pull resolve, adoption) accumulates per-rank census counts;
  5. the counts are summed over ranks (all_reduce) and every rank runs the
     identical census epilogue, then swaps.

Tie-breaks use global linear source indices ((row0 + y) * W + x), so the
result is bit-identical for any number of strips (tests/test_strips*.py).
Exchanges go through ``torch.distributed`` point-to-point operations
(NCCL over NVLink on GPUs, gloo on CPU), batched per exchange.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["StripPlan", "HaloComm", "StagedHaloComm", "DeviceStrip", "cuda_view"]


@dataclass(frozen=True)
class StripPlan:
    height: int
    width: int
    world: int

    def __post_init__(self):
        if self.world < 1 or self.height < self.world:
            raise ValueError("need at least one row per strip")

    def rows(self, rank: int) -> tuple[int, int]:
        """(row0, h): balanced split, the first H % world ranks one row longer."""
        base, extra = divmod(self.height, self.world)
        h = base + (1 if rank < extra else 0)
        row0 = rank * base + min(rank, extra)
        return row0, h

    def up(self, rank: int) -> int:
        """Rank owning global row row0 - 1."""
        return (rank - 1) % self.world

    def down(self, rank: int) -> int:
        """Rank owning global row row0 + h."""
        return (rank + 1) % self.world


class HaloComm:
    """Boundary-row exchange between vertically adjacent strips.

    ``exchange(first, last, ghost_top, ghost_bottom)``: this rank's first
    row goes to the upper neighbour (its ghost bottom), its last row to the
    lower neighbour (its ghost top); the ghosts are filled likewise.  Works
    on CUDA tensors (NCCL) and CPU tensors (gloo); with one rank it is a
    local wrap copy.  The order of the four operations is the same on every
    rank so that with two ranks (up == down) the per-peer matching is right.
    """

    def __init__(self, rank: int = 0, world: int = 1, group=None):
        self.rank, self.world, self.group = rank, world, group

    def exchange(self, first, last, ghost_top, ghost_bottom) -> None:
        if self.world == 1:
            ghost_bottom.copy_(first)
            ghost_top.copy_(last)
            return
        import torch.distributed as dist

        up = (self.rank - 1) % self.world
        down = (self.rank + 1) % self.world
        ops = [
            dist.P2POp(dist.isend, first.contiguous(), up, self.group),
            dist.P2POp(dist.isend, last.contiguous(), down, self.group),
            dist.P2POp(dist.irecv, ghost_bottom, down, self.group),
            dist.P2POp(dist.irecv, ghost_top, up, self.group),
        ]
        for r in dist.batch_isend_irecv(ops):
            r.wait()

    def sum_(self, t) -> None:
        if self.world == 1:
            return
        import torch.distributed as dist

        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)


class StagedHaloComm(HaloComm):
    """HaloComm over a host-side process group (gloo): device rows are staged
    through host memory around each exchange and reduction.  For runs whose
    ranks share a GPU or have no NCCL (tests, CPU-only launchers); the
    exchange pattern and results are those of the device path."""

    def exchange(self, first, last, ghost_top, ghost_bottom) -> None:
        if not first.is_cuda:
            return super().exchange(first, last, ghost_top, ghost_bottom)
        import torch

        torch.cuda.current_stream().synchronize()
        gt, gb = ghost_top.cpu(), ghost_bottom.cpu()
        super().exchange(first.cpu(), last.cpu(), gt, gb)
        ghost_top.copy_(gt)
        ghost_bottom.copy_(gb)

    def sum_(self, t) -> None:
        if not t.is_cuda:
            return super().sum_(t)
        import torch

        torch.cuda.current_stream().synchronize()
        h = t.cpu()
        super().sum_(h)
        t.copy_(h)


class _CudaArray:
    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


_TYPESTR = {np.float32: "<f4", np.int32: "<i4", np.uint8: "|u1", np.int64: "<i8"}


def cuda_view(ptr: int, shape, dtype):
    """A torch CUDA tensor aliasing device memory owned by the C ABI."""
    import torch

    return torch.as_tensor(_CudaArray(ptr, shape, _TYPESTR[dtype]), device="cuda")


class DeviceStrip:
    """One rank's strip on its GPU, stepped with halo exchanges."""

    FRONT = (("energy", 0), ("infra", 0), ("comm", 0), ("comm", 1), ("comm", 2))

    def __init__(self, plan: StripPlan, rank: int, capacity: int, hidden: int = 0, device: int = 0,
                 comm: HaloComm | None = None):
        from .device import DeviceSubstrate

        self.plan, self.rank = plan, rank
        self.row0, self.h = plan.rows(rank)
        self.W = plan.width
        self.dev = DeviceSubstrate(plan.width, self.h, capacity, hidden, device, row0=self.row0,
                                   height_global=plan.height)
        self.comm = comm or HaloComm(rank, plan.world)
        # field radiation's selection buffers are allocated now, as the single
        # context's binding does (engine.py: select_cells(0, 0.0)), not inside
        # the first radiation event of a run
        self.dev.count_occupied()
        self.dev.select_cells_at(0, 0.0, 0)

    # -- views ----------------------------------------------------------------
    def _plane(self, which: str, buffer: int, sub: int, dtype):
        ptr, stride = self.dev.plane_ptr(which, buffer)
        item = np.dtype(dtype).itemsize
        return cuda_view(ptr + sub * stride * item, (self.h + 2, self.W), dtype)

    def _rows(self, plane):
        return plane[1], plane[self.h], plane[0], plane[self.h + 1]  # first, last, ghost top, ghost bottom

    def _halo_buffers(self, which: int):
        """Persistent (2, planes * W) int32 device buffers: send [first; last]
        rows, recv [ghost above; ghost below] (evo_halo_pack / _unpack)."""
        import torch

        from ._lib import check

        bufs = self.__dict__.setdefault("_halo", {})
        if which not in bufs:
            import ctypes as C

            words = C.c_int64()
            check(self.dev.lib.evo_halo_row_words(self.dev.ctx, which, C.byref(words)))
            mk = lambda: torch.empty((2, words.value), dtype=torch.int32, device="cuda")  # noqa: E731
            bufs[which] = (mk(), mk())
        return bufs[which]

    def _exchange(self, which: int) -> None:
        import ctypes as C

        import torch

        from ._lib import check

        from .device import _stream

        send, recv = self._halo_buffers(which)
        stream = _stream(torch.cuda.current_stream().cuda_stream)  # 0 -> the legacy default stream
        check(self.dev.lib.evo_halo_pack(self.dev.ctx, which, C.c_void_p(send.data_ptr()), stream))
        self.comm.exchange(send[0], send[1], recv[0], recv[1])
        check(self.dev.lib.evo_halo_unpack(self.dev.ctx, which, C.c_void_p(recv.data_ptr()), stream))

    def exchange_front(self) -> None:
        """Ghost rows of the sensed front planes (before pass 1): one pack
        launch, one batched NCCL send/recv pair per neighbour, one unpack."""
        self._exchange(0)

    def exchange_mid(self) -> None:
        """Ghost rows of the pass-1 outputs pass 2 reads (proposal byte,
        quantity, post-death genome)."""
        self._exchange(1)

    def front_rows(self):
        """(first, last, ghost_top, ghost_bottom) views of the sensed front planes, each (5, W)."""
        return [self._rows(self._plane(w, 0, k, np.float32)) for w, k in self.FRONT]

    def mid_rows(self):
        return [self._rows(self._plane("mid_genome", 0, 0, np.int32)),
                self._rows(self._plane("mid_quantity", 0, 0, np.float32)),
                self._rows(self._plane("mid_proposal", 0, 0, np.uint8))]

    def step(self, scalars, t: int, flags: int = 0) -> None:
        import torch

        from . import _lib

        stream = torch.cuda.current_stream().cuda_stream
        if not flags & (_lib.F_UNFUSED | _lib.F_EXPORT_ACTIONS | _lib.F_INJECT_ACTIONS):
            # what evo_step passes to its pass 1: pass 2 and the swap follow (the
            # halo calls exchange record / texture rows when the step is fused / lazy)
            flags |= _lib.F_FUSE_MID | _lib.F_LAZY
        self.exchange_front()
        self.dev.pass1(scalars, t, flags=flags, stream=stream)
        self.exchange_mid()
        self.dev.pass2(t, flags=flags | _lib.F_NO_CENSUS, stream=stream)
        if not hasattr(self, "_counts"):
            ptr, _ = self.dev.plane_ptr("census_counts")
            self._counts = cuda_view(ptr, (self.dev.capacity,), np.int32)
        self.comm.sum_(self._counts)
        self.dev.census_finish(t, stream=stream)
        self.dev.swap()


    def field_radiation(self, pool, master_seed: int, t: int, p: float = 0.01, rates=None,
                        purpose: str = "field_radiation", wait=None) -> dict:
        """Config-3 field radiation over row strips (every rank calls it with
        an identical pool): the strip's occupied cells draw after those of
        the strips above it (an exclusive scan of the per-rank occupancy), so
        the union of the ranks' selections is the one-context selection; the
        per-slot parent counts are summed over the ranks, every rank admits
        the same children (deterministic host NEAT, planned before ``wait``
        is called and anything reads the device), expresses them on its
        own device and moves its own selected cells.  The caller folds the
        device census into ``pool`` first where deaths matter."""
        import torch

        from .neat import stream_key
        from .radiation import _plan_programs, admit_children, express_on, plan_field_radiation

        plan = plan_field_radiation(pool, master_seed, t, rates)  # host draws first: the step may still run
        if wait is not None:
            wait()
        world = self.plan.world
        occ = torch.zeros(world, dtype=torch.int64, device="cuda")
        occ[self.rank] = self.dev.count_occupied()
        self.comm.sum_(occ)
        first = int(occ[: self.rank].sum().item())
        counts, n_sel = self.dev.select_cells_at(stream_key(master_seed, t, purpose), p, first)
        tot = torch.from_numpy(counts.astype(np.int64)).cuda()
        self.comm.sum_(tot)
        counts = tot.cpu().numpy().astype(np.int32)
        slot_map, parents, children = admit_children(pool, counts, master_seed, t, rates, plan)
        express_on(self.dev, pool, children, _plan_programs(plan))
        self.dev.set_slots(np.asarray(pool.slot_states(), np.int8))
        self.dev.remap_selected(slot_map)
        return {"selected": int(counts.sum()), "parents": len(parents), "children": len(children)}


def step_local(strips, scalars, t: int, flags: int = 0) -> None:
    """Step several strips driven by ONE process (e.g. a single-GPU
    emulation of a multi-rank run, or peer devices in one process): the
    same two exchanges and census sum as ``DeviceStrip.step``, done with
    device-to-device copies between the strips' ghost rows."""
    import torch

    from . import _lib

    import ctypes as C

    from ._lib import check
    from .device import _stream

    n = len(strips)
    stream = torch.cuda.current_stream().cuda_stream
    cstream = _stream(stream)  # 0 -> the legacy default stream, as the passes use

    def ring(which):
        bufs = [s._halo_buffers(which) for s in strips]
        for s, (send, _) in zip(strips, bufs):
            check(s.dev.lib.evo_halo_pack(s.dev.ctx, which, C.c_void_p(send.data_ptr()), cstream))
        for r in range(n):
            up, down = bufs[(r - 1) % n][0], bufs[(r + 1) % n][0]
            recv = bufs[r][1]
            recv[0].copy_(up[1])    # ghost above <- upper neighbour's last row
            recv[1].copy_(down[0])  # ghost below <- lower neighbour's first row
        for s, (_, recv) in zip(strips, bufs):
            check(s.dev.lib.evo_halo_unpack(s.dev.ctx, which, C.c_void_p(recv.data_ptr()), cstream))

    if not flags & (_lib.F_UNFUSED | _lib.F_EXPORT_ACTIONS | _lib.F_INJECT_ACTIONS):
        flags |= _lib.F_FUSE_MID | _lib.F_LAZY  # as DeviceStrip.step
    ring(0)
    for s in strips:
        s.dev.pass1(scalars, t, flags=flags, stream=stream)
    ring(1)
    for s in strips:
        s.dev.pass2(t, flags=flags | _lib.F_NO_CENSUS, stream=stream)
    counts = [cuda_view(s.dev.plane_ptr("census_counts")[0], (s.dev.capacity,), np.int32) for s in strips]
    total = torch.stack(counts).sum(0, dtype=torch.int32)
    for c, s in zip(counts, strips):
        c.copy_(total)
        s.dev.census_finish(t, stream=stream)
        s.dev.swap()


def field_radiation_local(strips, pools, master_seed: int, t: int, p: float = 0.01, rates=None,
                          purpose: str = "field_radiation") -> dict:
    """``DeviceStrip.field_radiation`` for strips driven by ONE process (as
    ``step_local``): the occupancy scan and the parent-count sum are done on
    the host; ``pools`` holds one identical pool per strip."""
    from .neat import stream_key
    from .radiation import admit_children, express_on

    occ = [s.dev.count_occupied() for s in strips]
    counts = np.zeros(strips[0].dev.capacity, np.int64)
    first = 0
    for s, n in zip(strips, occ):
        c, _ = s.dev.select_cells_at(stream_key(master_seed, t, purpose), p, first)
        counts += c
        first += n
    counts = counts.astype(np.int32)
    out = None
    for s, pool in zip(strips, pools):
        slot_map, parents, children = admit_children(pool, counts, master_seed, t, rates)
        express_on(s.dev, pool, children)
        s.dev.set_slots(np.asarray(pool.slot_states(), np.int8))
        s.dev.remap_selected(slot_map)
        out = {"selected": int(counts.sum()), "parents": len(parents), "children": len(children)}
    return out
