"""Slot pool for device runs (subset of neuroevo.GenomePool).

The reference's ``GenomePool`` (/root/reference/pkg/src/evoca/neuroevo.py:
415-545) owns NEAT genomes, lineage records and cached dense params.  NEAT
genetics stay on the host and out of this package's scope; the engine only
needs the pool's slot table: ``capacity``, ``params(slot)``, liveness and
``update_census``.  ``SlotPool`` provides exactly that surface for the
BASELINE synthetic configurations (genomes = directly installed weight
tables).  Any object with the same methods - including the reference
``GenomePool`` itself - can be passed to the engine instead.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

__all__ = ["SlotPool", "SlotRecord"]


@dataclass
class SlotRecord:
    lineage_id: int
    slot: int
    birth_step: int
    death_step: Optional[int] = None
    peak_population: int = 0
    parents: tuple = ()


class SlotPool:
    def __init__(self, capacity: int, net_factory=None, counter=None):
        if capacity < 1:
            raise ValueError("pool capacity must be positive")
        from .neat import InnovationCounter

        self.capacity = capacity
        self.net_factory = net_factory
        self.innovations = counter if counter is not None else InnovationCounter()
        self._genomes = [None] * capacity
        self._death = np.full(capacity, -1, np.int64)
        self._params = [None] * capacity
        self._state = np.zeros(capacity, np.int8)  # 0 free, 1 live, 2 dead
        self._lineage = np.full(capacity, -1, np.int64)
        self.records: dict[int, SlotRecord] = {}
        self.next_lineage_id = 0
        self.version = 0  # bumped on every params/liveness change
        # apply_device_census: the device peak and the occupant it was last folded for, per slot
        self._seen_peak = np.full(capacity, -1, np.int64)
        self._seen_lineage = np.full(capacity, -2, np.int64)

    def install(self, slot: int, params, birth_step: int = 0, genome=None) -> int:
        """Put a parameter set (and optionally its pattern network) in a slot
        and mark it live (admission without NEAT)."""
        if not 0 <= slot < self.capacity:
            raise ValueError("slot outside the pool capacity")
        self._params[slot] = params
        self._genomes[slot] = genome
        self._state[slot] = 1
        lid = self.next_lineage_id
        self.next_lineage_id += 1
        self._lineage[slot] = lid
        self.records[lid] = SlotRecord(lid, slot, birth_step)
        self.version += 1
        return slot

    def params(self, slot: int):
        return self._params[slot]

    def genome(self, slot: int):
        g = self._genomes[slot]
        if g is None:
            raise KeyError(f"slot {slot} has no genome")
        return g

    def set_genome(self, slot: int, genome) -> None:
        self._genomes[slot] = genome

    # -- admission (GenomePool.can_admit / admit, neuroevo.py:451-487) ----------

    def can_admit(self) -> bool:
        return bool(np.any(self._state != 1))

    def admit(self, genome, parents: tuple = (), birth_step: int = 0) -> Optional[int]:
        """Lowest free slot, else evict the dead slot with the oldest death
        step (lowest index on ties); None when every slot is live.  Params come
        from ``net_factory(genome)`` (e.g. a device-expression placeholder)."""
        free = np.flatnonzero(self._state == 0)
        if len(free):
            idx = int(free[0])
        else:
            dead = np.flatnonzero(self._state == 2)
            if not len(dead):
                return None
            idx = int(dead[np.lexsort((dead, self._death[dead]))[0]])
        params = self.net_factory(genome) if self.net_factory is not None else None
        self._genomes[idx] = genome
        self._params[idx] = params
        self._state[idx] = 1
        self._death[idx] = -1
        lid = self.next_lineage_id
        self.next_lineage_id += 1
        self._lineage[idx] = lid
        self.records[lid] = SlotRecord(lid, idx, birth_step, parents=tuple(parents))
        self.version += 1
        return idx

    def admit_batch(self, genomes, parents, birth_step: int = 0) -> list:
        """``admit`` of each genome in order (same slot choice: lowest free
        slot, then the dead slot with the oldest death step, lowest index on
        ties; stops at the first refusal), with the slot search done once
        for the batch.  ``parents``: one tuple per genome.  Returns the slots."""
        free = np.flatnonzero(self._state == 0)
        dead = np.flatnonzero(self._state == 2)
        dead = dead[np.lexsort((dead, self._death[dead]))]
        order = np.concatenate([free, dead])[:len(genomes)]
        out = []
        for idx, genome, par in zip(order.tolist(), genomes, parents):
            params = self.net_factory(genome) if self.net_factory is not None else None
            self._genomes[idx] = genome
            self._params[idx] = params
            lid = self.next_lineage_id
            self.next_lineage_id += 1
            self._lineage[idx] = lid
            self.records[lid] = SlotRecord(lid, idx, birth_step, parents=tuple(par))
            out.append(idx)
        if out:
            sel = np.asarray(out, np.int64)
            self._state[sel] = 1
            self._death[sel] = -1
            self.version += 1
        return out

    def is_live(self, slot: int) -> bool:
        return 0 <= slot < self.capacity and self._state[slot] == 1

    def live_mask(self) -> np.ndarray:
        return self._state == 1

    def live_count(self) -> int:
        return int((self._state == 1).sum())

    def live_slots(self) -> list[int]:
        return [int(i) for i in np.flatnonzero(self._state == 1)]

    def lineage(self, slot: int) -> int:
        return int(self._lineage[slot])

    def record_for_slot(self, slot: int) -> SlotRecord:
        return self.records[int(self._lineage[slot])]

    def slot_states(self) -> np.ndarray:
        return self._state.copy()

    def peaks(self) -> np.ndarray:
        out = np.zeros(self.capacity, np.int32)
        for i in np.flatnonzero(self._lineage >= 0):
            out[i] = self.records[int(self._lineage[i])].peak_population
        return out

    def deaths_at(self, step: int) -> list[int]:
        """Lineages whose recorded death step is ``step`` (neuroevo.py:544-545)."""
        return [r.lineage_id for r in self.records.values() if r.death_step == step]

    def update_census(self, counts, step: int) -> list[int]:
        """Same contract as GenomePool.update_census (neuroevo.py:521-542)."""
        dead = []
        for i in np.flatnonzero(self._state == 1):
            c = int(counts[i])
            rec = self.records[int(self._lineage[i])]
            if c == 0:
                self._state[i] = 2
                self._death[i] = step
                rec.death_step = step
                dead.append(int(i))
            elif c > rec.peak_population:
                rec.peak_population = c
        return dead

    def apply_device_census(self, state: np.ndarray, death_step: np.ndarray, peak: np.ndarray) -> list[int]:
        """Fold the device's deferred census (slot state, first zero-count
        step, peak) into the records; equivalent to having called
        update_census every step."""
        dead = []
        live = np.flatnonzero(self._state == 1)
        state, peak = np.asarray(state), np.asarray(peak)
        # a live slot whose occupant and device peak are those of the last fold
        # has nothing new (its record already holds that peak): the records
        # are only visited for the others (a radiation event folds ~1000 slots)
        lin = self._lineage[live]
        pk = peak[live].astype(np.int64)
        todo = (state[live] == 2) | (pk != self._seen_peak[live]) | (lin != self._seen_lineage[live])
        for i in live[todo]:
            rec = self.records[int(self._lineage[i])]
            if peak[i] > rec.peak_population:
                rec.peak_population = int(peak[i])
            if state[i] == 2:
                self._state[i] = 2
                self._death[i] = int(death_step[i])
                rec.death_step = int(death_step[i])
                dead.append(int(i))
        self._seen_peak[live] = pk
        self._seen_lineage[live] = lin
        return dead
