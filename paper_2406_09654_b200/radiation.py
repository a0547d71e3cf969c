"""Radiation feed on the device path.

Host NEAT (mutation, crossover, pool admission) stays on the host
(north_star (6)); what moves to the GPU is everything around it:

* ``DeviceExpressed`` - the params object a pool's ``net_factory`` returns
  for an admitted genome (GenomePool.admit, neuroevo.py:476).  The engine
  turns every such slot into ONE batched ``evo_express_cppn`` launch (the
  reference calls hypernet.generate_network per admission on the CPU,
  hypernet.py:183-220); the host tables are fetched lazily, only if someone
  reads ``.w1``/``.w`` etc.  ``use_device_expression(state)`` installs it, so
  the reference's own ``apply_radiation`` (physics.py:346-392), run on the
  device-compacted adoption events, admits children whose weights are
  generated on the GPU.
* ``apply_radiation`` - the reference's adoption-driven radiation
  (physics.py:346-392) owned by this package: per device-compacted adoption
  event (ascending target), a merge roll and a mutation roll from the step's
  "radiation" stream, then ``neat.crossover`` / ``neat.mutate`` from the
  event's own "merge" / "mutate" stream, pool admission and installation of
  the child at the target.  The engine calls it whenever p_radiation or
  p_merge is non-zero (engine.py:244 in the reference).
* ``field_radiation`` - the BASELINE config-3 extension:
  every ``every`` steps, 1 % of occupied cells (device draw from the host
  Philox stream ``rng.stream(seed, t, "field_radiation")``, rng.py:19-33) are
  selected; one child per distinct parent slot is mutated on the host
  (native ``neat.mutate_batch``, each parent on ``stream(seed, t, "mutate",
  parent)``), admitted, its weights generated on the device, and the
  selected cells move to it.  The host draws do not depend on the
  selection: ``plan_field_radiation`` mutates (numbering deferred) and
  compiles a child for every live slot while the step before the event is
  still running on the device, and the event numbers and admits the
  children of the slots actually selected.
"""

from __future__ import annotations

import numpy as np

from . import neat

__all__ = ["DeviceExpressed", "device_net_factory", "use_device_expression", "stream_key", "apply_radiation",
           "field_radiation", "plan_field_radiation", "FieldRadiationPlan"]


stream_key = neat.stream_key


class DeviceExpressed:
    """Dense params of a pattern network, generated on the device.

    Reads of the table attributes (DenseParams ``w1, b1, w2, b2`` for a
    hidden-layer substrate, DirectParams ``w, b`` for the direct one) pull
    the slot's tables back with ``evo_get_params``."""

    def __init__(self, genome, hidden: int, tau: float = 0.2, w_max: float = 3.0):
        self.genome = genome
        self.hidden = int(hidden)
        self.tau = float(tau)
        self.w_max = float(w_max)
        self._dev = None
        self._slot = None
        self._tables = None

    @property
    def expressed(self) -> bool:
        return self._dev is not None

    def bind(self, dev, slot: int) -> None:
        self._dev, self._slot, self._tables = dev, int(slot), None

    def _fetch(self):
        if self._tables is None:
            if self._dev is None:
                raise RuntimeError("params not generated yet: the engine expresses them at its next step")
            w1, b1, w2, b2 = self._dev.get_params_arrays(self._slot, 1)
            self._tables = (None if w1 is None else w1[0], None if b1 is None else b1[0], w2[0], b2[0])
        return self._tables

    def __getattr__(self, name):
        # only the table attributes are synthesised; anything else is absent
        if name in ("w1", "b1", "w2", "b2") and self.__dict__.get("hidden", 0) > 0:
            return self._fetch()[("w1", "b1", "w2", "b2").index(name)]
        if name in ("w", "b") and self.__dict__.get("hidden", 1) == 0:
            return self._fetch()[2 if name == "w" else 3]
        raise AttributeError(name)


def device_net_factory(hidden: int, tau: float = 0.2, w_max: float = 3.0):
    def factory(genome):
        return DeviceExpressed(genome, hidden, tau, w_max)

    return factory


def use_device_expression(state, tau: float = 0.2, w_max: float = 3.0) -> None:
    """Route the pool's admissions through the device CPPN kernel."""
    from .engine import _hidden_of

    state.pool.net_factory = device_net_factory(_hidden_of(state), tau, w_max)


def apply_radiation(events, pool, rates, planes, master_seed: int, step: int) -> None:
    """Adoption-driven radiation on a host genome plane (physics.py:346-392).

    ``events``: AdoptionEvents of the step in ascending target order;
    ``pool``: a slot pool with ``live_mask / can_admit / admit / genome /
    lineage / innovations`` (SlotPool or the reference's GenomePool);
    ``rates``: ``p_merge``, ``p_radiation`` and the mutation rates;
    ``planes``: the PlaneSet whose genome plane receives the children (the
    back buffer, before the census).  Decisions are taken for all events
    first (the liveness of the defenders as it was when the step began), then
    children are admitted in target order until the pool is full."""
    n = len(events)
    if n == 0:
        return
    merge_roll, mutate_roll = neat.stream(master_seed, step, "radiation").random((2, n))
    winner = np.asarray(events.winner_slot, np.int64)
    defender = np.asarray(events.defender_slot, np.int64)
    live = np.asarray(pool.live_mask(), bool)
    merge_ok = (defender >= 0) & (defender != winner)
    merge_ok[merge_ok] = live[defender[merge_ok]]
    merge = merge_ok & (merge_roll < rates.p_merge)
    mutation = ~merge & (mutate_roll < rates.p_radiation)
    cells = planes.genome_index.reshape(-1)
    for k in np.flatnonzero(merge | mutation):
        if not pool.can_admit():
            break  # admissions only fill slots within one call
        tgt, win = int(events.target[k]), int(winner[k])
        if merge[k]:
            dfd = int(defender[k])
            child = neat.crossover(pool.genome(win), pool.genome(dfd), neat.stream(master_seed, step, "merge", tgt))
            parents = (pool.lineage(win), pool.lineage(dfd))
        else:
            child = neat.mutate(pool.genome(win), rates, neat.stream(master_seed, step, "mutate", tgt),
                                pool.innovations)
            parents = (pool.lineage(win),)
        slot = pool.admit(child, parents=parents, birth_step=step + 1)
        if slot is not None:
            cells[tgt] = slot


class FieldRadiationPlan:
    """The selection-independent host half of a field-radiation event at
    step ``t``: one deferred-numbering child (``neat.mutate_batch_deferred``,
    parent slot s on ``stream(seed, t, "mutate", s)``) and its compiled
    expression program for the first live slots (ascending) - as many as
    the pool has room for, plus a margin: an event admits children for the
    lowest parent slots only, until the pool is full."""

    def __init__(self, pool, master_seed: int, t: int, rates=None):
        self.master_seed, self.t = int(master_seed), int(t)
        self.rates = rates or neat.EvolutionRates()
        states = np.asarray(pool.slot_states())
        room = int(np.count_nonzero(states != 1))  # grows if the census fold finds deaths: the margin
        self.slots = np.flatnonzero(states == 1)[:room + max(32, room // 4)] if room else np.zeros(0, np.int64)
        self.genomes = [pool.genome(int(s)) for s in self.slots]
        self.children = neat.mutate_batch_deferred(
            self.genomes, self.rates, [stream_key(master_seed, t, "mutate", int(s)) for s in self.slots])
        self.programs = neat.compile_programs(self.children) if self.children else None
        self.admitted = None  # plan positions of the children an event admitted

    def positions(self, pool, master_seed: int, t: int, rates, take):
        """Plan positions of the parent slots ``take``, or None when the plan
        does not cover them unchanged (other step / seed / rates, a slot
        not live at planning or holding another genome since)."""
        if (int(master_seed), int(t)) != (self.master_seed, self.t) or (rates or neat.EvolutionRates()) != self.rates:
            return None
        take = np.asarray(take, np.int64)
        pos = np.searchsorted(self.slots, take)
        if len(take) and (pos.max() >= len(self.slots) or not np.array_equal(self.slots[pos], take)):
            return None
        if any(pool.genome(int(s)) is not self.genomes[int(i)] for s, i in zip(take, pos)):
            return None
        return pos


def plan_field_radiation(pool, master_seed: int, t: int, rates=None) -> FieldRadiationPlan:
    """Host NEAT of the field-radiation event at step ``t`` done ahead of the
    device selection (call it while the preceding step runs)."""
    return FieldRadiationPlan(pool, master_seed, t, rates)


def admit_children(pool, counts, master_seed: int, t: int, rates=None, plan: FieldRadiationPlan | None = None):
    """The host half of a field-radiation event (config-3 extension): one
    mutated child per parent slot with selected cells (``counts``, per slot),
    admitted in ascending parent order until the pool refuses; returns
    (slot_map: parent -> child or -1, parents, children).  Deterministic
    given the pool and counts, so every rank of a strip run admits the same
    children."""
    rates = rates or neat.EvolutionRates()
    parents = np.flatnonzero(counts)
    slot_map = np.full(pool.capacity, -1, np.int32)
    # admissions only fill slots, so the first `room` parents (ascending slot)
    # get children - exactly those a mutate/admit loop stopping at the first
    # refusal would mutate, consuming the innovation counter in that order
    room = int(np.count_nonzero(np.asarray(pool.slot_states()) != 1)) if hasattr(pool, "slot_states") else None
    take = [int(x) for x in (parents if room is None else parents[:room])]
    pos = plan.positions(pool, master_seed, t, rates, take) if plan is not None else None
    if pos is not None:  # the planned draws, numbered now in admission order
        kids = neat.number_deferred([plan.children[int(i)] for i in pos], pool.innovations)
    else:
        kids = neat.mutate_batch([pool.genome(par) for par in take], rates,
                                 [stream_key(master_seed, t, "mutate", par) for par in take], pool.innovations)
    if hasattr(pool, "admit_batch"):
        children = pool.admit_batch(kids, [(pool.lineage(par),) for par in take], birth_step=t)
        slot_map[np.asarray(take[:len(children)], np.int64)] = children
    else:
        children = []
        for par, child in zip(take, kids):
            slot = pool.admit(child, parents=(pool.lineage(par),), birth_step=t)
            if slot is None:
                break
            slot_map[par] = slot
            children.append(slot)
    if plan is not None:
        plan.admitted = pos[:len(children)] if pos is not None else None
    return slot_map, parents, list(children)


def express_on(dev, pool, slots, programs=None) -> None:
    """Device tables of newly admitted slots whose parameters are
    DeviceExpressed (one batched evo_express_cppn per (tau, w_max)), binding
    them to ``dev``.  ``programs``: the compiled programs of exactly
    ``slots``' genomes, in order (used when they form one batch)."""
    by_expr = {}
    for s in slots:
        prm = pool.params(s)
        if isinstance(prm, DeviceExpressed):
            by_expr.setdefault((prm.tau, prm.w_max), []).append((s, prm))
    whole = len(by_expr) == 1 and len(next(iter(by_expr.values()))) == len(slots)
    for (tau, w_max), items in by_expr.items():
        dev.express_cppn([s for s, _ in items], [prm.genome for _, prm in items], tau, w_max,
                         programs=programs if whole else None)
        for s, prm in items:
            prm.bind(dev, s)


def _plan_programs(plan):
    if plan is None or plan.admitted is None or plan.programs is None:
        return None
    return neat.subset_programs(plan.programs, plan.admitted)


def field_radiation(state, t: int, p: float = 0.01, rates: neat.EvolutionRates | None = None,
                    purpose: str = "field_radiation", wait=None) -> dict:
    """One config-3 radiation event on the state's device front (call between
    steps).  The host draws are planned first (``plan_field_radiation``), so
    they overlap a step still running on the device; ``wait`` (optional) is
    called after planning, before anything reads the device - e.g. the
    synchronisation of a caller's own stream.  Returns {"selected",
    "parents", "children"}."""
    from .engine import _binding, _fold_census

    b = _binding(state)
    dev = b.dev
    pool = state.pool
    plan = plan_field_radiation(pool, state.master_seed, t, rates) if hasattr(pool, "slot_states") else None
    if wait is not None:
        wait()
    dev_peak = _fold_census(state)  # admission must see the device's deaths (slot states, peaks)
    counts, n_sel = dev.select_cells(stream_key(state.master_seed, t, purpose), p)
    synced = getattr(pool, "version", None) is not None and b.pool_version == pool.version
    slot_map, parents, children = admit_children(pool, counts, state.master_seed, t, rates, plan)
    if synced and all(isinstance(pool.params(s), DeviceExpressed) for s in children):
        # only the children changed: express exactly those (one batched
        # evo_express_cppn) instead of sync_params' scan of every slot
        express_on(dev, pool, children, _plan_programs(plan))
        for s in children:
            b.param_ids[s] = pool.params(s)
        from .engine import _peaks, _slot_states

        if dev_peak is None:
            peaks = _peaks(pool)
        else:
            # the binding was in sync, so the device's peaks are the records'
            # (the fold just took them); only the children's slots start over
            peaks = np.array(dev_peak, np.int32)
            peaks[np.asarray(list(children), np.int64)] = 0
        dev.set_slots(_slot_states(pool), peaks)
        b.pool_version = pool.version
    else:
        b.sync_params(pool)  # one batched evo_express_cppn for every new slot
    dev.remap_selected(slot_map)
    b.device_ahead = True
    return {"selected": int(n_sel), "parents": len(parents), "children": len(children)}
