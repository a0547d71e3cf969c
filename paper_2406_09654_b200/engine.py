"""Step scheduler with the reference's API, backed by the device.

Drop-in for /root/reference/pkg/src/evoca/engine.py:
  * ``step(state)``   - one step of a host-resident state: upload the front
    planes, run the two device passes, download into the back planes, census,
    swap (engine.py:233-248).  Works on this package's ``SimState`` and on
    the reference's own ``SimState`` (duck-typed: ``substrate``, ``pool``,
    ``config``, ``master_seed``).
  * ``run(state, steps, hooks, should_stop)`` - the batch loop
    (engine.py:251-271), device-resident between hook points.
  * ``build_action_field(state)`` - device sense + controller, exported as an
    ``ActionField`` (engine.py:193-230).
  * ``digest(state)`` - FNV-1a over the front planes (engine.py:301-315).
  * ``new_state(config)`` / ``seed_initial_population`` (engine.py:94-139),
    ``gather_sensors`` (engine.py:142-161), ``describe_params`` /
    ``validate_param`` / ``apply_param`` live steering (engine.py:321-390).
Host NEAT radiation (physics.apply_radiation, physics.py:346-392) stays on
the host; when its probabilities are non-zero the engine records adoption
events on the device and hands them to a host callback per step.
"""

from __future__ import annotations

import logging
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _lib
from .device import DeviceSubstrate
from .hypernet import DenseParams, DirectParams
from .physics import ActionField, AdoptionEvents, PhysicsParams, step_scalars
from .pool import SlotPool
from .substrate import Substrate, create_substrate
from .synth import BASELINE_CONFIGS, synth_arrays, synth_params

__all__ = [
    "GridConfig", "HypernetConfig", "EvolutionRates", "RunConfig", "ServeConfig", "FieldRadiationConfig",
    "ExperimentConfig", "config_to_dict", "parse_config",
    "SimState", "Hook", "baseline_state", "new_state", "seed_initial_population", "gather_sensors", "step",
    "run", "build_action_field", "digest", "describe_params", "validate_param", "apply_param", "render_rgb",
    "device_of", "sync_to_host",
]

log = logging.getLogger(__name__)


DEFAULT_POOL_CAPACITY = 512  # neuroevo.py:50


@dataclass
class GridConfig:
    width: int = 256
    height: int = 256

    def validate(self) -> None:  # config.py:32-36
        if self.width < 4:
            raise ValueError("grid.width must be >= 4")
        if self.height < 4:
            raise ValueError("grid.height must be >= 4")


@dataclass
class HypernetConfig:
    hidden_size: int = 16  # 0 selects the BASELINE direct 45->13 controller
    tau: float = 0.2
    w_max: float = 3.0

    def validate(self) -> None:  # config.py:45-51 (hidden 0 = the direct-net extension)
        if self.hidden_size < 0:
            raise ValueError("hypernet.hidden_size must be >= 0")
        if not 0.0 <= self.tau < 1.0:
            raise ValueError("hypernet.tau must be in [0, 1)")
        if self.w_max <= 0:
            raise ValueError("hypernet.w_max must be positive")


@dataclass
class EvolutionRates:
    """neuroevo.py:170-203, with the reference's defaults (p_radiation 0.02,
    p_merge 0.2: adoption-driven radiation is on unless a config turns it
    off; the BASELINE synthetic configurations set both to 0)."""

    weight_perturb_prob: float = 0.8
    weight_perturb_sigma: float = 0.5
    weight_reset_prob: float = 0.05
    add_connection_prob: float = 0.05
    add_node_prob: float = 0.03
    toggle_enable_prob: float = 0.01
    c1: float = 1.0
    c2: float = 1.0
    c3: float = 0.4
    p_radiation: float = 0.02
    p_merge: float = 0.2

    def validate(self) -> None:  # neuroevo.py:186-203
        for name in ("weight_perturb_prob", "weight_reset_prob", "add_connection_prob", "add_node_prob",
                     "toggle_enable_prob", "p_radiation", "p_merge"):
            v = getattr(self, name)
            if not 0.0 <= v <= 1.0:
                raise ValueError(f"{name} must be in [0, 1], got {v}")
        if self.weight_perturb_sigma <= 0:
            raise ValueError("weight_perturb_sigma must be positive")
        for name in ("c1", "c2", "c3"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be non-negative")


@dataclass
class RunConfig:
    """config.py:55-72 (CLI cadence; carried for config/snapshot fidelity)."""

    steps: int = 1000
    metrics_every: int = 100
    snapshot_every: int = 0
    frame_every: int = 100

    def validate(self) -> None:
        if self.steps < 0:
            raise ValueError("run.steps must be >= 0")
        for name in ("metrics_every", "snapshot_every", "frame_every"):
            if getattr(self, name) < 0:
                raise ValueError(f"run.{name} must be >= 0")
        if self.metrics_every == 0:
            raise ValueError("run.metrics_every must be >= 1")
        if self.frame_every == 0:
            raise ValueError("run.frame_every must be >= 1")


@dataclass
class ServeConfig:
    """config.py:74-90 (steering server; carried for config/snapshot fidelity)."""

    host: str = "127.0.0.1"
    port: int = 8765
    frame_fps: float = 10.0
    telemetry_fps: float = 2.0
    max_steps_per_second: float = 0.0

    def validate(self) -> None:
        if not 0 <= self.port <= 65535:
            raise ValueError("serve.port must be in [0, 65535]")
        if self.frame_fps <= 0:
            raise ValueError("serve.frame_fps must be positive")
        if self.telemetry_fps <= 0:
            raise ValueError("serve.telemetry_fps must be positive")
        if self.max_steps_per_second < 0:
            raise ValueError("serve.max_steps_per_second must be >= 0")


@dataclass
class FieldRadiationConfig:
    """BASELINE config-3 extension: every ``every`` steps
    a fraction ``p`` of occupied cells moves to freshly mutated children of
    their genomes (radiation.field_radiation).  0 disables it."""

    every: int = 0
    p: float = 0.01

    def validate(self) -> None:
        if self.every < 0:
            raise ValueError("field_radiation.every must be >= 0")
        if not 0.0 <= self.p <= 1.0:
            raise ValueError("field_radiation.p must be in [0, 1]")


@dataclass
class ExperimentConfig:
    grid: GridConfig = field(default_factory=GridConfig)
    seed: int = 0
    initial_population: int = 64
    physics: PhysicsParams = field(default_factory=PhysicsParams)
    evolution: EvolutionRates = field(default_factory=EvolutionRates)
    hypernet: HypernetConfig = field(default_factory=HypernetConfig)
    run: RunConfig = field(default_factory=RunConfig)
    serve: ServeConfig = field(default_factory=ServeConfig)
    field_radiation: FieldRadiationConfig = field(default_factory=FieldRadiationConfig)

    def validate(self) -> None:  # config.py:104-121
        self.grid.validate()
        self.physics.validate()
        self.evolution.validate()
        self.hypernet.validate()
        self.run.validate()
        self.serve.validate()
        self.field_radiation.validate()
        if self.seed < 0:
            raise ValueError("seed must be >= 0")
        if self.initial_population < 0:
            raise ValueError("initial_population must be >= 0")
        if self.initial_population > DEFAULT_POOL_CAPACITY:
            raise ValueError(f"initial_population must be <= {DEFAULT_POOL_CAPACITY}")
        if self.initial_population > self.grid.width * self.grid.height:
            raise ValueError("initial_population must fit on the grid")


@dataclass
class SimState:
    """engine.py:61-91 fields plus the device handle (created lazily)."""

    substrate: Substrate
    pool: object
    config: object
    master_seed: int
    workers: int = 1
    last_adoptions: int = 0
    last_extinctions: int = 0
    radiation: Optional[Callable] = None

    @property
    def t(self) -> int:
        return self.substrate.step_counter

    @property
    def physics(self):
        return self.config.physics

    @property
    def rates(self):
        return self.config.evolution


@dataclass(frozen=True)
class Hook:
    """engine.py:87-91.  ``device=True`` (extension): the hook only uses
    device-side views (``render_rgb``, ``last_adoptions``) and fires during a
    device-resident ``run`` without downloading the planes."""

    every: int
    fn: Callable
    device: bool = False


_SECTIONS = {"grid": GridConfig, "physics": PhysicsParams, "evolution": EvolutionRates, "hypernet": HypernetConfig,
             "run": RunConfig, "serve": ServeConfig, "field_radiation": FieldRadiationConfig}
_SCALAR_KEYS = ("seed", "initial_population")


def _coerce(path: str, default, value):  # config.py:133-151
    if isinstance(default, bool):
        if not isinstance(value, bool):
            raise ValueError(f"{path} must be a boolean")
        return value
    if isinstance(default, int):
        if not isinstance(value, int) or isinstance(value, bool):
            raise ValueError(f"{path} must be an integer")
        return value
    if isinstance(default, float):
        if not isinstance(value, (int, float)) or isinstance(value, bool):
            raise ValueError(f"{path} must be a number")
        return float(value)
    if isinstance(default, str):
        if not isinstance(value, str):
            raise ValueError(f"{path} must be a string")
        return value
    return value


def parse_config(data: dict) -> ExperimentConfig:
    """Build and validate a config from a parsed JSON object (config.py:164-183);
    also accepts this package's ``field_radiation`` section."""
    if not isinstance(data, dict):
        raise ValueError("config root must be an object")
    cfg = ExperimentConfig()
    for key, value in data.items():
        if key in _SECTIONS:
            if not isinstance(value, dict):
                raise ValueError(f"{key} must be an object")
            if key == "physics" and "energy_source_map" in value:
                raise ValueError("physics.energy_source_map is not configurable from file")
            obj = _SECTIONS[key]()
            known = set(vars(obj))
            for k, v in value.items():
                if k not in known:
                    raise ValueError(f"unknown key {key}.{k}")
                setattr(obj, k, _coerce(f"{key}.{k}", getattr(obj, k), v))
            setattr(cfg, key, obj)
        elif key in _SCALAR_KEYS:
            setattr(cfg, key, _coerce(key, getattr(cfg, key), value))
        else:
            raise ValueError(f"unknown key {key}")
    cfg.validate()
    return cfg


def config_to_dict(cfg) -> dict:
    """JSON-ready dict that parse_config round-trips (config.py:194-198); the
    field-radiation extension is written only when enabled, so other configs
    stay loadable by the reference."""
    from dataclasses import asdict

    out = asdict(cfg)
    out["physics"].pop("energy_source_map", None)
    fr = out.get("field_radiation")
    if fr is not None and not fr.get("every"):
        out.pop("field_radiation")
    return out


# -- device binding -------------------------------------------------------------


class _Binding:
    """Per-state device context plus the host<->device coherence bookkeeping."""

    def __init__(self, state, device: int = 0):
        sub = state.substrate
        self.hidden = _hidden_of(state)
        self.capacity = int(state.pool.capacity)
        self.dev = DeviceSubstrate(sub.width, sub.height, self.capacity, self.hidden, device=device)
        self.param_ids = [None] * self.capacity
        self.pool_version = None
        self.device_ahead = False  # device front newer than the host mirror
        self.pinned = False
        fr = getattr(state.config, "field_radiation", None)
        if fr is not None and fr.every > 0:
            # field radiation selects cells on the device every `every` steps:
            # allocate its buffers now (a zero-probability selection) rather
            # than inside the first radiation step
            self.dev.select_cells(0, 0.0)

    def sync_params(self, pool) -> None:
        ver = getattr(pool, "version", None)
        if ver is not None and ver == self.pool_version:
            return
        from .radiation import DeviceExpressed

        changed, express = [], []
        for slot in range(self.capacity):
            p = pool.params(slot)
            if p is not None and self.param_ids[slot] is not p:
                if isinstance(p, DeviceExpressed):
                    express.append(slot)
                else:
                    changed.append(slot)
        if express:  # admitted pattern networks: one batched device expression
            ps = [pool.params(s) for s in express]
            by_expr = {}
            for s, p in zip(express, ps):
                by_expr.setdefault((p.tau, p.w_max), []).append((s, p))
            for (tau, w_max), items in by_expr.items():
                self.dev.express_cppn([s for s, _ in items], [p.genome for _, p in items], tau, w_max)
                for s, p in items:
                    p.bind(self.dev, s)
                    self.param_ids[s] = p
        # upload contiguous runs of changed slots
        i = 0
        while i < len(changed):
            j = i
            while j + 1 < len(changed) and changed[j + 1] == changed[j] + 1:
                j += 1
            lo, hi = changed[i], changed[j] + 1
            self.dev.set_params([_as_params(pool.params(s), self.hidden) for s in range(lo, hi)], slot0=lo)
            for s in range(lo, hi):
                self.param_ids[s] = pool.params(s)
            i = j + 1
        self.dev.set_slots(_slot_states(pool), _peaks(pool))
        self.pool_version = ver


def _hidden_of(state) -> int:
    hn = getattr(state.config, "hypernet", None)
    hidden = getattr(hn, "hidden_size", None)
    if hidden is None:
        raise ValueError("config.hypernet.hidden_size is required")
    # a reference config with DirectParams in the pool means the direct net
    from .radiation import DeviceExpressed

    for slot in range(int(state.pool.capacity)):
        p = state.pool.params(slot)
        if isinstance(p, DeviceExpressed):
            return p.hidden
        if p is not None:
            if isinstance(p, DirectParams) or (hasattr(p, "w") and not hasattr(p, "w1")):
                return 0
            return int(p.w1.shape[0])
    return int(hidden)


def _as_params(p, hidden):
    if hidden == 0:
        if isinstance(p, DirectParams):
            return p
        return DirectParams(np.asarray(p.w, np.float32), np.asarray(p.b, np.float32))
    if isinstance(p, DenseParams):
        return p
    return DenseParams(np.asarray(p.w1, np.float32), np.asarray(p.b1, np.float32),
                       np.asarray(p.w2, np.float32), np.asarray(p.b2, np.float32))


def _slot_states(pool) -> np.ndarray:
    if hasattr(pool, "slot_states"):
        return pool.slot_states()
    if hasattr(pool, "slots"):  # reference GenomePool
        code = {"free": 0, "live": 1, "dead": 2}
        return np.array([code[s.state] for s in pool.slots], np.int8)
    return np.asarray(pool.live_mask(), np.int8)


def _peaks(pool) -> np.ndarray:
    if hasattr(pool, "peaks"):
        return pool.peaks()
    out = np.zeros(int(pool.capacity), np.int32)
    if hasattr(pool, "slots"):
        for i, s in enumerate(pool.slots):
            if s.lineage_id >= 0 and s.lineage_id in pool.records:
                out[i] = pool.records[s.lineage_id].peak_population
    return out


def device_of(state, device: int = 0) -> DeviceSubstrate:
    """The state's device context (created on first use)."""
    b = getattr(state, "_evo_binding", None)
    if b is None:
        b = _Binding(state, device)
        state._evo_binding = b
    return b.dev


def _binding(state) -> _Binding:
    device_of(state)
    return state._evo_binding


def _radiation_active(state) -> bool:
    r = state.config.evolution
    return getattr(r, "p_radiation", 0.0) > 0.0 or getattr(r, "p_merge", 0.0) > 0.0


def _radiation_fn(state):
    """The host radiation callback: ``state.radiation`` if set, else this
    package's restatement of physics.apply_radiation (radiation.py)."""
    if getattr(state, "radiation", None) is not None:
        return state.radiation
    from .radiation import apply_radiation

    return apply_radiation


# -- the drop-in step -------------------------------------------------------------


def step(state) -> None:
    """One step of a host-resident state (engine.py:233-248)."""
    b = _binding(state)
    sub = state.substrate
    t = sub.step_counter
    b.sync_params(state.pool)
    if not b.pinned:  # page-lock the host planes once: uploads/downloads become direct DMA
        b.dev.pin(sub.front)
        b.dev.pin(sub.back)
        b.pinned = True
    if b.device_ahead:
        _download_front(state)
    phys = state.config.physics
    rad = _radiation_active(state)
    flags = (_lib.F_RECORD_EVENTS | _lib.F_NO_CENSUS) if rad else 0
    # upload front -> pass 1 -> pass 2 -> download into back, pipelined over
    # row bands inside the library (evo_step_host)
    counts, adoptions, _ = b.dev.step_host(sub.front, sub.back, step_scalars(t, phys), t, flags=flags,
                                           source_map=phys.energy_source_map)
    if rad:
        events = b.dev.read_events()
        if len(events):
            gi_before = sub.back.genome_index.copy()
            _radiation_fn(state)(events, state.pool, state.config.evolution, sub.back, state.master_seed, t)
            moved = np.flatnonzero(sub.back.genome_index.ravel() != gi_before.ravel())
            if len(moved):
                b.dev.patch_genomes(moved, sub.back.genome_index.ravel()[moved])
        gi = sub.back.genome_index
        counts = np.bincount(gi[gi >= 0], minlength=int(state.pool.capacity))
        b.dev.census_finish(t)  # resets the device accumulators
        newly_dead = state.pool.update_census(counts, t + 1)
        b.pool_version = None
        b.sync_params(state.pool)
    else:
        newly_dead = state.pool.update_census(counts, t + 1)
    sub.swap_buffers()
    state.last_adoptions = int(adoptions)
    state.last_extinctions = len(newly_dead)
    b.device_ahead = False
    fr = getattr(state.config, "field_radiation", None)
    if fr is not None and fr.every > 0 and sub.step_counter % fr.every == 0:
        from .radiation import field_radiation

        field_radiation(state, sub.step_counter, fr.p)
        _download_front(state)  # keep the host mirror current in host-resident mode


def _download_front(state) -> None:
    b = _binding(state)
    b.dev.download(state.substrate.front)
    _fold_census(state)
    b.device_ahead = False


def _fold_census(state):
    """Bring the device's deferred census into the host pool; returns the
    device's per-slot peaks (what the records of the live slots now hold)."""
    b = _binding(state)
    counts, st, death, peak = b.dev.read_census()
    pool = state.pool
    if isinstance(pool, SlotPool):
        # the device already holds these slot states; pool.version is not
        # bumped, so changes the host made since the last sync stay pending
        pool.apply_device_census(st, death, peak)
        return peak
    # foreign pool (e.g. the reference GenomePool): replay update_census in
    # death-step order, feeding each slot's peak so peaks update identically
    live = np.asarray(pool.live_mask(), bool)
    newly = [i for i in np.flatnonzero(live) if st[i] == 2]
    for d in sorted({int(death[i]) for i in newly}):
        feed = np.where(live, np.maximum(peak, 1), 0).astype(np.int64)
        for i in newly:
            if int(death[i]) <= d:
                feed[i] = 0
        pool.update_census(feed, d)
    feed = np.where(np.asarray(pool.live_mask(), bool), peak, 0).astype(np.int64)
    pool.update_census(np.maximum(feed, 1) * np.asarray(pool.live_mask(), np.int64), int(state.substrate.step_counter))


def sync_to_host(state) -> None:
    """Make the host mirror (front planes + pool census) current."""
    b = getattr(state, "_evo_binding", None)
    if b is not None and b.device_ahead:
        _download_front(state)


class _GenomePatches:
    """Stand-in for the back PlaneSet handed to the host radiation callback
    in a device-resident run: ``genome_index.ravel()`` / ``.reshape(-1)``
    return a recorder whose item assignments (children installed at adoption
    targets, physics.py:389-392) are collected and patched onto the device."""

    def __init__(self):
        self.cells: list = []
        self.slots: list = []

    @property
    def genome_index(self):
        return self

    def ravel(self):
        return self

    def reshape(self, *shape):
        return self

    def __setitem__(self, cell, slot):
        self.cells.append(int(cell))
        self.slots.append(int(slot))


def _device_radiation_step(state, b, t, phys) -> None:
    """One step with adoption-driven radiation, device-resident: the device
    steps with adoption events recorded and the census deferred; the host
    runs the radiation callback on the compacted events (physics.py:346-392),
    the children it installs are patched onto the device genome plane, and
    the census (physics.py:395-404) runs on the device's counts corrected for
    those patches; new slots are expressed on the device before the next step."""
    dev = b.dev
    dev.step_raw(step_scalars(t, phys), t, flags=_lib.F_RECORD_EVENTS | _lib.F_NO_CENSUS,
                 source_map=phys.energy_source_map)
    events = dev.read_events()
    counts = dev.census_take().astype(np.int64)
    if len(events):
        patches = _GenomePatches()
        _radiation_fn(state)(events, state.pool, state.config.evolution, patches, state.master_seed, t)
        if patches.cells:
            cells = np.asarray(patches.cells, np.int64)
            slots = np.asarray(patches.slots, np.int32)
            dev.patch_genomes(cells, slots)
            winner = dict(zip(events.target.tolist(), events.winner_slot.tolist()))
            for c, sl in zip(patches.cells, patches.slots):  # the target held the winner's slot
                counts[winner[c]] -= 1
                counts[sl] += 1
    newly_dead = state.pool.update_census(counts, t + 1)
    b.pool_version = None
    b.sync_params(state.pool)  # children expressed in one launch, slot table + peaks pushed
    state.last_adoptions = len(events)
    state.last_extinctions = len(newly_dead)


def run(state, steps: int, hooks=(), should_stop: Optional[Callable[[], bool]] = None) -> None:
    """engine.run (engine.py:251-271): device-resident between hooks, with
    adoption-driven radiation (when its probabilities are non-zero) on the
    host per step over device-compacted events."""
    rad = _radiation_active(state)
    b = _binding(state)
    sub = state.substrate
    b.sync_params(state.pool)
    if not b.device_ahead:
        b.dev.upload(sub.front)
    phys = state.config.physics
    fr = getattr(state.config, "field_radiation", None)
    periods = [h.every for h in hooks] + ([fr.every] if fr is not None and fr.every > 0 else [])
    done = 0
    while done < steps:
        if should_stop is not None and should_stop():
            break
        t = sub.step_counter
        n = 1
        if rad:
            _device_radiation_step(state, b, t, phys)
        else:
            if should_stop is None:
                # the steps up to the next hook / radiation event go down as one
                # evo_run (one CUDA graph launch per 128 steps: small worlds
                # are launch-bound)
                n = min([steps - done] + [e - t % e for e in periods])
            if n > 1:
                b.dev.run([step_scalars(t + j, phys) for j in range(n)], t, source_map=phys.energy_source_map)
            else:
                b.dev.step_raw(step_scalars(t, phys), t, source_map=phys.energy_source_map)
        sub.step_counter = t + n
        done += n
        b.device_ahead = True
        if fr is not None and fr.every > 0 and sub.step_counter % fr.every == 0:
            from .radiation import field_radiation

            field_radiation(state, sub.step_counter, fr.p)
        due = [h for h in hooks if sub.step_counter % h.every == 0]
        dev_due = [h for h in due if getattr(h, "device", False)]
        due = [h for h in due if not getattr(h, "device", False)]
        if dev_due:
            if not rad:
                adoptions, extinctions = b.dev.read_stats()
                state.last_adoptions, state.last_extinctions = int(adoptions), int(extinctions)
            _fire(state, dev_due)
        if due:
            _download_front(state)
            if not rad:
                adoptions, extinctions = b.dev.read_stats()
                state.last_adoptions, state.last_extinctions = int(adoptions), int(extinctions)
            _fire(state, due)
            b.sync_params(state.pool)
            b.dev.upload(sub.front)  # hooks may write the front
    if b.device_ahead:
        _download_front(state)
        if not rad:
            adoptions, extinctions = b.dev.read_stats()
            state.last_adoptions, state.last_extinctions = int(adoptions), int(extinctions)


def _fire(state, hooks) -> None:
    for h in hooks:
        if state.substrate.step_counter % h.every == 0:
            try:
                h.fn(state)
            except Exception:
                log.exception("hook failed at step %d", state.substrate.step_counter)


def build_action_field(state) -> ActionField:
    """Sense + controller on the device for every occupied front cell."""
    b = _binding(state)
    b.sync_params(state.pool)
    if b.device_ahead:
        _download_front(state)
    b.dev.upload(state.substrate.front)
    t = state.substrate.step_counter
    b.dev.pass1(step_scalars(t, state.config.physics), t, phases=0, flags=_lib.F_EXPORT_ACTIONS)
    cells, acts = b.dev.get_actions()
    if len(cells) == 0:
        return ActionField.empty()
    return ActionField.from_block(cells, acts)


_FNV_OFFSET = 0xCBF29CE484222325


def digest(state) -> int:
    """64-bit FNV-1a over every front plane in channel-table order, then
    genome, then rotation (engine.py:301-315)."""
    import ctypes as C

    sync_to_host(state)
    lib = _lib.load()
    front = state.substrate.front
    h = C.c_uint64(_FNV_OFFSET)
    arrays = []
    for spec in state.substrate.specs:
        arr = front.channels[spec.name]
        arrays.extend(arr[k] for k in range(spec.arity))
    arrays += [front.genome_index, front.rotation]
    for a in arrays:
        buf = np.ascontiguousarray(a).view(np.uint8).reshape(-1)
        _lib.check(lib.evo_fnv1a64(h.value, _lib.ptr(buf), buf.size, C.byref(h)))
    return int(h.value)


# -- state construction (engine.py:94-139) -------------------------------------------


def new_state(config: ExperimentConfig, workers: int = 1, seed_population: bool = True) -> SimState:
    """A ready-to-run state from a validated config (engine.py:94-107).  The
    pool's net factory defers expression to the device: admitted genomes are
    expressed in one batched CPPN launch (evo_express_cppn) when the state
    first steps, bit-identical to the reference's generate_network."""
    from .radiation import device_net_factory

    hyper = config.hypernet
    sub = create_substrate(config.grid.width, config.grid.height)
    pool = SlotPool(DEFAULT_POOL_CAPACITY, net_factory=device_net_factory(hyper.hidden_size, hyper.tau, hyper.w_max))
    state = SimState(substrate=sub, pool=pool, config=config, master_seed=config.seed, workers=workers)
    if seed_population and config.initial_population > 0:
        seed_initial_population(state, config.initial_population)
    return state


def seed_initial_population(state, count: int) -> None:
    """Scatter fresh organisms onto distinct front cells (engine.py:110-139):
    placement and headings from the "seed_cells" stream, each genome from its
    own "init_genome" stream, energy = infrastructure = 1."""
    from .neat import init_genome, stream

    sub = state.substrate
    if count > state.pool.capacity:
        raise ValueError("initial population exceeds pool capacity")
    if count > sub.width * sub.height:
        raise ValueError("initial population exceeds cell count")
    sync_to_host(state)
    t = sub.step_counter
    g = stream(state.master_seed, t, "seed_cells")
    cells = g.choice(sub.width * sub.height, size=count, replace=False)
    rots = g.integers(0, 8, size=count)
    front = sub.front
    gi = front.genome_index.reshape(-1)
    energy = front.channels["energy"][0].reshape(-1)
    infra = front.channels["infrastructure"][0].reshape(-1)
    rot = front.rotation.reshape(-1)
    for i in range(count):
        genome = init_genome(stream(state.master_seed, t, "init_genome", i), state.pool.innovations)
        slot = state.pool.admit(genome, parents=(), birth_step=t)
        if slot is None:
            raise RuntimeError("pool rejected a seed genome")
        c = int(cells[i])
        gi[c] = slot
        energy[c] = 1.0
        infra[c] = 1.0
        rot[c] = rots[i]


def gather_sensors(sub, x: int, y: int) -> np.ndarray:
    """Scalar sensor vector of one cell (engine.py:142-161): self then the
    eight neighbours in the cell's rotation order, channels E, I, C0..C2.
    (The device builds these vectors in shared memory; this host version is
    the reference's per-cell helper over the host front planes.)"""
    from .physics import KERNEL_OFFSETS, PERM_TABLE

    w, h = sub.width, sub.height
    front = sub.front
    planes = (front.channels["energy"][0], front.channels["infrastructure"][0], front.channels["communication"][0],
              front.channels["communication"][1], front.channels["communication"][2])
    r = int(front.rotation[y, x])
    out = np.empty(45, np.float32)
    coords = [(x, y)] + [((x + int(KERNEL_OFFSETS[j, 0])) % w, (y + int(KERNEL_OFFSETS[j, 1])) % h)
                         for j in PERM_TABLE[r]]
    for s, (cx, cy) in enumerate(coords):
        for ch, p in enumerate(planes):
            out[s * 5 + ch] = p[cy, cx]
    return out


# -- live parameter steering (engine.py:321-390) -------------------------------------

_PARAM_RANGES: dict[str, tuple[float, float]] = {
    "physics.cycle_amplitude": (0.0, 2.0),
    "physics.cycle_period": (2, 100000),
    "physics.drain_fraction": (0.0, 1.0),
    "physics.invest_rate": (0.0, 10.0),
    "physics.liquidate_rate": (0.0, 10.0),
    "physics.invest_efficiency": (0.0, 1.0),
    "physics.liquidate_efficiency": (0.0, 1.0),
    "physics.explore_fraction": (0.0, 1.0),
    "physics.upkeep": (0.0, 1.0),
    "physics.decay_on_starvation": (0.0, 1.0),
    "physics.death_threshold": (0.0, 1.0),
    "evolution.weight_perturb_prob": (0.0, 1.0),
    "evolution.weight_perturb_sigma": (1e-6, 5.0),
    "evolution.weight_reset_prob": (0.0, 1.0),
    "evolution.add_connection_prob": (0.0, 1.0),
    "evolution.add_node_prob": (0.0, 1.0),
    "evolution.toggle_enable_prob": (0.0, 1.0),
    "evolution.c1": (0.0, 10.0),
    "evolution.c2": (0.0, 10.0),
    "evolution.c3": (0.0, 10.0),
    "evolution.p_radiation": (0.0, 1.0),
    "evolution.p_merge": (0.0, 1.0),
    "hypernet.tau": (0.0, 0.99),
    "hypernet.w_max": (0.1, 10.0),
}
_INT_PARAMS = {"physics.cycle_period"}


def describe_params(state) -> list[dict]:
    """Steerable parameters with current values and ranges (engine.py:351-358)."""
    items = []
    for path, (lo, hi) in _PARAM_RANGES.items():
        section, name = path.split(".")
        items.append({"path": path, "value": getattr(getattr(state.config, section), name), "min": lo, "max": hi})
    return items


def validate_param(path: str, value):
    """Check a steering request without touching any state (engine.py:361-376)."""
    if path not in _PARAM_RANGES:
        raise ValueError(f"unknown parameter {path!r}")
    lo, hi = _PARAM_RANGES[path]
    if isinstance(value, bool) or not isinstance(value, (int, float)):
        raise ValueError(f"{path} expects a number")
    if path in _INT_PARAMS:
        if value != int(value):
            raise ValueError(f"{path} must be an integer")
        value = int(value)
    else:
        value = float(value)
    if not lo <= value <= hi:
        raise ValueError(f"{path} must be in [{lo}, {hi}]")
    return value


def apply_param(state, path: str, value) -> None:
    """Set one steerable parameter (engine.py:379-390).  Physics scalars are
    recomputed from the config at every step, so the next device step (or the
    next step of a device-resident run) uses the new value without a sync;
    hypernet tau / w_max apply to genomes expressed from now on."""
    value = validate_param(path, value)
    section, name = path.split(".")
    obj = getattr(state.config, section)
    old = getattr(obj, name)
    setattr(obj, name, value)
    try:
        obj.validate()
    except ValueError:
        setattr(obj, name, old)
        raise
    if section == "hypernet" and isinstance(state.pool, SlotPool):
        from .radiation import device_net_factory

        hyper = state.config.hypernet
        state.pool.net_factory = device_net_factory(_hidden_of(state), hyper.tau, hyper.w_max)


def render_rgb(state, norm_energy: float = 1.0, norm_infrastructure: float = 1.0):
    """RGBA frame of the state's front buffer (substrate.py:147-165).  When the
    newest planes are on the device (a device-resident run) the frame is
    rendered there and only 4 B/cell come back; otherwise the host mirror is
    rendered.  Both are bit-identical to the reference's frame."""
    from .substrate import RgbFrame
    from .substrate import render_rgb as host_render

    if norm_energy == 0 or norm_infrastructure == 0:
        raise ValueError("display norms must be non-zero")
    b = getattr(state, "_evo_binding", None)
    sub = state.substrate
    if b is not None and b.device_ahead:
        return RgbFrame(sub.width, sub.height, b.dev.render_rgb(norm_energy, norm_infrastructure))
    return host_render(sub, norm_energy, norm_infrastructure)


# -- BASELINE synthetic states -------------------------------------------------------


def baseline_state(name: str = "c2", seed: int = 0, width: int | None = None, height: int | None = None,
                   genomes: int | None = None) -> SimState:
    """A seeded BASELINE.json configuration (synth.py draw order), optionally
    resized (bounded CPU samples / parity windows)."""
    cfg = BASELINE_CONFIGS[name]
    w = width or cfg.width
    h = height or cfg.height
    g = genomes or cfg.genomes
    ec = ExperimentConfig(grid=GridConfig(w, h), seed=seed, hypernet=HypernetConfig(cfg.hidden),
                          evolution=EvolutionRates(p_radiation=0.0, p_merge=0.0))  # SURVEY.md §8d notes
    ec.physics.cycle_period = cfg.cycle_period
    ec.field_radiation = FieldRadiationConfig(cfg.radiation_every, cfg.radiation_p or 0.01)
    sub = create_substrate(w, h)
    E, I, Cm, gi, rot = synth_arrays(h, w, g, seed, cfg.sparse_infra)
    f = sub.front
    f.channels["energy"][0] = E
    f.channels["infrastructure"][0] = I
    f.channels["communication"][:] = Cm
    f.genome_index[:] = gi
    f.rotation[:] = rot
    cap = max(cfg.capacity, g)
    pool = SlotPool(cap)
    genomes = [None] * g
    if cfg.radiation_every:
        from .radiation import device_net_factory
        from .synth import synth_genomes

        from .neat import pack

        genomes, pool.innovations = synth_genomes(g, seed)
        for gen in genomes:  # flat arrays cached for the native radiation mutation
            pack(gen)
        pool.net_factory = device_net_factory(cfg.hidden)
    for i, p in enumerate(synth_params(g, cfg.hidden, seed)):
        pool.install(i, p, genome=genomes[i])
    return SimState(substrate=sub, pool=pool, config=ec, master_seed=seed)
