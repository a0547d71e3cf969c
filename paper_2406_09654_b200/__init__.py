"""B200-native (sm_100a) implementation of the evoca per-step substrate update.

Drop-in for the hot path of the reference package ``evoca``
(/root/reference/pkg/src/evoca, arXiv 2406.09654 "Coralai"): the same
experiment API (``Substrate``/``PlaneSet`` with named channels, the
rotation-ordered Moore sensing kernel, ``ActionField`` actuators,
``PhysicsParams``, ``step``/``run``/``digest``) executed by hand-written CUDA
kernels behind a C ABI (include/evoca_b200.h, libevoca_b200.so).  There is
no CPU fallback.
"""

from .engine import (  # noqa: F401
    EvolutionRates,
    ExperimentConfig,
    GridConfig,
    Hook,
    HypernetConfig,
    SimState,
    baseline_state,
    build_action_field,
    device_of,
    digest,
    run,
    step,
    sync_to_host,
)
from .hypernet import DenseParams, DirectParams  # noqa: F401
from .physics import ActionField, AdoptionEvents, PhysicsParams  # noqa: F401
from .pool import SlotPool  # noqa: F401
from .substrate import STANDARD_CHANNELS, ChannelSpec, PlaneSet, Substrate, create_substrate  # noqa: F401

__version__ = "0.1.0"
