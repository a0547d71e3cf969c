"""Seeded synthetic inputs for the BASELINE.json configurations.

Draw order (pinned so the oracle and the device see the same
state): g = default_rng(seed); E = g.random((H,W), f32); I = g.random((H,W),
f32) [config 5: then I[g.random((H,W)) < 0.9] = 0]; C = g.standard_normal
((3,H,W)).astype(f32); theta = g.random((H,W))*2*pi -> rot = floor(theta /
(pi/4)) mod 8; gi = g.integers(0, G, (H,W), int32).  Weights from
default_rng(seed+1), slot order: direct W = N(0,1)*0.5 (13,45), b = 0;
hidden W1 = N*0.3 (H,45), W2 = N*0.3 (13,H), biases 0.  ("N(0, s)" in
BASELINE.json is read as a standard deviation.)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .hypernet import DenseParams, DirectParams

__all__ = ["BaselineConfig", "BASELINE_CONFIGS", "synth_arrays", "synth_params", "synth_genomes"]


@dataclass(frozen=True)
class BaselineConfig:
    name: str
    width: int
    height: int
    genomes: int
    hidden: int
    steps: int
    sparse_infra: bool = False
    cycle_period: int = 20
    capacity: int = 0          # pool capacity (0: = genomes)
    radiation_every: int = 0   # field radiation period (config 3)
    radiation_p: float = 0.0   # fraction of occupied cells irradiated


# BASELINE.json "configs" (the multi-GPU layouts of configs 4/5 are handled
# by the callers; config 3's radiation by radiation.field_radiation).
BASELINE_CONFIGS = {
    "c1": BaselineConfig("c1-64x64-g8-direct", 64, 64, 8, 0, 100),
    "c2": BaselineConfig("c2-1024x1024-g64-direct", 1024, 1024, 64, 0, 1000),
    "c3": BaselineConfig("c3-4096x4096-g256-direct-rad50", 4096, 4096, 256, 0, 1000, capacity=2048,
                         radiation_every=50, radiation_p=0.01),
    "c4": BaselineConfig("c4-16384x16384-g1024-direct", 16384, 16384, 1024, 0, 500),
    "c5": BaselineConfig("c5-32768x32768-g4096-h128", 32768, 32768, 4096, 128, 200, sparse_infra=True),
}


def synth_arrays(height: int, width: int, genomes: int, seed: int = 0, sparse_infra: bool = False):
    g = np.random.default_rng(seed)
    E = g.random((height, width), dtype=np.float32)
    I = g.random((height, width), dtype=np.float32)
    if sparse_infra:
        I[g.random((height, width)) < 0.9] = 0
    C = g.standard_normal((3, height, width)).astype(np.float32)
    theta = g.random((height, width)) * (2.0 * np.pi)
    rot = (np.floor(theta / (np.pi / 4)) % 8).astype(np.uint8)
    gi = g.integers(0, genomes, (height, width), dtype=np.int32)
    return E, I, C, gi, rot


def synth_params(genomes: int, hidden: int = 0, seed: int = 0):
    g = np.random.default_rng(seed + 1)
    if hidden == 0:
        return [DirectParams((g.standard_normal((13, 45)) * 0.5).astype(np.float32), np.zeros(13, np.float32))
                for _ in range(genomes)]
    out = []
    for _ in range(genomes):
        w1 = (g.standard_normal((hidden, 45)) * 0.3).astype(np.float32)
        w2 = (g.standard_normal((13, hidden)) * 0.3).astype(np.float32)
        out.append(DenseParams(w1, np.zeros(hidden, np.float32), w2, np.zeros(13, np.float32)))
    return out


def synth_genomes(genomes: int, seed: int = 0, counter=None):
    """Config-3 pattern networks, one per initial slot, from default_rng(seed+2)
    (neat.init_c3_genome)."""
    from .neat import InnovationCounter, init_c3_genome

    g = np.random.default_rng(seed + 2)
    counter = counter if counter is not None else InnovationCounter()
    return [init_c3_genome(g, counter) for _ in range(genomes)], counter
