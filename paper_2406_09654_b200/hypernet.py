"""Controller parameter types (hypernet.py of the reference).

``DenseParams`` is the reference's 45->H(tanh)->13 parameter set
(/root/reference/pkg/src/evoca/hypernet.py:77-84).  ``DirectParams`` is the
BASELINE.json 45->13 direct controller, an extension the reference does not
have (config.py:46-47 requires hidden >= 1); its semantics are the
reference forward pass with the hidden layer removed: z = s.W^T + b, then
the same sigmoid sequence and clip (hypernet.py:245-251).
The forward pass itself runs only on the device (pass-1 kernel).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["N_SENSORS", "N_ACTUATORS", "DenseParams", "DirectParams", "pack_params"]

N_SENSOR_SLOTS = 9
N_SENSE_SUBCHANNELS = 5
N_SENSORS = N_SENSOR_SLOTS * N_SENSE_SUBCHANNELS  # hypernet.py:35-38
N_ACTUATORS = 13


@dataclass
class DenseParams:
    w1: np.ndarray  # (hidden, 45)
    b1: np.ndarray  # (hidden,)
    w2: np.ndarray  # (13, hidden)
    b2: np.ndarray  # (13,)


@dataclass
class DirectParams:
    w: np.ndarray  # (13, 45)
    b: np.ndarray  # (13,)


def pack_params(params_list, hidden: int):
    """Stack per-slot parameters into the C-ABI layout of evo_set_params.
    ``None`` entries (free slots) become zeros."""
    n = len(params_list)
    if hidden == 0:
        w2 = np.zeros((n, N_ACTUATORS, N_SENSORS), np.float32)
        b2 = np.zeros((n, N_ACTUATORS), np.float32)
        for i, p in enumerate(params_list):
            if p is None:
                continue
            if isinstance(p, DirectParams):
                w2[i], b2[i] = p.w, p.b
            else:
                raise TypeError("a direct (hidden=0) substrate needs DirectParams per slot")
        return None, None, w2, b2
    w1 = np.zeros((n, hidden, N_SENSORS), np.float32)
    b1 = np.zeros((n, hidden), np.float32)
    w2 = np.zeros((n, N_ACTUATORS, hidden), np.float32)
    b2 = np.zeros((n, N_ACTUATORS), np.float32)
    for i, p in enumerate(params_list):
        if p is None:
            continue
        if p.w1.shape != (hidden, N_SENSORS) or p.w2.shape != (N_ACTUATORS, hidden):
            raise ValueError("DenseParams shape does not match the substrate's hidden size")
        w1[i], b1[i], w2[i], b2[i] = p.w1, p.b1, p.w2, p.b2
    return w1, b1, w2, b2
