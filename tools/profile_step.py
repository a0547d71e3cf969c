"""Run a few device steps of a BASELINE config for profiling (ncu / launch lists).

    python tools/profile_step.py [--config c2] [--steps 6] [--flush]
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--flush", action="store_true")
    ap.add_argument("--genomes", type=int, default=None)
    ap.add_argument("--width", type=int, default=None)
    ap.add_argument("--height", type=int, default=None)
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--time", action="store_true", help="CUDA-event time per step")
    ap.add_argument("--run", type=int, default=0, help="time dev.run (evo_run) of this many steps, wall clock")
    args = ap.parse_args()
    import torch

    from paper_2406_09654_b200 import engine, physics

    st = engine.baseline_state(args.config, genomes=args.genomes, width=args.width, height=args.height)
    dev = engine.device_of(st)
    st._evo_binding.sync_params(st.pool)
    dev.upload(st.substrate.front)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if args.flush else None
    times = []
    for t in range(args.steps):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        dev.step_raw(physics.step_scalars(t, st.config.physics), t, flags=args.flags, stream=s.cuda_stream)
        e1.record(s)
        times.append((e0, e1))
    torch.cuda.synchronize()
    if args.run:
        import time

        k = args.run
        for rep in range(3):
            scs = [physics.step_scalars(args.steps + rep * k + i, st.config.physics) for i in range(k)]
            t0 = time.perf_counter()
            dev.run(scs, args.steps + rep * k, stream=s.cuda_stream)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            print(f"evo_run {k} steps: {dt / k * 1e6:.2f} us/step (EVO_NO_GRAPH={os.environ.get('EVO_NO_GRAPH')})")
    if args.time:
        ms = [a.elapsed_time(b) for a, b in times]
        n = st.substrate.width * st.substrate.height
        best = min(ms[1:] or ms)
        print(f"step ms: {[round(x, 3) for x in ms]}  best {best:.3f} ms  {n / best / 1e6:.2f} G cell-updates/s")
    print("adoptions", dev.read_stats())
    if os.environ.get("EVOCA_B200_LIB"):
        import ctypes as C

        import numpy as np

        from paper_2406_09654_b200 import _lib

        out = np.zeros(8, np.uint64)
        _lib.check(_lib.load().evo_debug_phase_cycles(_lib.ptr(out), 1))
        names = ["bucket", "controller", "physics", "commit", "setup"]
        tot = float(out[:5].sum())
        for i, n in enumerate(names):
            print(f"phase {n:10s} {int(out[i]):>14d} cycles  {out[i] / tot * 100:5.1f}%  "
                  f"{out[i] / args.steps / 148:10.0f} per CTA-step")
        if out[7]:
            print(f"distinct genome slots per controller warp-iteration: {out[6] / out[7]:.2f}")
        hc = np.zeros(8, np.uint64)
        _lib.check(_lib.load().evo_debug_hidden_cycles(_lib.ptr(hc), 1))
        if hc.sum():
            names = ["tile end + L1 issue", "wait L1 MMA", "stage A1 + fetch", "epilogue (tanh, layer 2)",
                     "exchange sync", "finish + store", "tile-end sync + restage", "-"]
            tot = float(hc.sum())
            for i, n in enumerate(names):
                print(f"hid {n:22s} {hc[i] / tot * 100:5.1f}%  {hc[i] / 148 / args.steps:12.0f} cycles/CTA-step")


if __name__ == "__main__":
    main()
