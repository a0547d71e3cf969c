"""Benchmark of the evoca substrate step on B200 (BASELINE.json metric:
cell-updates/sec of the full step, and % of the HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

Workload (default, the largest single-GPU BASELINE.json configuration,
configs[2]): 4096x4096 torus, 256 genomes (pool capacity 2048), direct
45->13 controller, field radiation every 50 steps (1 % of occupied cells move
to host-mutated children whose weights the device expresses); synthetic
seeded state (paper_2406_09654_b200/synth.py).  The timed window is placed so
that it contains one radiation step (or one per 50 steps for >= 50 steps).
--config c2 / c4 / c5 select the other BASELINE configurations.
A step = one full substrate update (pass 1 + pass 2, plus the radiation
event on its steps).  Each timed step is bracketed by CUDA events on the
launching stream, with an L2 flush (a 256 MiB memset, twice the 126 MB L2)
before it and outside the timed interval, so the state (839 MB for config 3,
52 MB for config 2) is read from HBM every step.  Multi-GPU: one process per
GPU (torchrun); the torus grows with the GPU count ((H*N) x W, weak scaling)
and is split into row strips, one per GPU, with NCCL halo exchanges and a
census all_reduce inside every timed step (paper_2406_09654_b200/strips.py);
the slowest rank's time is reported.  --strips forces that path on one GPU.

--impl reference times the reference algorithm on the host cores: the
oracle port (oracle/oracle.py; the reference is pure Python and cannot be
compiled), each step a bounded sample (a 1024x1024 window of the same
workload - all of config 2 - or 512x512 for runs over 100 steps) so the run stays within minutes.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_CELL = 50  # 25 B state read + 25 B written per cell-update
# split over the two launches of a step: pass 1 reads the 25 B
# state and writes the final E and C planes (16 B); pass 2 writes the final
# infrastructure, genome and rotation planes (9 B)
BYTES_PER_CELL_PASS1 = 25 + 16
BYTES_PER_CELL_PASS2 = 9
FLOP_PER_CELL_DIRECT = 2 * 45 * 13
L2_FLUSH_BYTES = 256 << 20


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured", d
    except Exception:
        return 6650.0, "fallback", {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._loop, daemon=True)

    def _loop(self):
        # NVML every 5 ms (a config-3 window of 20 steps lasts ~40 ms); the
        # nvidia-smi query below is the fallback (~50 ms per call)
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            bits = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append([str(sm), str(mx), ""] + ["Active" if r & b else "Not Active" for b in bits])
                self._stop.wait(0.005)
            return
        except Exception:
            pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and s[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def run_ours(args, rank, world, local):
    import torch

    from paper_2406_09654_b200 import _lib, engine, physics
    from paper_2406_09654_b200.synth import BASELINE_CONFIGS

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = BASELINE_CONFIGS[args.config]
    # strips: every rank holds the same seeded state (its strip of a
    # (H * world) x W torus) so that the pool - and with it config 3's
    # field radiation, which every rank applies identically - is shared
    state = engine.baseline_state(args.config, seed=args.seed if (world > 1 or args.strips) else args.seed + rank)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sh = stream.cuda_stream
    phys = state.config.physics
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    ncell = cfg.width * cfg.height
    strips = world > 1 or args.strips
    if strips:
        # weak scaling: a (H * world) x W torus, one H x W row strip per GPU,
        # NCCL halo exchanges + census all_reduce inside every step
        from paper_2406_09654_b200.strips import DeviceStrip, HaloComm, StripPlan

        plan = StripPlan(cfg.height * world, cfg.width, world)
        strip = DeviceStrip(plan, rank, state.pool.capacity, cfg.hidden, device=local, comm=HaloComm(rank, world))
        dev = strip.dev
        dev.set_params([state.pool.params(s) for s in range(state.pool.capacity)])
        dev.set_slots(state.pool.slot_states())
    else:
        dev = engine.device_of(state, device=local)
        state._evo_binding.sync_params(state.pool)
    dev.upload(state.substrate.front)
    dev.sync()

    radiate = cfg.radiation_every > 0  # config 3: field radiation every 50 steps, amortised

    def one_step(sc, t, e0=None, e1=None, e2=None):
        if e0 is not None:
            e0.record(stream)
        if strips:
            strip.step(sc, t)
            if e1 is not None:
                e1.record(stream)
            if radiate and (t + 1) % cfg.radiation_every == 0:
                # over the strips: global draw order, summed parent counts,
                # identical children on every rank (DeviceStrip.field_radiation)
                strip.field_radiation(state.pool, state.master_seed, t + 1, cfg.radiation_p, wait=stream.synchronize)
            if e2 is not None:
                e2.record(stream)
            return
        # the call engine.run makes; the library records its own event between
        # the two passes while profiling is on (evo_profile)
        dev.step_raw(sc, t, stream=sh)
        if radiate and (t + 1) % cfg.radiation_every == 0:
            from paper_2406_09654_b200 import radiation

            state.substrate.step_counter = t + 1
            # host NEAT planned while the step runs; then the radiation's
            # device calls (on the context's own stream) wait for the step
            radiation.field_radiation(state, t + 1, cfg.radiation_p, wait=stream.synchronize)
        if e2 is not None:
            e2.record(stream)

    # config 3's field radiation fires after every step t with (t+1) % 50 == 0;
    # start the clock so that one such step falls in the middle of the timed
    # window (windows of >= 50 steps hold one per 50 steps anyway)
    t = 0
    if radiate:
        every = cfg.radiation_every
        t = (every - 1 - min(args.steps, every) // 2 - args.warmup) % every
    for _ in range(args.warmup):
        flush.zero_()
        one_step(physics.step_scalars(t, phys), t)
        t += 1
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    scal = [physics.step_scalars(t + i, phys) for i in range(args.steps)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    if not strips:
        dev.profile(True)
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            flush.zero_()
            one_step(scal[i], t, *ev[i])
            t += 1
        torch.cuda.synchronize()
    if strips:
        k1 = sum(a.elapsed_time(m) for a, m, _ in ev)
        k2 = sum(m.elapsed_time(z) for _, m, z in ev)
        total_ms = k1 + k2
    else:
        # whole steps (radiation events included) between the bench's own
        # events; pass 1 from the library's per-step events, the rest is pass 2
        total_ms = sum(a.elapsed_time(z) for a, _, z in ev)
        k1, _, nprof = dev.profile_read()
        dev.profile(False)
        assert nprof == args.steps, (nprof, args.steps)
        k2 = total_ms - k1
    if world > 1:
        tt = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(tt.item())
    adoptions, _ = dev.read_stats()

    # e2e through the public API with host-resident planes, every step: H2D of
    # the front planes, the step, D2H of the new planes, census read-back.
    # One GPU: engine.step (the reference's drop-in entry point).  N GPUs: each
    # rank's row strip through DeviceStrip (halo exchanges + census
    # all_reduce inside), with its own page-locked host planes.
    e2e_steps = max(3, min(args.steps, 20))
    if strips:
        row0, h = plan.rows(rank)
        hf = state.substrate.front
        E = np.ascontiguousarray(hf.channels["energy"][0][:h])
        I = np.ascontiguousarray(hf.channels["infrastructure"][0][:h])
        Cm = np.ascontiguousarray(hf.channels["communication"][:, :h])
        gi = np.ascontiguousarray(hf.genome_index[:h])
        rot = np.ascontiguousarray(hf.rotation[:h])
        for arr in (E, I, Cm, gi, rot):
            dev.lib.evo_host_register(arr.ctypes.data_as(__import__("ctypes").c_void_p), arr.nbytes)

        def e2e_step(t):
            dev.upload_arrays(E, I, Cm, gi, rot)
            strip.step(physics.step_scalars(t, phys), t)
            dev.download_arrays(E, I, Cm, gi, rot)
            dev.read_census()

        e2e_step(0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(e2e_steps):
            e2e_step(i + 1)
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        for arr in (E, I, Cm, gi, rot):
            dev.lib.evo_host_unregister(arr.ctypes.data_as(__import__("ctypes").c_void_p))
        e2e_api = "DeviceStrip.step with evo_upload_planes / evo_download_planes of the rank's strip"
        e2e_cells = h * cfg.width
    else:
        e2e_state = engine.baseline_state(args.config, seed=args.seed + rank)
        engine.device_of(e2e_state, device=local)
        engine.step(e2e_state)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            engine.step(e2e_state)
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        e2e_api = "paper_2406_09654_b200.engine.step(state) on host-resident planes (evo_step_host, banded H2D/step/D2H)"
        e2e_cells = ncell
    if world > 1:
        tt = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(tt.item())

    if rank != 0:
        return None
    # which pass-1 pipeline the library ran (evo_pass1): the
    # per-tile fused kernel for small direct pools, the gather path for large
    # direct pools, genome-sorted rows + tcgen05 for hidden-layer nets
    cap = max(cfg.capacity, cfg.genomes)
    if cfg.hidden > 0:
        p1_name = ("pass-1 pipeline on genome-sorted rows (7 launches: sort x4, k_hid_sense, "
                   "k_hid_net tcgen05 3xTF32 MLP, k_physics_rows)")
        launches_per_step = 8
    elif cap > 68:
        p1_name = ("pass-1 pipeline, gather path, lazy fused evo_step (7 launches: k_gs_rank slot ranks - the "
                   "previous pass 2 wrote the sense texture -, k_gs_colscan, k_gs_scan_band, k_gs_scan_bands, "
                   "k_gs_scatter, k_gs_tilemap, k_direct_gather FFMA2 net + physics)" if not strips else
                   "pass-1 pipeline, gather path (8 launches: k_gs_count sense texture + slot ranks, "
                   "k_gs_colscan, k_gs_scan_band, k_gs_scan_bands, k_gs_scatter, k_gs_tilemap, "
                   "k_direct_gather FFMA2 net, k_physics_rows)")
        launches_per_step = 9 if strips else 8
    else:
        p1_name = "k_pass1_direct (pass 1: sense+net+physics)"
        launches_per_step = 2
    rows_path = cap > 68 or cfg.hidden > 0
    launches_per_step += 5 if strips else 0  # strips: halo pack/unpack x2, census epilogue
    n_rad = sum(1 for i in range(args.steps) if radiate and (t - args.steps + i + 1) % cfg.radiation_every == 0)
    hbm, hbm_kind, pk = peaks()
    step_s = total_ms / 1e3 / args.steps
    value = ncell * world / step_s
    achieved_gbs = ncell * BYTES_PER_CELL / step_s / 1e9
    k1_s, k2_s = k1 / 1e3 / args.steps, k2 / 1e3 / args.steps
    # DRAM read + write bytes of the dominant launch(es) per step, from an ncu
    # capture of this workload (profiles/ncu_traffic.json, tools/traffic_json.py):
    # the pass-1 pipeline's total on the gather / genome-sorted paths, the
    # fused kernel's on the tile path
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof) and not strips:
        try:
            rec = json.load(open(prof)).get(args.config, {})
            if rows_path:
                traffic = rec.get("pass1_dram_bytes_per_step")
            else:
                per = rec.get("per_kernel_dram_bytes_per_launch", {})
                traffic = next((v for k, v in per.items() if "k_pass1_direct" in k), None)
        except Exception:
            traffic = None
    clk = clocks.summary()
    sm_hz = (clk["sm_mhz"] or 1965.0) * 1e6
    fp32_peak = 148 * 128 * 2 * sm_hz / 1e12  # derived FP32 CUDA-core peak at the sampled clock
    line = {
        "metric": "cell-updates/sec (full step)",
        "value": value,
        "unit": "cell-updates/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": step_s * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (seeded, BASELINE.json config distributions)",
        "config": {"workload": cfg.name, "grid": [cfg.height, cfg.width], "genomes": cfg.genomes,
                   "net": "45->13 direct" if cfg.hidden == 0 else f"45->{cfg.hidden}->13",
                   "cells_per_gpu": ncell, "l2": "flushed before every timed step (256 MiB memset)",
                   "radiation_steps_timed": n_rad,
                   "parallelism": (f"row strips x{world} over a {cfg.height * world}x{cfg.width} torus, NCCL halo "
                                   "exchange + census all_reduce per step") if strips else "single GPU"},
        "roofline": {
            "kernel": (p1_name + ", dominant") if not strips else "strip step",
            "bound": "hbm",
            "achieved": (ncell * BYTES_PER_CELL_PASS1 / k1_s / 1e9) if not strips else achieved_gbs,
            "peak": hbm,
            "peak_kind": hbm_kind,
            "unit": "GB/s",
            "frac": ((ncell * BYTES_PER_CELL_PASS1 / k1_s / 1e9) if not strips else achieved_gbs) / hbm,
            "traffic": traffic,
            "traffic_over_algorithmic": (traffic / (ncell * BYTES_PER_CELL_PASS1)) if traffic else None,
            "algorithmic_bytes_per_cell": BYTES_PER_CELL_PASS1 if not strips else BYTES_PER_CELL,
            "units_per_launch": ncell,
            "step": {"achieved": achieved_gbs, "frac": achieved_gbs / hbm,
                     "algorithmic_bytes_per_cell": BYTES_PER_CELL},
            "kernels": [
                {"name": p1_name if not strips else
                 "strip step (exchanges + pass 1 + pass 2 + census)", "ms": k1_s * 1e3, "share": k1 / total_ms,
                 "fp32_tflops": ncell * FLOP_PER_CELL_DIRECT / k1_s / 1e12 if cfg.hidden == 0 else None,
                 "fp32_peak_tflops_derived": fp32_peak},
            ] + ([] if strips else [
                {"name": "k_resolve (pass 2: explore resolve+adoption+census"
                 + ("; writes the next step's sense texture)" if cap > 68 and cfg.hidden == 0 else ")")
                 + (" + field radiation every %d steps" % cfg.radiation_every if radiate else ""),
                 "ms": k2_s * 1e3, "share": k2 / total_ms},
            ]),
        },
        "e2e": {"value": ncell * world * e2e_steps / e2e_s, "unit": "cell-updates/s",
                "api": e2e_api,
                "h2d_bytes_per_step": (e2e_cells * 25 + state.pool.capacity * 9) * world,
                "d2h_bytes_per_step": (e2e_cells * 25 + state.pool.capacity * 4 + 16) * world},
        "gpu_launches": launches_per_step * args.steps + 6 * n_rad,
        "clocks": clk,
        "adoptions_last_step": int(adoptions),
    }
    if args.cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(args.config, budget_s=args.cpu_seconds)
    return line


def cpu_baseline(config: str, budget_s: float = 15.0, side: int | None = None, steps: int | None = None):
    """The oracle port (numpy + numba, like the reference) on the host cores,
    on a bounded sample of the workload: SURVEY.md §8d runs config 2 whole
    and the larger configs as 1024x1024 slices with the same distributions
    and genome counts."""
    from oracle import oracle as orc
    from paper_2406_09654_b200.synth import BASELINE_CONFIGS

    cfg = BASELINE_CONFIGS[config]
    side_h = min(cfg.height, side or 1024)
    side_w = min(cfg.width, side or 1024)
    p = orc.synth_planes(side_h, side_w, cfg.genomes, seed=0, sparse_infra=cfg.sparse_infra)
    net = orc.synth_net(cfg.genomes, cfg.hidden, seed=0)
    phys = orc.Phys(cycle_period=cfg.cycle_period)
    orc.step(orc.synth_planes(16, 16, cfg.genomes, seed=1), 0, net, phys)  # numba compile
    n = 0
    t0 = time.perf_counter()
    while True:
        p = orc.step(p, n, net, phys).planes
        n += 1
        el = time.perf_counter() - t0
        if (steps is not None and n >= steps) or (steps is None and el >= budget_s):
            break
    return {"value": side_h * side_w * n / el, "unit": "cell-updates/s", "cores": os.cpu_count(),
            "kind": "port", "sample": f"{n} oracle steps on a {side_h}x{side_w} window of {cfg.name} "
                                      f"(numpy/numba/BLAS, {os.cpu_count()} host threads)"}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    side = 1024 if args.steps <= 100 else 512
    from paper_2406_09654_b200.synth import BASELINE_CONFIGS

    cfg = BASELINE_CONFIGS[args.config]
    for _ in range(args.warmup):
        cpu_baseline(args.config, side=side, steps=1)
    cb = cpu_baseline(args.config, side=side, steps=args.steps)
    return {
        "impl": "reference",
        "metric": "cell-updates/sec (full step)",
        "value": cb["value"],
        "unit": "cell-updates/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (seeded, BASELINE.json config distributions)",
        "config": {"workload": cfg.name, "grid": [cfg.height, cfg.width], "genomes": cfg.genomes,
                   "sample_grid": [min(side, cfg.height), min(side, cfg.width)]},
        "cpu_baseline": cb,
        "e2e": {"value": cb["value"], "unit": "cell-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--strips", action="store_true", help="use the row-strip (multi-GPU) path even on one GPU")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank, world, local = dist_env()
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        line = run_ours(args, rank, world, local)
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
            dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
