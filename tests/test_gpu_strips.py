"""Strip mode of the CUDA kernels: the torus split into 1-4 row strips
(separate strip contexts on one GPU, ghost rows exchanged by device copies,
census summed) must reproduce the single-context step bit for bit, and the
oracle given the same actions."""

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2406_09654_b200 import _lib, physics
from paper_2406_09654_b200.hypernet import DenseParams, DirectParams
from paper_2406_09654_b200.strips import DeviceStrip, StripPlan, step_local
from tests.test_gpu_parity import download, make_dev

pytestmark = pytest.mark.gpu


def _params(net):
    if net.hidden == 0:
        return [DirectParams(net.w2[i], net.b2[i]) for i in range(net.capacity)]
    return [DenseParams(net.w1[i], net.b1[i], net.w2[i], net.b2[i]) for i in range(net.capacity)]


def _strips(p, net, world):
    H, W = p.shape
    plan = StripPlan(H, W, world)
    strips = []
    for r in range(world):
        s = DeviceStrip(plan, r, net.capacity, hidden=net.hidden)
        s.dev.set_params(_params(net))
        s.dev.set_slots(np.ones(net.capacity, np.int8))
        row0, h = plan.rows(r)
        s.dev.upload_arrays(p.E[row0:row0 + h], p.I[row0:row0 + h], p.C[:, row0:row0 + h],
                            p.gi[row0:row0 + h], p.rot[row0:row0 + h])
        strips.append(s)
    return plan, strips


def _gather(plan, strips, p_like):
    H, W = p_like.shape
    out = orc.Planes(np.empty((H, W), np.float32), np.empty((H, W), np.float32), np.empty((3, H, W), np.float32),
                     np.empty((H, W), np.int32), np.empty((H, W), np.uint8))
    for r, s in enumerate(strips):
        row0, h = plan.rows(r)
        E = np.empty((h, W), np.float32)
        I = np.empty((h, W), np.float32)
        Cm = np.empty((3, h, W), np.float32)
        gi = np.empty((h, W), np.int32)
        rot = np.empty((h, W), np.uint8)
        s.dev.download_arrays(E, I, Cm, gi, rot)
        out.E[row0:row0 + h], out.I[row0:row0 + h], out.C[:, row0:row0 + h] = E, I, Cm
        out.gi[row0:row0 + h], out.rot[row0:row0 + h] = gi, rot
    return out


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("shape", [(64, 64), (70, 33)])
@pytest.mark.parametrize("genomes", [8, 300])
def test_strips_match_single_context(world, shape, genomes):
    """1-4 row strips (ghost rows filled by the halo exchange) reproduce the
    single context bit for bit: 8 genomes run the per-tile kernel, 300 the
    gather path (sense texture from the exchanged ghost rows, TMA build on
    widths divisible by 4, the LSU build otherwise) - the path the weak-
    scaling bench runs with config 3 on every GPU."""
    import torch

    H, W = shape
    p0 = orc.synth_planes(H, W, genomes, seed=H + world)
    p0.I[np.random.default_rng(1).random((H, W)) < 0.3] = 0
    net = orc.synth_net(genomes, 0, seed=2)
    ref = make_dev(p0, genomes, net)
    plan, strips = _strips(p0, net, world)
    params = physics.PhysicsParams(cycle_period=20, explore_fraction=0.8)
    for t in range(6):
        sc = physics.step_scalars(t, params)
        ref.step_raw(sc, t)
        step_local(strips, sc, t)
        torch.cuda.synchronize()
        got = _gather(plan, strips, p0)
        want = download(ref)
        assert got.equal(want), f"world={world} t={t}"
        c_ref = ref.read_census()[0]
        for s in strips:
            assert np.array_equal(s.dev.read_census()[0], c_ref)
    for s in strips:
        s.dev.close()
    ref.close()


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("shape", [(64, 64), (35, 132)])
def test_lazy_strips_match_single_context(world, shape):
    """Strips run the fused, lazy gather step too: between downloads the E, I,
    C state of a strip lives in its sense texture, evo_halo_pack / unpack(0)
    exchange texture rows (ghost rows of the texture) and (1) the pass-1
    records' rows (kept behind the strip's last record row).  Five steps
    without touching the planes, with unoccupied and starving cells, then a
    download; twice; bit-identical to the single context and to EVO_F_UNFUSED
    strips."""
    import torch

    from paper_2406_09654_b200 import _lib

    H, W = shape
    genomes = 300
    p0 = orc.synth_planes(H, W, genomes, seed=3 * H + world)
    rng = np.random.default_rng(5)
    p0.gi[rng.random((H, W)) < 0.25] = -1
    p0.I[rng.random((H, W)) < 0.2] *= np.float32(0.002)
    net = orc.synth_net(genomes, 0, seed=4)
    ref = make_dev(p0, genomes, net)
    plan, strips = _strips(p0, net, world)
    plan2, unfused = _strips(p0, net, world)
    params = physics.PhysicsParams(cycle_period=6, explore_fraction=0.8)
    t = 0
    for _ in range(2):
        for _ in range(5):
            sc = physics.step_scalars(t, params)
            ref.step_raw(sc, t)
            step_local(strips, sc, t)
            step_local(unfused, sc, t, flags=_lib.F_UNFUSED)
            t += 1
        torch.cuda.synchronize()
        want = download(ref)
        assert _gather(plan, strips, p0).equal(want), f"world={world} t={t}"
        assert _gather(plan2, unfused, p0).equal(want), f"unfused world={world} t={t}"
        c_ref = ref.read_census()[0]
        for s in strips:
            assert np.array_equal(s.dev.read_census()[0], c_ref)
    for s in strips + unfused:
        s.dev.close()
    ref.close()


@pytest.mark.parametrize("world", [1, 2, 3])
def test_strips_tensor_core_hidden_net(world):
    """The config-5 net (45->128 tanh->13 on tcgen05) in strip mode: per-cell
    results do not depend on the strip / bucket / tile placement, so 1-3
    strips reproduce the single context bit for bit."""
    import torch

    H, W = 48, 40
    p0 = orc.synth_planes(H, W, 24, seed=world, sparse_infra=True)
    net = orc.synth_net(24, 128, seed=4)
    ref = make_dev(p0, 24, net)
    plan, strips = _strips(p0, net, world)
    params = physics.PhysicsParams(cycle_period=20)
    for t in range(3):
        sc = physics.step_scalars(t, params)
        ref.step_raw(sc, t)
        step_local(strips, sc, t)
        torch.cuda.synchronize()
        assert _gather(plan, strips, p0).equal(download(ref)), f"world={world} t={t}"
    for s in strips:
        s.dev.close()
    ref.close()


def _rank_worker(rank, world, port, outdir, t_steps, genomes=9):
    """One rank of a world-2 run: its own process and CUDA context on cuda:0,
    DeviceStrip.step with the halo exchanges and census all_reduce going
    through gloo (StagedHaloComm) - the rank's kernels never wait on the
    other rank's kernels, only the host waits on the exchange."""
    import os

    import torch.distributed as dist

    from paper_2406_09654_b200.strips import StagedHaloComm

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = orc.synth_planes(70, 48, genomes, seed=21)
        p.I[np.random.default_rng(2).random((70, 48)) < 0.4] = 0  # contention across the strip seams
        net = orc.synth_net(genomes, 0, seed=21)
        plan = StripPlan(70, 48, world)
        s = DeviceStrip(plan, rank, net.capacity, hidden=0, device=0, comm=StagedHaloComm(rank, world))
        s.dev.set_params(_params(net))
        s.dev.set_slots(np.ones(net.capacity, np.int8))
        row0, h = plan.rows(rank)
        s.dev.upload_arrays(p.E[row0:row0 + h], p.I[row0:row0 + h], p.C[:, row0:row0 + h], p.gi[row0:row0 + h],
                            p.rot[row0:row0 + h])
        params = physics.PhysicsParams(cycle_period=20)
        for t in range(t_steps):
            s.step(physics.step_scalars(t, params), t)
        E = np.empty((h, 48), np.float32)
        I = np.empty((h, 48), np.float32)
        Cm = np.empty((3, h, 48), np.float32)
        gi = np.empty((h, 48), np.int32)
        rot = np.empty((h, 48), np.uint8)
        s.dev.download_arrays(E, I, Cm, gi, rot)
        counts, state, _, _ = s.dev.read_census()
        np.savez(os.path.join(outdir, f"r{rank}.npz"), E=E, I=I, C=Cm, gi=gi, rot=rot, counts=counts, state=state,
                 meta=np.array([row0, h]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("genomes", [9, 300])
def test_device_strips_two_processes_match_single_context(genomes):
    """DeviceStrip.step itself with world size 2 (two processes, gloo-staged
    exchanges) equals the single-context device step bit for bit after
    several steps, census included (9 genomes: per-tile kernel; 300: the
    gather path with its TMA texture build)."""
    import os
    import socket
    import tempfile

    import torch.multiprocessing as mp

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    steps = 5
    p = orc.synth_planes(70, 48, genomes, seed=21)
    p.I[np.random.default_rng(2).random((70, 48)) < 0.4] = 0
    net = orc.synth_net(genomes, 0, seed=21)
    dev = make_dev(p, genomes, net)
    params = physics.PhysicsParams(cycle_period=20)
    for t in range(steps):
        dev.step_raw(physics.step_scalars(t, params), t)
    want = download(dev)
    counts_want, state_want, _, _ = dev.read_census()
    dev.close()
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rank_worker, args=(2, port, d, steps, genomes), nprocs=2, join=True)
        got = orc.Planes(np.empty((70, 48), np.float32), np.empty((70, 48), np.float32),
                         np.empty((3, 70, 48), np.float32), np.empty((70, 48), np.int32), np.empty((70, 48), np.uint8))
        for r in range(2):
            z = np.load(os.path.join(d, f"r{r}.npz"))
            row0, h = z["meta"].tolist()
            got.E[row0:row0 + h], got.I[row0:row0 + h], got.C[:, row0:row0 + h] = z["E"], z["I"], z["C"]
            got.gi[row0:row0 + h], got.rot[row0:row0 + h] = z["gi"], z["rot"]
            assert np.array_equal(z["counts"], counts_want) and np.array_equal(z["state"], state_want)
    assert got.equal(want)
