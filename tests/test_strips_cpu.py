"""Multi-rank strip decomposition on CPU (gloo, world sizes 1-3).

Each rank steps its row strip with the numpy model of the device's two-pass
decomposition (oracle/strip_model.py) and the package's HaloComm exchanging
ghost rows through torch.distributed (gloo); the census is an all_reduce.
The reassembled result must equal the full-grid oracle step bit for bit,
which checks the strip plan, the exchange pattern (including the two-rank
case where up == down), the global tie-break indices across strip seams and
the census reduction."""

import os
import socket
import tempfile

import numpy as np
import pytest

from oracle import oracle as orc
from oracle import strip_model as sm
from paper_2406_09654_b200.strips import HaloComm, StripPlan

H, W, G = 23, 17, 6


def test_plan_partition():
    for Hh, world in ((23, 1), (23, 2), (23, 3), (8, 8), (1024, 8)):
        plan = StripPlan(Hh, 5, world)
        rows = [plan.rows(r) for r in range(world)]
        assert rows[0][0] == 0
        for (a, ha), (b, _) in zip(rows, rows[1:]):
            assert a + ha == b
        assert rows[-1][0] + rows[-1][1] == Hh
        assert max(h for _, h in rows) - min(h for _, h in rows) <= 1
        assert plan.up(0) == world - 1 and plan.down(world - 1) == 0
    with pytest.raises(ValueError):
        StripPlan(2, 5, 3)


def _state():
    p = orc.synth_planes(H, W, G, seed=11)
    rng = np.random.default_rng(3)
    p.gi[rng.random((H, W)) < 0.2] = -1
    # strong contention across seams
    p.I[rng.random((H, W)) < 0.3] = 0
    return p, orc.synth_net(G, 0, seed=11)


def _strip_step(rank, world, comm, p, net, phys, t):
    import torch

    plan = StripPlan(H, W, world)
    row0, h = plan.rows(rank)
    ext_E = np.zeros((h + 2, W), np.float32)
    ext_I = np.zeros((h + 2, W), np.float32)
    ext_C = np.zeros((3, h + 2, W), np.float32)
    ext_E[1:h + 1] = p.E[row0:row0 + h]
    ext_I[1:h + 1] = p.I[row0:row0 + h]
    ext_C[:, 1:h + 1] = p.C[:, row0:row0 + h]
    # front halo exchange: E, I, C0..2 packed
    planes = [ext_E, ext_I, ext_C[0], ext_C[1], ext_C[2]]
    first = torch.from_numpy(np.stack([q[1] for q in planes]))
    last = torch.from_numpy(np.stack([q[h] for q in planes]))
    gt = torch.empty_like(first)
    gb = torch.empty_like(first)
    comm.exchange(first, last, gt, gb)
    for i, q in enumerate(planes):
        q[0] = gt[i].numpy()
        q[h + 1] = gb[i].numpy()
    E, Cm, mI, mgi, rp, q = sm.pass1(ext_E, ext_I, ext_C, p.gi[row0:row0 + h].copy(), p.rot[row0:row0 + h].copy(),
                                     net, phys, t, W)
    ext_gi = np.zeros((h + 2, W), np.int32)
    ext_rp = np.zeros((h + 2, W), np.uint8)
    ext_q = np.zeros((h + 2, W), np.float32)
    ext_gi[1:h + 1], ext_rp[1:h + 1], ext_q[1:h + 1] = mgi, rp, q
    first = torch.from_numpy(np.stack([ext_gi[1], ext_q[1].view(np.int32), ext_rp[1].astype(np.int32)]))
    last = torch.from_numpy(np.stack([ext_gi[h], ext_q[h].view(np.int32), ext_rp[h].astype(np.int32)]))
    gt = torch.empty_like(first)
    gb = torch.empty_like(first)
    comm.exchange(first, last, gt, gb)
    ext_gi[0], ext_gi[h + 1] = gt[0].numpy(), gb[0].numpy()
    ext_q[0], ext_q[h + 1] = gt[1].numpy().view(np.float32), gb[1].numpy().view(np.float32)
    ext_rp[0], ext_rp[h + 1] = gt[2].numpy().astype(np.uint8), gb[2].numpy().astype(np.uint8)
    I, gi, rot, adopted = sm.pass2(ext_gi, ext_rp, ext_q, mI, row0, H, W)
    counts = torch.from_numpy(np.bincount(gi[gi >= 0], minlength=G).astype(np.int64))
    comm.sum_(counts)
    return row0, h, E, I, Cm, gi, rot, counts.numpy(), adopted


def _worker(rank, world, port, outdir):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p, net = _state()
        phys = orc.Phys(cycle_period=20, explore_fraction=0.9)
        comm = HaloComm(rank, world)
        for t in (0, 20):  # day-free and night (float64 sin(2pi)) steps
            res = _strip_step(rank, world, comm, p, net, phys, t)
            np.savez(os.path.join(outdir, f"r{rank}_t{t}.npz"), *res[2:8], meta=np.array(res[:2] + (res[8],)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [1, 2, 3])
def test_gloo_strips_match_full_grid_oracle(world):
    import torch.multiprocessing as mp

    p, net = _state()
    phys = orc.Phys(cycle_period=20, explore_fraction=0.9)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        for t in (0, 20):
            ref = orc.step(p, t, net, phys)
            E = np.zeros((H, W), np.float32)
            I = np.zeros((H, W), np.float32)
            Cm = np.zeros((3, H, W), np.float32)
            gi = np.zeros((H, W), np.int32)
            rot = np.zeros((H, W), np.uint8)
            adopted = 0
            for r in range(world):
                z = np.load(os.path.join(d, f"r{r}_t{t}.npz"))
                row0, h, a = z["meta"].tolist()
                E[row0:row0 + h], I[row0:row0 + h] = z["arr_0"], z["arr_1"]
                Cm[:, row0:row0 + h] = z["arr_2"]
                gi[row0:row0 + h], rot[row0:row0 + h] = z["arr_3"], z["arr_4"]
                counts = z["arr_5"]
                adopted += a
                assert np.array_equal(counts, ref.counts), "census all_reduce"
            got = orc.Planes(E, I, Cm, gi, rot)
            assert got.equal(ref.planes), f"world={world} t={t}"
            assert adopted == len(ref.events)
