import numpy as np, sys
sys.path.insert(0, '.')
from oracle import oracle as orc
from paper_2406_09654_b200 import _lib, physics
from tests.test_gpu_parity import make_dev, rel_err, oracle_phys_to_params
for hidden, g in ((16, 6), (1, 3), (13, 4), (128, 5)):
    p0 = orc.synth_planes(48, 40, g, seed=hidden)
    net = orc.synth_net(g, hidden, seed=hidden)
    oa = orc.act(p0, net)
    res = []
    for flag in (0, _lib.F_CUDA_CORE_NET):
        dev = make_dev(p0, net.capacity, net)
        dev.step_raw(physics.step_scalars(0, oracle_phys_to_params(orc.Phys(cycle_period=20))), 0, flags=_lib.F_EXPORT_ACTIONS | flag)
        cells, acts = dev.get_actions()
        d = np.abs(acts.astype(np.float64) - oa.a) 
        res.append((rel_err(acts, oa.a), d.max(), float(np.max(d / np.maximum(np.abs(oa.a), 1.0)))))
        dev.close()
    print(hidden, "tc rel %.2e abs %.2e | cuda rel %.2e abs %.2e" % (res[0][0], res[0][1], res[1][0], res[1][1]))
