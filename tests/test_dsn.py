"""DevelSet-Net front end (configs[3]): network shapes (CPU), fused clip + AHF
init kernel and the end-to-end instant-OPC path (GPU)."""

import numpy as np
import pytest
import torch

from paper_2303_12529_b200 import dsn


def test_net_branches_shapes_cpu():
    net = dsn.build_net(base=4, depth=3, device="cpu")
    x = torch.randn(2, 1, 64, 64)
    with torch.no_grad():
        a, b = net(x)
    assert a.shape == (2, 1, 64, 64) and b.shape == (2, 1, 64, 64)
    net2 = dsn.build_net(base=4, depth=3, device="cpu")
    with torch.no_grad():
        a2, _ = net2(x)
    assert torch.equal(a, a2)  # seeded random init is reproducible


@pytest.mark.gpu
def test_dsn_init_matches_reference_clip_and_ahf():
    import paper_2303_12529_b200 as b2
    rng = np.random.default_rng(3)
    raw = (rng.standard_normal((64, 64)) * 300).astype(np.float32)
    mraw = (rng.standard_normal((64, 64)) * 0.1).astype(np.float32)
    cfg = b2.OptConfig()
    phi0, m = dsn.dsn_init(torch.from_numpy(raw).cuda(), torch.from_numpy(mraw).cuda(), cfg)
    assert np.array_equal(phi0.cpu().numpy(), np.clip(raw.astype(np.float64), cfg.d_lower, cfg.d_upper))
    # the same kernel arithmetic as levelset.ahf (levelset.py:147-151), bit for bit
    assert np.array_equal(m.cpu().numpy(), b2.ahf(mraw.astype(np.float64), cfg.epsilon))
    assert m.min() > 0 and m.max() < 1


@pytest.mark.gpu
def test_instant_opc_small_batch():
    import paper_2303_12529_b200 as b2
    from oracle import lsopc_oracle as o
    (fc, fw), (dc, dw) = o.synthetic_kernels(17, 4, 1)
    F = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(fc, fw)], "focus")
    D = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(dc, dw)], "defocus")
    targets = [o.rect_layout(256, [(40 + 10 * i, 60, 80, 40), (150, 120, 50, 90)]) for i in range(3)]
    net = dsn.build_net(base=8, depth=3)
    r = dsn.instant_opc(targets, F, D, b2.OptConfig(max_iters=8), net=net)
    assert len(r.results) == 3 and r.latency > 0
    # the refinement on two lanes (the default) equals one lane bit for bit
    import torch
    cfg = b2.OptConfig(max_iters=8)
    x = dsn.tsdf_batch(targets, cfg.d_upper, cfg.d_lower)
    phi0 = x.float().contiguous()
    m = torch.full_like(phi0, 0.5)
    r2 = dsn.refine_batch(targets, phi0, m, F, D, cfg, lanes=2)
    r1 = dsn.refine_batch(targets, phi0, m, F, D, cfg, lanes=1)
    for a, b in zip(r2, r1):
        assert np.array_equal(a.final_mask, b.final_mask) and np.array_equal(a.final_phi.phi, b.final_phi.phi)
        assert [h.l_dso for h in a.loss_history] == [h.l_dso for h in b.loss_history]
    for res, t in zip(r.results, targets):
        assert res.final_mask.shape == t.shape and set(np.unique(res.final_mask)) <= {0, 1}
        assert 1 <= res.iters_run <= 8
        assert all(np.isfinite([h.l_dso for h in res.loss_history]))
