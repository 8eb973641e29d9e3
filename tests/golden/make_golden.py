"""Generate golden vectors by running the REAL reference package.

Run in the build container only (the reference is not on the GPU box):

    cp -r /root/reference/pkg/src/lsopc /tmp/refpkg/
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py /tmp/refpkg [--big]

Outputs `tests/golden/*.npz`.  Each fixture records the reference function it
came from.  `--big` adds the 2048^2 / N_k=24 full-size samples (~3 min);
`--only modsearch` regenerates just `modsearch.npz`.
"""

import hashlib
import sys
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent


def main():
    ref_path = sys.argv[1] if len(sys.argv) > 1 else "/tmp/refpkg"
    big = "--big" in sys.argv
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
    sys.path.insert(0, ref_path)
    import lsopc
    from lsopc import levelset, litho, optimizer

    # ---- modulation_search (optimizer.py:294-341) -------------------------------
    ms = {}
    f, d = litho.gen_synthetic_kernels(9, 2, seed=2)
    t = np.zeros((64, 64), dtype=np.uint8)
    t[16:40, 20:44] = 1
    phi_gt = levelset.tsdf_from_mask(t)
    for tag, cfg in (("default", optimizer.OptConfig()), ("nocurvw", optimizer.OptConfig(curvature_weight=0.0))):
        r = optimizer.modulation_search(phi_gt, t, f, d, cfg, num_samples=5, eval_steps=3)
        ms[f"{tag}_candidates"] = np.array([[dh, l] for dh, l in r.candidates])
        ms[f"{tag}_best"] = np.array(r.best_delta_h)
    ms["target"] = t
    np.savez_compressed(OUT / "modsearch.npz", **ms)
    if only == "modsearch":
        return

    def kset_arrays(ks):
        return (np.stack([k.coeffs for k in ks.kernels]),
                np.array([k.weight for k in ks.kernels]))

    # ---- kernels (litho.gen_synthetic_kernels) -------------------------------
    kern = {}
    for side, n_k, seed in [(9, 2, 0), (9, 2, 3), (9, 2, 1), (17, 4, 1), (35, 8, 4), (7, 2, 0)]:
        f, d = litho.gen_synthetic_kernels(side, n_k, seed=seed)
        for tag, ks in (("f", f), ("d", d)):
            c, w = kset_arrays(ks)
            kern[f"{side}_{n_k}_{seed}_{tag}_c"] = c
            kern[f"{side}_{n_k}_{seed}_{tag}_w"] = w
    f, d = litho.gen_synthetic_kernels(35, 24, seed=4)
    for tag, ks in (("f", f), ("d", d)):
        c, w = kset_arrays(ks)
        kern[f"35_24_4_{tag}_sha"] = np.frombuffer(
            hashlib.sha256(c.tobytes()).digest(), dtype=np.uint8)
        kern[f"35_24_4_{tag}_w"] = w
        kern[f"35_24_4_{tag}_c0"] = c[:, 17, :]      # centre row of every kernel
    np.savez_compressed(OUT / "kernels.npz", **kern)

    # ---- forward model -------------------------------------------------------
    rng = np.random.default_rng(99)
    fwd = {}
    f, d = litho.gen_synthetic_kernels(9, 2, seed=3)
    m = rng.random((64, 64))
    fwd["rand64_mask"] = m
    fwd["rand64_I_nom"] = litho.aerial_intensity(m, f, litho.NOMINAL)
    fwd["rand64_I_out"] = litho.aerial_intensity(m, f, litho.OUTER)
    fwd["rand64_I_in"] = litho.aerial_intensity(m, d, litho.INNER)
    mb = (rng.random((32, 32)) < 0.5).astype(np.float64)
    fwd["bin32_mask"] = mb
    p = litho.print_corners(mb, f, d, optimizer.OptConfig(), binarize=False)
    fwd["bin32_Z_nom"], fwd["bin32_Z_in"], fwd["bin32_Z_out"] = p.nominal, p.inner, p.outer
    p = litho.print_corners(mb, f, d, optimizer.OptConfig(), binarize=True)
    fwd["bin32_H_nom"], fwd["bin32_H_in"], fwd["bin32_H_out"] = p.nominal, p.inner, p.outer
    np.savez_compressed(OUT / "forward.npz", **fwd)

    # ---- gradients (optimizer.ilt_gradient / pvb_gradient) --------------------
    grad = {}
    cfg = optimizer.OptConfig()
    for seed in (0, 3):
        target = np.zeros((64, 64), dtype=np.uint8)
        target[16:48, 21:42] = 1
        f, d = litho.gen_synthetic_kernels(9, 2, seed=seed)
        mask = target.astype(np.float64)
        pr = litho.print_corners(mask, f, d, cfg, binarize=False)
        grad[f"s{seed}_target"] = target
        grad[f"s{seed}_g_ilt"] = optimizer.ilt_gradient(mask, pr.nominal, target, f, cfg)
        grad[f"s{seed}_g_pvb"] = optimizer.pvb_gradient(mask, pr.inner, pr.outer, target, f, d, cfg)
        grad[f"s{seed}_l_ilt"] = optimizer.ilt_loss(pr.nominal, target)
        grad[f"s{seed}_l_pvb"] = optimizer.pvb_loss(pr.inner, pr.outer, target)
    np.savez_compressed(OUT / "gradients.npz", **grad)

    # ---- level set -----------------------------------------------------------
    ls = {}
    rng = np.random.default_rng(12345)
    phi = rng.standard_normal((32, 48)) * 5.0
    g = levelset.geometry_gradient(phi)
    ls["phi"] = phi
    for name in ("gx", "gy", "gxx", "gyy", "gxy"):
        ls[name] = getattr(g, name)
    ls["mag"] = g.magnitude
    mod = rng.random((32, 48))
    ls["mod"] = mod
    ls["kappa"] = levelset.curvature(phi, mod, 0.9)
    for i in range(4):
        mk = (rng.random((64, 64)) < rng.uniform(0.1, 0.9)).astype(np.uint8)
        ls[f"tsdf_mask{i}"] = mk
        ls[f"tsdf_phi{i}"] = levelset.tsdf_from_mask(mk).phi
    t = np.zeros((128, 128), dtype=np.uint8)
    t[30:80, 25:55] = 1
    t[60:100, 70:110] = 1
    ls["tsdf_two_rect"] = levelset.tsdf_from_mask(t, 20.0, -7.0).phi
    np.savez_compressed(OUT / "levelset.npz", **ls)

    # ---- optimize trajectories ----------------------------------------------
    opt = {}
    f, d = litho.gen_synthetic_kernels(17, 4, seed=1)
    for tag, kw in (("on", {}), ("off", {"use_curvature": False})):
        r = optimizer.optimize(t, f, d, optimizer.OptConfig(max_iters=15, **kw))
        opt[f"rect128_{tag}_hist"] = np.array([[h.l_ilt, h.l_pvb, h.l_dso, h.dt, h.max_v,
                                                h.max_step, h.max_grad_mag]
                                               for h in r.loss_history])
        opt[f"rect128_{tag}_phi"] = r.final_phi.phi
        opt[f"rect128_{tag}_mask"] = r.final_mask
        opt[f"rect128_{tag}_metrics"] = np.array([r.metrics.l2, r.metrics.pvband,
                                                  r.metrics.shots, r.iters_run])
    # AC-5 case: 512^2 two bars, K=35, N_k=8, seed 4, max_iters=50
    from lsopc import fileio
    tgt = fileio.parse_layout("SIZE 512\nRECT 150 120 70 270\nRECT 290 120 70 270\n")
    f, d = litho.gen_synthetic_kernels(35, 8, seed=4)
    for tag, kw in (("on", {}), ("off", {"use_curvature": False})):
        r = optimizer.optimize(tgt, f, d, optimizer.OptConfig(max_iters=50, **kw))
        opt[f"bar512_{tag}_hist"] = np.array([[h.l_ilt, h.l_pvb, h.l_dso, h.dt, h.max_v,
                                               h.max_step, h.max_grad_mag]
                                              for h in r.loss_history])
        opt[f"bar512_{tag}_mask_packed"] = np.packbits(r.final_mask)
        opt[f"bar512_{tag}_metrics"] = np.array([r.metrics.l2, r.metrics.pvband,
                                                 r.metrics.shots, r.iters_run])
    np.savez_compressed(OUT / "optimize.npz", **opt)

    # ---- fracture (metrics.fracture): rectangle lists on random masks ---------
    from lsopc import metrics
    fr = {}
    rng = np.random.default_rng(77)
    for i in range(12):
        h, w = int(rng.integers(3, 48)), int(rng.integers(3, 48))
        m = (rng.random((h, w)) < rng.uniform(0.2, 0.95)).astype(np.uint8)
        fr[f"mask{i}"] = m
        fr[f"rects{i}"] = np.array(metrics.fracture(m), dtype=np.int64).reshape(-1, 4)
    np.savez_compressed(OUT / "fracture.npz", **fr)

    if big:
        # full-size samples: 2048^2 iccad-like clip 0, N_k = 24, iteration 0
        sys.path.insert(0, str(OUT.parents[1]))
        from oracle.lsopc_oracle import iccad_like_clip
        clip = iccad_like_clip(0)
        f, d = litho.gen_synthetic_kernels(35, 24, seed=4)
        cfg = optimizer.OptConfig()
        mask = clip.astype(np.float64)
        pr = litho.print_corners(mask, f, d, cfg, binarize=False)
        hard = litho.print_corners(mask, f, d, cfg, binarize=True)
        g_ilt = optimizer.ilt_gradient(mask, pr.nominal, clip, f, cfg)
        g_pvb = optimizer.pvb_gradient(mask, pr.inner, pr.outer, clip, f, d, cfg)
        v = optimizer.velocity(g_ilt, g_pvb, cfg)
        rs = np.random.default_rng(5)
        ys = rs.integers(0, 2048, 4096)
        xs = rs.integers(0, 2048, 4096)
        big_out = {
            "ys": ys, "xs": xs,
            "z_nom": pr.nominal[ys, xs], "z_in": pr.inner[ys, xs], "z_out": pr.outer[ys, xs],
            "v": v[ys, xs],
            "v_absmax": np.abs(v).max(), "v_sum": v.sum(),
            "l_ilt": optimizer.ilt_loss(pr.nominal, clip),
            "l_pvb": optimizer.pvb_loss(pr.inner, pr.outer, clip),
            "hard_l2": lsopc.l2_error(hard.nominal, clip),
            "hard_pvb": lsopc.pvband(hard.inner, hard.outer),
        }
        np.savez_compressed(OUT / "clip2048.npz", **big_out)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
