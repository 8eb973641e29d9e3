"""Dump fp32-tier outputs (intensity at three corners, ILT gradient, a
6-iteration history and final mask of the 2048^2 clip) for a bit-for-bit
comparison between two library builds (dev check):
    LSOPC_B200_LIB=a python scripts/bitcheck.py out_a.npz; ... ; python scripts/bitcheck.py --cmp a.npz b.npz"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
if sys.argv[1] == "--cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    for k in a.files:
        same = np.array_equal(a[k], b[k])
        print(k, "identical" if same else f"DIFFERS max {np.abs(a[k] - b[k]).max():.3e}")
    sys.exit(0)
import paper_2303_12529_b200 as b2  # noqa: E402
from paper_2303_12529_b200 import _native as nv, inputs  # noqa: E402
nv.set_precision("fp32")
clip = inputs.iccad_like_clip(seed=0)
m = clip.astype(np.float64)
f, d = b2.gen_synthetic_kernels(35, 24, seed=4)
out = {c.label: b2.aerial_intensity(m, k, c) for k, c in ((f, b2.NOMINAL), (f, b2.OUTER), (d, b2.INNER))}
z = b2.print_corners(m, f, d, b2.OptConfig(), binarize=False).nominal
out["grad"] = b2.ilt_gradient(m, z, clip, f, b2.OptConfig())
r = b2.optimize(clip, f, d, b2.OptConfig(max_iters=6, stop_patience=10**9, precision="fp32"))
out["hist"] = np.array([[h.l_ilt, h.l_pvb, h.l_dso, h.dt, h.max_v] for h in r.loss_history])
out["mask"] = r.final_mask
np.savez(sys.argv[1], **out)
