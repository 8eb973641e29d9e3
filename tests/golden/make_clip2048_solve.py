"""Golden full solve at configs[1] size, made by the REAL reference (slow: the
reference spends ~80 s per 2048^2 iteration on one CPU core; ~35 min here).

    cp -r /root/reference/pkg/src/lsopc /tmp/refpkg/
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_clip2048_solve.py /tmp/refpkg

Writes tests/golden/clip2048_solve.npz: the loss history, iteration count,
metrics and the bit-packed final mask of optimize(iccad_like_clip(0),
gen_synthetic_kernels(35, 24, seed=4), OptConfig()).
"""

import sys
import time
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent


def main():
    sys.path.insert(0, sys.argv[1] if len(sys.argv) > 1 else "/tmp/refpkg")
    sys.path.insert(0, str(OUT.parents[1]))
    from lsopc import litho, optimizer
    from oracle import lsopc_oracle as o  # the App. B generator (pinned by test_oracle_golden)
    clip = o.iccad_like_clip(0)
    f, d = litho.gen_synthetic_kernels(35, 24, seed=4)
    t0 = time.time()
    r = optimizer.optimize(clip, f, d, optimizer.OptConfig())
    hist = np.array([[h.l_ilt, h.l_pvb, h.l_dso, h.dt, h.max_v, h.max_step, h.max_grad_mag] for h in r.loss_history])
    np.savez_compressed(OUT / "clip2048_solve.npz", hist=hist, iters=np.array(r.iters_run),
                        metrics=np.array([r.metrics.l2, r.metrics.pvband, r.metrics.shots]),
                        mask_packed=np.packbits(r.final_mask), seconds=np.array(time.time() - t0))
    print("iters", r.iters_run, "metrics", r.metrics.l2, r.metrics.pvband, r.metrics.shots, "s", time.time() - t0)


if __name__ == "__main__":
    main()
