"""optimize() time vs iteration count (dev probe): slope = per-iteration,
intercept = fixed cost of a call (upload, TSDF, session, finish, shots, D2H)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2303_12529_b200 as b2  # noqa: E402
from paper_2303_12529_b200 import _native as nv, inputs  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
nv.set_precision(prec)
clip = inputs.iccad_like_clip(seed=0)
focus, defocus = b2.gen_synthetic_kernels(35, 24, seed=4)
for K in (1, 2, 4, 8, 20, 40):
    cfg = b2.OptConfig(max_iters=K, stop_patience=10**9, precision=prec)
    b2.optimize(clip, focus, defocus, cfg)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        b2.optimize(clip, focus, defocus, cfg)
        ts.append(time.perf_counter() - t0)
    print(f"{prec} K={K}: optimize median {1e3 * np.median(ts):.2f} ms", flush=True)
