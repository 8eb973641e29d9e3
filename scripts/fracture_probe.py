"""Time the device shot count of the configs[1] solve's final mask (2048^2,
240 shots) and compare with the host implementation."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2303_12529_b200 import metrics  # noqa: E402

g = np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / "clip2048_solve.npz")
mask = np.unpackbits(g["mask_packed"])[:2048 * 2048].reshape(2048, 2048)
ys, xs = np.nonzero(mask)
print("box", ys.min(), ys.max(), xs.min(), xs.max())
md = torch.as_tensor(mask, device="cuda")
for name, fn in (("device", lambda: metrics.shot_count(md)), ("host", lambda: metrics.shot_count(mask))):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 5
    for _ in range(n):
        c = fn()
    print(name, c, f"{(time.perf_counter() - t0) / n * 1e3:.3f} ms")
