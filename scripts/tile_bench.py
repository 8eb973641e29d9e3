"""Per-iteration time of the configs[4] tile through optimize_tiled on one
process (strips per rank automatic unless given).
    python scripts/tile_bench.py [prec] [side] [strips_per_rank] [axis]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2303_12529_b200 as b2  # noqa: E402
from paper_2303_12529_b200 import inputs, tiled  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
m = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] != "auto" else None
axis = int(sys.argv[4]) if len(sys.argv) > 4 else None
g = T // 2048
mosaic = inputs.mosaic_tile(range(g * g), grid=(g, g))
focus, defocus = b2.gen_synthetic_kernels(35, 24, seed=4)
tiled.optimize_tiled(mosaic, focus, defocus, b2.OptConfig(max_iters=1, stop_patience=10**9, precision=prec),
                     axis=axis, strips_per_rank=m)
t0 = time.perf_counter()
r = tiled.optimize_tiled(mosaic, focus, defocus, b2.OptConfig(max_iters=6, stop_patience=10**9, precision=prec),
                         axis=axis, strips_per_rank=m)
torch.cuda.synchronize()
print(f"{prec} {T}^2: {r.strips} strips of {r.window}: {1e3 * r.loop_time / r.iters_run:.2f} ms/iter "
      f"(loop {r.loop_time:.3f} s, {r.iters_run} iters, wall {time.perf_counter() - t0:.1f} s), "
      f"l_dso {r.loss_history[-1].l_dso:.6g}", flush=True)
