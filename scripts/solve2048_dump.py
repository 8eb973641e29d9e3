"""Full default solve of iccad_like_clip(0) (configs[1]) in both tiers; dumps
history / metrics / packed mask to gpurun_out/ for comparison with the
reference's golden solve (dev probe)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2303_12529_b200 as b2
from paper_2303_12529_b200 import _native as nv
from oracle import lsopc_oracle as o
(fc, fw), (dc, dw) = o.synthetic_kernels(35, 24, 4)
F = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(fc, fw)], "focus")
D = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(dc, dw)], "defocus")
clip = o.iccad_like_clip(0)
for prec in ("fp64", "fp32"):
    r = b2.optimize(clip, F, D, b2.OptConfig(precision=prec))
    hist = np.array([[h.l_ilt, h.l_pvb, h.l_dso, h.dt, h.max_v, h.max_step, h.max_grad_mag] for h in r.loss_history])
    np.savez_compressed(f"gpurun_out/solve2048_{prec}.npz", hist=hist, iters=r.iters_run,
                        metrics=np.array([r.metrics.l2, r.metrics.pvband, r.metrics.shots]),
                        mask_packed=np.packbits(r.final_mask))
    print(prec, r.iters_run, r.metrics.l2, r.metrics.pvband, r.metrics.shots, f"{r.wall_time:.3f}s")
