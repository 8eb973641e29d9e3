"""cProfile of optimize() on the GPU box (dev probe)."""
import cProfile, pstats, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2303_12529_b200 as b2
from paper_2303_12529_b200 import _native as nv, inputs
nv.set_precision("fp32")
clip = inputs.iccad_like_clip(seed=0)
(fc, fw), (dc, dw) = inputs.synthetic_kernel_arrays(35, 24, 4)
focus = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(fc, fw)], "focus")
defocus = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(dc, dw)], "defocus")
cfg = b2.OptConfig(max_iters=50, stop_patience=10**9, precision="fp32")
b2.optimize(clip, focus, defocus, cfg); torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(3):
    b2.optimize(clip, focus, defocus, cfg)
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
