"""Break down the end-to-end optimize() time on one GPU (dev probe)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2303_12529_b200 as b2
from paper_2303_12529_b200 import _native as nv, inputs
from paper_2303_12529_b200.metrics import shot_count

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
nv.set_precision(prec)
clip = inputs.iccad_like_clip(seed=0)
(fc, fw), (dc, dw) = inputs.synthetic_kernel_arrays(35, 24, 4)
focus = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(fc, fw)], "focus")
defocus = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(dc, dw)], "defocus")
t = time.perf_counter(); fk = focus.device(clip.shape); dk = defocus.device(clip.shape); torch.cuda.synchronize()
print(f"spectra build (both sets): {time.perf_counter()-t:.3f} s")
for rep in range(3):
    cfg = b2.OptConfig(max_iters=50, stop_patience=10**9, precision=prec)
    torch.cuda.synchronize(); t = time.perf_counter()
    r = b2.optimize(clip, focus, defocus, cfg)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"optimize 50 iters: {dt:.3f} s  ({50/dt:.1f} iters/s), wall_time {r.wall_time:.3f}")
t = time.perf_counter(); n = shot_count(r.final_mask); print(f"shot_count: {time.perf_counter()-t:.3f} s ({n} shots)")
td = nv.to_dev(clip, np.uint8)
for rep in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    lsf = b2.tsdf_from_mask(clip)
    print(f"tsdf_from_mask (host API): {time.perf_counter()-t:.4f} s")
