"""A few 8192^2 DSO iterations (ncu target for the config-5 column passes)."""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2303_12529_b200 as b2
from paper_2303_12529_b200 import _native as nv, inputs
nv.set_precision("fp32")
w = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
clip = np.ascontiguousarray(inputs.mosaic_tile(range(16), grid=(4, 4))[:, :w])
(fc, fw), (dc, dw) = inputs.synthetic_kernel_arrays(35, 24, 4)
focus = b2.KernelSet([b2.OpticalKernel(c, float(x)) for c, x in zip(fc, fw)], "focus")
defocus = b2.KernelSet([b2.OpticalKernel(c, float(x)) for c, x in zip(dc, dw)], "defocus")
b2.optimize(clip, focus, defocus, b2.OptConfig(max_iters=2, stop_patience=10**9, precision="fp32"))
