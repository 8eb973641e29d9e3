"""The opt-in tensor-core F1 (csrc/f1_tc.cu, LSOPC_B200_TCF1=1: the column
pass as a tcgen05 split-TF32 contraction over the kernel taps) against the
oracle at the fp32 tier's tolerances, in a subprocess (the switch is read
once per process).  It is measured and not adopted; this keeps
it correct."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
import paper_2303_12529_b200 as b2
from paper_2303_12529_b200 import _native as nv
from oracle import lsopc_oracle as o
nv.set_precision("fp32")
f, d = o.synthetic_kernels(35, 24, 4)
F = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(*f)], "focus")
D = b2.KernelSet([b2.OpticalKernel(c, float(w)) for c, w in zip(*d)], "defocus")
rng = np.random.default_rng(3)
t = np.zeros((512, 256), np.uint8)
for _ in range(12):
    h, w = rng.integers(20, 90, size=2)
    y, x = rng.integers(0, 512 - h), rng.integers(0, 256 - w)
    t[y:y + h, x:x + w] = 1
m = t.astype(np.float64)
hf = o.spectra(f[0], t.shape)
worst = 0.0
for cond, arrs in ((b2.NOMINAL, f), (b2.OUTER, f)):
    ref = o.intensity(m, arrs[0], arrs[1], cond.dose, hf)
    worst = max(worst, np.abs(b2.aerial_intensity(m, F, cond) - ref).max() / np.abs(ref).max())
z = o.corners(m, f, d, binarize=False, hf_focus=hf, hf_defocus=o.spectra(d[0], t.shape))["nominal"]
g = b2.ilt_gradient(m, z, t, F, b2.OptConfig())
gr = o.ilt_grad(m, z, t, f, hf=hf)
print("RESULT", worst, np.abs(g - gr).max() / np.abs(gr).max())
"""


def test_tensor_core_f1_vs_oracle():
    env = {**os.environ, "LSOPC_B200_TCF1": "1"}
    p = subprocess.run([sys.executable, "-c", SCRIPT.format(root=str(ROOT))], env=env, capture_output=True,
                       text=True, timeout=600, cwd=str(ROOT))
    assert p.returncode == 0, p.stderr[-3000:]
    line = [x for x in p.stdout.splitlines() if x.startswith("RESULT")][-1]
    ierr, gerr = (float(v) for v in line.split()[1:])
    assert ierr <= 1e-5, ierr
    assert gerr <= 2e-5, gerr
