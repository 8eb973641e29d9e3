"""DevelSet-Net front end (BASELINE configs[3]).

The paper's DSN is a two-branch UNet: the level-set branch
predicts the initial level set phi0 for DSO, the modulation branch predicts
phi_m whose approximated Heaviside H_eps(phi_m) is the
curvature modulation m of the DSO evolution.  The reference package excludes
the network (`SPEC.md:8`); its boundary is `optimize(..., phi0=, modulation=)`
(`optimizer.py:204-228`).  This module supplies a random-initialised network
of that shape (no trained weights exist offline) so the end-to-end
"instant OPC" latency of configs[3] can be measured:

    targets --TSDF (device)--> DSN (bf16, cuDNN) --clip + AHF (one fused
    device pass, lsopc_dsn_init)--> phi0, m (float64, device) --> DSO loop

The network is PyTorch library code (convolutions through cuDNN); it is the
front end of the hot path, not part of it.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _native as nv


def _torch():
    return nv.torch()


def build_net(base=16, depth=4, seed=0, device="cuda"):
    """Random-initialised two-branch UNet: input 1 channel (the target's
    TSDF / 100), outputs 2 channels (phi0 in TSDF units, phi_m)."""
    import torch
    import torch.nn as nn

    torch.manual_seed(seed)

    def block(cin, cout):
        return nn.Sequential(nn.Conv2d(cin, cout, 3, padding=1), nn.BatchNorm2d(cout), nn.ReLU(inplace=True),
                             nn.Conv2d(cout, cout, 3, padding=1), nn.BatchNorm2d(cout), nn.ReLU(inplace=True))

    class DevelSetNet(nn.Module):
        def __init__(self):
            super().__init__()
            ch = [base * (2 ** i) for i in range(depth)]
            self.down = nn.ModuleList([block(1 if i == 0 else ch[i - 1], ch[i]) for i in range(depth)])
            self.pool = nn.MaxPool2d(2)
            self.up = nn.ModuleList([nn.ConvTranspose2d(ch[i], ch[i - 1], 2, stride=2) for i in range(depth - 1, 0, -1)])
            self.dec = nn.ModuleList([block(2 * ch[i - 1], ch[i - 1]) for i in range(depth - 1, 0, -1)])
            self.head_phi = nn.Conv2d(ch[0], 1, 1)   # level-set branch
            self.head_m = nn.Conv2d(ch[0], 1, 1)     # modulation branch

        def forward(self, x):
            skips = []
            for i, d in enumerate(self.down):
                x = d(x)
                if i < len(self.down) - 1:
                    skips.append(x)
                    x = self.pool(x)
            for up, dec in zip(self.up, self.dec):
                x = up(x)
                x = dec(torch.cat([x, skips.pop()], dim=1))
            return self.head_phi(x), self.head_m(x)

    return DevelSetNet().to(device).eval()


def tsdf_batch(targets, d_upper=900.0, d_lower=-100.0):
    """Device TSDFs (float64) of a list of uint8 targets (levelset.py:86-101)."""
    torch = _torch()
    out = []
    for t in targets:
        td = nv.to_dev(np.ascontiguousarray((np.asarray(t) != 0).astype(np.uint8)), np.uint8)
        phi = nv.empty(t.shape, np.float64)
        nv.check(nv.lib().lsopc_tsdf(t.shape[0], t.shape[1], nv.ptr(td), float(d_upper), float(d_lower),
                                     nv.ptr(phi), nv.stream()))
        out.append(phi)
    return torch.stack(out)


def dsn_init(phi_raw, m_raw, cfg):
    """Fused clip + AHF of the network outputs (float32, any shape) into the
    DSO initial state (float64 device tensors)."""
    torch = _torch()
    phi_raw = phi_raw.float().contiguous()
    m_raw = m_raw.float().contiguous()
    phi0 = torch.empty(phi_raw.shape, dtype=torch.float64, device="cuda")
    m = torch.empty(m_raw.shape, dtype=torch.float64, device="cuda")
    nv.check(nv.lib().lsopc_dsn_init(phi_raw.numel(), nv.ptr(phi_raw), nv.ptr(m_raw), float(cfg.d_lower),
                                     float(cfg.d_upper), float(cfg.epsilon), nv.ptr(phi0), nv.ptr(m), nv.stream()))
    return phi0, m


@dataclass
class InstantOPCResult:
    results: list          # OptimizationResult per target
    t_tsdf: float
    t_net: float
    t_init: float
    t_dso: float

    @property
    def latency(self):
        return self.t_tsdf + self.t_net + self.t_init + self.t_dso


def refine_batch(targets, phi0, m, focus_kernels, defocus_kernels, cfg, lanes=2):
    """The device level-set refinement of each target from its device phi0 /
    modulation, on `lanes` worker threads with their own CUDA streams and work
    buffers (like parallel.optimize_batch): one clip's host-side gaps overlap
    another's device loop.  Results do not depend on `lanes`."""
    from .optimizer import _assemble, _optimize_device
    torch = _torch()
    results = [None] * len(targets)

    def run_lane(idx):
        # each clip is assembled (waiting for its host shot count) after the
        # lane's next clip has run, so the count never stalls the lane
        pending = None
        for i in idx:
            parts = _optimize_device(targets[i], focus_kernels, defocus_kernels, cfg, phi0=phi0[i], modulation=m[i],
                                     shots_on="host")
            if pending is not None:
                results[pending[0]] = _assemble(pending[1], cfg)
            pending = (i, parts)
        if pending is not None:
            results[pending[0]] = _assemble(pending[1], cfg)

    lanes = max(1, min(int(lanes), len(targets)))
    if lanes == 1:
        run_lane(range(len(targets)))
        return results
    from concurrent.futures import ThreadPoolExecutor
    from . import _native as nv
    dev = torch.cuda.current_device()
    producer = torch.cuda.current_stream()

    def worker(lane):
        nv.set_lane(lane)
        torch.cuda.set_device(dev)
        stream = torch.cuda.Stream()
        stream.wait_stream(producer)  # phi0 / m were written on the caller's stream
        with torch.cuda.stream(stream):
            run_lane(range(lane, len(targets), lanes))
        stream.synchronize()

    with ThreadPoolExecutor(max_workers=lanes) as pool:
        for f in [pool.submit(worker, lane) for lane in range(lanes)]:
            f.result()
    return results


def instant_opc(targets, focus_kernels, defocus_kernels, cfg, net=None, lanes=2):
    """configs[3]: DSN prediction for a batch of targets followed by the GPU
    level-set refinement of each target.  Stage times are device-synchronised.
    The refinements run on `lanes` worker threads with their own CUDA streams
    and work buffers (like parallel.optimize_batch), so one clip's host-side
    gaps overlap another's device loop; results do not depend on `lanes`."""
    torch = _torch()
    net = net or build_net()

    def sync():
        torch.cuda.synchronize()

    sync()
    t0 = time.perf_counter()
    x = tsdf_batch(targets, cfg.d_upper, cfg.d_lower)
    sync()
    t1 = time.perf_counter()
    with torch.no_grad(), torch.autocast("cuda", dtype=torch.bfloat16):
        phi_raw, m_raw = net((x / 100.0).float().unsqueeze(1))
    sync()
    t2 = time.perf_counter()
    # the level-set branch predicts in TSDF units around the target's TSDF
    phi0, m = dsn_init(x.float() + 100.0 * phi_raw.float().squeeze(1), m_raw.float().squeeze(1), cfg)
    sync()
    t3 = time.perf_counter()
    results = refine_batch(targets, phi0, m, focus_kernels, defocus_kernels, cfg, lanes)
    sync()
    t4 = time.perf_counter()
    return InstantOPCResult(results, t1 - t0, t2 - t1, t3 - t2, t4 - t3)
