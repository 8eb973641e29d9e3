"""Golden kernel spectra from the REAL reference: `KernelSet.stacked_ffts`
(litho.py:71-82: Hf = FFT2(embed_kernel(h)), Hrot_f = FFT2(h(-u)), sigma).

Run in the build container only (the reference is not on the GPU box):

    cp -r /root/reference/pkg/src/lsopc /tmp/refpkg/
    python tests/golden/make_spectra.py /tmp/refpkg

Writes tests/golden/spectra.npz.
"""
import sys
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent


def main():
    sys.path.insert(0, sys.argv[1] if len(sys.argv) > 1 else "/tmp/refpkg")
    from lsopc import litho
    out = {}
    for side, n_k, seed, shape in [(9, 2, 3, (32, 64)), (17, 4, 1, (64, 64)), (7, 2, 0, (16, 128))]:
        f, d = litho.gen_synthetic_kernels(side, n_k, seed=seed)
        for tag, ks in (("f", f), ("d", d)):
            hf, hrot, sigma = ks.stacked_ffts(shape)
            key = f"{side}_{n_k}_{seed}_{tag}_{shape[0]}x{shape[1]}"
            out[key + "_hf"] = hf
            out[key + "_hrot"] = hrot
            out[key + "_sigma"] = sigma
    np.savez_compressed(OUT / "spectra.npz", **out)
    print("wrote", OUT / "spectra.npz", sorted(out)[:3], "...")


if __name__ == "__main__":
    main()
