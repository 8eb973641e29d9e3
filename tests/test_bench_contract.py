"""bench.py's contract pieces that run without a GPU: the SURVEY §8(d)
algorithmic byte count behind `roofline.achieved`, the per-pass byte model,
the workload config both arms print, and the default flags the driver relies
on (N = 1, a K / W that finish in minutes, W >= 3)."""

import importlib.util
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _bench():
    spec = importlib.util.spec_from_file_location("bench_contract", ROOT / "bench.py")
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_algorithmic_bytes_match_survey():
    b = _bench()
    n = 2048 * 2048
    assert b.algorithmic_bytes_per_iter(n, 48, "fp32") == n * (64 * 24 + 170) == 7155482624
    assert b.algorithmic_bytes_per_iter(n, 48, "fp64") == n * (128 * 24 + 230)


def test_pass_byte_model_covers_every_pass():
    b = _bench()
    n = 2048 * 2048
    per = b.pass_bytes(n, 48, 2, "fp32")
    assert len(per) == len(b.PASS_NAMES) == 8
    # the four spectral passes move (2 N_k + small) complex fields each: T_k / U_k round trips
    for i in (1, 2, 4, 5):
        assert per[i] >= 96 * 8 * n
    # their sum is what ncu measures per iteration (profiles/traffic_fp32.json: 13.3 GB)
    assert 12.5e9 < sum(per) < 14.0e9


def test_default_flags_and_config(monkeypatch):
    b = _bench()
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    a = b.parse()
    assert (a.gpus, a.impl, a.precision) == (1, "b200", "fp32")
    assert a.warmup >= 3 and 1 <= a.steps <= 100
    cfg = b.workload_config(1)
    assert cfg["clip_side"] == 2048 and cfg["kernels_per_set"] == 24 and cfg["kernel_side"] == 35
    assert "l2_flush" in cfg and "model" not in cfg
