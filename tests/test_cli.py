"""The CLI and file formats (reference cli.py,
fileio.py, tests test_io_cli.py / test_acceptance.py:250-271):

* CPU: byte-exact formats and their error messages, config precedence and
  exit codes, host subcommands (gen-kernels, fracture).
* GPU: `optimize` over several targets in one process equals the library
  bit for bit per target, and the SOCS spectra (K0) are built once per
  shape -- the second target of a shape does not rebuild them.
"""

import json
import struct

import numpy as np
import pytest

from paper_2303_12529_b200 import cli, fileio
from paper_2303_12529_b200.errors import FormatError


# ---------------------------------------------------------------------------
# file formats (CPU)


def test_field_dump_bytes_and_round_trip(tmp_path, rng):
    p = tmp_path / "f.f64"
    fileio.dump_field(p, np.array([[1.0, 2.0], [3.0, 4.0]]))
    assert p.read_bytes() == b"DVLF1\x00" + struct.pack("<II", 2, 2) + struct.pack("<4d", 1.0, 2.0, 3.0, 4.0)
    f = rng.standard_normal((33, 17))
    fileio.dump_field(p, f)
    out = fileio.load_field(p)
    assert out.dtype == np.float64 and np.array_equal(out, f)


def test_field_errors(tmp_path):
    p = tmp_path / "f.f64"
    p.write_bytes(b"NOPE!\x00" + b"\x00" * 40)
    with pytest.raises(FormatError, match="DVLF1"):
        fileio.load_field(p)
    fileio.dump_field(p, np.zeros((4, 4)))
    data = p.read_bytes()
    p.write_bytes(data[:-8])
    with pytest.raises(FormatError, match=str(len(data))):
        fileio.load_field(p)


def test_pgm_round_trip_threshold_comments(tmp_path, rng):
    p = tmp_path / "m.pgm"
    m = (rng.random((32, 48)) < 0.5).astype(np.uint8)
    fileio.save_pgm(p, m)
    assert np.array_equal(fileio.load_pgm(p), m)
    p.write_bytes(b"P5\n3 1\n255\n" + bytes([0, 127, 128]))
    assert np.array_equal(fileio.load_pgm(p), [[0, 0, 1]])
    p.write_bytes(b"P5\n# a comment\n2 1\n255\n" + bytes([255, 0]))
    assert np.array_equal(fileio.load_pgm(p), [[1, 0]])
    p.write_bytes(b"P6\n1 1\n255\n\x00\x00\x00")
    with pytest.raises(FormatError):
        fileio.load_pgm(p)
    p.write_bytes(b"P5\n4 4\n255\n" + bytes(3))
    with pytest.raises(FormatError, match="truncated"):
        fileio.load_pgm(p)


def test_layout_parsing():
    g = fileio.parse_layout("SIZE 64\nRECT 10 10 20 8\n")
    assert g.shape == (64, 64) and g[10:18, 10:30].all() and g.sum() == 160
    assert fileio.parse_layout("SIZE 32\nRECT 0 0 10 10\nRECT 5 5 10 10\n").sum() == 175
    g = fileio.parse_layout("# header\nSIZE 16\n\nRECT 1 2 3 4  # inline\n")
    assert g[2:6, 1:4].all() and g.sum() == 12
    with pytest.raises(FormatError, match="line 2"):
        fileio.parse_layout("SIZE 16\nRECT 1 2 three 4\n")
    with pytest.raises(FormatError, match="line 1"):
        fileio.parse_layout("CIRCLE 1 2 3\n")
    with pytest.raises(ValueError, match="line 2"):
        fileio.parse_layout("SIZE 16\nRECT 10 10 10 10\n")
    with pytest.raises(ValueError):
        fileio.parse_layout("SIZE 16\nRECT 1 1 0 5\n")


def test_loss_csv(tmp_path):
    from paper_2303_12529_b200.optimizer import IterationRecord
    p = tmp_path / "loss.csv"
    fileio.write_loss_csv(p, [IterationRecord(1.5, 2.5, 20.25, 0.1, 8.5, 0.2, 1.0)])
    lines = p.read_text().splitlines()
    assert lines == ["iter,L_ilt,L_pvb,L_DSO,dt,max_v", "0,1.5,2.5,20.25,0.1,8.5"]


# ---------------------------------------------------------------------------
# CLI on the host (CPU)


def test_config_file_parsing_and_precedence(tmp_path):
    cfgf = tmp_path / "run.cfg"
    cfgf.write_text("max_iters = 0   # comment\nlambda = 0.5\nuse_curvature = no\n")
    args = cli.build_parser().parse_args(["optimize", "--target", "t", "--kernels", "k", "--out-dir", "o",
                                          "--config", str(cfgf), "--max-iters", "3"])
    cfg = cli.config_from_args(args)
    assert (cfg.max_iters, cfg.curvature_weight, cfg.use_curvature) == (3, 0.5, False)
    bad = tmp_path / "bad.cfg"
    bad.write_text("warp_speed = 9\n")
    with pytest.raises(FormatError, match="bad.cfg:1"):
        cli.read_config_file(bad)


def test_exit_codes_and_host_subcommands(tmp_path, capsys):
    assert cli.main([]) == 1
    assert cli.main(["fracture", "--bogus", "x"]) == 1
    assert cli.main(["fracture", "--mask", str(tmp_path / "nope.pgm")]) == 1
    a, b = tmp_path / "a.dvlk", tmp_path / "b.dvlk"
    assert cli.main(["gen-kernels", "--side", "35", "--count", "24", "--seed", "7", "--out", str(a)]) == 0
    assert cli.main(["gen-kernels", "--side", "35", "--count", "24", "--seed", "7", "--out", str(b)]) == 0
    assert a.read_bytes() == b.read_bytes()
    m = fileio.parse_layout("SIZE 64\nRECT 5 5 20 30\nRECT 30 10 10 10\n")
    mp = tmp_path / "m.pgm"
    fileio.save_pgm(mp, m)
    out = tmp_path / "shots.csv"
    assert cli.main(["fracture", "--mask", str(mp), "--out", str(out)]) == 0
    from paper_2303_12529_b200.metrics import fracture
    lines = out.read_text().splitlines()
    assert lines[0] == "x,y,w,h"
    assert [tuple(int(v) for v in ln.split(",")) for ln in lines[1:]] == fracture(m)


# ---------------------------------------------------------------------------
# GPU: batch optimize == library, spectra built once per shape


@pytest.fixture
def workspace(tmp_path):
    from paper_2303_12529_b200 import gen_synthetic_kernels, save_kernels
    lay = []
    for i, text in enumerate(("SIZE 128\nRECT 25 30 30 50\nRECT 70 60 40 40\n",
                              "SIZE 128\nRECT 20 20 70 24\nRECT 40 60 24 50\n",
                              "SIZE 256\nRECT 60 70 90 40\nRECT 120 130 40 80\n")):
        p = tmp_path / f"t{i}.lay"
        p.write_text(text)
        lay.append(p)
    k = tmp_path / "syn.dvlk"
    f, d = gen_synthetic_kernels(17, 4, seed=1)
    save_kernels(k, f, d)
    return tmp_path, lay, k


@pytest.mark.gpu
def test_batch_optimize_equals_library_and_builds_spectra_once(workspace):
    from paper_2303_12529_b200 import _native as nv
    from paper_2303_12529_b200 import load_kernels, optimize, OptConfig
    nv.set_precision("fp64")
    tmp, lay, k = workspace
    out = tmp / "batch"
    before = nv.DeviceKernelSet.builds
    assert cli.main(["optimize", "--target", str(lay[0]), str(lay[1]), "--kernels", str(k), "--size", "128",
                     "--out-dir", str(out), "--max-iters", "6"]) == 0
    # two targets of one shape: focus + defocus spectra built once
    assert nv.DeviceKernelSet.builds - before == 2
    focus, defocus = load_kernels(k)
    summary = json.loads((out / "batch.json").read_text())
    assert [s["target"] for s in summary] == [str(lay[0]), str(lay[1])]
    for p in lay[:2]:
        run = out / p.stem
        target = fileio.parse_layout(p.read_text(), 128)
        r = optimize(target, focus, defocus, OptConfig(max_iters=6))
        m = json.loads((run / "metrics.json").read_text())
        assert (m["l2"], m["pvband"], m["shots"], m["iters"]) == (r.metrics.l2, r.metrics.pvband, r.metrics.shots,
                                                                   r.iters_run)
        assert np.array_equal(fileio.load_pgm(run / "mask.pgm"), r.final_mask)
        assert np.array_equal(fileio.load_field(run / "phi.f64"), r.final_phi.phi)
        rows = (run / "loss.csv").read_text().splitlines()[1:]
        assert [float(x.split(",")[3]) for x in rows] == [h.l_dso for h in r.loss_history]
    # a third target of another shape builds that shape's spectra only
    before = nv.DeviceKernelSet.builds
    assert cli.main(["optimize", "--target", str(lay[0]), str(lay[2]), "--kernels", str(k), "--size", "128",
                     "--out-dir", str(tmp / "b2"), "--max-iters", "2"]) == 0
    assert nv.DeviceKernelSet.builds - before == 4


@pytest.mark.gpu
def test_cli_single_target_subcommands_match_library(workspace, capsys):
    from paper_2303_12529_b200 import (OptConfig, l2_error, load_kernels, print_corners, pvband, shot_count,
                                       tsdf_from_mask)
    from paper_2303_12529_b200 import _native as nv
    nv.set_precision("fp64")
    tmp, lay, k = workspace
    target = fileio.parse_layout(lay[0].read_text(), 128)
    assert cli.main(["optimize", "--target", str(lay[0]), "--kernels", str(k), "--size", "128",
                     "--out-dir", str(tmp / "one"), "--max-iters", "4"]) == 0
    for name in ("mask.pgm", "phi.f64", "metrics.json", "loss.csv"):
        assert (tmp / "one" / name).exists()
    assert cli.main(["tsdf", "--target", str(lay[0]), "--size", "128", "--out-dir", str(tmp / "ts")]) == 0
    assert np.array_equal(fileio.load_field(tmp / "ts" / "phi.f64"), tsdf_from_mask(target).phi)
    mp = tmp / "mask.pgm"
    fileio.save_pgm(mp, target)
    capsys.readouterr()
    assert cli.main(["metrics", "--mask", str(mp), "--target", str(lay[0]), "--kernels", str(k),
                     "--size", "128"]) == 0
    got = json.loads(capsys.readouterr().out)
    focus, defocus = load_kernels(k)
    prints = print_corners(target.astype(np.float64), focus, defocus, OptConfig(), binarize=True)
    assert got["l2"] == l2_error(prints.nominal, target) and got["pvband"] == pvband(prints.inner, prints.outer)
    assert got["shots"] == shot_count(target)
    assert cli.main(["simulate", "--target", str(lay[0]), "--kernels", str(k), "--size", "128",
                     "--out-dir", str(tmp / "sim")]) == 0
    assert np.array_equal(fileio.load_pgm(tmp / "sim" / "nominal.pgm"), prints.nominal)
    bad = tmp / "bad.dvlk"
    bad.write_bytes(b"garbage")
    assert cli.main(["simulate", "--target", str(lay[0]), "--kernels", str(bad), "--size", "128",
                     "--out-dir", str(tmp / "y")]) == 1
