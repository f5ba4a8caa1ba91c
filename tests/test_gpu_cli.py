"""CLI deconv / blur / bench through the GPU path, checked against direct
library calls (proj/tests/test_cli.cpp:58-155,196-230)."""
import numpy as np
import pytest

from paper_1304_7211_b200 import OperatorKind as K, RlConfig, cli, convolve, rlDeconvolve, rlDeconvolveSelective
from paper_1304_7211_b200.pgm import readPgmFile, writePgm, writePgmFile
from paper_1304_7211_b200.psf import makeBoxPsf, makeDiscPsf

pytestmark = pytest.mark.gpu


def scene(w=48, h=40, seed=3):
    rng = np.random.default_rng(seed)
    return np.clip(np.round(rng.uniform(20, 230, (h, w))), 0, 255)


def test_cli_deconv_byte_identical_to_library(tmp_path):
    p = tmp_path / "b.pgm"
    writePgmFile(str(p), scene())
    img = readPgmFile(str(p))
    out = tmp_path / "r.pgm"
    assert cli.main(["deconv", "--in", str(p), "--psf", "disc:9", "--iters", "15", "--out", str(out)]) == 0
    lib = rlDeconvolve(img, makeDiscPsf(9), RlConfig(iterations=15)).image
    assert out.read_bytes() == writePgm(lib)


def test_cli_selective_deconv_matches_library(tmp_path, capsys):
    p = tmp_path / "b.pgm"
    writePgmFile(str(p), scene(seed=4))
    img = readPgmFile(str(p))
    out = tmp_path / "r.pgm"
    assert cli.main(["deconv", "--in", str(p), "--psf", "disc:9", "--iters", "12", "--op", "naive", "--thin", "0.5",
                     "--out", str(out)]) == 0
    assert "omitted=" in capsys.readouterr().out
    lib = rlDeconvolveSelective(img, makeDiscPsf(9), RlConfig(iterations=12, op=K.Naive), 0.5, 10).image
    assert out.read_bytes() == writePgm(lib)


def test_cli_blur_replicate_matches_operator(tmp_path):
    p = tmp_path / "g.pgm"
    writePgmFile(str(p), scene(seed=5))
    out = tmp_path / "b.pgm"
    assert cli.main(["blur", "--in", str(p), "--psf", "box:5x3", "--mode", "replicate", "--out", str(out)]) == 0
    ref = convolve(readPgmFile(str(p)), makeBoxPsf(5, 3), K.Auto)
    assert out.read_bytes() == writePgm(ref)


def test_cli_incompatible_operator_exits_1(tmp_path):
    p = tmp_path / "t.pgm"
    writePgmFile(str(p), scene(8, 8))
    assert cli.main(["deconv", "--in", str(p), "--psf", "box:3x3", "--op", "box1d-sliding", "--iters", "1",
                     "--out", str(tmp_path / "o.pgm")]) == 1


def test_cli_bench_tables(tmp_path):
    p = tmp_path / "g.pgm"
    writePgmFile(str(p), scene(24, 20, seed=6))
    t1 = tmp_path / "t1.csv"
    assert cli.main(["bench", "--experiment", "table1", "--in", str(p), "--reps", "1", "--iters", "1",
                     "--out", str(t1)]) == 0
    lines = t1.read_text().splitlines()
    assert len(lines) == 1 + 8 * 8
    assert any(l.startswith("table1,box2d-sliding,box:9x9,") and l.split(",")[3] for l in lines)
    assert any(l.startswith("table1,box1d-sliding,disc:9,,,") for l in lines)  # incompatible cell stays empty
    t2 = tmp_path / "t2.csv"
    assert cli.main(["bench", "--experiment", "table2", "--in", str(p), "--reps", "1", "--iters", "2",
                     "--thresholds", "0", "0.1", "--out", str(t2)]) == 0
    rows = [l.split(",") for l in t2.read_text().splitlines()[1:]]
    assert [r[1] for r in rows] == ["naive", "naive:thin=0", "naive:thin=0.1"]
    assert rows[1][7] == "inf"  # threshold 0 == the unthinned reference (rl.hpp threshold-0 equivalence)
