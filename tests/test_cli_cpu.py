"""CLI callers of the GPU path, host-only parts: PGM I/O (pgm.hpp), snrDb,
PSF spec grammar and the sparse text format (fastdeconv_cli.cpp, psf.hpp),
the bench CSV format (bench.hpp emitCsv) and CLI exit codes that need no
device.  Mirrors proj/tests/test_image.cpp:85-186, test_bench.cpp:129-174,
test_cli.cpp:47-57,107-195."""
import math

import numpy as np
import pytest

from paper_1304_7211_b200 import cli
from paper_1304_7211_b200.pgm import PgmParseError, readPgm, snrDb, writePgm, writePgmFile
from paper_1304_7211_b200.psf import (formatSparsePsf, makeDiscPsf, parsePsfSpec, parseSparsePsf, taps_of,
                                      toSparse)


def test_snr_closed_form_and_identity():
    assert abs(snrDb(np.full((10, 10), 10.0), np.full((10, 10), 11.0)) - 20.0) < 1e-12
    img = np.random.default_rng(13).uniform(1, 255, (6, 6))
    assert math.isinf(snrDb(img, img)) and snrDb(img, img) > 0
    with pytest.raises(ValueError):
        snrDb(np.ones((3, 3)), np.ones((4, 3)))
    with pytest.raises(ValueError):
        snrDb(np.zeros((3, 3)), np.ones((3, 3)))


def test_read_minimal_p5_and_p2_with_comments():
    img = readPgm(b"P5 2 2 255 " + bytes([0, 64, 128, 255]))
    np.testing.assert_array_equal(img, [[0, 64], [128, 255]])
    img = readPgm(b"P2\n# a comment\n3 1\n# another\n255\n0 127 255\n")
    np.testing.assert_array_equal(img, [[0, 127, 255]])


def test_write_rounds_and_clamps_and_round_trips():
    back = readPgm(writePgm(np.array([[255.4, -3.0], [300.0, 127.5001]])))
    np.testing.assert_array_equal(back, [[255, 0], [255, 128]])
    assert readPgm(writePgm(np.array([[0.5, 1.5, 2.5]])))[0].tolist() == [1, 2, 3]  # lround: half away from 0
    rng = np.random.default_rng(15)
    for _ in range(25):
        img = rng.integers(0, 256, (rng.integers(1, 18), rng.integers(1, 18))).astype(np.float64)
        np.testing.assert_array_equal(readPgm(writePgm(img)), img)
    with pytest.raises(ValueError):
        writePgm(np.array([[np.nan]]))
    with pytest.raises(ValueError):
        writePgm(np.zeros((0, 0)))


@pytest.mark.parametrize("data,needle", [(b"P6 1 1 255 x", "magic"), (b"P5 2 2 65535 ", "maxval"),
                                         (b"P5 2 2 255 \x00", "byte"), (b"P5 2", "end of input"),
                                         (b"P2 2 1 100\n50 101\n", "exceeds maxval")])
def test_read_errors(data, needle):
    with pytest.raises(PgmParseError, match=needle):
        readPgm(data)


def test_psf_spec_grammar():
    assert parsePsfSpec("line:15").width == 15
    assert parsePsfSpec("box:3x5").height == 5
    assert parsePsfSpec("diag:5").supportCount == 5
    assert len(taps_of(parsePsfSpec("disc:9"))) == len(taps_of(makeDiscPsf(9)))
    for spec, msg in [("line", "bad PSF spec"), ("line:0", "bad PSF size"), ("line:3a", "bad PSF size"),
                      ("box:3", "bad box spec"), ("blob:9", "unknown PSF kind"), ("file:/nonexistent", "cannot open")]:
        with pytest.raises(RuntimeError, match=msg):
            parsePsfSpec(spec)


def test_sparse_text_round_trip(tmp_path):
    psf = toSparse(makeDiscPsf(9))
    text = formatSparsePsf(psf)
    assert text.startswith("# dx dy weight\n")
    back = parseSparsePsf(text)
    assert [(dx, dy) for dx, dy, _ in back.taps] == [(dx, dy) for dx, dy, _ in psf.taps]
    np.testing.assert_allclose([w for *_, w in back.taps], [w for *_, w in psf.taps], rtol=1e-13)  # renormalised on load
    p = tmp_path / "d9.txt"
    p.write_text(text)
    assert parsePsfSpec(f"file:{p}").supportCount == psf.supportCount
    for bad, msg in [("0 0\n", "expected 'dx dy weight'"), ("0 0 -1\n", "positive"),
                     ("0 0 1\n0 0 2\n", "duplicate tap"), ("# only\n", "no taps")]:
        with pytest.raises(RuntimeError, match=msg):
            parseSparsePsf(bad)


def test_emit_csv_format():
    assert cli.emit_csv([]) == "experiment,operator,psf,mean_s,stddev_s,omitted_pct,snr_orig_db,snr_ref_db,speedup\n"
    csv = cli.emit_csv([cli._row("table1", "naive", "line:9", 0.048, 0.001)])
    assert csv.count("\n") == 2 and "table1,naive,line:9,0.05,0.00,,,,\n" in csv
    csv = cli.emit_csv([cli._row("table2", "naive:thin=0", "disc:9", 3.771, 0.0049, 0.0, 13.308, math.inf, 0.994)])
    assert "table2,naive:thin=0,disc:9,3.77,0.00,0.00,13.31,inf,0.99\n" in csv


def test_cli_host_only_commands_and_exit_codes(tmp_path, capsys):
    a = tmp_path / "a.pgm"
    writePgmFile(str(a), np.arange(12, dtype=np.float64).reshape(3, 4) + 1)
    assert cli.main(["snr", "--ref", str(a), "--test", str(a)]) == 0
    assert capsys.readouterr().out.strip() == "inf"
    out = tmp_path / "p.txt"
    assert cli.main(["psf-gen", "--psf", "disc:9", "--out", str(out)]) == 0
    assert "taps" in capsys.readouterr().out and parseSparsePsf(out.read_text()).supportCount > 0
    assert cli.main(["snr", "--ref", str(tmp_path / "nope.pgm"), "--test", str(a)]) == 1
    assert cli.main(["blur", "--in", str(a), "--psf", "blob:9", "--out", str(tmp_path / "o.pgm")]) == 1
    with pytest.raises(SystemExit) as e:
        cli.main(["snr", "--bogus", "x"])
    assert e.value.code == 2
    with pytest.raises(SystemExit) as e:
        cli.main([])
    assert e.value.code == 2
    with pytest.raises(SystemExit) as e:
        cli.main(["--help"])
    assert e.value.code == 0
