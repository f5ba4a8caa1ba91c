"""Command-line front end over the B200 path, mirroring the reference's
``fastdeconv`` tool (proj/tools/fastdeconv_cli.cpp:101-270): the same
subcommands, options, defaults, output lines and CSV format, with every
convolution and RL run going through libfdgpu (there is no CPU fallback).

    python -m paper_1304_7211_b200.cli blur    --in g.pgm --psf disc:9 [--mode cyclic|replicate] --out b.pgm
    python -m paper_1304_7211_b200.cli deconv  --in b.pgm --psf disc:9 [--iters 100] [--op auto]
                                               [--eps 1e-8] [--thin T [--reactivate 10]] --out r.pgm
    python -m paper_1304_7211_b200.cli snr     --ref a.pgm --test b.pgm
    python -m paper_1304_7211_b200.cli psf-gen --psf disc:9 --out disc9.txt
    python -m paper_1304_7211_b200.cli bench   --experiment table1|table2 --in g.pgm --out t.csv
                                               [--reps 100] [--iters 100] [--thresholds ...] [--mode cyclic]

Errors print ``error: <message>`` and exit 1, like the reference's main().
"""
import argparse
import math
import sys
import time
from typing import List, Optional

import numpy as np

from .convolve import OperatorKind, dispatch, operatorAcceptsPsf, operatorKindFromName, operatorName
from .pgm import readPgmFile, snrDb, writePgmFile
from .psf import (formatSparsePsf, makeBoxPsf, makeDiagonalPsf, makeDiscPsf, makeLinePsf, parsePsfSpec,
                  toSparse)
from .rl import BoundaryMode, RlConfig, blurImage, rlDeconvolve, rlDeconvolveSelective


def _mode(name: str) -> BoundaryMode:
    if name == "cyclic":
        return BoundaryMode.Cyclic
    if name == "replicate":
        return BoundaryMode.Replicate
    raise RuntimeError(f"bad boundary mode '{name}' (expected cyclic or replicate)")


def _timed(fn):
    t0 = time.perf_counter()
    out = fn()
    return out, time.perf_counter() - t0


def run_blur(a) -> int:
    img = readPgmFile(a.input)
    psf = parsePsfSpec(a.psf)
    out, secs = _timed(lambda: blurImage(img, psf, _mode(a.mode)))
    writePgmFile(a.out, out)
    print(f"blur: psf={a.psf} mode={a.mode} {img.shape[1]}x{img.shape[0]} {secs:.3f} s -> {a.out}")
    return 0


def run_deconv(a) -> int:
    img = readPgmFile(a.input)
    psf = parsePsfSpec(a.psf)
    cfg = RlConfig(iterations=a.iters, op=operatorKindFromName(a.op), epsilonDiv=a.eps)
    if a.thin is not None:
        res, secs = _timed(lambda: rlDeconvolveSelective(img, psf, cfg, a.thin, a.reactivate))
        writePgmFile(a.out, res.image)
        print(f"deconv: {a.iters} iterations operator={a.op} thin={a.thin:g} "
              f"omitted={res.trace.omittedPercent():.2f}% {secs:.3f} s -> {a.out}")
    else:
        resolved = dispatch(psf, cfg.op)
        res, secs = _timed(lambda: rlDeconvolve(img, psf, cfg))
        writePgmFile(a.out, res.image)
        print(f"deconv: {a.iters} iterations operator={operatorName(resolved)} {secs:.3f} s -> {a.out}")
    return 0


def run_snr(a) -> int:
    v = snrDb(readPgmFile(a.ref), readPgmFile(a.test))
    print("inf" if math.isinf(v) else f"{v:.2f}")
    return 0


def run_psf_gen(a) -> int:
    psf = parsePsfSpec(a.psf)
    sparse = toSparse(psf)
    try:
        with open(a.out, "w") as fh:
            fh.write(formatSparsePsf(sparse))
    except OSError:
        raise RuntimeError(f"cannot open for writing: {a.out}") from None
    print(f"psf-gen: {a.psf} -> {a.out} ({sparse.supportCount} taps)")
    return 0


# ------------------------------------------------------------ bench tables
TABLE1_PSFS = [("line:9", lambda: makeLinePsf(9)), ("line:17", lambda: makeLinePsf(17)),
               ("box:9x9", lambda: makeBoxPsf(9, 9)), ("box:17x17", lambda: makeBoxPsf(17, 17)),
               ("diag:9", lambda: makeDiagonalPsf(9)), ("diag:17", lambda: makeDiagonalPsf(17)),
               ("disc:9", lambda: makeDiscPsf(9)), ("disc:17", lambda: makeDiscPsf(17))]
TABLE1_OPS = [OperatorKind.Naive, OperatorKind.Fourier, OperatorKind.List, OperatorKind.GenericBox,
              OperatorKind.Box2dSliding, OperatorKind.Box2dCumulated, OperatorKind.Box1dSliding,
              OperatorKind.Box1dCumulated]
DEFAULT_THRESHOLDS = [0.0, 0.005, 0.01, 0.02, 0.05, 0.1, 0.2, 0.5]


def _mean(xs):
    return sum(xs) / len(xs) if xs else 0.0


def _std(xs):
    if len(xs) < 2:
        return 0.0
    m = _mean(xs)
    return math.sqrt(sum((x - m) ** 2 for x in xs) / len(xs))


def _row(exp, op, psf, mean=None, std=None, omitted=None, snr_o=None, snr_r=None, speedup=None):
    return [exp, op, psf, mean, std, omitted, snr_o, snr_r, speedup]


def emit_csv(rows) -> str:
    """bench.hpp emitCsv: fixed columns, 2-decimal cells, empty when absent."""
    def cell(v):
        if v is None or isinstance(v, str):
            return "" if v is None else v
        if math.isinf(v):
            return "inf" if v > 0 else "-inf"
        return f"{v:.2f}"
    out = ["experiment,operator,psf,mean_s,stddev_s,omitted_pct,snr_orig_db,snr_ref_db,speedup"]
    for r in rows:
        out.append(",".join(cell(x) for x in r))
    return "\n".join(out) + "\n"


def run_table1(original, iters: int, reps: int, mode: BoundaryMode):
    rows = []
    blurred = [(label, mk(), None) for label, mk in TABLE1_PSFS]
    blurred = [(label, psf, np.maximum(blurImage(original, psf, mode), 0.0)) for label, psf, _ in blurred]
    for op in TABLE1_OPS:
        for label, psf, img in blurred:
            if operatorAcceptsPsf(op, psf):
                cfg = RlConfig(iterations=iters, op=op)
                samples = [_timed(lambda: rlDeconvolve(img, psf, cfg))[1] for _ in range(reps)]
                rows.append(_row("table1", operatorName(op), label, _mean(samples), _std(samples)))
            else:
                rows.append(_row("table1", operatorName(op), label))
    return rows


def run_table2(original, iters: int, reps: int, mode: BoundaryMode, thresholds: List[float]):
    psf = makeDiscPsf(9)
    blurred = np.maximum(blurImage(original, psf, mode), 0.0)
    cfg = RlConfig(iterations=iters, op=OperatorKind.Naive)
    reference, t0 = _timed(lambda: rlDeconvolve(blurred, psf, cfg).image)
    ref_s = [t0] + [_timed(lambda: rlDeconvolve(blurred, psf, cfg))[1] for _ in range(reps - 1)]
    ref_mean = _mean(ref_s)
    rows = [_row("table2", "naive", "disc:9", ref_mean, _std(ref_s), 0.0, snrDb(original, reference), math.inf,
                 1.0)]
    for t in thresholds:
        run, s0 = _timed(lambda: rlDeconvolveSelective(blurred, psf, cfg, t))
        samples = [s0] + [_timed(lambda: rlDeconvolveSelective(blurred, psf, cfg, t))[1] for _ in range(reps - 1)]
        rows.append(_row("table2", f"naive:thin={t:g}", "disc:9", _mean(samples), _std(samples),
                         run.trace.omittedPercent(), snrDb(original, run.image), snrDb(reference, run.image),
                         ref_mean / _mean(samples)))
    return rows


def run_bench(a) -> int:
    if a.experiment not in ("table1", "table2"):
        raise RuntimeError(f"bad experiment '{a.experiment}' (expected table1 or table2)")
    if a.iters < 1:
        raise ValueError("bench: iterations must be >= 1")
    if a.reps < 1:
        raise ValueError("bench: repetitions must be >= 1")
    original = readPgmFile(a.input)
    mode = _mode(a.mode)
    if a.experiment == "table1":
        rows = run_table1(original, a.iters, a.reps, mode)
    else:
        rows = run_table2(original, a.iters, a.reps, mode, a.thresholds or DEFAULT_THRESHOLDS)
    try:
        with open(a.out, "w", newline="\n") as fh:
            fh.write(emit_csv(rows))
    except OSError:
        raise RuntimeError(f"cannot open for writing: {a.out}") from None
    print(f"bench: {a.experiment} image={a.input} reps={a.reps} iters={a.iters} -> {a.out} ({len(rows)} rows)")
    return 0


def parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="fastdeconv-b200", description="Richardson-Lucy deconvolution with "
                                "PSF-specialized convolution operators (B200 path)")
    sub = p.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("blur", help="Convolve an image with a PSF")
    b.add_argument("--in", dest="input", required=True)
    b.add_argument("--psf", required=True)
    b.add_argument("--mode", default="cyclic")
    b.add_argument("--out", required=True)
    b.set_defaults(fn=run_blur)
    d = sub.add_parser("deconv", help="Richardson-Lucy deconvolution")
    d.add_argument("--in", dest="input", required=True)
    d.add_argument("--psf", required=True)
    d.add_argument("--iters", type=int, default=100)
    d.add_argument("--op", default="auto")
    d.add_argument("--eps", type=float, default=1e-8)
    d.add_argument("--thin", type=float, default=None)
    d.add_argument("--reactivate", type=int, default=10)
    d.add_argument("--out", required=True)
    d.set_defaults(fn=run_deconv)
    s = sub.add_parser("snr", help="Signal-to-noise ratio between two images (dB)")
    s.add_argument("--ref", required=True)
    s.add_argument("--test", required=True)
    s.set_defaults(fn=run_snr)
    g = sub.add_parser("psf-gen", help="Write a PSF as a sparse tap-list file")
    g.add_argument("--psf", required=True)
    g.add_argument("--out", required=True)
    g.set_defaults(fn=run_psf_gen)
    t = sub.add_parser("bench", help="Run a benchmark experiment, emit CSV")
    t.add_argument("--experiment", required=True)
    t.add_argument("--in", dest="input", required=True)
    t.add_argument("--reps", type=int, default=100)
    t.add_argument("--iters", type=int, default=100)
    t.add_argument("--thresholds", type=float, nargs="*", default=None)
    t.add_argument("--mode", default="cyclic")
    t.add_argument("--out", required=True)
    t.set_defaults(fn=run_bench)
    return p


def main(argv: Optional[List[str]] = None) -> int:
    args = parser().parse_args(argv)
    try:
        return args.fn(args)
    except Exception as e:  # the reference's main(): "error: <what>", exit 1
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
