"""Spans-engine probe: RL Mpx*it/s of the device loop per PSF and engine.

usage: python scripts/spans_probe.py W H ITERS PSF [PSF ...]
PSF = a workloads name (disc10, oblique21) or a parsePsfSpec spec (disc:9,
diag:17 -> converted to UniformConvexPsf rows).  Per PSF: GenericBox on the
default spans kernel, on the runtime-table kernel (spans mode 3), on the
per-tap engine (FDG_NO_SPANS) and Naive, in microseconds per pass.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1304_7211_b200 import OperatorKind as K, RlConfig, RlSolver, workloads as W  # noqa: E402
from paper_1304_7211_b200._lib import lib  # noqa: E402
from paper_1304_7211_b200.psf import UniformConvexPsf, parsePsfSpec, taps_of  # noqa: E402


def convex(psf):
    rows = {}
    for dx, dy, _ in taps_of(psf):
        lo, hi = rows.get(dy, (dx, dx))
        rows[dy] = (min(lo, dx), max(hi, dx))
    return UniformConvexPsf([(dy, rows[dy][0], rows[dy][1]) for dy in sorted(rows)])


def rate(psf, op, w, h, iters):
    dev = torch.device("cuda", 0)
    pitch = (w + 3) // 4 * 4
    g = torch.Generator(device=dev).manual_seed(0)
    f = torch.rand((h, pitch), device=dev, generator=g) * 0.8 + 0.2
    u = torch.empty_like(f)
    solver = RlSolver(psf, RlConfig(iterations=iters, op=op), w, h, batch=1, device=0)
    st = torch.cuda.current_stream(dev)
    solver.use_stream(st.cuda_stream)
    for _ in range(2):
        solver.run(f, u, iters)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record(st)
    for _ in range(reps):
        solver.run(f, u, iters)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return w * h * iters / (ms * 1e-3) / 1e6, ms / (2 * iters) * 1e3


def main():
    w, h, iters = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    for name in sys.argv[4:]:
        psf = W.make_psf(name) if ":" not in name else convex(parsePsfSpec(name))
        out = []
        for label, op, mode, nospans in (("spans", K.GenericBox, 0, False), ("spanr", K.GenericBox, 3, False),
                                         ("taps", K.GenericBox, 0, True), ("naive", K.Naive, 0, False)):
            if nospans:
                os.environ["FDG_NO_SPANS"] = "1"
            prev = lib().fdg_set_option(b"spans", mode)
            try:
                v, us = rate(psf, op, w, h, iters)
            finally:
                lib().fdg_set_option(b"spans", prev)
                os.environ.pop("FDG_NO_SPANS", None)
            out.append(f"{label} {v:9.0f} ({us:6.1f} us/pass)")
        print(f"{name:10s} {w}x{h} {iters} it: " + " | ".join(out), flush=True)


if __name__ == "__main__":
    main()
