"""Case list of the golden fixtures (tests/golden/golden_v1.npz), shared by
scripts/gen_golden.py (which runs the reference) and tests/test_oracle.py."""
from oracle.pyoracle import (AUTO, BOX1D_CUMUL, BOX1D_SLIDING, BOX2D_CUMUL, BOX2D_SLIDING, GENERIC_BOX, LIST,
                             NAIVE)
from paper_1304_7211_b200 import psf as P
from paper_1304_7211_b200 import workloads as W


def make_psf(spec: str):
    kind, _, arg = spec.partition(":")
    if kind == "line":
        return P.makeLinePsf(int(arg))
    if kind == "box":
        a, b = arg.split("x")
        return P.makeBoxPsf(int(a), int(b))
    if kind == "disc":
        return P.makeDiscPsf(int(arg))
    if kind == "diag":
        return P.makeDiagonalPsf(int(arg))
    if kind == "densedisc":
        return P.DensePsf(*_dense_of(P.makeDiscPsf(int(arg))))
    if kind == "asym":
        return P.SparsePsf([(2, -1, 1.0), (0, 0, 2.0), (-3, 1, 0.5)])
    if kind == "blob":
        return P.DensePsf(3, 1, 1, 0, [1.0, 2.0, 1.0])
    if kind == "gauss":
        return W.gaussian31(seed=5, size=int(arg))
    if kind == "oblique":
        return W.oblique_line()
    if kind == "disc10":
        return W.disc_r10()
    raise ValueError(spec)


def _dense_of(convex):
    xs = [x for _, lo, hi in convex.rows for x in range(lo, hi + 1)] + [0]
    ys = [r[0] for r in convex.rows] + [0]
    x0, x1, y0, y1 = min(xs), max(xs), min(ys), max(ys)
    w, h = x1 - x0 + 1, y1 - y0 + 1
    g = [0.0] * (w * h)
    for dy, lo, hi in convex.rows:
        for dx in range(lo, hi + 1):
            g[(dy - y0) * w + (dx - x0)] = 1.0
    return w, h, -x0, -y0, g


CONV_CASES = {
    "line5_s": ("line:5", BOX1D_SLIDING, (7, 23)),
    "line4_c": ("line:4", BOX1D_CUMUL, (9, 17)),
    "line15_list": ("line:15", LIST, (5, 40)),
    "box5x3_s": ("box:5x3", BOX2D_SLIDING, (21, 19)),
    "box3x5_c": ("box:3x5", BOX2D_CUMUL, (13, 30)),
    "box9_g": ("box:9x9", GENERIC_BOX, (25, 25)),
    "disc9_g": ("disc:9", GENERIC_BOX, (33, 29)),
    "disc4_list": ("disc:4", LIST, (11, 14)),
    "disc5_naive": ("disc:5", NAIVE, (17, 12)),
    "diag7_list": ("diag:7", LIST, (20, 31)),
    "diag5_g": ("diag:5", GENERIC_BOX, (16, 16)),
    "asym_list": ("asym", LIST, (7, 11)),
    "asym_naive": ("asym", NAIVE, (9, 13)),
    "blob_auto": ("blob", AUTO, (6, 10)),
    "gauss7_naive": ("gauss:7", NAIVE, (24, 19)),
    "oblique_g": ("oblique", GENERIC_BOX, (40, 44)),
    "disc10_g": ("disc10", GENERIC_BOX, (30, 36)),
    "disc9_auto": ("disc:9", AUTO, (15, 15)),
    "box1_naive": ("box:1x1", NAIVE, (5, 5)),
}

RL_CASES = {
    "line9_auto": ("line:9", AUTO, (20, 33), 15),
    "line15_slide": ("line:15", BOX1D_SLIDING, (16, 40), 12),
    "box3x5_slide": ("box:3x5", BOX2D_SLIDING, (25, 22), 10),
    "disc5_auto": ("disc:5", AUTO, (24, 27), 12),
    "diag5_list": ("diag:5", LIST, (18, 21), 10),
    "gauss7_naive": ("gauss:7", NAIVE, (22, 20), 8),
    "oblique_g": ("oblique", GENERIC_BOX, (30, 32), 6),
}

SEL_CASES = {
    "densedisc3_naive": ("densedisc:3", NAIVE, (24, 24), 25, 0.002, 10, 0),
    "diag5_list": ("diag:5", LIST, (20, 26), 22, 0.003, 10, 0),
    "gauss7_from5": ("gauss:7", NAIVE, (21, 19), 30, 0.001, 10, 5),
    "densedisc3_inf": ("densedisc:3", NAIVE, (24, 24), 25, float("inf"), 10, 0),
}
