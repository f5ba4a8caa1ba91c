"""PSF data model for the Python face of the B200 Richardson-Lucy path.

Mirrors the three representations of the reference
(/root/reference/proj/include/fastdeconv/psf.hpp:26-173) -- same names,
argument meaning and validation errors -- because they are the *inputs* of
the hot path: the representation decides the operator (convolve.hpp:627-633).
Classification, conversion and the adjoint are done by the native library
(paper_1304_7211_b200/csrc/plan.cpp) when a plan is built; this module only
validates, normalises and marshals.
"""
from __future__ import annotations

import math
import re
from typing import Iterable, List, Sequence, Tuple

import numpy as np

DENSE, CONVEX, SPARSE = 0, 1, 2


def _normalise(ws: Sequence[float]) -> List[float]:
    # sequential double sum exactly as the reference ctors (psf.hpp:38-45);
    # builtin sum() is compensated since Python 3.12, so sum by hand.
    total = 0.0
    for w in ws:
        total += w
    return [w / total for w in ws]


class DensePsf:
    """Grid with an anchor; cell (ix, iy) acts at (ix-anchorX, iy-anchorY). psf.hpp:26-70"""

    def __init__(self, width: int, height: int, anchorX: int, anchorY: int, weights: Iterable[float]):
        weights = [float(w) for w in np.asarray(list(weights) if not isinstance(weights, np.ndarray)
                                                else weights, dtype=np.float64).ravel()]
        if width < 1 or height < 1:
            raise ValueError("DensePsf: dimensions must be at least 1x1")
        if not (0 <= anchorX < width and 0 <= anchorY < height):
            raise ValueError("DensePsf: anchor must lie inside the grid")
        if len(weights) != width * height:
            raise ValueError("DensePsf: weight count does not match dimensions")
        for w in weights:
            if not (w >= 0.0) or not math.isfinite(w):
                raise ValueError("DensePsf: weights must be finite and nonnegative")
        total = 0.0
        for w in weights:
            total += w
        if total <= 0.0:
            raise ValueError("DensePsf: total weight must be positive")
        self._raw = weights
        self.width, self.height, self.anchorX, self.anchorY = width, height, anchorX, anchorY
        self.weights = np.array(_normalise(weights), dtype=np.float64)

    def raw(self):
        return {"repr": DENSE, "width": self.width, "height": self.height, "anchor_x": self.anchorX,
                "anchor_y": self.anchorY, "weights": np.array(self._raw, dtype=np.float64)}

    def extents(self) -> Tuple[int, int, int, int]:
        return (-self.anchorX, self.width - 1 - self.anchorX, -self.anchorY, self.height - 1 - self.anchorY)


class UniformConvexPsf:
    """Row-convex uniform PSF: one [xMin, xMax] span per contiguous dy. psf.hpp:75-120"""

    def __init__(self, rows: Iterable[Tuple[int, int, int]]):
        rows = [(int(a), int(b), int(c)) for a, b, c in rows]
        if not rows:
            raise ValueError("UniformConvexPsf: at least one support row required")
        count = 0
        for i, (dy, lo, hi) in enumerate(rows):
            if lo > hi:
                raise ValueError("UniformConvexPsf: row interval is empty")
            if i > 0 and dy != rows[i - 1][0] + 1:
                raise ValueError("UniformConvexPsf: row offsets must be contiguous and increasing")
            count += hi - lo + 1
        self.rows = rows
        self.supportCount = count
        self.uniformWeight = 1.0 / float(count)

    def raw(self):
        a = np.array(self.rows, dtype=np.int32).reshape(-1, 3)
        return {"repr": CONVEX, "rows": (a[:, 0].copy(), a[:, 1].copy(), a[:, 2].copy())}

    def extents(self):
        return (min(r[1] for r in self.rows), max(r[2] for r in self.rows), self.rows[0][0], self.rows[-1][0])


class SparsePsf:
    """Tap list (dx, dy, w); positive weights, unique offsets. psf.hpp:124-170"""

    def __init__(self, taps: Iterable[Tuple[int, int, float]]):
        taps = [(int(dx), int(dy), float(w)) for dx, dy, w in taps]
        if not taps:
            raise ValueError("SparsePsf: at least one tap required")
        for _, _, w in taps:
            if not (w > 0.0) or not math.isfinite(w):
                raise ValueError("SparsePsf: weights must be finite and positive")
        if len({(dx, dy) for dx, dy, _ in taps}) != len(taps):
            raise ValueError("SparsePsf: duplicate tap coordinates")
        self._raw = taps
        ws = _normalise([w for _, _, w in taps])
        self.taps = [(dx, dy, w) for (dx, dy, _), w in zip(taps, ws)]

    @property
    def supportCount(self):
        return len(self.taps)

    def raw(self):
        a = np.array([(dx, dy) for dx, dy, _ in self._raw], dtype=np.int32).reshape(-1, 2)
        return {"repr": SPARSE, "taps": (a[:, 0].copy(), a[:, 1].copy(),
                                         np.array([w for _, _, w in self._raw], dtype=np.float64))}

    def extents(self):
        return (min(t[0] for t in self.taps), max(t[0] for t in self.taps),
                min(t[1] for t in self.taps), max(t[1] for t in self.taps))


Psf = (DensePsf, UniformConvexPsf, SparsePsf)


# ---------------------------------------------------------------- generators
def makeLinePsf(length: int) -> DensePsf:
    """Horizontal uniform line, anchor floor(length/2). psf.hpp:179-183"""
    if length < 1:
        raise ValueError("makeLinePsf: length must be at least 1")
    return DensePsf(length, 1, length // 2, 0, [1.0] * length)


def makeBoxPsf(mx: int, my: int) -> DensePsf:
    """Uniform mx x my rectangle, anchor (mx//2, my//2). psf.hpp:186-191"""
    if mx < 1 or my < 1:
        raise ValueError("makeBoxPsf: dimensions must be at least 1")
    return DensePsf(mx, my, mx // 2, my // 2, [1.0] * (mx * my))


def makeDiscPsf(diameter: int) -> UniformConvexPsf:
    """Pixel centres within diameter/2 of the d x d grid centre. psf.hpp:196-217"""
    if diameter < 1:
        raise ValueError("makeDiscPsf: diameter must be at least 1")
    c = diameter / 2.0
    r2 = c * c
    anchor = diameter // 2
    rows = []
    for j in range(diameter):
        yd = (j + 0.5) - c
        inside = [i for i in range(diameter) if ((i + 0.5) - c) ** 2 + yd * yd <= r2]
        if inside:
            rows.append((j - anchor, min(inside) - anchor, max(inside) - anchor))
    return UniformConvexPsf(rows)


def makeDiagonalPsf(length: int) -> SparsePsf:
    """45-degree diagonal of `length` taps centred on the anchor. psf.hpp:220-229"""
    if length < 1:
        raise ValueError("makeDiagonalPsf: length must be at least 1")
    a = length // 2
    return SparsePsf([(i - a, i - a, 1.0) for i in range(length)])


def taps_of(psf) -> List[Tuple[int, int, float]]:
    """(dx, dy, w) list with normalised weights (psfTaps, psf.hpp:378)."""
    if isinstance(psf, DensePsf):
        out = []
        for iy in range(psf.height):
            for ix in range(psf.width):
                w = psf.weights[iy * psf.width + ix]
                if w > 0.0:
                    out.append((ix - psf.anchorX, iy - psf.anchorY, float(w)))
        return out
    if isinstance(psf, UniformConvexPsf):
        return [(dx, dy, psf.uniformWeight) for dy, lo, hi in psf.rows for dx in range(lo, hi + 1)]
    return list(psf.taps)


def adjoint(psf):
    """Reflect about the origin, (dx,dy) -> (-dx,-dy). psf.hpp:280-308"""
    if isinstance(psf, DensePsf):
        w, h = psf.width, psf.height
        g = np.array(psf._raw, dtype=np.float64).reshape(h, w)[::-1, ::-1]
        return DensePsf(w, h, w - 1 - psf.anchorX, h - 1 - psf.anchorY, g.ravel())
    if isinstance(psf, UniformConvexPsf):
        return UniformConvexPsf([(-dy, -hi, -lo) for dy, lo, hi in reversed(psf.rows)])
    return SparsePsf([(-dx, -dy, w) for dx, dy, w in psf._raw])


# ------------------------------------------------- sparse text format (CLI)
def parseSparsePsf(text: str) -> SparsePsf:
    """One "dx dy weight" triple per line, '#' comment and blank lines ignored,
    weights renormalised on load (psf.hpp:231-262).  Errors name the line."""
    taps, seen = [], set()
    for line_no, line in enumerate(text.split("\n"), start=1):
        if line.endswith("\r"):
            line = line[:-1]
        s = line.lstrip(" \t")
        if not s or s.startswith("#"):
            continue
        parts = line.split()
        try:
            if len(parts) != 3:
                raise ValueError
            dx, dy, w = int(parts[0]), int(parts[1]), float(parts[2])
        except ValueError:
            raise RuntimeError(f"sparse PSF: line {line_no}: expected 'dx dy weight'") from None
        if not (w > 0.0) or not math.isfinite(w):
            raise RuntimeError(f"sparse PSF: line {line_no}: weight must be positive")
        if (dx, dy) in seen:
            raise RuntimeError(f"sparse PSF: line {line_no}: duplicate tap ({dx}, {dy})")
        seen.add((dx, dy))
        taps.append((dx, dy, w))
    if not taps:
        raise RuntimeError("sparse PSF: no taps found")
    return SparsePsf(taps)


def formatSparsePsf(psf: SparsePsf) -> str:
    """Inverse of parseSparsePsf, 17 significant digits (psf.hpp:264-271)."""
    out = ["# dx dy weight"]
    for dx, dy, w in psf.taps:
        out.append(f"{dx} {dy} {w:.17g}")
    return "\n".join(out) + "\n"


def toSparse(psf) -> SparsePsf:
    """Non-zero taps of any representation, in the reference's toSparse order."""
    return SparsePsf([(dx, dy, w) for dx, dy, w in taps_of(psf) if w != 0.0])


def parsePsfSpec(spec: str):
    """CLI PSF grammar line:<M> | box:<MX>x<MY> | disc:<D> | diag:<M> |
    file:<path> (fastdeconv_cli.cpp:16-58), same error messages."""
    if ":" not in spec:
        raise RuntimeError(f"bad PSF spec '{spec}' (expected line:<M>, box:<MX>x<MY>, disc:<D>, diag:<M>, "
                           "or file:<path>)")
    kind, arg = spec.split(":", 1)

    def size(s: str) -> int:  # std::stoi consuming the whole argument, value >= 1
        ok = re.fullmatch(r"[ \t\n\v\f\r]*[+-]?[0-9]+", s) is not None
        v = int(s) if ok else 0
        if v < 1 or v > 2**31 - 1:
            raise RuntimeError(f"bad PSF size '{s}' in spec '{spec}'")
        return v

    if kind == "line":
        return makeLinePsf(size(arg))
    if kind == "disc":
        return makeDiscPsf(size(arg))
    if kind == "diag":
        return makeDiagonalPsf(size(arg))
    if kind == "box":
        if "x" not in arg:
            raise RuntimeError(f"bad box spec '{spec}' (expected box:<MX>x<MY>)")
        a, b = arg.split("x", 1)
        return makeBoxPsf(size(a), size(b))
    if kind == "file":
        try:
            with open(arg) as fh:
                text = fh.read()
        except OSError:
            raise RuntimeError(f"cannot open PSF file: {arg}") from None
        return parseSparsePsf(text)
    raise RuntimeError(f"unknown PSF kind '{kind}' in spec '{spec}'")
