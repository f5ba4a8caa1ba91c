"""Seeded synthetic inputs and PSFs of the BASELINE.json configurations.

The paper measures on the 256x256 "cameraman" photograph, which is not in
this container; BASELINE.json defines five synthetic configurations instead.
Every choice the configs leave open is frozen here (the manifest; see
DESIGN.md section "Workloads"):

* scene: background 0.2; rectangles then disks painted in order, each with
  intensity U[0.1, 1]; rectangle width and height drawn independently from
  U{8..128}, top-left corner U{0..W-1} x U{0..H-1}, clipped; disk radius
  U{4..40}, centre U{0..W-1} x U{0..H-1}, pixels with (x-cx)^2+(y-cy)^2 <= r^2.
  RNG: numpy PCG64 seeded with the config seed; draws in the order listed.
* observation: f = g (x) h with replicate boundary (blurImage(g, h,
  Replicate), rl.hpp:264), plus N(0, sigma^2) noise from the same
  generator, clamped to >= 1e-6, stored as float32.  The blur is evaluated
  in float64 on the CPU (separable cumulative sums for boxes, direct
  per-row sums otherwise) so that the input is identical for the oracle and
  the GPU; large inputs may instead be blurred on the GPU (bench only).
* PSFs: horizontal 1x15 / 1x31 boxes (makeLinePsf), the separable 15x15 box
  (makeBoxPsf), the r<=10 integer disc (317 taps, UniformConvexPsf rows
  xMax = floor(sqrt(100 - dy^2))), the 21 px @ 30 deg oblique line
  (origin-symmetric rasteriser: t in [-10.5, 10.5] step 1/8, (lround(t cos),
  -lround(t sin)), row-convex, UniformConvexPsf), and the 31x31 perturbed
  Gaussian (sigma 5, weight x (1 + 0.2 U[0,1]) from PCG64(1003), DensePsf
  anchor (15,15)).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Tuple

import numpy as np

from .psf import DensePsf, UniformConvexPsf, makeBoxPsf, makeLinePsf, taps_of


# ------------------------------------------------------------------- PSFs
def disc_r10() -> UniformConvexPsf:
    rows = []
    for dy in range(-10, 11):
        xm = int(math.isqrt(100 - dy * dy))
        rows.append((dy, -xm, xm))
    return UniformConvexPsf(rows)


def _round_half_away(v: float) -> int:
    return int(math.floor(v + 0.5)) if v >= 0 else -int(math.floor(-v + 0.5))


def oblique_line(length: int = 21, angle_deg: float = 30.0) -> UniformConvexPsf:
    th = math.radians(angle_deg)
    half = length / 2.0
    pts = set()
    n = int(round(2 * half * 8))
    for i in range(n + 1):
        t = -half + i / 8.0
        pts.add((_round_half_away(t * math.cos(th)), -_round_half_away(t * math.sin(th))))
    by_row = {}
    for dx, dy in pts:
        by_row.setdefault(dy, []).append(dx)
    rows = []
    for dy in sorted(by_row):
        xs = sorted(by_row[dy])
        if xs != list(range(xs[0], xs[-1] + 1)):
            raise AssertionError("oblique rasteriser produced a non-convex row")
        rows.append((dy, xs[0], xs[-1]))
    return UniformConvexPsf(rows)


def gaussian31(seed: int = 1003, sigma: float = 5.0, size: int = 31) -> DensePsf:
    rng = np.random.Generator(np.random.PCG64(seed))
    u = rng.random(size * size)
    a = size // 2
    w = []
    for iy in range(size):
        for ix in range(size):
            dx, dy = ix - a, iy - a
            w.append(math.exp(-(dx * dx + dy * dy) / (2.0 * sigma * sigma)) * (1.0 + 0.2 * u[iy * size + ix]))
    return DensePsf(size, size, a, a, w)


# ------------------------------------------------------------------ scene
def scene(width: int, height: int, seed: int, n_rect: int, n_disk: int,
          rng: np.random.Generator = None) -> np.ndarray:
    rng = rng or np.random.Generator(np.random.PCG64(seed))
    g = np.full((height, width), 0.2, dtype=np.float64)
    for _ in range(n_rect):
        rw = int(rng.integers(8, 129))
        rh = int(rng.integers(8, 129))
        x0 = int(rng.integers(0, width))
        y0 = int(rng.integers(0, height))
        v = float(rng.uniform(0.1, 1.0))
        g[y0:min(height, y0 + rh), x0:min(width, x0 + rw)] = v
    for _ in range(n_disk):
        r = int(rng.integers(4, 41))
        cx = int(rng.integers(0, width))
        cy = int(rng.integers(0, height))
        v = float(rng.uniform(0.1, 1.0))
        ya, yb = max(0, cy - r), min(height, cy + r + 1)
        xa, xb = max(0, cx - r), min(width, cx + r + 1)
        yy, xx = np.mgrid[ya:yb, xa:xb]
        m = (xx - cx) ** 2 + (yy - cy) ** 2 <= r * r
        g[ya:yb, xa:xb][m] = v
    return g


def blur_replicate(g: np.ndarray, psf) -> np.ndarray:
    """f = g (x) h, replicate boundary, float64 (correlation, convolve.hpp:17-21)."""
    h, w = g.shape
    taps = taps_of(psf)
    xs = [t[0] for t in taps]
    ys = [t[1] for t in taps]
    l, r, t_, b = max(0, -min(xs)), max(0, max(xs)), max(0, -min(ys)), max(0, max(ys))
    p = np.pad(g, ((t_, b), (l, r)), mode="edge")
    rect = _as_rect(taps)
    if rect is not None:
        mx, my, x0, y0 = rect
        c = np.cumsum(np.pad(p, ((0, 0), (1, 0))), axis=1)
        hs = c[:, l + x0 + mx: l + x0 + mx + w] - c[:, l + x0: l + x0 + w]
        c2 = np.cumsum(np.pad(hs, ((1, 0), (0, 0))), axis=0)
        return (c2[t_ + y0 + my: t_ + y0 + my + h] - c2[t_ + y0: t_ + y0 + h]) / (mx * my)
    out = np.zeros((h, w), dtype=np.float64)

    def rows(y0, y1):  # every output pixel accumulates its taps in tap order
        o = out[y0:y1]
        for dx, dy, wt in taps:
            o += wt * p[t_ + dy + y0: t_ + dy + y1, l + dx: l + dx + w]

    blk = 64
    if h * w < (1 << 20):
        rows(0, h)
    else:  # row blocks on a thread pool (numpy releases the GIL): same bits
        import os
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
            list(ex.map(lambda y: rows(y, min(h, y + blk)), range(0, h, blk)))
    return out


def _as_rect(taps):
    xs = sorted({t[0] for t in taps})
    ys = sorted({t[1] for t in taps})
    ws = {t[2] for t in taps}
    if len(ws) != 1 or len(taps) != len(xs) * len(ys):
        return None
    if xs != list(range(xs[0], xs[-1] + 1)) or ys != list(range(ys[0], ys[-1] + 1)):
        return None
    return len(xs), len(ys), xs[0], ys[0]


def observe(g: np.ndarray, psf, sigma: float, rng: np.random.Generator) -> np.ndarray:
    f = blur_replicate(g, psf) + rng.normal(0.0, sigma, size=g.shape)
    return np.maximum(f, 1e-6).astype(np.float32)


# ---------------------------------------------------------------- configs
@dataclass(frozen=True)
class Config:
    name: str
    width: int
    height: int
    seed: int
    n_rect: int
    n_disk: int
    psf: str
    op: str
    iterations: int
    sigma: float
    batch: int = 1


CONFIGS = {
    "cfg0": Config("cfg0", 512, 512, 0, 64, 32, "line15", "box1d-sliding", 100, 0.01),
    "cfg1": Config("cfg1", 1024, 1024, 1, 64, 32, "oblique21", "generic-box", 200, 0.005),
    "cfg2": Config("cfg2", 2048, 2048, 2, 256, 128, "disc10", "generic-box", 200, 0.01),
    "cfg3": Config("cfg3", 4096, 4096, 3, 64, 32, "gauss31", "naive", 150, 0.01),
    "cfg4": Config("cfg4", 16384, 16384, 4, 4096, 2048, "box15x15", "box2d-sliding", 100, 0.01),
    "cfg4b": Config("cfg4b", 2048, 2048, 100, 64, 32, "line31", "box1d-sliding", 100, 0.01, batch=64),
}


# Config 3 thinning thresholds (absolute max|du|), calibrated once on the
# oracle over the real 4096^2 input so that the mean active fraction over
# 1-based iterations 21..150 is ~50 % / ~25 % (
# profiles/r01_cfg3_thresholds.json records the calibration run).
CFG3_THRESHOLDS = {"active50": 3.959644988918793e-05, "active25": 0.00010181517217181817}
CFG3_THIN_START = 20
CFG3_PERIOD = 10


def make_psf(name: str):
    return {"line15": lambda: makeLinePsf(15), "line31": lambda: makeLinePsf(31),
            "box15x15": lambda: makeBoxPsf(15, 15), "disc10": disc_r10, "oblique21": oblique_line,
            "gauss31": gaussian31}[name]()


def make_input(cfg: Config, width: int = None, height: int = None, image: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    """(g, f) for one image of a config (optionally at a reduced size, same
    seed / counts scaled by area so the scene density stays the same)."""
    w = width or cfg.width
    h = height or cfg.height
    scale = (w * h) / float(cfg.width * cfg.height)
    n_rect = max(1, int(round(cfg.n_rect * scale))) if scale < 1 else cfg.n_rect
    n_disk = max(1, int(round(cfg.n_disk * scale))) if scale < 1 else cfg.n_disk
    seed = cfg.seed + image
    rng = np.random.Generator(np.random.PCG64(seed))
    g = scene(w, h, seed, n_rect, n_disk, rng)
    f = observe(g, make_psf(cfg.psf), cfg.sigma, rng)
    return g, f


def psnr(u: np.ndarray, g: np.ndarray) -> float:
    """PSNR with peak 1 (images live in [0, ~1.05]): 10 log10(1 / MSE)."""
    mse = float(np.mean((np.asarray(u, np.float64) - np.asarray(g, np.float64)) ** 2))
    return float("inf") if mse == 0 else 10.0 * math.log10(1.0 / mse)


def max_rel(a: np.ndarray, ref: np.ndarray) -> float:
    """max |a - ref| / |ref| (ref > 0 on these inputs)."""
    a = np.asarray(a, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.max(np.abs(a - ref) / np.maximum(np.abs(ref), 1e-30)))
