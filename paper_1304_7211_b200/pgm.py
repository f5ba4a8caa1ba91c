"""PGM image I/O (pgm.hpp) and image metrics (image.hpp snrDb) for the CLI
callers of the GPU path.  Host-side file plumbing, no device work.

Semantics follow the reference:
* ``readPgm`` (pgm.hpp:63-110): binary P5 or ASCII P2, maxval <= 255, '#'
  comments in the header, exactly one whitespace byte after maxval for P5;
  errors are ``PgmParseError`` naming the byte offset.
* ``writePgm`` (pgm.hpp:114-130): P5, maxval 255, each pixel rounded half away
  from zero (``std::lround``) and clamped to [0, 255]; non-finite pixels and
  empty images raise ``ValueError`` (std::invalid_argument).
* ``snrDb`` (image.hpp:149-167): 10 log10(sum r^2 / sum (r - t)^2), +inf for
  identical images.
"""
import math
from typing import Union

import numpy as np

__all__ = ["PgmParseError", "readPgm", "writePgm", "readPgmFile", "writePgmFile", "snrDb"]


class PgmParseError(RuntimeError):
    """Malformed PGM input; the message names the byte offset (pgm.hpp:13-16)."""


class _Cursor:
    def __init__(self, data: bytes):
        self.b = data
        self.pos = 0

    def at_end(self) -> bool:
        return self.pos >= len(self.b)

    def peek(self) -> int:
        return self.b[self.pos]

    @staticmethod
    def is_space(c: int) -> bool:
        return c in (0x20, 0x09, 0x0D, 0x0A, 0x0B, 0x0C)

    def skip_space_and_comments(self):
        while not self.at_end():
            c = self.peek()
            if self.is_space(c):
                self.pos += 1
            elif c == ord("#"):
                while not self.at_end() and self.peek() != ord("\n"):
                    self.pos += 1
            else:
                break

    def parse_uint(self, what: str) -> int:
        self.skip_space_and_comments()
        if self.at_end():
            raise PgmParseError(f"PGM: unexpected end of input at byte {self.pos} while reading {what}")
        if not (ord("0") <= self.peek() <= ord("9")):
            raise PgmParseError(f"PGM: expected {what} at byte {self.pos}")
        v = 0
        while not self.at_end() and ord("0") <= self.peek() <= ord("9"):
            v = v * 10 + (self.peek() - ord("0"))
            self.pos += 1
            if v > 1000000000:
                raise PgmParseError(f"PGM: {what} out of range at byte {self.pos}")
        return v


def readPgm(data: Union[bytes, bytearray]) -> np.ndarray:
    """Image (H x W float64) from PGM bytes."""
    data = bytes(data)
    if len(data) < 2 or data[0] != ord("P") or data[1] not in (ord("2"), ord("5")):
        raise PgmParseError("PGM: expected magic 'P2' or 'P5' at byte 0")
    binary = data[1] == ord("5")
    cur = _Cursor(data)
    cur.pos = 2
    width = cur.parse_uint("width")
    height = cur.parse_uint("height")
    maxval = cur.parse_uint("maxval")
    if width < 1 or height < 1:
        raise PgmParseError(f"PGM: dimensions must be positive (at byte {cur.pos})")
    if maxval < 1 or maxval > 255:
        raise PgmParseError(f"PGM: unsupported maxval {maxval} at byte {cur.pos} (expected <= 255)")
    count = width * height
    if binary:
        if cur.at_end() or not _Cursor.is_space(cur.peek()):
            raise PgmParseError(f"PGM: expected single whitespace after maxval at byte {cur.pos}")
        cur.pos += 1
        if len(data) - cur.pos < count:
            raise PgmParseError(f"PGM: truncated pixel data at byte {len(data)} (expected {count} bytes "
                                f"after byte {cur.pos})")
        px = np.frombuffer(data, dtype=np.uint8, count=count, offset=cur.pos).astype(np.float64)
    else:
        px = np.empty(count, dtype=np.float64)
        for i in range(count):
            v = cur.parse_uint("pixel value")
            if v > maxval:
                raise PgmParseError(f"PGM: sample value {v} exceeds maxval at byte {cur.pos}")
            px[i] = v
    return px.reshape(height, width)


def writePgm(img) -> bytes:
    """P5 bytes of an image (rounded half away from zero, clamped to [0, 255])."""
    a = np.asarray(img, dtype=np.float64)
    if a.ndim != 2 or a.size == 0:
        raise ValueError("writePgm: empty image")
    if not np.all(np.isfinite(a)):
        raise ValueError("writePgm: non-finite pixel value")
    q = np.clip(np.sign(a) * np.floor(np.abs(a) + 0.5), 0, 255).astype(np.uint8)  # std::lround
    h, w = a.shape
    return f"P5\n{w} {h}\n255\n".encode() + q.tobytes()


def readPgmFile(path: str) -> np.ndarray:
    try:
        with open(path, "rb") as fh:
            data = fh.read()
    except OSError:
        raise RuntimeError(f"cannot open for reading: {path}") from None
    return readPgm(data)


def writePgmFile(path: str, img) -> None:
    data = writePgm(img)
    try:
        with open(path, "wb") as fh:
            fh.write(data)
    except OSError:
        raise RuntimeError(f"cannot open for writing: {path}") from None


def snrDb(reference, test) -> float:
    r = np.asarray(reference, dtype=np.float64)
    t = np.asarray(test, dtype=np.float64)
    if r.shape != t.shape:
        raise ValueError("snrDb: image dimensions differ")
    signal = float(np.sum(r * r))
    error = float(np.sum((r - t) ** 2))
    if signal == 0.0:
        raise ValueError("snrDb: reference image is identically zero")
    if error == 0.0:
        return math.inf
    return 10.0 * math.log10(signal / error)
