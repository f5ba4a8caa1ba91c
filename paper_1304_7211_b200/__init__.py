"""B200-native Richardson-Lucy hot path of arXiv 1304.7211 (fastdeconv).

Python face of the C-ABI library ``libfdgpu.so`` (include/fdgpu.h).  Names
follow the reference API (/root/reference/proj/include/fastdeconv): the PSF
model lives in :mod:`.psf`, operators in :mod:`.convolve`, the RL drivers in
:mod:`.rl`.  There is no CPU fallback: calls that need the device raise
``FdgError`` when the library or a CUDA device is missing.
"""
from .psf import (DensePsf, UniformConvexPsf, SparsePsf, makeLinePsf, makeBoxPsf, makeDiscPsf,
                  makeDiagonalPsf, adjoint, taps_of, toSparse, parseSparsePsf, formatSparsePsf, parsePsfSpec)
from .pgm import PgmParseError, readPgm, writePgm, readPgmFile, writePgmFile, snrDb
from .convolve import (OperatorKind, operatorName, operatorKindFromName, supportsMasking,
                       operatorAcceptsPsf, dispatch, ConvCounters, ConvPlan, convolve, maskedConvolve)
from .rl import (RlConfig, RlIterationRecord, RlTrace, RlResult, rlDeconvolve, rlDeconvolveBatch, rlDeconvolveSelective,
                 rlStep, blurImage, BoundaryMode, RlSolver)
from ._lib import FdgError, lib_path

__all__ = [n for n in dir() if not n.startswith("_")]
