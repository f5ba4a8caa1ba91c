"""Phase breakdown of the host-buffer API (FDG_PROFILE=1: per-phase ms from
inside fdg_rl_deconvolve) for small configs.  usage: e2e_probe2.py cfg1 [cfg2 ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FDG_PROFILE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1304_7211_b200 import OperatorKind as K, RlConfig, rlDeconvolve, workloads as W  # noqa: E402
from paper_1304_7211_b200._lib import Context  # noqa: E402

OPS = {"box1d-sliding": K.Box1dSliding, "box2d-sliding": K.Box2dSliding, "generic-box": K.GenericBox,
       "naive": K.Naive}
for name in sys.argv[1:]:
    cfg = W.CONFIGS[name]
    psf = W.make_psf(cfg.psf)
    _, f = W.make_input(cfg)
    fp = torch.from_numpy(np.ascontiguousarray(f, dtype=np.float32)).pin_memory().numpy()
    ctx = Context(0)
    rc = RlConfig(iterations=cfg.iterations, op=OPS[cfg.op])
    for rep in range(3):
        t = time.perf_counter()
        r = rlDeconvolve(fp, psf, rc, ctx=ctx)
        print(name, rep, f"{(time.perf_counter() - t) * 1e3:.2f} ms", flush=True)
