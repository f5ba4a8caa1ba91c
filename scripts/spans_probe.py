"""Spans-engine probe: RL Mpx*it/s of the device loop for a PSF/size pair.
usage: python scripts/spans_probe.py {disc10|oblique21} W H [iters]
(engine variant via FDG_SPANS_TILE etc., read once per process)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1304_7211_b200 import OperatorKind as K, RlConfig, RlSolver, workloads as W  # noqa: E402

psf_name, w, h = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 20
psf = W.make_psf(psf_name)
dev = torch.device("cuda", 0)
pitch = (w + 3) // 4 * 4
g = torch.Generator(device=dev).manual_seed(0)
f = torch.rand((h, pitch), device=dev, generator=g) * 0.8 + 0.2
u = torch.empty_like(f)
solver = RlSolver(psf, RlConfig(iterations=iters, op=K.GenericBox), w, h, batch=1, device=0)
st = torch.cuda.current_stream(dev)
solver.use_stream(st.cuda_stream)
for _ in range(2):
    solver.run(f, u, iters)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
reps = 3
for _ in range(reps):
    solver.run(f, u, iters)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"{psf_name} {w}x{h} {iters} it: {w * h * iters / (ms * 1e-3) / 1e6:.0f} Mpx*it/s "
      f"({ms / (2 * iters) * 1e3:.1f} us/pass) tile={os.environ.get('FDG_SPANS_TILE', '-')}")
