"""Single-GPU measurement of the sharded schedule (fdg_shard_group_*):
`world` row strips of a cfg4-sized image run in one process with the
production row ranges and kernels; per strip, device time of the interior
launch, the boundary-band launch and the (emulated, device-copy) halo
exchange, against the whole-image fused iteration.

usage: python scripts/shard_probe.py [world] [iterations] [size]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1304_7211_b200 import OperatorKind as K, RlConfig, RlSolver  # noqa: E402
from paper_1304_7211_b200.psf import makeBoxPsf  # noqa: E402
from paper_1304_7211_b200.sharded import ShardGroup  # noqa: E402

world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
n = int(sys.argv[3]) if len(sys.argv) > 3 else 16384
psf = makeBoxPsf(15, 15)
cfg = RlConfig(iterations=iters, op=K.Box2dSliding)
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
f = torch.rand((n, n), device=dev, generator=g) * 0.8 + 0.2
u = torch.empty_like(f)

# whole image, same iterations (graph-replayed solver)
solver = RlSolver(psf, cfg, n, n)
st = torch.cuda.current_stream(dev)
solver.use_stream(st.cuda_stream)
solver.run(f, u)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
solver.run(f, u)
e1.record(st)
torch.cuda.synchronize()
whole_ms = e0.elapsed_time(e1) / iters

grp = ShardGroup(psf, cfg, n, n, world)
grp.ctx.set_stream(st.cuda_stream)
grp.run(f, u)
torch.cuda.synchronize()
e0.record(st)
grp.run(f, u)
e1.record(st)
torch.cuda.synchronize()
group_ms = e0.elapsed_time(e1) / iters
rows = []
for r in range(world):
    t = grp.timing(r)
    info = grp.infos[r]
    rows.append({"rank": r, "core": info["core"], "halo": info["halo"],
                 "interior_us": 1e3 * t["interior_ms"] / iters, "bands_us": 1e3 * t["bands_ms"] / iters,
                 "exchange_us": 1e3 * t["exchange_ms"] / max(iters - 1, 1),
                 "halo_bytes_per_iteration": info["halo_bytes_per_iteration"]})
mid = rows[world // 2]

# one rank of `world` alone with the production multi-stream schedule
# (loopback exchange of its own edge rows): its per-iteration device time
# is what each GPU of a world-GPU run spends, minus NVLink
from paper_1304_7211_b200._lib import lib  # noqa: E402
from paper_1304_7211_b200.sharded import ShardedRl  # noqa: E402

lib().fdg_set_option(b"shard_loopback", 1)
rank = world // 2
lib().fdg_set_option(b"shard_bands", int(os.environ.get("BANDS", "0")))
sh = ShardedRl(psf, cfg, n, n, rank, world)
sh.ctx.set_stream(st.cuda_stream)
core = sh.info["core"]
fs = f[:core].contiguous()
us = torch.empty_like(fs)
sh.run(fs, us)
torch.cuda.synchronize()
e0.record(st)
sh.run(fs, us)
e1.record(st)
torch.cuda.synchronize()
rank_ms = e0.elapsed_time(e1) / iters
t = sh.timing()
loop = {"rank": rank, "us_per_iteration": 1e3 * rank_ms, "interior_us": 1e3 * t["interior_ms"] / iters,
        "bands_us": 1e3 * t["bands_ms"] / iters, "exchange_us": 1e3 * t["exchange_ms"] / max(iters - 1, 1),
        "parallel_efficiency_model": whole_ms / (world * rank_ms)}
out = {"world": world, "size": n, "iterations": iters, "whole_image_us_per_iteration": 1e3 * whole_ms,
       "group_us_per_iteration_all_strips_serial": 1e3 * group_ms,
       "ideal_strip_us": 1e3 * whole_ms / world,
       "interior_strip": mid,
       "one_rank_loopback": loop,
       "band_plus_exchange_over_interior": (mid["bands_us"] + mid["exchange_us"]) / max(mid["interior_us"], 1e-9),
       "band_over_interior": mid["bands_us"] / max(mid["interior_us"], 1e-9),
       "strips": rows}
print(json.dumps(out, indent=1))
