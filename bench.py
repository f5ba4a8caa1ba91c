#!/usr/bin/env python
"""Benchmark of the B200 Richardson-Lucy hot path (metric: RL Mpixel-iterations/s).

Default workload: BASELINE config 4 -- one 16384 x 16384 fp32 image (seed 4,
4096 rectangles, 2048 disks), separable 15x15 uniform box, box2d-sliding,
100 RL iterations; row-strip sharded over N GPUs with a 7-row halo exchange
per iteration (torch.distributed / NCCL).  `--config cfg4b` runs the batch
of 64 2048^2 images (1x31 box, sharded by image); cfg0..cfg3 are accepted
for diagnostics.

A "step" is one full RL deconvolution (all iterations) of the workload.
value : px*it of all ranks / max-over-ranks device time, inputs resident in HBM
e2e   : the same through the public host API (rlDeconvolve on host arrays;
        H2D of f and D2H of u inside every step), N = 1 path per rank
--impl reference : the reference CPU implementation (oracle/_ref, compiled
        from the unmodified reference headers) on this host's cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

B_PER_PXIT = 24  # algorithmic HBM bytes per px*it (2 passes x (2 reads + 1 write) x fp32)


# FP32 FMA throughput measured on this pool's B200 (scripts/ffma2_probe.cu,
# profiles/r01_ffma2_probe.md): 74.1 TFLOP/s = 148 SMs x 128 lanes x 2 x 1.965 GHz
FP32_TFLOPS_MEASURED = 74.1
DENSE_FLOP_PER_PXIT = 2 * 2 * 961  # two 31x31 correlations, one FMA per tap


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML
    every 10 ms in a thread (an nvidia-smi loop needs ~0.3 s to start and
    missed sub-second runs), plus one sample at start() and at stop()."""

    # NVML clocks-event reason bits
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index=0, period_s=0.01):
        self.index = index
        self.period = period_s
        self.rows = []
        self._stop = threading.Event()
        self._th = None
        self._h = None
        self._max = None

    def _sample(self):
        import pynvml
        try:
            sm = pynvml.nvmlDeviceGetClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            try:
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:
                r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
            self.rows.append((sm, r))
        except Exception:
            pass

    def _loop(self):
        while not self._stop.wait(self.period):
            self._sample()

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self._max = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._sample()
            self._th = threading.Thread(target=self._loop, daemon=True)
            self._th.start()
        except Exception:
            self._h = None

    def stop(self):
        if self._h is not None:
            self._stop.set()
            if self._th:
                self._th.join(1.0)
            self._sample()
        sm = [r[0] for r in self.rows]
        reasons = sorted({name for _, bits in self.rows for b, name in self.REASONS.items() if bits & b})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self._max,
                "reasons": reasons, "samples": len(self.rows), "source": "nvml (10 ms)"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# --------------------------------------------------------------- reference
WORKLOAD_KEYS = ("workload", "width", "height", "batch", "psf", "op", "iterations")


def workload_config(cfg, iterations=None):
    """The `config` object of both arms: the workload only (engine details
    go to `engine_info`), so the driver sees identical configs."""
    return {"workload": cfg.name, "width": cfg.width, "height": cfg.height, "batch": cfg.batch,
            "psf": cfg.psf, "op": cfg.op, "iterations": iterations or cfg.iterations}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# single-core cost of the reference per px*it on the B200 host (r01), by
# reference operator (sizes the bounded samples)
REF_US_PER_PXIT = {"box1d-sliding": 0.011, "box1d-cumul": 0.012, "box2d-sliding": 0.016, "box2d-cumul": 0.014,
                   "generic-box": 0.08, "naive": 1.7}
REF_OPS = {"naive": 0, "list": 1, "generic-box": 2, "box2d-sliding": 3, "box2d-cumul": 4, "box1d-sliding": 5,
           "box1d-cumul": 6}
AUTO_OP = {"line15": "box1d-cumul", "line31": "box1d-cumul", "box15x15": "box2d-cumul", "disc10": "generic-box",
           "oblique21": "generic-box", "gauss31": "naive"}  # dispatch(Auto), convolve.hpp:628-633


def reference_sample(cfg, op_name=None, budget_s=10.0):
    """(rows per strip, iterations): about `budget_s` of single-core
    reference work per thread at the config's width (full-width strips: the
    per-pixel cost is what the metric needs; BASELINE.md 3 times 3-5
    iterations of the long configs)."""
    per_px_it_us = REF_US_PER_PXIT[op_name or cfg.op]
    px_it = budget_s * 1e6 / per_px_it_us
    iters = cfg.iterations
    rows = int(px_it / iters / cfg.width)
    if rows < 32:  # expensive operators / huge rows: fewer iterations instead of thinner strips
        rows = 32
        iters = max(2, int(px_it / rows / cfg.width))
    return min(rows, cfg.height), min(iters, cfg.iterations)


def ref_rate(cfg, op_name, threads, budget_s, pin_core=None):
    """Mpx*it/s of the reference rlDeconvolve(op) on `threads` independent
    full-width strips (one per thread; `pin_core`: the calling thread and
    its strip thread pinned to that core), and the sample description."""
    from oracle import pyoracle as O
    from paper_1304_7211_b200 import workloads as W
    psf = W.make_psf(cfg.psf)
    strip_rows, iters = reference_sample(cfg, op_name, budget_s)
    rows = min(cfg.height, strip_rows + 64)
    _, f = W.make_input(cfg, cfg.width, rows)
    prev = os.sched_getaffinity(0) if pin_core is not None else None
    try:
        if pin_core is not None:
            os.sched_setaffinity(0, {pin_core})
        secs, pxit = O.ref_bench_strips(f.astype(np.float64), psf, REF_OPS[op_name], iters, threads, strip_rows)
    finally:
        if prev is not None:
            os.sched_setaffinity(0, prev)
    sample = (f"reference rlDeconvolve({op_name}) x {threads} independent {strip_rows}x{cfg.width} strips, "
              f"{iters} iterations, {secs:.1f} s" + (f", pinned to core {pin_core}" if pin_core is not None else ""))
    return pxit / secs / 1e6, sample


def run_reference(args, cfg, world, rank):
    """The reference's own CPU implementation of the path (oracle/_ref, the
    unmodified headers) on all host threads of this box, rank 0 only."""
    from oracle import pyoracle as O

    if rank != 0:
        return 0
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libfdref.so not built"}))
        return 0
    threads = len(os.sched_getaffinity(0)) or 1
    vals, sample = [], ""
    for i in range(args.warmup + args.steps):
        v, sample = ref_rate(cfg, cfg.op, threads, budget_s=5.0)
        if i >= args.warmup:
            vals.append(v)
    value = statistics.median(vals)
    sample += f"; host {cpu_model()}, nproc {os.cpu_count()}"
    line = {"metric": "RL Mpixel*iterations/s", "value": value, "unit": "Mpx*it/s", "impl": "reference",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "ms_per_step": None, "scaling": "strong" if cfg.batch == 1 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded BASELINE generator)",
            "config": workload_config(cfg, args.iterations),
            "cpu_baseline": {"value": value, "unit": "Mpx*it/s", "cores": threads, "kind": "reference",
                             "sample": sample, "cpu_model": cpu_model(), "nproc": os.cpu_count()},
            "e2e": {"value": value, "unit": "Mpx*it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def cpu_baseline(cfg):
    """the reference (oracle/_ref) single-threaded as designed,
    pinned to one core, with the config's named operator (the headline
    value) and the Auto-dispatched one; plus all host threads on
    independent strips as a separately labelled aggregate.  ~20 s total."""
    try:
        from oracle import pyoracle as O
        if not O.ref_available():
            return None
        core = sorted(os.sched_getaffinity(0))[-1]
        named, s_named = ref_rate(cfg, cfg.op, 1, budget_s=6.0, pin_core=core)
        auto_op = AUTO_OP[cfg.psf]
        auto, s_auto = ref_rate(cfg, auto_op, 1, budget_s=6.0, pin_core=core)
        threads = len(os.sched_getaffinity(0)) or 1
        agg, s_agg = ref_rate(cfg, cfg.op, threads, budget_s=5.0)
        return {"value": named, "unit": "Mpx*it/s", "cores": 1, "kind": "reference",
                "sample": s_named + " (1 core of " + str(os.cpu_count()) + ")",
                "cpu_model": cpu_model(), "nproc": os.cpu_count(),
                "auto_operator": {"op": auto_op, "value": auto, "cores": 1, "sample": s_auto},
                "all_threads": {"value": agg, "cores": threads, "sample": s_agg}}
    except Exception as e:  # the baseline is reported, never required
        return {"value": None, "error": str(e)}


# ---------------------------------------------------------------- our path
def run_ours(args, cfg, world, rank, local):
    import torch
    import torch.distributed as dist

    from paper_1304_7211_b200 import ConvPlan, RlConfig, RlSolver, OperatorKind as K, rlDeconvolve, workloads as W
    from paper_1304_7211_b200 import sharded as S
    from paper_1304_7211_b200._lib import Context

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    op = {"box1d-sliding": K.Box1dSliding, "box2d-sliding": K.Box2dSliding, "generic-box": K.GenericBox,
          "naive": K.Naive}[cfg.op]
    psf = W.make_psf(cfg.psf)
    iters = args.iterations or cfg.iterations
    rl_cfg = RlConfig(iterations=iters, op=op)
    W_, H_ = cfg.width, cfg.height
    pitch = (W_ + 3) // 4 * 4

    # ---- inputs (built once per rank, then resident in HBM)
    t0 = time.time()
    strips = world > 1 and cfg.batch == 1  # row strips: libfdgpu's sharded runner (NCCL halo exchange)
    shard = None
    if cfg.batch == 1:
        f_full = make_input_gpu(cfg, psf, dev)
        if strips:
            ctx_sh = Context(local)
            ctx_sh.set_stream(torch.cuda.current_stream(dev).cuda_stream)
            shard = S.ShardedRl(psf, rl_cfg, W_, H_, rank, world, S.comm_unique_id(), ctx=ctx_sh)
            r0, core = shard.info["r0"], shard.info["core"]
        else:
            r0, core = 0, H_
        f_dev = torch.zeros((core, pitch), dtype=torch.float32, device=dev)
        f_dev[:, :W_] = f_full[r0:r0 + core]
        f_host = f_full[r0:r0 + core].cpu().numpy() if world == 1 or strips else None
        del f_full
        nimg = 1
        px_local = W_ * core
    else:
        share = S.batch_share(cfg.batch, world, rank)
        nimg = len(share)
        f_dev = torch.stack([make_input_gpu(cfg, psf, dev, image=i) for i in share])
        f_host = f_dev.cpu().numpy() if world == 1 else None
        s = None
        px_local = W_ * H_ * nimg
    setup_s = time.time() - t0
    u_dev = torch.empty_like(f_dev)
    stream = torch.cuda.current_stream(dev)
    if shard is not None:
        solver = None

        def step():  # per iteration: halo exchange (NCCL, comm stream) || interior, then the bands
            shard.run(f_dev, u_dev, iters)

        def launch_count():
            return shard.ctx.launch_count()
    else:
        solver = RlSolver(psf, rl_cfg, W_, H_, batch=nimg, device=local)
        solver.use_stream(stream.cuda_stream)

        def step():  # one process, whole image(s): the C driver loop, replayed as a CUDA graph
            solver.run(f_dev, u_dev, iters)

        def launch_count():
            return solver.launches()

    # ---- warmup
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    # ---- kernel-only timing of the pass loop (roofline "achieved")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    sampler = ClockSampler(local)
    sampler.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    launches0 = launch_count()
    ev[0].record(stream)
    for _ in range(args.steps):
        step()
    ev[1].record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    launches = launch_count() - launches0
    ms_total = ev[0].elapsed_time(ev[1])
    if world > 1:
        t = torch.tensor([ms_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
        n = torch.tensor([launches], device=dev, dtype=torch.float64)
        dist.all_reduce(n)
        launches = int(n.item())
    ms_step = ms_total / args.steps
    total_pxit = W_ * H_ * iters * (cfg.batch if cfg.batch > 1 else 1)
    value = total_pxit / (ms_step * 1e-3) / 1e6

    # dominant-kernel duration: the step is back-to-back launches of one
    # engine (two pass launches per iteration, one fused launch per
    # iteration, or one row-resident launch per run); its average launch time
    # is the step time over the launches (incl. halo exchanges when world > 1)
    # (row strips on several ranks run the two-pass solver passes)
    engine = shard.info["engine"] if shard is not None else solver.engine()
    # launches of the dominant kernel per step (the step also has one tiny
    # start-stamp kernel for the per-iteration trace; sharded runs add the
    # boundary-band launches)
    per_step = {"fused": iters, "rowres": 1}.get(engine, 2 * iters)
    kern_ms = ms_step / per_step
    pxit_per_launch = px_local * iters / per_step
    # algorithmic bytes: SURVEY 8d's canonical 24 B/px*it (two passes x (2
    # reads + 1 write) x fp32) is kept as the denominator for every engine;
    # the fused kernel moves 12 B/px*it, the row-resident one 8 B/px per run
    kbytes = B_PER_PXIT * pxit_per_launch
    peak, peak_kind = peaks()
    achieved = kbytes / (kern_ms * 1e-3) / 1e9
    hbm_bytes = {"fused": 12.0, "rowres": 8.0 / iters}.get(engine, 24.0)
    kernel_desc = {"fused": "k_fused (whole RL iteration per launch, 12 B/px*it through HBM)",
                   "rowres": "k_rowres (all iterations per launch, rows resident in shared memory)",
                   "box": "k_rect (fused conv + RL epilogue, 12 B/px per pass launch)"}.get(
        engine, f"k_{engine} (fused conv pass, 12 B/px per pass launch)")
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(cfg.name)
        except Exception:
            traffic = None

    # the dense 31x31 engine (cfg3) is FP32-FMA bound: its roofline is FLOP/s
    roof = None
    if engine == "dense":
        # one correlation per launch: pxit_per_launch is half an iteration's px*it
        tf = DENSE_FLOP_PER_PXIT * pxit_per_launch / (kern_ms * 1e-3) / 1e12
        roof = {"bound": "fp32", "achieved": tf, "peak": FP32_TFLOPS_MEASURED, "unit": "TFLOP/s",
                "frac": tf / FP32_TFLOPS_MEASURED, "traffic": traffic,
                "peak_kind": "measured FFMA throughput (profiles/r01_ffma2_probe.md)",
                "kernel": "k_dense (31x31 correlation + RL epilogue, 2*961 FLOP/px per launch)",
                "engine": engine, "kernel_ms": kern_ms, "launches_per_step": per_step,
                "algorithmic_flop_per_launch": DENSE_FLOP_PER_PXIT * pxit_per_launch,
                "hbm_frac_canonical": achieved / peak}

    # ---- e2e through the public host API (rank-local, N = 1 semantics per rank)
    e2e = None
    if cfg.batch == 1 and world == 1:
        f_pinned = torch.from_numpy(f_host).pin_memory().numpy()
        u_pinned = torch.empty(f_host.shape, dtype=torch.float32).pin_memory().numpy()  # the result lands here
        ctx = Context(local)
        for _ in range(max(2, min(args.warmup, 3))):  # warm: allocations, solver, captured graph, first replay
            rlDeconvolve(f_pinned, psf, rl_cfg, ctx=ctx, out=u_pinned)
        e_t = []
        for _ in range(max(1, min(args.steps, 3))):
            torch.cuda.synchronize(dev)
            a = time.perf_counter()
            res = rlDeconvolve(f_pinned, psf, rl_cfg, ctx=ctx, out=u_pinned)
            e_t.append(time.perf_counter() - a)
        e2e_s = statistics.median(e_t)
        e2e = {"value": W_ * H_ * iters / e2e_s / 1e6, "unit": "Mpx*it/s", "h2d_bytes_per_step": int(f_host.nbytes),
               "d2h_bytes_per_step": int(res.image.nbytes),
               "api": "paper_1304_7211_b200.rlDeconvolve (C ABI fdg_rl_deconvolve, page-locked host buffers in and out)"}
        ns = ctx.last_schedule()
        e2e["schedule"] = (f"time-skewed pipeline over {ns} row strips (uploads / downloads overlap the iterations)"
                           if ns else "upload, iterate, download")
    elif shard is not None:
        # this rank's strip through the sharded entry point with host buffers
        # (H2D of its f rows, D2H of its u rows every step); max over ranks
        f_pinned = torch.from_numpy(f_host).pin_memory().numpy()
        u_pinned = torch.empty(f_host.shape, dtype=torch.float32).pin_memory().numpy()
        for _ in range(2):
            shard.run(f_pinned, u_pinned, iters)
        e_t = []
        for _ in range(max(1, min(args.steps, 3))):
            dist.barrier()
            a = time.perf_counter()
            shard.run(f_pinned, u_pinned, iters)
            e_t.append(time.perf_counter() - a)
        tt = torch.tensor([statistics.median(e_t)], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        hb = torch.tensor([float(f_host.nbytes)], device=dev, dtype=torch.float64)
        dist.all_reduce(hb)
        e2e = {"value": W_ * H_ * iters / float(tt.item()) / 1e6, "unit": "Mpx*it/s",
               "h2d_bytes_per_step": int(hb.item()), "d2h_bytes_per_step": int(hb.item()),
               "api": "paper_1304_7211_b200.sharded.ShardedRl.run (C ABI fdg_shard_run, host buffers), max over ranks"}
    elif world == 1:
        # batch: per-image host API calls (pinned inputs), all images each step
        from paper_1304_7211_b200 import rlDeconvolveBatch
        ctx = Context(local)
        f_pinned = torch.from_numpy(f_host).pin_memory().numpy()
        u_pinned = torch.empty(f_host.shape, dtype=torch.float32).pin_memory().numpy()
        for _ in range(2):  # warm: the batched solver, streams and planes
            rlDeconvolveBatch(f_pinned, psf, rl_cfg, ctx=ctx, out=u_pinned)
        e_t = []
        for _ in range(max(1, min(args.steps, 3))):
            torch.cuda.synchronize(dev)
            a = time.perf_counter()
            res = rlDeconvolveBatch(f_pinned, psf, rl_cfg, ctx=ctx, out=u_pinned)
            e_t.append(time.perf_counter() - a)
        e2e_s = statistics.median(e_t)
        e2e = {"value": W_ * H_ * iters * f_host.shape[0] / e2e_s / 1e6, "unit": "Mpx*it/s",
               "h2d_bytes_per_step": int(f_host.nbytes), "d2h_bytes_per_step": int(res.image.nbytes),
               "api": "paper_1304_7211_b200.rlDeconvolveBatch (C ABI fdg_rl_deconvolve_batch, page-locked host "
                      "buffers; uploads / downloads of neighbouring chunks overlap the iterations)"}

    # ---- CPU baseline (rank 0, N = 1 only; bounded sample)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg)

    if rank == 0:
        line = {
            "metric": "RL Mpixel*iterations/s", "value": value, "unit": "Mpx*it/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if cfg.batch == 1 else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded BASELINE generator)",
            "config": workload_config(cfg, iters),
            "engine_info": {"engine": engine,
                            "parallelism": f"rowstrip{world}" if cfg.batch == 1 else f"image-shard{world}",
                            "l2": "working set 3 planes >> 126 MB L2 (no flush needed)" if W_ * H_ * 12 * nimg > 4e8
                            else "working set L2-resident (no flush: the RL loop re-reads its own planes)",
                            "setup_s": round(setup_s, 2)},
            "sharding": ({"kind": "row strips, NCCL send/recv halo exchange on a comm stream overlapping the "
                                  "strip interior (libfdgpu fdg_shard_run)",
                          "halo_rows": shard.info["halo"],
                          "exchanges_per_iteration": shard.info["exchanges_per_iteration"],
                          "halo_bytes_per_iteration_rank0": shard.info["halo_bytes_per_iteration"]}
                         if shard is not None else None),
            "per_gpu_value": value / world,
            "roofline": roof if roof else {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": kernel_desc, "engine": engine, "kernel_ms": kern_ms,
                         "launches_per_step": per_step,
                         "algorithmic_bytes_per_launch": kbytes,
                         "model": "canonical 24 B/px*it (SURVEY 8d)",
                         "engine_hbm_bytes_per_pxit": hbm_bytes},
            "hbm_roofline_mpxit": peak * 1e9 / B_PER_PXIT / 1e6 * world,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def make_input_gpu(cfg, psf, dev, image=0):
    """The workloads.make_input observation built on the device: the seeded
    scene is painted on the host, the replicate blur runs on the device (fp32,
    Auto operator) and the N(0, sigma^2) noise comes from a seeded torch
    generator on the device (the float64 CPU path takes ~45 s and ~10 GB of
    host memory at 16384^2; every rank builds the same image).  Returns the
    observation as a (H, W) float32 CUDA tensor."""
    import torch
    from paper_1304_7211_b200 import ConvPlan, workloads as W
    from paper_1304_7211_b200._lib import Context
    seed = cfg.seed + image
    rng = np.random.Generator(np.random.PCG64(seed))
    g = W.scene(cfg.width, cfg.height, seed, cfg.n_rect, cfg.n_disk, rng)
    gd = torch.from_numpy(g.astype(np.float32)).to(dev)
    del g
    bd = torch.empty_like(gd)
    ctx = Context(dev.index)
    ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
    plan = ConvPlan(psf, ctx=ctx)
    plan.apply_device(gd.data_ptr(), bd.data_ptr(), cfg.width, cfg.height, cfg.width)
    del gd
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    noise = torch.randn(bd.shape, generator=gen, device=dev, dtype=torch.float32) * cfg.sigma
    f = torch.clamp_min(bd + noise, 1e-6)
    torch.cuda.synchronize(dev)
    return f


def run_thinned(args, cfg, world, rank, local):
    """Thinned (selective) RL on config 3: the free-running
    GPU masks (rl.hpp:187-257 with deactivation held off for iterations
    < 20, reactivation every 10), thresholds calibrated to ~50 % / ~25 %
    active (profiles/r01_cfg3_thresholds.json).  Headline = effective rate
    (full-image px x iterations / device loop time); also the active-pixel
    rate and the unthinned rate of the same input on the same GPU."""
    import numpy as np
    import torch

    from paper_1304_7211_b200 import OperatorKind as K, RlConfig, rlDeconvolve, rlDeconvolveSelective
    from paper_1304_7211_b200 import workloads as W
    from paper_1304_7211_b200._lib import Context

    if world > 1:
        if rank == 0:
            print(json.dumps({"metric": "RL Mpixel*iterations/s", "unavailable":
                              "thinned config 3 is a single-image replica (SURVEY 8e)"}))
        return 0
    torch.cuda.set_device(local)
    thr = W.CFG3_THRESHOLDS[args.thin]
    iters = args.iterations or cfg.iterations
    psf = W.make_psf(cfg.psf)
    _, f = W.make_input(cfg)
    ctx = Context(local)
    rc = RlConfig(iterations=iters, op=K.Naive)
    for _ in range(args.warmup):
        rlDeconvolveSelective(f, psf, RlConfig(iterations=min(iters, 25), op=K.Naive), thr, 10, thin_start=20,
                              ctx=ctx)
    loops, walls, act = [], [], None
    sampler = ClockSampler(local)
    sampler.start()
    launches0 = ctx.launch_count()
    for _ in range(args.steps):
        a = time.perf_counter()
        r = rlDeconvolveSelective(f, psf, rc, thr, 10, thin_start=20, ctx=ctx)
        walls.append(time.perf_counter() - a)
        loops.append(r.trace.totalSeconds())
        inact = np.array([x.inactiveFraction for x in r.trace.records])
        act = float(1 - inact[20:].mean()) if iters > 20 else 1.0
    clocks = sampler.stop()
    launches = ctx.launch_count() - launches0
    loop_s = statistics.median(loops)
    un = [rlDeconvolve(f, psf, rc, ctx=ctx).trace.totalSeconds() for _ in range(2)]
    un_s = min(un)
    pxit = cfg.width * cfg.height * iters
    value = pxit / loop_s / 1e6
    # FLOP actually needed: full 2 x 961 FMA for the unthinned iterations, the
    # active fraction of it afterwards (3844 a FLOP per px*it)
    a_mean = (min(iters, 20) + max(0, iters - 20) * act) / iters
    tf = DENSE_FLOP_PER_PXIT * a_mean * pxit / loop_s / 1e12
    line = {"metric": "RL Mpixel*iterations/s (effective, thinned)", "value": value, "unit": "Mpx*it/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": loop_s * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded BASELINE generator)",
            "config": dict(workload_config(cfg, iters), workload=f"cfg3-{args.thin}"),
            "engine_info": {"op": "naive (masked dense)", "threshold": thr, "period": 10, "thin_start": 20,
                            "masks": "free-running on the GPU", "engine": "dense (masked)"},
            "active_fraction_it21_on": act, "active_px_rate_mpxit": value * a_mean,
            "unthinned_value": pxit / un_s / 1e6, "speedup_vs_unthinned": un_s / loop_s,
            "roofline": {"bound": "fp32", "achieved": tf, "peak": FP32_TFLOPS_MEASURED, "unit": "TFLOP/s",
                         "frac": tf / FP32_TFLOPS_MEASURED, "traffic": None,
                         "kernel": "k_dense (masked: compacted active 4x4 blocks per 64x64 tile)",
                         "model": "3844 x active fraction FLOP per px*it (SURVEY 8d)"},
            "e2e": {"value": pxit / statistics.median(walls) / 1e6, "unit": "Mpx*it/s",
                    "h2d_bytes_per_step": int(f.nbytes), "d2h_bytes_per_step": int(f.nbytes),
                    "api": "paper_1304_7211_b200.rlDeconvolveSelective (host buffers)"},
            "cpu_baseline": None, "gpu_launches": launches, "clocks": clocks}
    print(json.dumps(line))
    return 0


def run_dry(args, cfg, world, rank):
    """--dry-run: the N-rank plumbing without a GPU (gloo): every rank
    reports its row strip (or image share) and rank 0 prints the table --
    proves that --gpus N starts N ranks with the sharding bench.py uses."""
    import torch.distributed as dist

    from paper_1304_7211_b200 import sharded as S, workloads as W
    if world > 1:
        dist.init_process_group("gloo")
    psf = W.make_psf(cfg.psf)
    if cfg.batch == 1:
        halo = S.fused_halo(psf) if cfg.psf == "box15x15" else S.psf_halo(psf)
        s = S.strip_of(cfg.height, world, rank, halo if world > 1 else 0)
        mine = {"rank": rank, "rows": [s.r0, s.r0 + s.core], "halo": s.halo}
    else:
        sh = S.batch_share(cfg.batch, world, rank)
        mine = {"rank": rank, "images": [sh.start, sh.stop]}
    table = [None] * world
    if world > 1:
        dist.all_gather_object(table, mine)
    else:
        table = [mine]
    if rank == 0:
        halo_bytes = 0
        if cfg.batch == 1 and world > 1:  # per iteration, both directions, all inner edges
            halo_bytes = 2 * (world - 1) * table[0]["halo"] * cfg.width * 4
        print(json.dumps({"dry_run": True, "n_gpus": world, "config": workload_config(cfg, args.iterations),
                          "shards": table, "halo_bytes_per_iteration": halo_bytes}))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def relaunch(n):
    """`bench.py --gpus N` outside torchrun: re-exec under
    torch.distributed.run with N local ranks (the driver's own launch)."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--iterations", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--thin", default=None, choices=["active50", "active25"],
                    help="config 3 thinned (selective RL) at the calibrated active fraction")
    ap.add_argument("--dry-run", action="store_true",
                    help="rank plumbing only (gloo, no GPU): print each rank's shard")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch(args.gpus)
    from paper_1304_7211_b200 import workloads as W
    cfg = W.CONFIGS[args.config]
    world, rank, local = dist_env()
    if args.dry_run:
        return run_dry(args, cfg, world, rank)
    if args.impl == "reference":
        return run_reference(args, cfg, world, rank)
    if args.thin:
        return run_thinned(args, W.CONFIGS["cfg3"], world, rank, local)
    return run_ours(args, cfg, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
