"""bench.py contract checks that need no GPU: the reference arm (the
reference's own CPU implementation, oracle/_ref) prints one JSON line with
the driver's keys, and --help / argument parsing work."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libfdref.so")


@pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built (needs /root/reference)")
def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "cfg0", "--steps", "1",
                          "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "scaling", "vs_baseline",
              "dtype", "config", "impl", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["config"]["workload"] == "cfg0"
    import importlib
    sys.path.insert(0, ROOT)
    assert tuple(line["config"]) == importlib.import_module("bench").WORKLOAD_KEYS
    assert line["cpu_baseline"]["nproc"] >= 1 and line["cpu_baseline"]["cpu_model"]
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0


def test_bench_help():
    out = subprocess.run([sys.executable, "bench.py", "--help"], cwd=ROOT, capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and "--impl" in out.stdout and "--gpus" in out.stdout


def test_gpus_flag_launches_ranks():
    """`bench.py --gpus 2` re-launches itself under torch.distributed.run with
    2 ranks (the driver's own launch); --dry-run shows each rank's shard."""
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run"], cwd=ROOT, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and [s["rank"] for s in line["shards"]] == [0, 1]
    assert line["shards"][0]["rows"] == [0, 8192] and line["shards"][1]["rows"] == [8192, 16384]
    assert line["shards"][0]["halo"] == 14  # fused strips: 2 x the 7-row PSF radius
    assert line["halo_bytes_per_iteration"] == 2 * 14 * 16384 * 4
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "4", "--dry-run", "--config", "cfg4b"], cwd=ROOT,
                         capture_output=True, text=True, timeout=300)
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert [s["images"] for s in line["shards"]] == [[0, 16], [16, 32], [32, 48], [48, 64]]


def test_config_keys_identical_in_both_arms():
    import importlib
    sys.path.insert(0, ROOT)
    bench = importlib.import_module("bench")
    from paper_1304_7211_b200 import workloads as W
    c = bench.workload_config(W.CONFIGS["cfg4"])
    assert tuple(c) == bench.WORKLOAD_KEYS


@pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built (needs /root/reference)")
def test_cpu_baseline_single_core_pinned():
    import importlib
    sys.path.insert(0, ROOT)
    bench = importlib.import_module("bench")
    from paper_1304_7211_b200 import workloads as W
    core = sorted(os.sched_getaffinity(0))[0]
    before = os.sched_getaffinity(0)
    v, sample = bench.ref_rate(W.CONFIGS["cfg0"], "box1d-cumul", 1, budget_s=0.2, pin_core=core)
    assert v > 0 and f"pinned to core {core}" in sample
    assert os.sched_getaffinity(0) == before  # restored
