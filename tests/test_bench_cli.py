"""bench.py's launch contract on CPU: --gpus N spawns N ranks through
torch.distributed.run on 127.0.0.1, and refuses (non-zero exit) instead of
printing a smaller-N number when the box has fewer GPUs."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _run(args, env=None):
    e = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, BENCH, *args], capture_output=True, text=True,
                          timeout=300, env=e)


def test_spawn_command():
    p = _run(["--gpus", "4", "--steps", "3", "--dry-run-spawn"])
    assert p.returncode == 0, p.stderr
    cmd = json.loads(p.stdout.strip().splitlines()[-1])["spawn"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[cmd.index(BENCH) + 1:] == ["--gpus", "4", "--steps", "3", "--dry-run-spawn"]


@pytest.mark.skipif(__import__("torch").cuda.device_count() >= 2, reason="box has >= 2 GPUs")
def test_more_gpus_than_devices_is_an_error():
    p = _run(["--gpus", "2", "--steps", "1", "--warmup", "3"])
    assert p.returncode != 0
    assert "CUDA devices" in p.stderr
    assert '"metric"' not in p.stdout


@pytest.mark.skipif(__import__("torch").cuda.device_count() >= 2, reason="box has >= 2 GPUs")
def test_torchrun_rank_without_its_gpu_is_an_error():
    env = {"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1", "MASTER_ADDR": "127.0.0.1",
           "MASTER_PORT": "29555"}
    p = _run(["--gpus", "2"], env)
    assert p.returncode != 0 and '"metric"' not in p.stdout


def test_c4_phase_schedule():
    sys.path.insert(0, ROOT)
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", BENCH)
    argv = sys.argv
    sys.argv = ["bench.py"]
    try:
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
    finally:
        sys.argv = argv
    t = mod.c4_phase_targets(5, 20, 5)
    # warm-up: one low / high cycle ending high; timed: 8, 64, 8, 64 (5 steps each)
    assert t == [8] * 2 + [64] * 3 + [8] * 5 + [64] * 5 + [8] * 5 + [64] * 5
    assert mod.c4_phase_targets(2, 4, 2) == [64] * 2 + [8] * 2 + [64] * 2
    assert mod.WL is mod.WORKLOADS["c4"]


@pytest.mark.gpu
def test_bench_line_contract():
    """One short c4 run prints ONE JSON line with the contract's keys: the
    BASELINE metric, device value, roofline (with ncu traffic), e2e through
    host buffers with its copy bytes, clocks, our own kernel launches, and
    the CPU baseline."""
    p = _run(["--steps", "4", "--warmup", "3", "--phase-steps", "2", "--no-sweep", "--no-c3"])
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert d["metric"] == "slab paged-decode attention HBM GB/s" and d["unit"] == "GB/s"
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["warmup"] == 3 and d["higher_is_better"]
    assert d["config"]["workload"].startswith("c4")
    assert d["value"] > 0 and d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] <= 1.2 and r["peak"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["value"] < d["value"] * 1.05  # through PCIe: not faster than the device leg
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    cb = d["cpu_baseline"]
    assert cb["value"] > 0 and cb["kind"] == "port" and cb["cores"] >= 1
    assert base  # BASELINE.json readable next to the bench
