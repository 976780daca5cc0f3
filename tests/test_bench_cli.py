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
