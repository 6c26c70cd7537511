"""bench.py host logic on CPU (-m "not gpu"): the reference arm's JSON line (config 0, whole oracle
iterations), the N-GPU self-launch command, the rank-to-GPU mapping of the gloo test mode and the
default-config rule."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_reference_arm_line_config0():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "0",
                        "--steps", "3", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["steps"] == 3 and d["warmup"] == 1
    assert d["unit"] == "iters/s" and d["value"] > 0 and d["higher_is_better"] is True
    assert abs(d["value"] - 1000.0 / d["ms_per_step"]) <= 1e-9 * d["value"]   # whole iterations, no scaling
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and "no sampling or scaling" in cb["sample"]
    assert set(cb["stage_s"]) == {"forward", "loss_l1", "backward"}
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_relaunch_command(monkeypatch):
    b = _bench()
    seen = {}

    def fake_call(cmd, env):
        seen["cmd"], seen["env"] = cmd, env
        return 0
    monkeypatch.setattr(b.subprocess, "call", fake_call)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "7"])
    args = b.parse()
    assert b.relaunch(args) == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert "--master-addr=127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "4", "--steps", "7"]
    assert seen["env"]["NCCL_DEBUG"] == "INFO" and seen["env"]["NCCL_DEBUG_FILE"] == "/dev/stderr"


def test_dist_env_gloo_maps_ranks_onto_visible_gpus(monkeypatch):
    b = _bench()
    import torch
    monkeypatch.setenv("WORLD_SIZE", "4")
    monkeypatch.setenv("RANK", "3")
    monkeypatch.setenv("LOCAL_RANK", "3")
    monkeypatch.setenv("GS_BENCH_BACKEND", "gloo")
    monkeypatch.setattr(torch.cuda, "device_count", lambda: 1)
    assert b.dist_env() == (4, 3, 0)
    monkeypatch.setenv("GS_BENCH_BACKEND", "nccl")
    assert b.dist_env() == (4, 3, 3)


def test_parse_default_config_is_left_to_the_world_size(monkeypatch):
    b = _bench()
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    a = b.parse()
    assert a.config is None and a.gpus == 1 and a.impl == "ours"
