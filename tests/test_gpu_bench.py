"""bench.py's contract on a GPU box (-m gpu): the default N = 1 line carries every key the driver
reads, and the N-rank flow (`--gpus 2`: self-launch under torch.distributed.run, config-4 keyframe
sharding, the collectives, max over ranks, one JSON line) runs end to end. This pool's boxes have one
GPU, so the 2-rank run uses gloo with both ranks on cuda:0 (GS_BENCH_BACKEND=gloo); the driver's
multi-GPU run uses NCCL, one GPU per rank."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(args, env=None):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=900, env=dict(os.environ, **(env or {})), cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_default_line_schema():
    d = _line(["--steps", "5", "--warmup", "3", "--no-cpu-baseline"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "clocks", "gpu_launches", "e2e", "roofline"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["value"] > 0 and d["gpu_launches"] == 8   # zero, project, bin_coop, emit, fwd, prologue, bwd tiles, gaussian_bwd
    assert d["config"]["workload"].startswith("config 2")
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    assert d["e2e"]["d2h_bytes_per_step"] >= 14 * 4 * d["config"]["n_gaussians"]


def test_two_rank_sharded_mapping_flow():
    d = _line(["--gpus", "2", "--steps", "2", "--warmup", "1"], env={"GS_BENCH_BACKEND": "gloo"})
    assert d["n_gpus"] == 2 and d["unit"] == "mapping iters/s" and d["scaling"] == "strong"
    assert d["config"]["keyframes"] == 8 and d["config"]["keyframes_per_rank"] == 4
    assert d["value"] > 0 and d["e2e"]["value"] > 0
