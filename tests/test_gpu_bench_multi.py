"""bench.py's N>1 paths end to end on one GPU (BS_RING_SAME_GPU=1: every rank on cuda:0,
time-sliced -- a functional check, the numbers mean nothing): `--gpus 2` self-launches two
ranks under torch.distributed.run, runs the C2 ring with the fused cross-GPU exchange and
the C3 sequence split as the headline, and rank 0 prints one JSON line with n_gpus 2 and no
NVLink roofline (no byte crossed NVLink)."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("config", ["c2", "c3"])
def test_bench_two_ranks_same_gpu(config):
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["BS_RING_SAME_GPU"] = "1"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
                        "--warmup", "3", "--no-cpu-baseline", "--config", config],
                       capture_output=True, text=True, timeout=1200, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    res = json.loads(lines[0])
    assert res["n_gpus"] == 2 and res["value"] > 0 and res["gpu_launches"] > 0
    assert res.get("roofline_migrate") is None   # same GPU: nothing crossed NVLink
    assert "ALL RANKS ON ONE GPU" in json.dumps(res["config"])   # labelled functional check
