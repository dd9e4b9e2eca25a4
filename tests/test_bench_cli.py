"""bench.py's multi-GPU launch contract (`--gpus 8` without torchrun silently
measured 1 GPU): without a torchrun environment, --gpus N > 1 launches N ranks itself, and
fails loudly -- a JSON error line and a non-zero exit -- when fewer GPUs are visible."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus_beyond_visible_devices_fails_loudly():
    import torch

    n = max(torch.cuda.device_count(), 1)  # ask for one more GPU than visible (>= 2)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", str(n + 1), "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 2, r.stdout + r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert "error" in line and f"--gpus {n + 1}" in line["error"]


def test_world_size_mismatch_is_rejected():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0 and "does not match WORLD_SIZE" in r.stderr


@pytest.mark.parametrize("cfg", ["c4", "c6_seqsplit", "c3_16k"])
def test_configs_exist(cfg):
    sys.path.insert(0, ROOT)
    import bench

    c = bench.CONFIGS[cfg]
    assert c["d"] == 128 and c["Hq"] % c["Hkv"] == 0
