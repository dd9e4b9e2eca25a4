"""bench.py's N-rank code path on a 1-GPU box (the CUDA kernels had never run
inside an N > 1 bench process group).

`bench.py --gpus 2` without a torchrun environment launches 2 ranks itself; with
HYDRA_BENCH_SHARED_GPU=1 both ranks map to the visible GPU and talk over gloo (NCCL refuses two
ranks on one device).  Head sharding has no data-path collective, so the ranks' kernels
never wait on one another; the sequence split stages its all-to-all through host memory under
gloo (dist.py).  Checked: the self-launch, the per-rank shard, the barriers and the max-over-ranks
timing all complete, and rank 0 prints ONE JSON line that says n_gpus = 2, the shard, and that it
is a shared-GPU test line, not a measurement."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*extra, timeout=900):
    env = dict(os.environ, HYDRA_BENCH_SHARED_GPU="1")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3",
                        "--no-cpu-baseline", "--e2e-steps", "1", *extra],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-6000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 only
    return json.loads(lines[0])


def test_head_shard_two_ranks():
    line = _bench("--config", "c2", "--paged-page-size", "0")
    assert line["n_gpus"] == 2 and "shared_gpu_test" in line
    assert line["config"]["parallelism"] == "kv-head shard x2" and line["config"]["heads_per_gpu"] == 16
    assert line["value"] > 0 and line["ms_per_step"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0


def test_seqsplit_two_ranks():
    line = _bench("--config", "c6_seqsplit", "--batch-sweep", "64")
    assert line["n_gpus"] == 2 and "shared_gpu_test" in line
    assert line["config"]["parallelism"] == "prefix sequence split x2"
    assert line["config"]["batch_shard"] == [0, 32]
    assert line["value"] > 0
