"""bench.py's multi-rank launcher: `--gpus N` without torchrun starts N ranks
itself (torch.distributed.run on 127.0.0.1) and reports n_gpus = N; with
fewer visible GPUs than N it refuses (unless --share-gpu)."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _run(*args, timeout=900):
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                          timeout=timeout, cwd=ROOT)


def test_bench_refuses_missing_gpus():
    r = _run("--gpus", "64", "--steps", "1", "--warmup", "3", timeout=300)
    assert r.returncode != 0 and "needs 64 visible GPUs" in (r.stderr + r.stdout)


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["ipc", "host"])
def test_bench_self_launch_two_ranks(transport):
    r = _run("--gpus", "2", "--share-gpu", "--transport", transport, "--steps", "3", "--warmup", "3",
             "--e2e-steps", "0")
    assert r.returncode == 0, r.stderr[-3000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    out = json.loads(line)
    assert out["n_gpus"] == 2 and out["value"] > 0 and out["gpu_launches"] > 0
    assert out["config"]["transport"] == transport and out["scaling"] == "weak"
