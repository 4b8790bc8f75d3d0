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


@pytest.mark.gpu
@pytest.mark.slow
def test_bench_line_contract():
    """The default bench line carries every key the driver and the judge read:
    metric/value/unit, timing fields, roofline (bound, achieved, peak, unit,
    frac, traffic), cpu_baseline (value, unit, cores, kind, sample), e2e (value,
    unit, h2d/d2h bytes), gpu_launches, clocks."""
    r = _run("--steps", "5", "--warmup", "3", "--e2e-steps", "1", "--no-parity", timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in out, k
    assert out["n_gpus"] == 1 and out["steps"] == 5 and out["value"] > 1e10 and out["gpu_launches"] == 10
    rl = out["roofline"]
    assert rl["bound"] == "hbm" and rl["unit"] == "GB/s" and 0 < rl["frac"] < 1.5
    assert abs(rl["frac"] - rl["achieved"] / rl["peak"]) < 1e-3
    cb = out["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] > 0 and "sample" in cb
    e2e = out["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] == 2 * 512 ** 3 * 4 and e2e["d2h_bytes_per_step"] == 512 ** 3 * 4
    assert "sm_mhz" in out["clocks"] and "reasons" in out["clocks"]
    assert out["fp32_roofline"]["frac"] > 0
