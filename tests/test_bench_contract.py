"""bench.py's driver contract: the JSON line's keys (GPU), and the launcher's refusal to time fewer
GPUs than --gpus asks for (CPU: no GPU in the container, so --gpus 2 must fail loudly)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None, timeout=600):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=timeout)


def test_gpus_mismatch_with_launcher_fails_loudly():
    """Under a launcher (WORLD_SIZE set) that started fewer ranks than --gpus, no line is printed."""
    r = _run(["--gpus", "2", "--steps", "1"], {"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"}, timeout=300)
    assert r.returncode != 0
    assert "WORLD_SIZE" in (r.stderr + r.stdout)
    assert '"value"' not in r.stdout


def test_gpus_beyond_the_node_fails_loudly():
    """Without a launcher, --gpus N spawns N ranks, and refuses when the node has fewer GPUs."""
    torch = pytest.importorskip("torch")
    if torch.cuda.device_count() >= 64:
        pytest.skip("node with 64 GPUs")
    r = _run(["--gpus", "64", "--steps", "1"], timeout=300)
    assert r.returncode != 0
    assert "GPU" in (r.stderr + r.stdout)
    assert '"value"' not in r.stdout


@pytest.mark.gpu
def test_bench_line_has_the_contract_keys():
    r = _run(["--steps", "2", "--warmup", "3", "--no-cpu-baseline"])
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks", "gpu_launches"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["steps"] == 2 and line["warmup"] >= 3
    assert line["value"] > 0 and line["gpu_launches"] > 0
    assert "workload" in line["config"]
    roof = line["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in roof, k
    assert 0 < roof["frac"] <= 1.0
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in line["clocks"] and "reasons" in line["clocks"]
