"""bench.py's JSON-line contract (the driver parses it): one line with every required key, on a small
configuration, for both arms and the training workload.  GPU (the reference arm runs on the host but
the test is grouped with the bench)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         cwd=ROOT, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_has_the_contract_keys():
    d = run("--config", "0", "--steps", "3", "--warmup", "3", "--cpu-seconds", "1")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["config"]["workload"].startswith("cfg0")
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in d["cpu_baseline"], k
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["clocks"] and "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert d["gpu_launches"] > 0


def test_training_workload_line():
    d = run("--workload", "train", "--config", "0", "--steps", "2", "--warmup", "1", "--iters", "3", "--train-T", "200",
            "--cpu-seconds", "1")
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["config"]["workload"] == "train-cfg0"


def test_gathered_block_and_gpus_beyond_the_node_fail_loudly():
    import torch
    d = run("--config", "0", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--no-bound-off")
    g = d["gathered"]
    assert g["mixtures"] == 1 and len(g["rank_ms"]) == 1 and len(g["d_hat_digest"]) == 16
    n = torch.cuda.device_count() + 1      # more ranks than GPUs: every rank refuses, the launch fails
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--config", "0",
                          "--steps", "3", "--warmup", "3"], capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert out.returncode != 0 and "visible GPUs" in out.stderr + out.stdout
