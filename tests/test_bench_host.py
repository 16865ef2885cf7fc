"""Host-side parts of bench.py's contract (no GPU): the reference arm (the oracle on the host cores)
prints the JSON line with the same `config` as our arm, and `--gpus N` outside torchrun re-launches
bench.py under torch.distributed.run with N ranks (127.0.0.1 rendezvous)."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1206_6468_b200 import synth  # noqa: E402


def test_reference_arm_line_and_config_match():
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "0",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, cwd=ROOT, timeout=600,
                         env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["cores"] == min(len(os.sched_getaffinity(0)), synth.config(0).M)
    args = argparse.Namespace(config=0, gpus=1)
    assert d["config"] == bench.config_line(args, synth.config(0), synth.config(0).iters)


def test_reference_arm_other_ranks_exit_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--config", "0", "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                         cwd=ROOT, timeout=300, env=env)
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_gpus_n_relaunches_under_torchrun():
    cmd = bench.relaunch_command(["--gpus", "4", "--steps", "3"], 4, 29512)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29512" in cmd
    assert cmd[-3:] == ["--gpus", "4", "--steps", "3"] or cmd[-4:-1] == ["--gpus", "4", "--steps"]
    assert os.path.basename(cmd[cmd.index("--master-port=29512") + 1]) == "bench.py"


def test_world_size_mismatch_fails_loudly():
    env = dict(os.environ, RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "0"],
                         capture_output=True, text=True, cwd=ROOT, timeout=300, env=env)
    assert out.returncode != 0 and "WORLD_SIZE" in (out.stderr + out.stdout)
