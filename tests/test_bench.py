"""bench.py keeps the driver's JSON-line contract: a short run of our arm on the GPU and
the reference arm on the host (the latter uses the CPU decoder only)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _line(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _line(["--impl", "reference", "--steps", "1", "--warmup", "1"], timeout=600)
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.gpu
def test_our_arm_line():
    d = _line(["--steps", "1", "--warmup", "3", "--frames", "4000", "--no-cpu-baseline"], timeout=900)
    assert BASE_KEYS <= set(d) and d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 3
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and d["dtype"] == "f32"
    r = d["roofline"]
    assert r["bound"] == "alu" and 0 < r["frac"] < 1 and r["peak"] > 0
    assert "sm_mhz" in d["clocks"] and isinstance(d["clocks"]["reasons"], list)
    assert d["config"]["frames_per_step"] == 7 * 4000


def test_gpus_n_relaunches_one_rank_per_gpu():
    """`bench.py --gpus N` outside torchrun starts N ranks (torch.distributed.run on
    127.0.0.1); the reference arm then runs on rank 0 only and prints one line."""
    sys.path.insert(0, ROOT)
    import bench
    cmd = bench.launch_command(["--gpus", "4", "--steps", "2"], 4, 29555)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[-3:] == ["--gpus", "4", "--steps", "2"][-3:]
    d = _line(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1"], timeout=900)
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0


@pytest.mark.gpu
def test_our_arm_under_torchrun_uses_nccl():
    """One rank launched by torchrun takes the multi-GPU path: NCCL process group, the
    counters all-reduce and the max-over-ranks timing."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr=127.0.0.1", "--master-port=29517", os.path.join(ROOT, "bench.py"), "--gpus", "1",
           "--steps", "1", "--warmup", "3", "--frames", "2000", "--no-cpu-baseline", "--no-e2e"]
    env = dict(os.environ, NCCL_DEBUG="INFO")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    d = json.loads(lines[-1])
    assert d["n_gpus"] == 1 and d["config"]["frames_per_step"] == 7 * 2000
    assert "NCCL" in r.stdout + r.stderr
    assert d["gen_decode"]["counters_equal_decode_only"]
