"""bench.py's output contract (the driver parses it): one JSON line with the
metric, value, roofline, cpu_baseline, e2e, clocks and launch count; the
reference arm's line with impl/cpu_baseline/e2e."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args,
                         capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "1", "--cells", "6"])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "atom-steps/s"
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["higher_is_better"] is True


@pytest.mark.gpu
def test_device_line():
    d = _run(["--steps", "20", "--warmup", "3", "--cells", "16", "--no-cpu-baseline"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "gpu_launches", "clocks", "e2e"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 20 and d["warmup"] == 3
    assert d["value"] > 0 and d["gpu_launches"] >= 20
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["e2e"]["value"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert "workload" in d["config"] and "sm_mhz" in d["clocks"]


def _torchrun(args, env_extra, timeout=600):
    env = dict(os.environ, **env_extra)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + os.getpid() % 300),
           os.path.join(ROOT, "bench.py")] + args
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]           # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.gpu
def test_two_rank_line():
    """The N-GPU path (torchrun, DistMD, max-over-ranks timing) with two ranks
    sharing one GPU over gloo (PC_BENCH_BACKEND; the driver runs NCCL)."""
    d = _torchrun(["--gpus", "2", "--cells", "16", "--steps", "10", "--warmup", "3"],
                  {"PC_BENCH_BACKEND": "gloo"})
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    assert d["config"]["global_atoms"] == 2 * d["config"]["atoms_per_gpu"]
    assert d["config"]["parallelism"] == "domain x2"


def test_reference_arm_under_torchrun():
    d = _torchrun(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1",
                   "--cells", "6"], {})
    assert d["impl"] == "reference" and d["value"] > 0
