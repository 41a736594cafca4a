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
    d = _run(["--steps", "20", "--warmup", "3", "--cells", "16", "--no-cpu-baseline",
              "--e2e-steps", "20"])
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
    assert d["config"]["global_atoms"] == 4 * 16 ** 3 == d["config"]["atoms_per_gpu"]
    for key in ("roofline_step", "roofline_build"):
        q = d[key]
        assert 0 < q["frac"] < 1 and abs(q["frac"] - q["achieved"] / q["peak"]) < 1e-9


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
@pytest.mark.parametrize("scaling,transport", [("strong", "nccl"), ("weak", "nccl"),
                                               ("strong", "p2p")])
def test_two_rank_line(scaling, transport):
    """The N-GPU path (torchrun, DistMD, max-over-ranks timing) with two ranks
    sharing one GPU over gloo (PC_BENCH_BACKEND; the driver runs NCCL).
    strong: the 16^3-cell system split over 2x1x1; weak: a 16^3-cell block per
    rank (32x16x16 global); p2p: the per-step halo by peer-memory stores
    (dist.P2PTransport) instead of the all-to-all."""
    d = _torchrun(["--gpus", "2", "--cells", "16", "--steps", "10", "--warmup", "3",
                   "--scaling", scaling, "--transport", transport],
                  {"PC_BENCH_BACKEND": "gloo"})
    assert d["config"]["halo_transport"] == transport
    assert d["n_gpus"] == 2 and d["scaling"] == scaling and d["value"] > 0
    n = 4 * 16 ** 3 * (2 if scaling == "weak" else 1)
    c = d["config"]
    assert c["global_atoms"] == n and c["atoms_per_gpu"] == n / 2
    assert 0.4 * n < c["rank0_owned_atoms"] < 0.6 * n
    assert c["parallelism"] == "domain x2"
    assert abs(d["value"] - n * 10 / (d["ms_per_step"] * 10e-3)) < 1e-6 * d["value"]
    # end-to-end leg through DistMD(state=host block) at N ranks
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] == 40


def test_reference_arm_under_torchrun():
    d = _torchrun(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1",
                   "--cells", "6"], {})
    assert d["impl"] == "reference" and d["value"] > 0
