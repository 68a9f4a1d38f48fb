"""bench.py launch contract on CPU (no GPU needed): `python bench.py --gpus N` without a launcher
starts N ranks itself (torch.distributed.run, one process per GPU) and rank 0 alone prints one
JSON line with n_gpus == N; the reference arm runs on rank 0 only."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*argv):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *argv], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_self_launches_two_ranks():
    d = _run("--gpus", "2", "--impl", "reference", "--scale", "12", "--steps", "3", "--warmup", "3")
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["scaling"] == "strong"                     # configs[4]: one graph over the N GPUs
    assert d["cpu_baseline"]["cores"] == len(os.sched_getaffinity(0))  # not torchrun's 1 thread
    assert d["cpu_baseline"]["serial"]["cores"] == 1
    assert "generator" in d["config"]["layout"]         # the CPU arm never relabels
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_reference_arm_one_rank():
    d = _run("--impl", "reference", "--scale", "12", "--steps", "3", "--warmup", "3")
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["unit"] == "GTEPS"
