"""bench.py's N > 1 path end to end on a 1-GPU box: `--gpus 2 --transport gloo` starts two ranks
that share the GPU and exchange through the host transport plugin (NCCL refuses two ranks on one
device); rank 0 measures the one-GPU reference point first, then both ranks run the partitioned
traversals.  The numbers are meaningless (two ranks on one GPU); the plumbing is what is checked:
one JSON line, n_gpus, strong scaling, the layout, the one-GPU point, launches, e2e."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_through_the_transport():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--transport",
                        "gloo", "--scale", "14", "--steps", "4", "--warmup", "3"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["steps"] == 4
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["e2e"]["value"] > 0
    assert "block-diagonal" in d["config"]["layout"] and d["config"]["partitions"] == 2
    one = d["detail"]["one_gpu"]
    assert one["generator_ids"]["value"] > 0 and one["degree_ordered"]["value"] > 0
    assert d["detail"]["exchange_bytes_per_step"] > 0
