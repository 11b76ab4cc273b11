"""The multi-rank path of bench.py (--gpus N: the ranks spawned through torch.distributed.run,
config 5's fixed batch sharded B/G per rank, barriers, max over ranks, one JSON line from rank 0)
run end to end on a one-GPU box: SC_BENCH_SHARE_GPU=1 puts both ranks on GPU 0 with a gloo
group (batch shards never wait on each other's kernels). A plumbing test, not a measurement."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.timeout(600)
def test_bench_two_ranks_share_config5():
    env = dict(os.environ, SC_BENCH_SHARE_GPU="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--steps", "10", "--warmup", "3", "--e2e-calls", "1"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert out.returncode == 0, out.stderr[-2000:]
    assert len(lines) == 1, out.stdout  # rank 0 prints, rank 1 does not
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 10 and d["scaling"] == "strong"
    assert d["config"]["cloths_per_gpu"] == 2048 and d["config"]["cloths"] == 4096
    assert "shared_gpu" in d["config"]
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["e2e"]["finite"]
