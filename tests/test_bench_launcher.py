"""bench.py's multi-GPU launcher on the CPU (-m "not gpu"): `python bench.py --gpus N` without a
torchrun environment launches N ranks itself (rendezvous on 127.0.0.1), the ranks meet at the
barrier / max-over-ranks path, and exactly ONE JSON line reaches stdout (rank 0).  --dry-run
replaces the GPU work with nothing, so this checks the plumbing only."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n", [2, 4])
def test_self_launch_n_ranks_one_json_line(n):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--dry-run",
                          "--steps", "3", "--warmup", "3"], capture_output=True, text=True, timeout=600, env=env,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["world_size"] == n and d["ranks_seen"] == n
    assert d["max_over_ranks"] == float(n)          # rank r contributes 1 + r: the MAX arrived
    assert d["steps"] == 3 and d["warmup"] == 3
