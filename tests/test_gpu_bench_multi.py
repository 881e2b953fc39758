"""bench.py's N > 1 code paths on one GPU (-m gpu): `--force-multi` runs the process group,
NCCL B1 (C++), the sampled oracle checks and the NCCL init-line capture in a world of one
process, so a first multi-GPU SCALE run does not meet them untested.  The N > 1 launcher itself
is covered on the CPU (tests/test_bench_launcher.py); one process per GPU at N >= 2 by
tests/test_gpu_multiproc_parity.py on a box with several GPUs."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")
def test_force_multi_line():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--force-multi", "--no-sweep",
                          "--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]           # one JSON line on stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["value"] > 0
    assert d["verified_sampled_vs_oracle"] is True       # sampled columns vs the oracle (N > 1 form)
    assert d["nccl"]["verified_sampled_vs_oracle"] is True and d["nccl"]["us_per_call"] > 0
    assert d["nccl_init"]["ranks_reporting"] == 1
    assert any("Init COMPLETE" in ln for ln in d["nccl_init"]["lines"])
    assert d["roofline"]["bound"] in ("hbm", "nvlink") and 0 < d["roofline"]["frac"] <= 1.1
    assert d["gpu_launches"] == 3


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")
def test_force_multi_sweep():
    """The p = N per-size sweep (every mpxa variant vs NCCL B1, largest points checked against
    the oracle) at N = 1."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--force-multi",
                          "--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    ns = d["nccl_sweep"]
    assert ns["p"] == 1
    for op, n in (("alltoall", 12), ("allgather", 25)):
        rows = ns[op]
        assert len(rows) == n
        for r in rows:                      # [bytes, t_roof, nccl_us, best_us, best, frac, speedup, by_variant]
            assert r[2] > 0 and r[3] > 0 and r[4] in r[7]
        assert ns[f"{op}_largest_verified_sampled_vs_oracle"] is True
