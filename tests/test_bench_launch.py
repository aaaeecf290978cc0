"""bench.py's launch path on CPU: `--gpus N` without a launcher re-executes
under torch.distributed.run and really forms N ranks (gloo dry run, no GPU)."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _run(*args):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                         timeout=240, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # exactly one JSON line on stdout
    return json.loads(lines[0])


@pytest.mark.timeout(300)
@pytest.mark.parametrize("n", [1, 2])
def test_gpus_flag_forms_that_many_ranks(n):
    d = _run("--gpus", str(n), "--dry-run")
    assert d["n_gpus"] == n and d["ranks"] == list(range(n))
    assert ("dp%d" % n in d["config"]["parallelism"]) if n > 1 else d["config"]["parallelism"] == "single GPU"


def test_world_mismatch_is_an_error():
    env_run = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run"],
                             capture_output=True, text=True, timeout=120, cwd=ROOT,
                             env={**__import__("os").environ, "WORLD_SIZE": "1", "RANK": "0"})
    assert env_run.returncode != 0 and "launcher started 1" in env_run.stderr


def test_reference_and_ours_share_the_config():
    sys.path.insert(0, str(ROOT))
    import bench

    for n in (1, 8):
        assert bench.config(n, "zslab", 4) == bench.config(n, "zslab", 4)
        assert set(bench.config(n, "angle", 4)) == set(bench.config(1, "zslab", 4))
