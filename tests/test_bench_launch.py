"""bench.py's launch contract on CPU: `--gpus N` outside torchrun re-executes
itself as N torch.distributed ranks (127.0.0.1 rendezvous) and rank 0 reports
n_gpus = N; a torchrun launch whose WORLD_SIZE disagrees with --gpus is refused."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _run(args, env=None, timeout=180):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True,
                          text=True, timeout=timeout, env=e, cwd=str(ROOT))


def _last_json(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out
    return json.loads(lines[-1])


@pytest.mark.parametrize("n", [2, 3])
def test_self_launch_spawns_n_ranks(n):
    r = _run(["--gpus", str(n), "--dry-run"])
    assert r.returncode == 0, r.stderr[-2000:]
    line = _last_json(r.stdout)
    assert line == {"dry_run": True, "n_gpus": n, "ranks_in_allreduce": n}


def test_single_gpu_runs_in_process():
    r = _run(["--gpus", "1", "--dry-run"])
    assert r.returncode == 0, r.stderr[-2000:]
    assert _last_json(r.stdout)["n_gpus"] == 1


def test_world_size_mismatch_is_refused():
    r = _run(["--gpus", "4", "--dry-run"], env={"WORLD_SIZE": "2", "RANK": "0"})
    assert r.returncode != 0
    assert "WORLD_SIZE=2" in (r.stderr + r.stdout)


@pytest.mark.gpu
def test_two_rank_bench_shares_one_gpu():
    """The N > 1 measurement path end to end on a one-GPU box: both ranks on
    cuda:0 over gloo (LW_BENCH_SHARE_GPU, a code-path check, never a number)."""
    r = _run(["--gpus", "2", "--scale", "16", "--steps", "3", "--warmup", "3",
              "--no-cpu-baseline", "--no-power"], env={"LW_BENCH_SHARE_GPU": "1"}, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = _last_json(r.stdout)
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert line["config"]["parallelism"] == "rows2"
