"""bench.py's multi-rank launch on CPU: with --gpus N and no WORLD_SIZE it starts N ranks itself
(torch.distributed.run, one process per GPU); the reference arm runs them over gloo, every rank
checks in and rank 0 alone prints the line.  A WORLD_SIZE that disagrees with --gpus is refused."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _env(**extra):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                            "MASTER_PORT")}
    env.update(extra)
    return env


def test_bench_self_launches_two_gloo_ranks():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--steps", "1", "--warmup", "0", "--ref-batch", "4", "--ref-cores", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env=_env())
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["ranks"] == 2
    assert line["value"] > 0 and line["cpu_baseline"]["cores"] == 1


def test_bench_refuses_world_size_mismatch():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300, cwd=ROOT,
                         env=_env(WORLD_SIZE="1", RANK="0"))
    assert out.returncode != 0 and "WORLD_SIZE=1" in out.stderr
