"""bench.py's multi-GPU launch contract on CPU: `--gpus N` without a launcher re-runs itself under
torch.distributed.run with N ranks (rendezvous on 127.0.0.1), rank 0 alone prints the JSON line with
n_gpus == N, and a WORLD_SIZE that disagrees with --gpus is refused.  The reference arm (the fp64 oracle
on the host) is the one arm that runs without a GPU, so it drives the launcher here."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None, timeout=600):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=e,
                          capture_output=True, text=True, timeout=timeout)


def test_gpus2_spawns_two_ranks_and_rank0_prints_one_line():
    r = _run(["--gpus", "2", "--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "0",
              "--cpu-seconds", "0.3"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["n_gpus"] == 2 and line["impl"] == "reference"
    assert line["value"] > 0 and line["unit"] == "queries/s"


def test_world_size_must_match_gpus():
    r = _run(["--gpus", "1", "--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "0"],
             env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2
    assert "WORLD_SIZE" in r.stderr
