"""bench.py plumbing on CPU: `--gpus N` launches N ranks by itself (the way
the driver's BENCH command calls it without torchrun), and a WORLD_SIZE that
disagrees with --gpus is refused instead of silently reporting fewer GPUs."""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(REPO, "bench.py")] + args,
                          capture_output=True, text=True, env=e, timeout=240)


def test_gpus_flag_spawns_that_many_ranks():
    p = _run(["--gpus", "2", "--dry-run"])
    assert p.returncode == 0, p.stderr
    line = json.loads([l for l in p.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["ranks_reporting"] == 2


def test_world_size_mismatch_is_refused():
    p = _run(["--gpus", "4", "--dry-run"], {"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert p.returncode == 2
    assert "WORLD_SIZE=1" in p.stderr
