"""bench.py's multi-GPU plumbing through bench.py itself, on CPU (gloo): `--gpus 2` re-executes
under torch.distributed.run with one process per rank, `--shard` splits the batch with
parallel.shard (strong scaling), and the per-image records / statistic rows all-gathered to
rank 0 give the same aggregates as one process.  `--launcher-probe` replaces only the library
calls (no GPU here) by host-made records."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _probe(*args, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--launcher-probe", *args],
                       capture_output=True, text=True, timeout=240, env=e)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [json.loads(x) for x in p.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, p.stdout           # rank 0 alone prints
    return lines[0], p.stderr


def test_self_launch_two_ranks_sharded_equals_one():
    one, _ = _probe("--gpus", "1", "--batch", "11", "--shard")
    two, err = _probe("--gpus", "2", "--batch", "11", "--shard")
    assert "process group gloo with 2 ranks" in err
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2 and two["scaling"] == "strong"
    assert two["shards"] == [6, 5] and sum(two["shards"]) == 11
    assert two["stats"] == one["stats"] and two["stats"]["images"] == 11
    assert two["row_means"] == one["row_means"]


def test_weak_mode_every_rank_its_own_batch():
    two, _ = _probe("--gpus", "2", "--batch", "5")
    assert two["scaling"] == "weak" and two["stats"]["images"] == 10


def test_world_size_must_match_gpus():
    e = dict(os.environ, WORLD_SIZE="3", RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--launcher-probe", "--gpus", "2"],
                       capture_output=True, text=True, timeout=120, env=e)
    assert p.returncode != 0 and "WORLD_SIZE=3" in (p.stderr + p.stdout)
