"""bench.py's JSON line on a real GPU (small batch): the contract's keys, a consistent roofline
block, the result checks all true, clocks sampled, library launches counted, and the CPU-oracle
baseline with its single-core per-call times; plus the default run's LMR block."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "gpu_launches", "clocks", "e2e", "roofline", "cpu_baseline"]


def _run(*args):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [x for x in p.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    return json.loads(lines[0])


def _check_line(d, block=False):
    for k in KEYS:
        if block and k in ("n_gpus", "steps", "warmup", "higher_is_better", "vs_baseline", "data"):
            continue                                          # the lmr block carries its own measurement only
        assert k in d, k
    assert d["value"] > 0 and d["unit"] == "Mpixel/s"
    if not block:
        assert d["n_gpus"] == 1 and d["higher_is_better"] is True
    r = d["roofline"]
    assert r["bound"] in ("alu", "hbm") and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["gpu_launches"] > 0 and d["clocks"]["samples"] > 0
    assert all(v is True or (isinstance(v, dict) and all(v.values())) for v in d["checks"].values())
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["matches_device"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0
    assert cb["single_core"]["cores"] == 1 and set(cb["single_core"]["per_call_ms"]) == {
        "encode", "hide", "extract", "recover", "sse"}


def test_default_line_with_lmr_block():
    d = _run("--steps", "3", "--warmup", "3", "--batch", "16", "--cpu-seconds", "2", "--e2e-steps", "3")
    _check_line(d)
    assert d["config"]["method"] == "emr" and d["config"]["batch_per_gpu"] == 16
    _check_line(d["lmr"], block=True)
    assert d["lmr"]["config"]["method"] == "lmr" and d["lmr"]["config"]["config_index"] == 3
    assert d["lmr"]["checks"]["recovered_equals_original"] is True


def test_shard_mode_one_rank():
    d = _run("--config", "4", "--shard", "--batch", "20", "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
             "--no-security", "--e2e-steps", "2")
    assert d["scaling"] == "strong" and d["config"]["global_batch"] == 20 and d["stats"]["images"] == 20


def test_two_ranks_sharded_match_one_rank():
    """The multi-rank bench path on the hardware at hand: torchrun self-launch, shard split (ragged:
    11 + 10 images), the record and statistics all-gathers and max-over-ranks timing. On a box with
    fewer GPUs than ranks the ranks share a GPU over gloo (a functional run, flagged in the line);
    the aggregates must equal the one-rank run's, image for image."""
    import torch

    common = ("--config", "4", "--shard", "--batch", "21", "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
              "--e2e-steps", "2")
    one = _run(*common)
    two = _run("--gpus", "2", *common)
    assert two["n_gpus"] == 2 and two["scaling"] == "strong" and two["config"]["global_batch"] == 21
    assert ("shared_gpus" in two) == (torch.cuda.device_count() < 2)
    assert all(v is True or (isinstance(v, dict) and all(v.values())) for v in two["checks"].values())
    assert two["stats"] == one["stats"]
    assert two["security"] == one["security"]                # per-image statistics are deterministic
