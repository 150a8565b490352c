"""One-off wide fuzz of the CUDA path against the oracle (GPU box only; not a pytest test).

Draws cases like tests/test_gpu_random_parity.py but from other seeds and a wider space: batch
sizes 1..17 (incl. multiples of 8), sides 16..1024 and coder tiles 3..9, and runs the test's own
body on each (every output of the four calls bit-exact against the oracle) until the time budget
is spent.  Failures are logged with the case tuple so that they can be replayed as a test.

    python tools/fuzz_parity.py --seconds 600 --seed 1 > gpurun_out/fuzz.log
"""
import argparse
import os
import sys
import time
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import test_gpu_random_parity as T  # noqa: E402


def cases(seed):
    rng = np.random.default_rng(seed)
    i = 0
    while True:
        H = int(2 ** rng.integers(4, 11))
        W = int(2 ** rng.integers(4, 11))
        if H * W > 512 * 1024:                     # keep the oracle's share of a case under a second or two
            continue
        method = int(rng.integers(0, 2))
        t = int(rng.integers(3, 10))
        emin = int(rng.integers(0, 4)) if method == 1 else 0
        rounds = int(rng.choice([20, 20, 12, 8]))
        B = int(rng.choice([1, 2, 3, 5, 8, 9, 16, 17]))
        if B * H * W > 2 << 20:
            B = max(1, (2 << 20) // (H * W))
        kinds = [T.KINDS[int(k)] for k in rng.integers(0, len(T.KINDS), B)]
        mode = int(rng.integers(0, 4))
        yield (100000 * seed + i, H, W, method, t, emin, rounds, kinds, mode)
        i += 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=600.0)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    t0 = time.time()
    n = bad = skipped = 0
    for c in cases(a.seed):
        if time.time() - t0 > a.seconds:
            break
        try:
            T.test_random_parity(c)
        except T.G.MmsbError as e:                  # a shape outside the envelope: refused loudly, not a mismatch
            skipped += 1
            print("REFUSED", c[:7], len(c[7]), c[8], str(e)[:120], flush=True)
            continue
        except Exception:
            bad += 1
            print("FAIL", c, flush=True)
            traceback.print_exc(file=sys.stdout)
        n += 1
        if n % 50 == 0:
            print(f"# {n} cases, {bad} failed, {skipped} refused, {time.time() - t0:.0f} s", flush=True)
    print(f"DONE cases={n} failed={bad} refused={skipped} seconds={time.time() - t0:.0f}", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
