"""Times the both-keys receiver (mmsb_receiver_both: one launch, recovery + extraction CTAs) against
the two separate receiver calls (extract, then recover) on the same marked batch, CUDA events,
median of 20 after 5 warm-ups.

  python tools/both_keys_probe.py [--config 2] [--method emr]
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_07992_b200 import mmsb as G  # noqa: E402
from paper_2302_07992_b200 import synth as S  # noqa: E402


def timed(fn, reps=20):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--method", default=None)
    a = ap.parse_args()
    cfg = S.CONFIGS[a.config]
    method = a.method or ("lmr" if cfg["method"] == "lmr" else "emr")
    mid = G.EMR if method == "emr" else G.LMR
    imgs, k1, k2 = S.batch(a.config)
    B, H, W = imgs.shape
    I, K1, K2 = (torch.from_numpy(x).cuda() for x in (imgs, k1, k2))
    ws = G.Workspace(mid, B, H, W)
    enc, b, cap, st = G.encode(mid, I, K1, ws)
    nb = (cap - 32).clamp(min=0)
    stride = int(((int(nb.max()) + 7) // 8 + 4 + 15) // 16 * 16)
    msgs = torch.from_numpy(np.stack([S.payload(S.image_seed(a.config, j), stride) for j in range(B)])).cuda()
    marked, _ = G.embed(mid, enc, K2, msgs, nb, ws)
    mo, rec = torch.zeros(B, stride, dtype=torch.uint8, device="cuda"), torch.empty_like(I)

    def separate():
        G.extract(mid, marked, K2, stride, ws, out=mo)
        G.recover(mid, marked, K1, ws, out=rec)

    def both():
        G.receive_both(mid, marked, K1, K2, stride, ws, msg_out=mo, rec_out=rec)

    t_sep, t_both = timed(separate), timed(both)
    px = B * H * W
    print(json.dumps({"config": a.config, "method": method, "images": B, "separate_ms": t_sep, "both_ms": t_both,
                      "speedup": t_sep / t_both, "both_gpx_s": px / t_both / 1e6}))


if __name__ == "__main__":
    main()
