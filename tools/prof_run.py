"""Small driver for ncu captures: N steps of the hot path on a config-2-like batch."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_07992_b200 import mmsb as G  # noqa: E402
from paper_2302_07992_b200 import synth as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--batch", type=int, default=128)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--method", default="emr")
a = ap.parse_args()
cfg = S.CONFIGS[a.config]
H, W, B = cfg["H"], cfg["W"], a.batch
mid = G.EMR if a.method == "emr" else G.LMR
imgs, k1, k2 = S.batch(a.config, n=B)
I, K1, K2 = (torch.from_numpy(x).cuda() for x in (imgs, k1, k2))
ws = G.Workspace(mid, B, H, W)
enc, b, cap, st = G.encode(mid, I, K1, ws)
nb = (cap - 32).clamp(min=0)
stride = int(((int(nb.max()) + 7) // 8 + 4 + 15) // 16 * 16)
msgs = torch.from_numpy(np.stack([S.payload(S.image_seed(a.config, j), stride) for j in range(B)])).cuda()
for _ in range(a.steps):
    enc, b, cap, st = G.encode(mid, I, K1, ws, out=enc)
    marked, _ = G.embed(mid, enc, K2, msgs, nb, ws)
    mo, nbo, _ = G.extract(mid, marked, K2, stride, ws)
    rec, _, sse = G.recover(mid, marked, K1, ws, original=I)       # + statistics (SSE), as bench.py
torch.cuda.synchronize()
assert torch.equal(nbo, nb), "round trip"
print("ok", G.kernel_launches())
