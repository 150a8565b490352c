"""Config 1 (one 512x512 image, EMR; BASELINE.json configs[1]): latency of the four calls + statistics,
launched eagerly and as a CUDA Graph replay ("for config 1, also report latency in us
with CUDA-Graph replay").  Prints one JSON line.

  python tools/latency_config1.py [--method emr|lmr] [--reps 200]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_07992_b200 import mmsb as G  # noqa: E402
from paper_2302_07992_b200 import synth as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--method", default="emr")
ap.add_argument("--reps", type=int, default=200)
a = ap.parse_args()
mid = G.EMR if a.method == "emr" else G.LMR
imgs, k1, k2 = S.batch(1, n=1)
I, K1, K2 = (torch.from_numpy(x).cuda() for x in (imgs, k1, k2))
H, W = imgs.shape[1:]
ws = G.Workspace(mid, 1, H, W)
enc, marked, rec = (torch.empty_like(I) for _ in range(3))
_, b, cap, _ = G.encode(mid, I, K1, ws, out=enc)
n = max(int(cap.item()) - 32, 0)
stride = ((n + 7) // 8 + 4 + 15) // 16 * 16
MSG = torch.from_numpy(S.payload(S.image_seed(1, 0), stride)[None]).cuda()
NB = torch.tensor([n], dtype=torch.int64, device="cuda")
MOUT = torch.zeros(1, stride, dtype=torch.uint8, device="cuda")
SSE = torch.empty(1, dtype=torch.int64, device="cuda")


def step():
    G.encode(mid, I, K1, ws, out=enc)
    G.embed(mid, enc, K2, MSG, NB, ws, out=marked)
    G.extract(mid, marked, K2, stride, ws, out=MOUT)
    G.recover(mid, marked, K1, ws, out=rec, original=I, sse_out=SSE)     # + statistics (SSE)


def timed(fn, reps):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


eager_us = timed(step, a.reps)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    step()                                   # warm the allocator on the capture stream
torch.cuda.current_stream().wait_stream(s)
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph):
    step()
graph_us = timed(graph.replay, a.reps)
ok = int(G.extract(mid, marked, K2, stride, ws)[1].item()) == n
print(json.dumps({"config": "BASELINE.json configs[1]: 1 x 512x512, " + a.method.upper(), "eager_us_per_step": eager_us,
                  "graph_us_per_step": graph_us, "graph_Mpx_per_s": H * W / graph_us, "payload_round_trip": ok,
                  "launches_per_step": "8 (EMR)" if mid == G.EMR else "LMR coder waves"}))
