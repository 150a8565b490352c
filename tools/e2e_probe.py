"""Diagnostic for bench.py's e2e leg: the same 2-lane sub-batch pipeline (host->device copies of
images + payload on the lane streams, device->host copies of the outputs on one stream, lanes
streaming across steps) with and without the compute between the copies, at config-2 sizes.

  python tools/e2e_probe.py [--steps 20] [--nsub 2]
"""
import argparse
import json

import torch

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--nsub", type=int, default=2)
ap.add_argument("--compute_ms", type=float, default=0.0, help="a busy kernel of this length per sub-batch")
ap.add_argument("--lanes", type=int, default=2)
ap.add_argument("--msg_bytes", type=int, default=180480, help="payload row bytes per image (0: images only)")
a = ap.parse_args()
B, HW = 1000, 512 * 512
MSGB = a.msg_bytes
dev = torch.device("cuda")
hI = torch.empty(B * HW, dtype=torch.uint8).pin_memory()
hM = torch.empty(max(B * MSGB, 1), dtype=torch.uint8).pin_memory()
hR = torch.empty(B * HW, dtype=torch.uint8).pin_memory()
hMO = torch.empty(max(B * MSGB, 1), dtype=torch.uint8).pin_memory()
sub = B // a.nsub


class Lane:
    def __init__(self):
        self.s = torch.cuda.Stream()
        self.I = torch.empty(sub * HW, dtype=torch.uint8, device=dev)
        self.M = torch.empty(max(sub * MSGB, 1), dtype=torch.uint8, device=dev)
        self.R = torch.empty(sub * HW, dtype=torch.uint8, device=dev)
        self.MO = torch.empty(max(sub * MSGB, 1), dtype=torch.uint8, device=dev)
        self.copied = None
        self.computed = torch.cuda.Event()


lanes = [Lane() for _ in range(a.lanes)]
counter = [0]
d2h = torch.cuda.Stream()
spin = torch.empty(1, device=dev)


def step(compute):
    for i in range(a.nsub):
        L = lanes[counter[0] % len(lanes)]                # lanes rotate over sub-batches across steps
        counter[0] += 1
        x, y = i * sub * HW, (i + 1) * sub * HW
        u, v = i * sub * MSGB, (i + 1) * sub * MSGB
        with torch.cuda.stream(L.s):
            L.I.copy_(hI[x:y], non_blocking=True)
            if MSGB:
                L.M.copy_(hM[u:v], non_blocking=True)
            if L.copied is not None:
                L.s.wait_event(L.copied)
            if compute:
                L.R.copy_(L.I)                     # device-side work standing in for the five calls
                if MSGB:
                    L.MO.copy_(L.M)
                if a.compute_ms > 0:
                    torch.cuda._sleep(int(a.compute_ms * 1.9e6))
            L.computed.record(L.s)
        d2h.wait_event(L.computed)
        with torch.cuda.stream(d2h):
            hR[x:y].copy_(L.R, non_blocking=True)
            if MSGB:
                hMO[u:v].copy_(L.MO, non_blocking=True)
            L.copied = torch.cuda.Event()
            L.copied.record(d2h)


def run(compute):
    step(compute)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    e0.record(cur)
    for L in lanes:
        L.s.wait_event(e0)
    for _ in range(a.steps):
        step(compute)
    for L in lanes:
        cur.wait_stream(L.s)
    cur.wait_stream(d2h)
    e1.record(cur)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    byt = B * (HW + MSGB)
    return {"ms_per_step": ms, "GBps_each_way": byt / ms / 1e6, "Gpx_s": B * HW / ms / 1e6}


print(json.dumps({"copies_only": run(False), "with_device_copies": run(True), "nsub": a.nsub,
                  "lanes": a.lanes, "compute_ms": a.compute_ms}))
