"""Copy-engine ceiling of the e2e pipeline shape (8 sub-batches over 3 streams, config-2 sizes):
host->device and device->host copies with 0, 4 or 16 device-to-device copies as stand-in compute."""
import torch, json
B, HW, stride = 1000, 512*512, 46592
hI = torch.empty(B, HW, dtype=torch.uint8).pin_memory()
hM = torch.empty(B, stride, dtype=torch.uint8).pin_memory()
hR = torch.empty(B, HW, dtype=torch.uint8).pin_memory()
hMo = torch.empty(B, stride, dtype=torch.uint8).pin_memory()
nsub, sub = 8, 125
class L:
    def __init__(s):
        s.st = torch.cuda.Stream(); s.I = torch.empty(sub, HW, dtype=torch.uint8, device='cuda'); s.M = torch.empty(sub, stride, dtype=torch.uint8, device='cuda')
        s.R = torch.empty_like(s.I); s.Mo = torch.empty_like(s.M)
lanes = [L() for _ in range(3)]
def step(compute):
    for i in range(nsub):
        l = lanes[i % 3]; a, z = i*sub, (i+1)*sub
        with torch.cuda.stream(l.st):
            l.I.copy_(hI[a:z], non_blocking=True); l.M.copy_(hM[a:z], non_blocking=True)
            if compute:
                for _ in range(compute): l.R.copy_(l.I)
            hR[a:z].copy_(l.R, non_blocking=True); hMo[a:z].copy_(l.Mo, non_blocking=True)
cur = torch.cuda.current_stream()
for compute in (0, 4, 16):
    step(compute); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    for l in lanes: l.st.wait_event(e0)
    for _ in range(5): step(compute)
    for l in lanes:
        ev = torch.cuda.Event(); ev.record(l.st); cur.wait_event(ev)
    e1.record(cur); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    byt = (hI.numel() + hM.numel())
    print(json.dumps({"compute_copies": compute, "ms_per_step": ms, "GBps_each_dir": byt / ms / 1e6, "Gpx_s": B*HW/ms/1e6}))
