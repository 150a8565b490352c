"""Performance probe of the fused encode / recover kernels: builds variants of libmmsb.so with
only the keystream CTAs (1) or only the worker CTAs (2, no waiting; +4: no row look-back; +8: no
cell transform in recovery) and times each call with CUDA events next to the normal build (3).  Outputs are garbage in the probe builds: timing only.

  python tools/role_probe.py [--build] [--batch 1000]
"""
import argparse
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build_variant(mask):
    from paper_2302_07992_b200 import build as B

    out = os.path.join(B.PKG, f"libmmsb_probe{mask}.so")
    objs = []
    os.makedirs(os.path.join(B.OBJ, f"probe{mask}"), exist_ok=True)
    for src in B._sources():
        obj = os.path.join(B.OBJ, f"probe{mask}", os.path.basename(src)[:-3] + ".o")
        subprocess.check_call([B.NVCC, *B.ARCH, *B.FLAGS, f"-DMMSB_PROBE_ROLES={mask}", "-c", src, "-o", obj])
        objs.append(obj)
    subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-o", out, *objs, "-lcudart"])
    return out


def run(mask, batch, config=2, reps=10):
    import numpy as np
    import torch

    from paper_2302_07992_b200 import mmsb as G
    from paper_2302_07992_b200 import synth as S

    imgs, k1, k2 = S.batch(config, n=batch)
    I, K1 = torch.from_numpy(imgs).cuda(), torch.from_numpy(k1).cuda()
    ws = G.Workspace(G.EMR, batch, imgs.shape[1], imgs.shape[2])
    enc = torch.empty_like(I)
    rec = torch.empty_like(I)
    res = {}
    for name, fn in (("encode", lambda: G.encode(G.EMR, I, K1, ws, out=enc)),
                     ("recover", lambda: G.recover(G.EMR, enc, K1, ws, out=rec))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        res[name] = a.elapsed_time(b) / reps
    print(f"mask={mask}", {k: round(v, 4) for k, v in res.items()}, flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--build", action="store_true")
    ap.add_argument("--batch", type=int, default=1000)
    ap.add_argument("--mask", type=int, default=None)
    ap.add_argument("--config", type=int, default=2)
    a = ap.parse_args()
    if a.build:
        for m in (1, 2):
            print(build_variant(m))
        sys.exit(0)
    if a.mask is not None:
        run(a.mask, a.batch, a.config)
        sys.exit(0)
    from paper_2302_07992_b200 import build as B

    for m in (3, 1, 2):
        env = dict(os.environ)
        if m != 3:
            env["MMSB_LIB"] = os.path.join(B.PKG, f"libmmsb_probe{m}.so")
        subprocess.run([sys.executable, __file__, "--mask", str(m), "--batch", str(a.batch), "--config", str(a.config)], env=env, timeout=120)
