"""No call writes outside its workspace or its output tensors: the workspace is carved from a
larger buffer whose guard bytes (before and after) must survive every call, for EMR and LMR at a
batch large enough that per-image strides matter."""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_2302_07992_b200 import mmsb as G
from paper_2302_07992_b200 import synth as S

pytestmark = pytest.mark.gpu

GUARD = 1 << 20


class _GuardedWs:
    def __init__(self, method, B, H, W):
        self.shape = G._shape(method, B, H, W, 7, 0)
        self.nbytes = G.lib().mmsb_workspace_bytes(C.byref(self.shape))
        self.raw = torch.full((self.nbytes + 2 * GUARD,), 0xA5, dtype=torch.uint8, device="cuda")
        self.buf = self.raw[GUARD:GUARD + self.nbytes]

    def intact(self):
        return bool((self.raw[:GUARD] == 0xA5).all()) and bool((self.raw[GUARD + self.nbytes:] == 0xA5).all())


@pytest.mark.parametrize("B,H,W", [(96, 128, 128), (8, 256, 1024), (2, 2048, 2048), (3, 64, 32)])
@pytest.mark.parametrize("method", [G.EMR, G.LMR])
def test_calls_stay_inside_the_workspace(method, B, H, W):
    kinds = ["smooth", "textured", "noise", "smooth"]
    imgs = np.stack([S.random_image(1200 + j, H, W, kinds[j % 4]) for j in range(B)])
    k1 = np.stack([np.frombuffer(S.key(1200 + j, 1), np.uint8) for j in range(B)])
    k2 = np.stack([np.frombuffer(S.key(1200 + j, 2), np.uint8) for j in range(B)])
    stride = S.msg_stride(H, W)
    msgs = np.stack([S.payload(j, stride) for j in range(B)])
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    ws = _GuardedWs(method, B, H, W)
    assert ws.nbytes > 0
    guarded = []

    def out(*shape):                                   # an output tensor with guard bytes around it
        n = int(np.prod(shape))
        raw = torch.full((n + 2 * GUARD,), 0x5A, dtype=torch.uint8, device="cuda")
        guarded.append((raw, n))
        return raw[GUARD:GUARD + n].view(*shape)

    enc, b, cap, st = G.encode(method, dev(imgs), dev(k1), ws, out=out(B, H, W))
    marked, _ = G.embed(method, enc, dev(k2), dev(msgs), (cap - 32).clamp(min=0), ws, out=out(B, H, W))
    G.extract(method, marked, dev(k2), stride, ws, out=out(B, stride))
    G.recover(method, marked, dev(k1), ws, out=out(B, H, W))
    G.receive_both(method, marked, dev(k1), dev(k2), stride, ws, msg_out=out(B, stride), rec_out=out(B, H, W))
    G.capacity(method, marked, ws)
    torch.cuda.synchronize()
    assert ws.intact()
    for raw, n in guarded:
        assert bool((raw[:GUARD] == 0x5A).all()) and bool((raw[GUARD + n:] == 0x5A).all())
