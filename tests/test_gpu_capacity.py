"""GPU <-> oracle parity for the capacity query (mmsb_capacity): b and C
of encrypted and marked images as the hider derives them, equal to the encoder's outputs and to
O.capacity; FORMAT / BADCASE headers."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2302_07992_b200 import mmsb as G
from paper_2302_07992_b200 import synth as S

pytestmark = pytest.mark.gpu


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("method", [G.EMR, G.LMR])
@pytest.mark.parametrize("H,W", [(128, 128), (16, 32768), (32768, 16)])
def test_capacity_matches_encoder_and_oracle(method, H, W):
    kinds = ["smooth", "textured", "noise", "constant", "quantised", "smooth"]
    imgs = np.stack([S.random_image(500 + j, H, W, k) for j, k in enumerate(kinds)])
    k1 = np.stack([np.frombuffer(S.key(500 + j, 1), np.uint8) for j in range(len(kinds))])
    k2 = np.stack([np.frombuffer(S.key(500 + j, 2), np.uint8) for j in range(len(kinds))])
    ws = G.Workspace(method, len(kinds), H, W)
    enc, b, cap, st = G.encode(method, _dev(imgs), _dev(k1), ws)
    stride = S.msg_stride(H, W)
    msgs = np.stack([S.payload(j, stride) for j in range(len(kinds))])
    marked, _ = G.embed(method, enc, _dev(k2), _dev(msgs), (cap - 32).clamp(min=0), ws)
    for X in (enc, marked):
        bq, cq, sq = G.capacity(method, X, ws)
        torch.cuda.synchronize()
        Xh = X.cpu().numpy()
        for j in range(len(kinds)):
            so, bo, co = O.capacity(method, Xh[j])
            assert (int(sq[j]), int(bq[j]), int(cq[j])) == (so, bo, co), (j, int(sq[j]), int(bq[j]), int(cq[j]), so, bo, co)
            if int(st[j]) == O.OK:                      # the hider sees what the owner computed
                assert (int(bq[j]), int(cq[j])) == (int(b[j]), int(cap[j]))


@pytest.mark.parametrize("method", [G.EMR, G.LMR])
def test_capacity_format_cases(method):
    H = W = 64
    rng = np.random.default_rng(7)
    X = rng.integers(0, 256, size=(4, H, W), dtype=np.uint8)
    X[0, 0, :3] |= 1                                     # EMR b-field 7 -> FORMAT
    X[1, 0, :3] &= 0xFE                                  # EMR b-field 0 -> b = 2
    bq, cq, sq = G.capacity(method, _dev(X))
    torch.cuda.synchronize()
    for j in range(4):
        so, bo, co = O.capacity(method, X[j])
        assert (int(sq[j]), int(bq[j]), int(cq[j])) == (so, bo, co), (j, int(sq[j]), so)
