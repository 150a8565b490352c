"""mmsb_receiver_recover_sse: the K1 recovery fused with the statistics call's SSE.
The recovered image and status must equal mmsb_receiver_recover's bit for bit and the SSE must
equal the oracle's sum of squared differences (and mmsb_stats), for EMR (finite PSNR) and LMR
(SSE 0, PSNR infinite), at several tile geometries and a FORMAT image."""
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
@pytest.mark.parametrize("H,W", [(16, 16), (32, 64), (128, 128), (512, 512)])
def test_recover_sse_matches_recover_and_oracle(method, H, W):
    kinds = ["smooth", "textured", "quantised", "constant"]
    B = len(kinds)
    imgs = np.stack([S.random_image(5100 + j, H, W, k) for j, k in enumerate(kinds)])
    k1 = np.stack([np.frombuffer(S.key(5100 + j, 1), np.uint8) for j in range(B)])
    k2 = np.stack([np.frombuffer(S.key(5100 + j, 2), np.uint8) for j in range(B)])
    stride = S.msg_stride(H, W)
    msgs = np.stack([S.payload(j, stride) for j in range(B)])
    I, K1, K2 = _dev(imgs), _dev(k1), _dev(k2)
    ws = G.Workspace(method, B, H, W)
    enc, b, cap, st = G.encode(method, I, K1, ws)
    marked, _ = G.embed(method, enc, K2, _dev(msgs), (cap - 32).clamp(min=0), ws)
    if method == G.EMR:
        marked[3, 0, :3] ^= 0x01            # header b-2 field > 5 on one image: FORMAT, zero output
        marked[3, 0, :3] |= 0x01
    ref, st_ref = G.recover(method, marked, K1, ws)
    sse_ref = G.stats(I, ref)
    rec, st_s, sse = G.recover(method, marked, K1, ws, original=I)
    torch.cuda.synchronize()
    assert torch.equal(rec, ref) and torch.equal(st_s, st_ref)
    assert torch.equal(sse, sse_ref)
    R = rec.cpu().numpy()
    for j in range(B):
        assert int(sse[j]) == O.sse(imgs[j], R[j])
        if method == G.LMR and int(st_s[j]) == 0:
            assert int(sse[j]) == 0
