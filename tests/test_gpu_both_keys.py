"""The both-keys receiver (mmsb_receiver_both, P:842-843 / P:1066-1067):
its payload, length, recovered image and status equal those of the separate K2 extraction and
K1 recovery calls -- and the oracle's -- for EMR and LMR, including a wrong-key image."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2302_07992_b200 import mmsb as G
from paper_2302_07992_b200 import synth as S

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("method,H,W", [(G.EMR, 128, 128), (G.EMR, 64, 256), (G.LMR, 128, 128), (G.LMR, 256, 64),
                                        (G.EMR, 16, 32768), (G.LMR, 16, 32768), (G.EMR, 32768, 16),
                                        (G.LMR, 32768, 16)])   # the envelope's edges (XL kernels)
def test_both_equals_separate_calls_and_oracle(method, H, W):
    kinds = ["smooth", "textured", "smooth", "constant", "smooth"]
    B = len(kinds)
    imgs = np.stack([S.random_image(7000 + j, H, W, k) for j, k in enumerate(kinds)])
    k1 = np.stack([np.frombuffer(S.key(7000 + j, 1), np.uint8) for j in range(B)])
    k2 = np.stack([np.frombuffer(S.key(7000 + j, 2), np.uint8) for j in range(B)])
    k2_rx = k2.copy()
    k2_rx[2] ^= 0x5A                                                   # receiver's K2 wrong for image 2
    stride = S.msg_stride(H, W)
    msgs = np.stack([S.payload(900 + j, stride) for j in range(B)])
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    ws = G.Workspace(method, B, H, W)
    enc, b, cap, st_e = G.encode(method, dev(imgs), dev(k1), ws)
    marked, st_h = G.embed(method, enc, dev(k2), dev(msgs), (cap - 32).clamp(min=0), ws)
    mo, nb, st_x = G.extract(method, marked, dev(k2_rx), stride, ws)
    rec, st_r = G.recover(method, marked, dev(k1), ws)
    mo2, nb2, rec2, st2 = G.receive_both(method, marked, dev(k1), dev(k2_rx), stride, ws)
    torch.cuda.synchronize()
    assert torch.equal(nb, nb2) and torch.equal(rec, rec2)
    C = cap.cpu().numpy()
    for j in range(B):
        region = 4 * ((int(C[j]) - 32 + 31) // 32) if C[j] > 32 else 0
        assert torch.equal(mo[j, :region], mo2[j, :region])
        expect = int(st_x[j]) if int(st_x[j]) != 0 else int(st_r[j])
        assert int(st2[j]) == expect
        # and against the oracle (the receiver holds both keys)
        Em = marked[j].cpu().numpy()
        sx, mo_o, nbo = O.extract(method, Em, k2_rx[j].tobytes(), stride)
        sr, R = O.recover(method, Em, k1[j].tobytes())
        assert int(nb2[j]) == nbo and np.array_equal(rec2[j].cpu().numpy(), R)
        assert np.array_equal(mo2[j, :region].cpu().numpy(), mo_o[:region])
        assert int(st2[j]) == (sx if sx != O.OK else sr)
    assert int(st2[2]) == O.E_INTEGRITY or int(nb2[2]) != int((cap[2] - 32).item())


@pytest.mark.parametrize("config,method", [(2, G.EMR), (3, G.LMR)])
def test_both_full_batch_equals_separate_calls(config, method):
    """The fused receiver at the benched size (1000 x 512^2, one launch with three CTA roles):
    every image's payload words, bit count, recovered image and status equal the separate calls'."""
    imgs, k1, k2 = S.batch(config)
    B, H, W = imgs.shape
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    I, K1, K2 = dev(imgs), dev(k1), dev(k2)
    ws = G.Workspace(method, B, H, W)
    enc, b, cap, st_e = G.encode(method, I, K1, ws)
    nb = (cap - 32).clamp(min=0)
    stride = int(((int(nb.max()) + 7) // 8 + 4 + 15) // 16 * 16)
    msgs = torch.randint(0, 256, (B, stride), dtype=torch.uint8, generator=torch.Generator().manual_seed(config)).cuda()
    marked, st_h = G.embed(method, enc, K2, msgs, nb, ws)
    mo, nbo, st_x = G.extract(method, marked, K2, stride, ws)
    rec, st_r = G.recover(method, marked, K1, ws)
    mo2, nb2, rec2, st2 = G.receive_both(method, marked, K1, K2, stride, ws)
    torch.cuda.synchronize()
    assert torch.equal(nbo, nb2) and torch.equal(nb2, nb)
    assert torch.equal(rec, rec2) and torch.equal(mo, mo2)
    assert int((st2 != 0).sum()) == 0 and int((st_x != 0).sum()) == 0 and int((st_r != 0).sum()) == 0
