"""GPU <-> oracle parity with the reduced-round keystream option (mmsb_shape.cipher_rounds = 12 / 8;
SURVEY §8(f) NEXT 4): every output of the four calls bit-exact against the oracle run with the same
rounds, for EMR and LMR; and the option really changes the keystream (ChaCha20 outputs differ)."""
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
@pytest.mark.parametrize("rounds", [8, 12])
def test_reduced_rounds_parity(method, rounds):
    H = W = 128
    kinds = ["smooth", "textured", "smooth", "quantised"]
    imgs = np.stack([S.random_image(800 + j, H, W, k) for j, k in enumerate(kinds)])
    k1 = np.stack([np.frombuffer(S.key(800 + j, 1), np.uint8) for j in range(len(kinds))])
    k2 = np.stack([np.frombuffer(S.key(800 + j, 2), np.uint8) for j in range(len(kinds))])
    stride = S.msg_stride(H, W)
    msgs = np.stack([S.payload(j, stride) for j in range(len(kinds))])
    ws = G.Workspace(method, len(kinds), H, W, cipher_rounds=rounds)
    enc, b, cap, st = G.encode(method, _dev(imgs), _dev(k1), ws)
    nb = (cap - 32).clamp(min=0)
    marked, st_h = G.embed(method, enc, _dev(k2), _dev(msgs), nb, ws)
    mo, nbo, st_x = G.extract(method, marked, _dev(k2), stride, ws)
    rec, st_r = G.recover(method, marked, _dev(k1), ws)
    torch.cuda.synchronize()
    ws20 = G.Workspace(method, len(kinds), H, W)
    enc20 = G.encode(method, _dev(imgs), _dev(k1), ws20)[0]
    torch.cuda.synchronize()
    assert not torch.equal(enc20, enc)                    # a different keystream
    try:
        O.set_cipher_rounds(rounds)
        for j in range(len(kinds)):
            so, E, bo, Co = O.encode(method, imgs[j], k1[j].tobytes())
            assert (int(st[j]), int(b[j]), int(cap[j])) == (so, bo, Co)
            assert np.array_equal(enc[j].cpu().numpy(), E)
            if so != O.OK:
                continue
            n = int(nb[j])
            _, Em = O.hide(method, E, k2[j].tobytes(), msgs[j], n)
            assert np.array_equal(marked[j].cpu().numpy(), Em)
            sx, mox, nbx = O.extract(method, Em, k2[j].tobytes(), stride)
            assert int(nbo[j]) == nbx and int(st_x[j]) == sx
            region = 4 * ((Co - 32 + 31) // 32) if Co > 32 else 0
            assert np.array_equal(mo[j].cpu().numpy()[:region], mox[:region])
            sr, R = O.recover(method, Em, k1[j].tobytes())
            assert int(st_r[j]) == sr and np.array_equal(rec[j].cpu().numpy(), R)
    finally:
        O.set_cipher_rounds(20)
