"""GPU <-> oracle parity on altered inputs: receivers fed images whose headers, coded-stream tables
or payload were changed after encoding must produce exactly the oracle's statuses and outputs
(FORMAT / BADCASE / INTEGRITY, and for LMR streams that no longer match their tables, the same
decoded garbage -- the decoder reads bytes past a stream's end as 0, O15)."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2302_07992_b200 import mmsb as G
from paper_2302_07992_b200 import synth as S

pytestmark = pytest.mark.gpu


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _marked(method, n, H=128, W=128, seed=900):
    imgs = np.stack([S.random_image(seed + j, H, W, "smooth") for j in range(n)])
    k1 = np.stack([np.frombuffer(S.key(seed + j, 1), np.uint8) for j in range(n)])
    k2 = np.stack([np.frombuffer(S.key(seed + j, 2), np.uint8) for j in range(n)])
    stride = S.msg_stride(H, W)
    msgs = np.stack([S.payload(seed + j, stride) for j in range(n)])
    out = []
    for j in range(n):
        st, E, b, C = O.encode(method, imgs[j], k1[j].tobytes())
        assert st == O.OK
        _, Em = O.hide(method, E, k2[j].tobytes(), msgs[j], C - 32)
        out.append(Em)
    return np.stack(out), k1, k2, stride


def _set_msb_bits(img, r0, bits):
    """overwrite the MSB-plane bits r0.. (pixel r's MSB = plane bit r, raster order)"""
    flat = img.ravel()
    for i, bit in enumerate(bits):
        flat[r0 + i] = (flat[r0 + i] & 0x7F) | (bit << 7)


def _receivers_match(method, X, k1, k2, stride):
    B = X.shape[0]
    mo, nb, st_x = G.extract(method, _dev(X), _dev(k2), stride)
    rec, st_r = G.recover(method, _dev(X), _dev(k1))
    bq, cq, sq = G.capacity(method, _dev(X))
    torch.cuda.synchronize()
    for j in range(B):
        sx, mox, nbx = O.extract(method, X[j], k2[j].tobytes(), stride)
        assert (int(st_x[j]), int(nb[j])) == (sx, nbx), (j, int(st_x[j]), sx, int(nb[j]), nbx)
        if sx == O.OK:
            n = int(nbx)
            assert np.array_equal(mo[j].cpu().numpy()[: (n + 7) // 8], mox[: (n + 7) // 8])
        sr, R = O.recover(method, X[j], k1[j].tobytes())
        assert int(st_r[j]) == sr, (j, int(st_r[j]), sr)
        assert np.array_equal(rec[j].cpu().numpy(), R), (j, np.argwhere(rec[j].cpu().numpy() != R)[:5])
        assert (int(sq[j]), int(bq[j]), int(cq[j])) == O.capacity(method, X[j])


def test_emr_altered_inputs():
    X, k1, k2, stride = _marked(G.EMR, 4)
    X = X.copy()
    X[0, 0, :3] |= 1                                   # b-field 7: FORMAT
    k2 = k2.copy()
    k2[1] ^= 0x5A                                      # wrong K2: the decrypted length is garbage (INTEGRITY)
    X[2].ravel()[1000:1400] ^= 1                       # LSBs (map / carriers) flipped
    _receivers_match(G.EMR, X, k1, k2, stride)


def test_lmr_altered_headers_and_tables():
    X, k1, k2, stride = _marked(G.LMR, 6)
    X = X.copy()
    H, W = X.shape[1:]
    T = O.tile_count(H, W, 7)
    _set_msb_bits(X[0], 3, [1, 0, 0, 1])               # t field 9 != 7: FORMAT
    _set_msb_bits(X[1], 0, [1, 1, 1])                  # b-field 7: BADCASE
    # a stream length changed: later streams shift, the decoder runs past ends / into neighbours
    sz_bits = [int(b) for b in format(5, "016b")]
    _set_msb_bits(X[2], 7, sz_bits)                    # first eta tile length := 5 bytes
    _set_msb_bits(X[3], 7 + 16 * T, [1] * 16)          # first map tile length := 65535: over the plane -> FORMAT
    X[4].ravel()[7 + 32 * T + 64:7 + 32 * T + 512] ^= 0x80   # coded bytes flipped
    _receivers_match(G.LMR, X, k1, k2, stride)
