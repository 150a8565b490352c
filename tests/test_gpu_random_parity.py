"""Seeded random sweep of the parameter space (shape incl. non-square and 16-pixel sides, method,
coder tile size, LMR schedule, cipher rounds, image kind, message length incl. empty / partial /
over capacity): every output of the four calls bit-exact against the oracle."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2302_07992_b200 import mmsb as G
from paper_2302_07992_b200 import synth as S

pytestmark = pytest.mark.gpu

KINDS = ["smooth", "textured", "noise", "constant", "quantised"]


def _cases(n=64, seed=31337):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        H = int(2 ** rng.integers(4, 10))
        W = int(2 ** rng.integers(4, 10))
        method = int(rng.integers(0, 2))
        t = int(rng.integers(3, 8))
        emin = int(rng.integers(0, 4)) if method == 1 else 0
        rounds = int(rng.choice([20, 20, 12, 8]))
        kinds = [KINDS[int(k)] for k in rng.integers(0, len(KINDS), 3)]
        mode = int(rng.integers(0, 4))             # 0 full, 1 partial, 2 empty, 3 one bit over
        out.append((i, H, W, method, t, emin, rounds, kinds, mode))
    return out


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"c{c[0]}_{c[1]}x{c[2]}_m{c[3]}_t{c[4]}_e{c[5]}_r{c[6]}")
def test_random_parity(case):
    i, H, W, method, t, emin, rounds, kinds, mode = case
    B = len(kinds)
    imgs = np.stack([S.random_image(4000 + 10 * i + j, H, W, k) for j, k in enumerate(kinds)])
    k1 = np.stack([np.frombuffer(S.key(4000 + 10 * i + j, 1), np.uint8) for j in range(B)])
    k2 = np.stack([np.frombuffer(S.key(4000 + 10 * i + j, 2), np.uint8) for j in range(B)])
    stride = S.msg_stride(H, W)
    msgs = np.stack([S.payload(4000 + 10 * i + j, stride) for j in range(B)])
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    ws = G.Workspace(method, B, H, W, tile_log2=t, lmr_emin=emin, cipher_rounds=rounds)
    enc, b, cap, st = G.encode(method, dev(imgs), dev(k1), ws, tile_log2=t)
    torch.cuda.synchronize()
    c = cap.cpu().numpy().astype(np.int64)
    nbits = {0: np.maximum(c - 32, 0), 1: np.maximum(c - 32, 0) // 3, 2: np.zeros_like(c), 3: c - 31}[mode]
    nbits = np.where(c > 0, nbits, 0)
    marked, st_h = G.embed(method, enc, dev(k2), dev(msgs), dev(nbits), ws, tile_log2=t)
    mo, nb_out, st_x = G.extract(method, marked, dev(k2), stride, ws, tile_log2=t)
    rec, st_r = G.recover(method, marked, dev(k1), ws, tile_log2=t)
    torch.cuda.synchronize()
    try:
        O.set_cipher_rounds(rounds)
        for j in range(B):
            so, E, bo, Co = O.encode(method, imgs[j], k1[j].tobytes(), tile_log2=t, lmr_emin=emin)
            assert (int(st[j]), int(b[j]), int(cap[j])) == (so, bo, Co), (j, "encode")
            assert np.array_equal(enc[j].cpu().numpy(), E), (j, "I_e")
            sh, Em = O.hide(method, E, k2[j].tobytes(), msgs[j], int(nbits[j]), tile_log2=t)
            assert int(st_h[j]) == sh, (j, "hide status", int(st_h[j]), sh)
            if sh in (O.OK, O.E_CAPACITY):
                assert np.array_equal(marked[j].cpu().numpy(), Em), (j, "I_e'")
            else:
                Em = marked[j].cpu().numpy()
            sx, mox, nbx = O.extract(method, Em, k2[j].tobytes(), stride, tile_log2=t)
            assert (int(st_x[j]), int(nb_out[j])) == (sx, nbx), (j, "extract")
            if sx == O.OK:
                assert np.array_equal(mo[j].cpu().numpy()[: (nbx + 7) // 8], mox[: (nbx + 7) // 8]), (j, "payload")
            sr, R = O.recover(method, Em, k1[j].tobytes(), tile_log2=t, lmr_emin=emin)
            assert int(st_r[j]) == sr, (j, "recover status")
            assert np.array_equal(rec[j].cpu().numpy(), R), (j, "I'")
    finally:
        O.set_cipher_rounds(20)
