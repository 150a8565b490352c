"""GPU <-> oracle parity for LMR-RDHEI through the C ABI (bit-exact on every output):
encrypted image with the coded maps in the MSB plane, b, capacity, status (incl. BADCASE),
marked image, extracted payload and the losslessly recovered image."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2302_07992_b200 import mmsb as G
from paper_2302_07992_b200 import synth as S

pytestmark = pytest.mark.gpu


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _run(imgs, k1, k2, msgs, t, nbits=None):
    B, H, W = imgs.shape
    stride = msgs.shape[1]
    ws = G.Workspace(G.LMR, B, H, W, tile_log2=t)
    I, K1, K2 = _dev(imgs), _dev(k1), _dev(k2)
    enc, b, cap, st_e = G.encode(G.LMR, I, K1, ws, tile_log2=t)
    nb = _dev(np.asarray(nbits, np.int64)) if nbits is not None else (cap - 32).clamp(min=0)
    marked, st_h = G.embed(G.LMR, enc, K2, _dev(msgs), nb, ws, tile_log2=t)
    mo, nb_out, st_x = G.extract(G.LMR, marked, K2, stride, ws, tile_log2=t)
    rec, st_r = G.recover(G.LMR, marked, K1, ws, tile_log2=t)
    torch.cuda.synchronize()
    c = lambda x: x.cpu().numpy()
    return dict(enc=c(enc), b=c(b), cap=c(cap), st_e=c(st_e), nbits=c(nb), marked=c(marked), st_h=c(st_h),
                msg=c(mo), nb_out=c(nb_out), st_x=c(st_x), rec=c(rec), st_r=c(st_r))


def _check(imgs, k1, k2, msgs, t, out):
    stride = msgs.shape[1]
    for j in range(imgs.shape[0]):
        st, E, b, C = O.encode(O.LMR, imgs[j], k1[j].tobytes(), tile_log2=t)
        assert out["st_e"][j] == st, (j, out["st_e"][j], st)
        assert out["b"][j] == b and out["cap"][j] == C, (j, out["b"][j], b, out["cap"][j], C)
        assert np.array_equal(out["enc"][j], E), (j, np.argwhere(out["enc"][j] != E)[:5])
        n = int(out["nbits"][j])
        st2, Em = O.hide(O.LMR, E, k2[j].tobytes(), msgs[j], n, tile_log2=t)
        assert out["st_h"][j] == st2, (j, out["st_h"][j], st2)
        if st2 in (O.OK, O.E_CAPACITY):
            assert np.array_equal(out["marked"][j], Em), (j, np.argwhere(out["marked"][j] != Em)[:5])
        else:
            Em = out["marked"][j]
        st3, mo, nbo = O.extract(O.LMR, Em, k2[j].tobytes(), stride, tile_log2=t)
        assert out["st_x"][j] == st3 and out["nb_out"][j] == nbo, (j, out["st_x"][j], st3, out["nb_out"][j], nbo)
        region = 4 * ((C - 32 + 31) // 32) if C > 32 else 0
        assert np.array_equal(out["msg"][j][:region], mo[:region])
        st4, R = O.recover(O.LMR, Em, k1[j].tobytes(), tile_log2=t)
        assert out["st_r"][j] == st4
        assert np.array_equal(out["rec"][j], R), (j, np.argwhere(out["rec"][j] != R)[:5])
        if st4 == O.OK:
            assert np.array_equal(R, imgs[j])                  # lossless


@pytest.mark.parametrize("H,W,t", [(32, 32, 7), (64, 64, 7), (128, 128, 7), (64, 256, 7), (256, 64, 6), (128, 128, 5),
                                   (64, 64, 3), (256, 256, 7), (16, 16, 7)])
def test_lmr_parity_small(H, W, t):
    kinds = ["smooth", "smooth", "textured", "constant", "noise", "quantised"]
    imgs = np.stack([S.random_image(300 + j, H, W, k) for j, k in enumerate(kinds)])
    k1 = np.stack([np.frombuffer(S.key(300 + j, 1), np.uint8) for j in range(len(kinds))])
    k2 = np.stack([np.frombuffer(S.key(300 + j, 2), np.uint8) for j in range(len(kinds))])
    stride = S.msg_stride(H, W)
    msgs = np.stack([S.payload(700 + j, stride) for j in range(len(kinds))])
    _check(imgs, k1, k2, msgs, t, _run(imgs, k1, k2, msgs, t))


def test_lmr_parity_512_config3_sample():
    imgs, k1, k2 = S.batch(3, n=4)                    # alternating smooth / textured (alpha 2 / 1)
    stride = S.msg_stride(512, 512)
    msgs = np.stack([S.payload(S.image_seed(3, j), stride) for j in range(4)])
    out = _run(imgs, k1, k2, msgs, 7)
    _check(imgs, k1, k2, msgs, 7, out)
    assert (out["st_r"] == 0).all() and np.array_equal(out["rec"], imgs)


def test_lmr_partial_and_capacity():
    H = W = 128
    imgs = np.stack([S.random_image(40 + j, H, W, "smooth") for j in range(4)])
    k1 = np.stack([np.frombuffer(S.key(40 + j, 1), np.uint8) for j in range(4)])
    k2 = np.stack([np.frombuffer(S.key(40 + j, 2), np.uint8) for j in range(4)])
    stride = S.msg_stride(H, W)
    msgs = np.stack([S.payload(60 + j, stride) for j in range(4)])
    caps = [O.encode(O.LMR, imgs[j], k1[j].tobytes())[3] for j in range(4)]
    nbits = [0, caps[1] - 32, caps[2] - 31, caps[3] // 2]
    out = _run(imgs, k1, k2, msgs, 7, nbits)
    assert out["st_h"][2] == O.E_CAPACITY
    _check(imgs, k1, k2, msgs, 7, out)


@pytest.mark.parametrize("emin", [1, 2, 3])
def test_lmr_schedule_variants_parity(emin):
    """Tab. LMR_block_size schedules: rotation blocks {2^e_min..}, bit-exact with the oracle."""
    H = W = 128
    kinds = ["smooth", "textured", "smooth", "constant"]
    imgs = np.stack([S.random_image(9100 + j, H, W, k) for j, k in enumerate(kinds)])
    k1 = np.stack([np.frombuffer(S.key(9100 + j, 1), np.uint8) for j in range(len(kinds))])
    k2 = np.stack([np.frombuffer(S.key(9100 + j, 2), np.uint8) for j in range(len(kinds))])
    stride = S.msg_stride(H, W)
    msgs = np.stack([S.payload(j, stride) for j in range(len(kinds))])
    ws = G.Workspace(G.LMR, len(kinds), H, W, lmr_emin=emin)
    enc, b, cap, st_e = G.encode(G.LMR, _dev(imgs), _dev(k1), ws)
    marked, st_h = G.embed(G.LMR, enc, _dev(k2), _dev(msgs), (cap - 32).clamp(min=0), ws)
    rec, st_r = G.recover(G.LMR, marked, _dev(k1), ws)
    torch.cuda.synchronize()
    for j in range(len(kinds)):
        st, E, bo, Co = O.encode(O.LMR, imgs[j], k1[j].tobytes(), lmr_emin=emin)
        assert int(st_e[j]) == st and int(b[j]) == bo and int(cap[j]) == Co
        assert np.array_equal(enc[j].cpu().numpy(), E)
        if st != O.OK:
            continue
        _, Em = O.hide(O.LMR, E, k2[j].tobytes(), msgs[j], Co - 32)
        assert np.array_equal(marked[j].cpu().numpy(), Em)
        _, R = O.recover(O.LMR, Em, k1[j].tobytes(), lmr_emin=emin)
        assert np.array_equal(rec[j].cpu().numpy(), R) and np.array_equal(R, imgs[j])
