"""GPU <-> oracle parity for EMR-RDHEI through the C ABI (bit-exact on every output).

Inputs come from paper_2302_07992_b200.synth (seeded); expected values from oracle/ only.
Sizes span several 64x64 tiles, several 8192-pixel scan chunks and the small-tile
templates (16x16, 32x32), plus non-square and full-size (512^2, 4096^2) images.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2302_07992_b200 import mmsb as G
from paper_2302_07992_b200 import synth as S

pytestmark = pytest.mark.gpu


def _batch(shapes_kind, H, W, seed0):
    imgs, k1, k2 = [], [], []
    for j, kind in enumerate(shapes_kind):
        imgs.append(S.random_image(seed0 + j, H, W, kind))
        k1.append(np.frombuffer(S.key(seed0 + j, 1), np.uint8))
        k2.append(np.frombuffer(S.key(seed0 + j, 2), np.uint8))
    return np.stack(imgs), np.stack(k1), np.stack(k2)


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _run_gpu(imgs, k1, k2, msgs, nbits, stride):
    B, H, W = imgs.shape
    ws = G.Workspace(G.EMR, B, H, W)
    I, K1, K2 = _dev(imgs), _dev(k1), _dev(k2)
    enc, b, cap, st_e = G.encode(G.EMR, I, K1, ws)
    nb = _dev(np.asarray(nbits, np.int64)) if nbits is not None else (cap - 32).clamp(min=0)
    marked, st_h = G.embed(G.EMR, enc, K2, _dev(msgs), nb, ws)
    msg_out, nb_out, st_x = G.extract(G.EMR, marked, K2, stride, ws)
    rec, st_r = G.recover(G.EMR, marked, K1, ws)
    sse = G.stats(I, rec)
    torch.cuda.synchronize()
    c = lambda t: t.cpu().numpy()
    return dict(enc=c(enc), b=c(b), cap=c(cap), st_e=c(st_e), nbits=c(nb), marked=c(marked), st_h=c(st_h),
                msg=c(msg_out), nb_out=c(nb_out), st_x=c(st_x), rec=c(rec), st_r=c(st_r), sse=c(sse))


def _check_against_oracle(imgs, k1, k2, msgs, stride, out, idx=None):
    B = imgs.shape[0]
    for j in (range(B) if idx is None else idx):
        st, E, b, C = O.encode(O.EMR, imgs[j], k1[j].tobytes())
        assert out["st_e"][j] == st
        assert out["b"][j] == b, (j, out["b"][j], b)
        assert out["cap"][j] == C, (j, out["cap"][j], C)
        assert np.array_equal(out["enc"][j], E), (j, np.argwhere(out["enc"][j] != E)[:5])
        n = int(out["nbits"][j])
        st2, Em = O.hide(O.EMR, E, k2[j].tobytes(), msgs[j], n)
        assert out["st_h"][j] == st2, (j, out["st_h"][j], st2)
        assert np.array_equal(out["marked"][j], Em), (j, np.argwhere(out["marked"][j] != Em)[:5])
        st3, mo, nbo = O.extract(O.EMR, Em, k2[j].tobytes(), stride)
        assert out["st_x"][j] == st3 and out["nb_out"][j] == nbo, (j, out["st_x"][j], st3, out["nb_out"][j], nbo)
        region = 4 * ((C - 32 + 31) // 32) if C > 32 else 0
        assert np.array_equal(out["msg"][j][:region], mo[:region])
        st4, R = O.recover(O.EMR, Em, k1[j].tobytes())
        assert out["st_r"][j] == st4
        assert np.array_equal(out["rec"][j], R), (j, np.argwhere(out["rec"][j] != R)[:5])
        assert out["sse"][j] == O.sse(imgs[j], R)


@pytest.mark.parametrize("H,W", [(16, 16), (32, 32), (64, 64), (128, 128), (64, 256), (256, 64), (16, 128),
                                 (256, 256)])
def test_emr_parity_small(H, W):
    kinds = ["smooth", "textured", "noise", "constant", "quantised", "smooth"]
    imgs, k1, k2 = _batch(kinds, H, W, 1000 + H + W)
    stride = S.msg_stride(H, W)
    msgs = np.stack([S.payload(500 + j, stride) for j in range(len(kinds))])
    out = _run_gpu(imgs, k1, k2, msgs, None, stride)
    _check_against_oracle(imgs, k1, k2, msgs, stride, out)


def test_emr_parity_partial_messages_and_capacity():
    H = W = 128
    imgs, k1, k2 = _batch(["smooth"] * 6, H, W, 77)
    stride = S.msg_stride(H, W)
    msgs = np.stack([S.payload(900 + j, stride) for j in range(6)])
    caps = [O.encode(O.EMR, imgs[j], k1[j].tobytes())[3] for j in range(6)]
    nbits = [0, 1, caps[2] - 32, caps[3] - 31, 12345 % max(caps[4] - 32, 1), caps[5] // 3]
    out = _run_gpu(imgs, k1, k2, msgs, nbits, stride)
    assert out["st_h"][3] == O.E_CAPACITY and np.array_equal(out["marked"][3], out["enc"][3])
    _check_against_oracle(imgs, k1, k2, msgs, stride, out)


def test_emr_parity_512_config2_sample():
    imgs, k1, k2 = S.batch(2, n=6)
    stride = S.msg_stride(512, 512)
    msgs = np.stack([S.payload(S.image_seed(2, j), stride) for j in range(6)])
    out = _run_gpu(imgs, k1, k2, msgs, None, stride)
    _check_against_oracle(imgs, k1, k2, msgs, stride, out)
    der, psnr = G.der_psnr(512, 512, out["cap"], out["sse"])
    for j in range(6):
        d, p = O.der_psnr(512, 512, int(out["cap"][j]), int(out["sse"][j]))
        assert der[j] == pytest.approx(d, rel=1e-12) and psnr[j] == pytest.approx(p, rel=1e-12)
        assert abs(psnr[j] - 51.1411) < 0.15


def test_emr_wrong_key_and_bad_header():
    H = W = 64
    imgs, k1, k2 = _batch(["smooth"] * 3, H, W, 5)
    stride = S.msg_stride(H, W)
    msgs = np.stack([S.payload(j, stride) for j in range(3)])
    out = _run_gpu(imgs, k1, k2, msgs, None, stride)
    marked = out["marked"].copy()
    marked[2].ravel()[0] |= 1
    marked[2].ravel()[1] |= 1                         # b-field 6: FORMAT
    bad_k2 = k2.copy()
    bad_k2[0, 0] ^= 1
    ws = G.Workspace(G.EMR, 3, H, W)
    mo, nb, st = G.extract(G.EMR, _dev(marked), _dev(bad_k2), stride, ws)
    rec, st_r = G.recover(G.EMR, _dev(marked), _dev(k1), ws)
    torch.cuda.synchronize()
    for j in range(3):
        so, mo_o, nbo = O.extract(O.EMR, marked[j], bad_k2[j].tobytes(), stride)
        assert st.cpu()[j] == so and nb.cpu()[j] == nbo
        _, E, _, C = O.encode(O.EMR, imgs[j], k1[j].tobytes())
        region = 4 * ((C - 32 + 31) // 32) if C > 32 else 0
        if so != O.E_FORMAT:
            assert np.array_equal(mo.cpu().numpy()[j][:region], mo_o[:region])
        sr, R = O.recover(O.EMR, marked[j], k1[j].tobytes())
        assert st_r.cpu()[j] == sr and np.array_equal(rec.cpu().numpy()[j], R)


@pytest.mark.slow
def test_emr_parity_4096_config5_sample():
    img = S.image(5, 0)[None]
    seed = S.image_seed(5, 0)
    k1 = np.frombuffer(S.key(seed, 1), np.uint8)[None]
    k2 = np.frombuffer(S.key(seed, 2), np.uint8)[None]
    stride = S.msg_stride(4096, 4096)
    msgs = S.payload(seed, stride)[None]
    out = _run_gpu(img, k1, k2, msgs, None, stride)
    _check_against_oracle(img, k1, k2, msgs, stride, out)


@pytest.mark.parametrize("method", [G.EMR, G.LMR])
def test_embed_in_place_equals_out_of_place(method):
    """mmsb_hider_embed with marked aliasing encrypted: the same marked image and
    statuses as out of place, including a CAPACITY image (left unchanged) and an empty message."""
    H = W = 128
    kinds = ["smooth", "textured", "smooth", "quantised"]
    imgs = np.stack([S.random_image(950 + j, H, W, k) for j, k in enumerate(kinds)])
    k1 = np.stack([np.frombuffer(S.key(950 + j, 1), np.uint8) for j in range(len(kinds))])
    k2 = np.stack([np.frombuffer(S.key(950 + j, 2), np.uint8) for j in range(len(kinds))])
    stride = S.msg_stride(H, W)
    msgs = np.stack([S.payload(j, stride) for j in range(len(kinds))])
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    enc, b, cap, st = G.encode(method, dev(imgs), dev(k1))
    nb = (cap - 32).clamp(min=0)
    nb[1] = cap[1] - 31                                  # one bit over: CAPACITY
    nb[3] = 0
    ref, st_ref = G.embed(method, enc, dev(k2), dev(msgs), nb)
    inplace = enc.clone()
    out, st_in = G.embed(method, inplace, dev(k2), dev(msgs), nb, out=inplace)
    torch.cuda.synchronize()
    assert out.data_ptr() == inplace.data_ptr()
    assert torch.equal(st_in, st_ref) and torch.equal(inplace, ref)
    assert int(st_ref[1]) == O.E_CAPACITY and torch.equal(ref[1], enc[1])
