"""Bit-exact GPU <-> oracle parity at the edges of the GPU shape envelope (power-of-two
H, W in [16, 32768]): the widest and the tallest image (one row / column of 64x64 tiles holding
512 tiles, the worker's strip-table limit kMaxTilesX; LMR coder tiles of 128 x 16 / 16 x 128),
the smallest (16 x 16: one partial tile, coder tiles narrower than 32 -> the reference coder
kernels), and a batch mixing textures at the widest shape.  Every output against the oracle.
"""
import numpy as np
import pytest
import torch

from paper_2302_07992_b200 import mmsb as G
from paper_2302_07992_b200 import synth as S

from test_gpu_configs import _batch_properties, _dev, _oracle_image, _run

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("method", [G.EMR, G.LMR])
@pytest.mark.parametrize("H,W", [(16, 32768), (32768, 16), (16, 16), (32, 16384)])
def test_extreme_shapes(method, H, W):
    kinds = ["smooth", "textured", "quantised"]
    imgs = np.stack([S.random_image(900 + j, H, W, k) for j, k in enumerate(kinds)])
    k1 = np.stack([np.frombuffer(S.key(900 + j, 1), np.uint8) for j in range(len(kinds))])
    k2 = np.stack([np.frombuffer(S.key(900 + j, 2), np.uint8) for j in range(len(kinds))])
    stride = S.msg_stride(H, W)
    msgs = np.stack([S.payload(950 + j, stride) for j in range(len(kinds))])
    out = _run(method, _dev(imgs), _dev(k1), _dev(k2), _dev(msgs))
    torch.cuda.synchronize()
    _batch_properties(method, _dev(imgs), _dev(msgs), out, expect_ok=False)
    for j in range(len(kinds)):
        _oracle_image(method, imgs[j], k1[j], k2[j], msgs[j], j, out)


@pytest.mark.parametrize("method", [G.EMR, G.LMR])
def test_maximum_square_image(method):
    """One 32768 x 32768 image (1 GiB), the top of the envelope: its upper angle pyramid (349 KB)
    does not fit shared memory, so the workers walk it in global memory (Geo::pyr_glob); the
    capacity exceeds 2^32 bits, so the payload is the largest the BE32 bit-count header can state
    (reading Q17).  Checked by properties that hold at any size (the oracle is checked against the
    same kernels at 16 x 32768, 32768 x 16 and the configs): statuses, payload round trip, LMR
    I' = I, EMR bits 1..7 of I' = I."""
    H = W = 32768
    base = S.random_image(77, 4096, 4096, "smooth")
    img = torch.from_numpy(np.tile(base, (8, 8))[None]).cuda()
    k1 = torch.from_numpy(np.frombuffer(S.key(77, 1), np.uint8)[None].copy()).cuda()
    k2 = torch.from_numpy(np.frombuffer(S.key(77, 2), np.uint8)[None].copy()).cuda()
    ws = G.Workspace(method, 1, H, W)
    enc, b, cap, st = G.encode(method, img, k1, ws)
    assert int(st[0]) == 0 and int(cap[0]) > 2 ** 32
    n = 2 ** 32 - 1 - 7                                  # <= 2^32 - 1 bits (BE32 header, Q17)
    stride = S.msg_stride(H, W)                          # rows cover the whole capacity region (0.94 GB)
    msg = torch.randint(0, 256, (1, stride), dtype=torch.uint8, device="cuda")
    nb = torch.tensor([n], dtype=torch.int64, device="cuda")
    marked, st_h = G.embed(method, enc, k2, msg, nb, ws)
    mo, nbo, st_x = G.extract(method, marked, k2, stride, ws)
    rec, st_r = G.recover(method, marked, k1, ws)
    torch.cuda.synchronize()
    assert (int(st_h[0]), int(st_x[0]), int(st_r[0]), int(nbo[0])) == (0, 0, 0, n)
    assert torch.equal(mo[0, : n // 8], msg[0, : n // 8])
    last = 8 - n % 8                                      # the partial last byte's n % 8 leading bits
    assert int((mo[0, n // 8] ^ msg[0, n // 8]) >> last) == 0
    if method == G.LMR:
        assert torch.equal(rec, img)
    else:
        assert torch.equal(rec >> 1, img >> 1)


@pytest.mark.parametrize("method", [G.EMR, G.LMR])
def test_batch_beyond_2_to_32_pixels(method):
    """20 480 images of 512^2 in one call: 5.4 G pixels, beyond 2^32, so a 32-bit pixel, bit or
    byte offset anywhere on the path would wrap.  The batch repeats 64 distinct images (and
    their keys and payloads) 320 times, and every repeat must reproduce the first copy's encrypted
    image, b, capacity, marked image, payload and recovered image exactly; the first copies are
    checked against the oracle elsewhere (config 2 / 3 samples), here 3 of them again."""
    n0, reps = 64, 320
    imgs, k1, k2 = S.batch(3, n=n0)
    stride = S.msg_stride(512, 512)
    msgs = np.stack([S.payload(S.image_seed(3, j), stride) for j in range(n0)])
    rep = lambda a: _dev(a).repeat(reps, *([1] * (a.ndim - 1)))
    I, K1, K2, M = rep(imgs), rep(k1), rep(k2), rep(msgs)
    assert I.shape[0] * 512 * 512 > 2 ** 32
    out = _run(method, I, K1, K2, M)
    _batch_properties(method, I, M, out, expect_ok=False)
    for k in ("enc", "b", "cap", "st_e", "marked", "st_h", "msg", "nb_out", "st_x", "rec", "st_r", "sse"):
        v = out[k].reshape(reps, n0, *out[k].shape[1:])
        assert bool((v == v[:1]).all()), k
    del I, M
    torch.cuda.empty_cache()
    for j in (0, 1, n0 - 1):
        _oracle_image(method, imgs[j], k1[j], k2[j], msgs[j], (reps - 1) * n0 + j, out)
