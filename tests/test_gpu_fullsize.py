"""Full-size parity in the launch configuration bench.py times: BASELINE.json configs 2 (1000 x 512^2,
EMR) and 3 (1000 x 512^2, LMR) as ONE batch per call (the fused kernels' role grid, lead rows and
image groups at full size), checked on sampled images against the oracle image by image, plus
batch-wide properties (payload round trip, LMR losslessness, EMR bits 1..7 intact).  Also: two
batches on two streams at once (the library keeps no state between calls besides the caller's
workspace)."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2302_07992_b200 import mmsb as G
from paper_2302_07992_b200 import synth as S

pytestmark = pytest.mark.gpu


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("config,method", [(2, G.EMR), (3, G.LMR)])
def test_full_batch_sampled_parity(config, method):
    imgs, k1, k2 = S.batch(config)
    B, H, W = imgs.shape
    I, K1, K2 = _dev(imgs), _dev(k1), _dev(k2)
    ws = G.Workspace(method, B, H, W)
    enc, b, cap, st_e = G.encode(method, I, K1, ws)
    nb = (cap - 32).clamp(min=0)
    stride = int(((int(nb.max()) + 7) // 8 + 4 + 15) // 16 * 16)
    rng = np.random.default_rng(config)
    msgs = rng.integers(0, 256, size=(B, stride), dtype=np.uint8)
    marked, st_h = G.embed(method, enc, K2, _dev(msgs), nb, ws)
    mo, nbo, st_x = G.extract(method, marked, K2, stride, ws)
    rec, st_r = G.recover(method, marked, K1, ws)
    torch.cuda.synchronize()
    assert (st_e == 0).all() and (st_h == 0).all() and (st_x == 0).all() and (st_r == 0).all()
    assert torch.equal(nbo, nb)
    # payload round trip for every image: the extracted bits equal the embedded ones
    bits_in = np.unpackbits(msgs, axis=1)
    bits_out = np.unpackbits(mo.cpu().numpy(), axis=1)
    nbn = nb.cpu().numpy()
    for j in range(0, B, 37):
        assert np.array_equal(bits_in[j, :nbn[j]], bits_out[j, :nbn[j]])
    R = rec.cpu().numpy()
    if method == G.LMR:
        assert np.array_equal(R, imgs)                                     # lossless
    else:
        assert np.array_equal(R >> 1, imgs >> 1)                           # only LSBs differ
    # sampled images against the oracle, every output
    for j in sorted(set(rng.integers(0, B, size=4).tolist()) | {0, B - 1}):
        st, E, bo, Co = O.encode(method, imgs[j], k1[j].tobytes())
        assert (int(b[j]), int(cap[j])) == (bo, Co) and np.array_equal(enc[j].cpu().numpy(), E)
        _, Em = O.hide(method, E, k2[j].tobytes(), msgs[j], int(nbn[j]))
        assert np.array_equal(marked[j].cpu().numpy(), Em)
        _, R_o = O.recover(method, Em, k1[j].tobytes())
        assert np.array_equal(R[j], R_o)


def test_two_streams_at_once():
    H = W = 256
    out = []
    for seed0 in (11000, 12000):
        imgs = np.stack([S.random_image(seed0 + j, H, W, "smooth") for j in range(24)])
        k1 = np.stack([np.frombuffer(S.key(seed0 + j, 1), np.uint8) for j in range(24)])
        out.append((imgs, k1))
    ref = []
    for imgs, k1 in out:                                                     # sequential reference
        enc, _, _, _ = G.encode(G.EMR, _dev(imgs), _dev(k1))
        rec, _ = G.recover(G.EMR, enc, _dev(k1))
        ref.append((enc.cpu(), rec.cpu()))
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    res = [None, None]
    inputs = [(_dev(i), _dev(k)) for i, k in out]
    wss = [G.Workspace(G.EMR, 24, H, W), G.Workspace(G.EMR, 24, H, W)]
    torch.cuda.synchronize()
    for r in range(3):
        for s in (0, 1):
            with torch.cuda.stream(streams[s]):
                I, K = inputs[s]
                enc, _, _, _ = G.encode(G.EMR, I, K, wss[s])
                rec, _ = G.recover(G.EMR, enc, K, wss[s])
                res[s] = (enc, rec)
        torch.cuda.synchronize()
        for s in (0, 1):
            assert torch.equal(res[s][0].cpu(), ref[s][0]) and torch.equal(res[s][1].cpu(), ref[s][1])
