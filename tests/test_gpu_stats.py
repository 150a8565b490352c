"""GPU <-> oracle parity of the paper's statistics: histograms (-> entropy,
chi^2), difference counts (-> NPCR, UACI, PSNR) exact; SSIM within 1e-9 relative (fp64 both sides,
different summation orders).  Inputs: the images of the protocol (I, I_e, I_e', I') at several
sizes, plus the closed-form cases of tests/test_oracle_stats.py."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2302_07992_b200 import mmsb as G
from paper_2302_07992_b200 import synth as S

pytestmark = pytest.mark.gpu


def _protocol_images(H, W, n=3):
    imgs = np.stack([S.random_image(8000 + j, H, W, ["smooth", "textured", "noise"][j % 3]) for j in range(n)])
    k1 = np.stack([np.frombuffer(S.key(8000 + j, 1), np.uint8) for j in range(n)])
    k2 = np.stack([np.frombuffer(S.key(8000 + j, 2), np.uint8) for j in range(n)])
    stride = S.msg_stride(H, W)
    msgs = np.stack([S.payload(j, stride) for j in range(n)])
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    I = dev(imgs)
    enc, b, cap, _ = G.encode(G.EMR, I, dev(k1))
    marked, _ = G.embed(G.EMR, enc, dev(k2), dev(msgs), (cap - 32).clamp(min=0))
    rec, _ = G.recover(G.EMR, marked, dev(k1))
    return I, enc, marked, rec


@pytest.mark.parametrize("H,W", [(16, 16), (64, 64), (128, 256), (512, 512), (16, 32768), (32768, 16)])
def test_histogram_entropy_chi2_and_differences(H, W):
    I, enc, marked, rec = _protocol_images(H, W)
    for X in (I, enc, marked, rec):
        h = G.histogram(X).cpu().numpy()
        ent, chi = G.entropy_chi2(H, W, h)
        for j in range(X.shape[0]):
            x = X[j].cpu().numpy()
            assert np.array_equal(h[j], np.bincount(x.ravel(), minlength=256))
            assert ent[j] == pytest.approx(O.entropy(x), rel=1e-12, abs=1e-15)
            assert chi[j] == pytest.approx(O.chi2(x), rel=1e-9, abs=1e-9)
    for A, B in ((I, enc), (I, marked), (I, rec), (enc, marked)):
        sse, nd, ad = (t.cpu().numpy() for t in G.diff_stats(A, B))
        npcr, uaci = G.npcr_uaci(H, W, nd, ad)
        for j in range(A.shape[0]):
            a, b = A[j].cpu().numpy(), B[j].cpu().numpy()
            assert sse[j] == O.sse(a, b)
            n_o, u_o = O.npcr_uaci(a, b)
            assert npcr[j] == pytest.approx(n_o, rel=1e-12) and uaci[j] == pytest.approx(u_o, rel=1e-12)


@pytest.mark.parametrize("H,W", [(16, 16), (64, 64), (128, 256), (256, 64), (16, 4096), (4096, 16)])
def test_ssim_parity(H, W):
    I, enc, marked, rec = _protocol_images(H, W)
    for A, B in ((I, rec), (I, enc), (I, I), (marked, rec)):
        s = G.ssim(A, B).cpu().numpy()
        for j in range(A.shape[0]):
            ref = O.ssim(A[j].cpu().numpy(), B[j].cpu().numpy())
            assert s[j] == pytest.approx(ref, rel=1e-9, abs=1e-12)
    assert np.all(G.ssim(I, I).cpu().numpy() == pytest.approx(1.0, abs=1e-12))


def test_ssim_is_reproducible():
    """The per-image SSIM sum is accumulated in fixed point: repeated calls (and any CTA finishing
    order) give the same bits."""
    g = torch.Generator().manual_seed(11)
    A = torch.randint(0, 256, (4, 512, 512), generator=g, dtype=torch.uint8).cuda()
    B = (A.int() + torch.randint(-20, 21, A.shape, generator=g).cuda()).clamp(0, 255).to(torch.uint8)
    runs = [G.ssim(A, B).cpu() for _ in range(5)]
    assert all(torch.equal(r, runs[0]) for r in runs[1:])


def test_closed_forms_on_gpu():
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    const = dev(np.full((2, 512, 512), 17, np.uint8))
    ent, chi = G.entropy_chi2(512, 512, G.histogram(const).cpu().numpy())
    assert list(ent) == [0.0, 0.0] and list(chi) == [255 * 262144] * 2
    bw = (np.random.default_rng(3).integers(0, 2, size=(1, 64, 64)) * 255).astype(np.uint8)
    _, nd, ad = G.diff_stats(dev(bw), dev(255 - bw))
    npcr, uaci = G.npcr_uaci(64, 64, nd.cpu().numpy(), ad.cpu().numpy())
    assert npcr[0] == 100.0 and uaci[0] == 100.0
