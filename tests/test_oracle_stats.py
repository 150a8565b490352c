"""Pins of the oracle's security / quality statistics: Shannon entropy and
chi^2, NPCR / UACI (reading Q26: sigma = 1 where pixels differ), SSIM
(11x11 Gaussian window sigma 1.5, K1 0.01, K2 0.03, L 255; mean over the
windows inside the image).  Closed forms, worked examples, algebraic identities and an
independent numpy/scipy evaluation of the same definitions."""
import math

import numpy as np
import pytest
from scipy.signal import correlate2d

import oracle as O
from paper_2302_07992_b200 import synth as S


def test_entropy_closed_forms():
    assert O.entropy(np.full((64, 64), 200, np.uint8)) == 0.0                 # constant image -> 0
    half = np.zeros((64, 64), np.uint8)
    half[:32] = 255
    assert O.entropy(half) == 1.0                                             # exact 50/50 -> 1 bit
    uni = np.arange(256 * 256, dtype=np.int64).reshape(256, 256).astype(np.uint8)
    assert abs(O.entropy(uni) - 8.0) < 1e-12                                  # every level equally often
    for k in (1, 2, 5):
        img = (np.arange(4096) % (1 << k)).astype(np.uint8).reshape(64, 64)
        assert abs(O.entropy(img) - k) < 1e-12


def test_chi2_worked_example_and_identity():
    assert O.chi2(np.full((512, 512), 17, np.uint8)) == 255 * 262144         # 66,846,720
    uni = np.arange(256 * 64, dtype=np.int64).reshape(128, 128).astype(np.uint8)
    assert O.chi2(uni) == 0.0
    rng = np.random.default_rng(5)
    for _ in range(5):
        img = rng.integers(0, 256, size=(96, 80), dtype=np.uint8)
        obs = np.bincount(img.ravel(), minlength=256).astype(np.float64)
        E = img.size / 256.0
        classic = float(((obs - E) ** 2 / E).sum())                           # sum (O - E)^2 / E
        assert abs(O.chi2(img) - classic) <= 1e-9 * max(1.0, classic)


def test_npcr_uaci_closed_forms():
    rng = np.random.default_rng(6)
    a = rng.integers(0, 256, size=(64, 64), dtype=np.uint8)
    assert O.npcr_uaci(a, a) == (0.0, 0.0)
    bw = (rng.integers(0, 2, size=(64, 64)) * 255).astype(np.uint8)
    assert O.npcr_uaci(bw, 255 - bw) == (100.0, 100.0)                        # binary image vs complement
    b = np.zeros((512, 512), np.uint8)
    c = b.copy()
    c[100, 200] = 255
    npcr, uaci = O.npcr_uaci(b, c)
    assert npcr == 100.0 / 262144 and abs(uaci - 100.0 / 262144) < 1e-18
    x = rng.integers(0, 256, size=(40, 40), dtype=np.uint8)
    y = rng.integers(0, 256, size=(40, 40), dtype=np.uint8)
    assert O.npcr_uaci(x, y) == O.npcr_uaci(y, x)                             # symmetric


def _ssim_numpy(a, b):
    g = np.exp(-((np.arange(11) - 5) ** 2) / (2 * 1.5 ** 2))
    w = np.outer(g, g)
    w /= w.sum()
    a, b = a.astype(np.float64), b.astype(np.float64)
    f = lambda x: correlate2d(x, w, mode="valid")
    ma, mb = f(a), f(b)
    va, vb, cab = f(a * a) - ma * ma, f(b * b) - mb * mb, f(a * b) - ma * mb
    C1, C2 = (0.01 * 255) ** 2, (0.03 * 255) ** 2
    return float(np.mean((2 * ma * mb + C1) * (2 * cab + C2) / ((ma * ma + mb * mb + C1) * (va + vb + C2))))


def test_ssim_identity_constants_symmetry_and_numpy():
    a = S.random_image(31, 48, 64, "smooth")
    assert O.ssim(a, a) == 1.0
    for c1, c2 in ((10, 200), (128, 128), (0, 255)):
        x, y = np.full((32, 32), c1, np.uint8), np.full((32, 32), c2, np.uint8)
        C1 = (0.01 * 255) ** 2
        closed = (2 * c1 * c2 + C1) / (c1 * c1 + c2 * c2 + C1)                 # sigma = 0: contrast term 1
        assert abs(O.ssim(x, y) - closed) < 1e-12
    b = S.random_image(32, 48, 64, "textured")
    assert O.ssim(a, b) == pytest.approx(O.ssim(b, a), rel=1e-12)
    for kind in ("smooth", "noise", "quantised"):
        x, y = S.random_image(40, 40, 56, kind), S.random_image(41, 40, 56, "smooth")
        assert O.ssim(x, y) == pytest.approx(_ssim_numpy(x, y), rel=1e-10, abs=1e-12)


def test_ssim_of_emr_recovery_in_the_papers_range():
    # EMR loses only the LSB plane: SSIM close to 1, the paper's BOWS-2 range 0.9746-0.9997
    img = S.image(2, 0)[:128, :128].copy()
    k1, k2 = S.key(1, 1), S.key(1, 2)
    st, E, b, C = O.encode(O.EMR, img, k1)
    _, Em = O.hide(O.EMR, E, k2, S.payload(1, S.msg_stride(128, 128)), C - 32)
    _, R = O.recover(O.EMR, Em, k1)
    assert 0.97 < O.ssim(img, R) < 1.0
