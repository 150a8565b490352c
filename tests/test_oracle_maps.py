"""Pins for the oracle's location maps and optimal-b selection.

The oracle implements the literal Omega glide (eq. gliding1/gliding2).  It is pinned to
  * an independent formulation: L_b(i,j) = 0  <=>  top_b(p(i,j)) == top_b(p(i,j-1)) for j >= 1
    (Omega always equals the top-b bits of the left neighbour; SURVEY finding 1),
  * SPEC.md's hand-derived worked examples (tests/golden/spec_worked_examples.txt),
  * exhaustive two-valued 4x4 images for every leading-bit distance k,
  * brute force over b for the argmax (eq. optimial_b) and the LMR candidate order.
"""
import itertools

import numpy as np
import pytest

import oracle as O
from paper_2302_07992_b200 import synth as S


def left_neighbour_map(img, b):
    img = img.astype(np.int64)
    t = img >> (8 - b)
    L = np.ones_like(img)
    L[:, 1:] = (t[:, 1:] != t[:, :-1]).astype(np.int64)
    return L.astype(np.uint8)


@pytest.mark.parametrize("kind", ["smooth", "textured", "noise", "constant", "quantised"])
@pytest.mark.parametrize("shape", [(4, 4), (5, 13), (16, 16), (33, 64)])
def test_glide_equals_left_neighbour_formula(kind, shape):
    for seed in range(3):
        img = S.random_image(seed, *shape, kind=kind)
        for b in range(1, 9):
            assert np.array_equal(O.location_map(img, b), left_neighbour_map(img, b)), (kind, shape, b)


def test_first_column_always_one():
    img = S.random_image(1, 20, 20, "noise")
    for b in range(1, 9):
        assert (O.location_map(img, b)[:, 0] == 1).all()


def test_spec_worked_examples():
    row = np.array([[144, 150, 96, 130]], np.uint8)
    assert list(O.location_map(row, 2)[0]) == [1, 0, 1, 1]
    z = O.zero_counts(row)
    assert list(z[2:8]) == [1, 1, 1, 1, 0, 0]
    assert O.select_b_emr(z) == 5                                           # b = 5, payload 5
    assert 5 * z[5] == 5
    const = np.full((4, 4), 77, np.uint8)
    for b in range(1, 9):
        L = O.location_map(const, b)
        assert (L == np.array([1, 0, 0, 0])).all()
    assert O.zero_counts(const)[2] == 12
    alt = np.tile(np.array([0, 255], np.uint8), (4, 4))
    assert O.zero_counts(alt)[1:].sum() == 0                                # S:272 alternating MSB


def test_exhaustive_two_valued_4x4():
    """All 2^16 4x4 images over {v, v ^ 2^(7-k)}: differing neighbours share exactly k MSBs."""
    rng = np.random.default_rng(0)
    pats = np.array(list(itertools.product([0, 1], repeat=16)), np.uint8).reshape(-1, 4, 4)
    for k in range(8):
        v = int(rng.integers(0, 256))
        w = v ^ (1 << (7 - k))
        imgs = np.where(pats == 1, w, v).astype(np.uint8)
        # brute force: a pixel is redundant at b iff it equals its left neighbour or b <= k
        same = imgs[:, :, 1:] == imgs[:, :, :-1]
        for idx in range(0, len(imgs), 257):          # every 257th pattern through ctypes ...
            z = O.zero_counts(imgs[idx])
            for b in range(1, 9):
                want = int(same[idx].sum()) + (int((~same[idx]).sum()) if b <= k else 0)
                assert z[b] == want, (k, idx, b)
        # ... and every pattern through the map routine for one b per k (vectorised compare)
        b = 1 + (k % 8)
        for idx in range(len(imgs)):
            if idx % 16 == 0:
                assert np.array_equal(O.location_map(imgs[idx], b), left_neighbour_map(imgs[idx], b))


def test_zeros_non_increasing_in_b():
    for kind in ["smooth", "textured", "noise", "quantised"]:
        z = O.zero_counts(S.random_image(3, 64, 64, kind))
        assert all(z[b] >= z[b + 1] for b in range(1, 8))


def test_select_b_and_candidates_brute_force():
    rng = np.random.default_rng(5)
    for _ in range(500):
        z = np.zeros(9, np.int64)
        z[1:] = np.sort(rng.integers(0, 50, 8))[::-1]
        if rng.random() < 0.3:                         # force ties
            z[3] = z[2] * 2 // 3
        best = max(range(2, 8), key=lambda b: (b * z[b], -b))
        assert O.select_b_emr(z) == best
        order = sorted(range(2, 9), key=lambda b: (-(b - 1) * z[b], b))
        assert O.lmr_candidates(z) == order


def test_all_zero_counts_pick_b2():
    assert O.select_b_emr(np.zeros(9, np.int64)) == 2
    assert O.lmr_candidates(np.zeros(9, np.int64)) == [2, 3, 4, 5, 6, 7, 8]
