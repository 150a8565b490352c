"""Pins for the oracle's multi-scale block rotation (PAPER.md P:659-671 eq. roration,
P:819-835 eq. roration2; readings Q6-Q11).

Pinned against numpy.rot90 per block (a library routine), the worked example S:218, the
block partition of Fig. fig:blocks, exhaustive angle injection on a 4x4
two-level schedule, and the group properties (round trip, permutation / multiset)."""
import itertools

import numpy as np
import pytest

import oracle as O


def np_angles(s, e):
    n = 1 << e
    M, N = s.shape
    BM, BN = M // n, N // n
    blocks = s[:BM * n, :BN * n].astype(np.int64).reshape(BM, n, BN, n)
    return (blocks.sum(axis=(1, 3)) % 4).astype(np.uint8)


def np_pass(grid, e, ang, inverse):
    n = 1 << e
    g = grid.copy()
    for by in range(ang.shape[0]):
        for bx in range(ang.shape[1]):
            blk = g[by * n:(by + 1) * n, bx * n:(bx + 1) * n]
            k = int(ang[by, bx])
            g[by * n:(by + 1) * n, bx * n:(bx + 1) * n] = np.rot90(blk, k if inverse else -k)
    return g


def test_worked_example_s218():
    g = np.array([[1, 2], [3, 4]], np.uint8)
    assert O.rotate_pass(g, 1, np.array([[1]], np.uint8), False).tolist() == [[3, 1], [4, 2]]
    assert O.rotate_pass(g, 1, np.array([[0]], np.uint8), False).tolist() == [[1, 2], [3, 4]]


def test_fig_blocks_partition_8x8():
    s = np.zeros((8, 8), np.uint8)
    assert [O.block_angles(s, e).size for e in (1, 2, 3)] == [16, 4, 1]
    assert O.emax(8, 8) == 3 and O.emax(512, 512) == 9 and O.emax(4096, 4096) == 12
    assert O.emax(5, 13) == 2 and O.emax(64, 256) == 6


@pytest.mark.parametrize("shape", [(8, 8), (16, 32), (13, 21), (64, 64)])
def test_angles_and_passes_vs_numpy(shape):
    rng = np.random.default_rng(sum(shape))
    for _ in range(5):
        s = rng.integers(0, 256, shape, dtype=np.uint8)
        g = rng.integers(0, 256, shape, dtype=np.uint8)
        for e in range(1, O.emax(*shape) + 1):
            a = O.block_angles(s, e)
            assert np.array_equal(a, np_angles(s, e))
            for inv in (False, True):
                assert np.array_equal(O.rotate_pass(g, e, a, inv), np_pass(g, e, a, inv))


@pytest.mark.parametrize("shape,emin", [((64, 64), 1), ((64, 64), 4), ((32, 128), 1), ((13, 21), 1), ((512, 512), 4)])
def test_rotate_all_composition_and_round_trip(shape, emin):
    rng = np.random.default_rng(shape[0] + emin)
    s = rng.integers(0, 256, shape, dtype=np.uint8)
    g = rng.integers(0, 256, shape, dtype=np.uint8)
    want = g.copy()
    for e in range(emin, O.emax(*shape) + 1):                 # ascending passes, clockwise
        want = np_pass(want, e, np_angles(s, e), False)
    fwd = O.rotate_all(g, s, emin, False)
    assert np.array_equal(fwd, want)
    assert np.array_equal(np.sort(fwd.ravel()), np.sort(g.ravel()))       # multiset invariant
    assert np.array_equal(O.rotate_all(fwd, s, emin, True), g)             # round trip
    # remainder strips (non-power-of-two sides) never move ("retain the remaining pixels")
    n = 1 << O.emax(*shape)
    M, N = shape
    if M % 2 or N % 2:
        assert np.array_equal(fwd[(M // 2) * 2:, :], g[(M // 2) * 2:, :])


def test_exhaustive_two_level_4x4():
    g = np.arange(16, dtype=np.uint8).reshape(4, 4)
    for combo in itertools.product(range(4), repeat=5):
        a1 = np.array(combo[:4], np.uint8).reshape(2, 2)
        a2 = np.array(combo[4:], np.uint8).reshape(1, 1)
        got = O.rotate_pass(O.rotate_pass(g, 1, a1, False), 2, a2, False)
        want = np_pass(np_pass(g, 1, a1, False), 2, a2, False)
        assert np.array_equal(got, want)
        back = O.rotate_pass(O.rotate_pass(got, 2, a2, True), 1, a1, True)
        assert np.array_equal(back, g)
