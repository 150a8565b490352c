"""Pins for the oracle's EMR / LMR calls, coder and statistics.

What fixes the answers here is the paper and the mathematics, not the oracle:
  * extract(hide(m)) = m; separability (extract takes K2 only, recover K1 only);
  * EMR: bits 1..7 of the recovered image equal the original; the PSNR equals
    10 log10(65025 MN / n_mis) EXACTLY, n_mis predicted at encode from independently pinned
    pieces (keystream, rotation); ~51.14 dB at 512^2;
  * LMR: recovery is bit-exact (PSNR +inf); the hider never touches the MSB plane
    (P:991); capacity = (b-1)/b of EMR's at the same b;
  * the capacity boundary is exact; a constant image gives b = 7;
  * coder round trip (exhaustive 4x4, random planes), the ideal-code-length bound;
  * statistics closed forms.
"""
import itertools
import math

import numpy as np
import pytest

import oracle as O
from paper_2302_07992_b200 import synth as S


def _keys(seed):
    return S.key(seed, 1), S.key(seed, 2)


def _roundtrip(method, img, seed, nbits=None):
    k1, k2 = _keys(seed)
    st, E, b, C = O.encode(method, img, k1)
    M, N = img.shape
    stride = S.msg_stride(M, N)
    msg = S.payload(seed, stride)
    if st != O.OK:
        return st, E, b, C, None, msg, None
    n = max(C - 32, 0) if nbits is None else nbits
    st2, Em = O.hide(method, E, k2, msg, n)
    return st, E, b, C, (st2, Em), msg, n


def _msg_bits(buf, n):
    return np.unpackbits(buf)[:n]


@pytest.mark.parametrize("shape", [(16, 16), (32, 32), (64, 64), (32, 128), (24, 40)])
@pytest.mark.parametrize("kind", ["smooth", "textured", "noise", "constant", "quantised"])
def test_emr_round_trip_and_lsb_only_loss(shape, kind):
    for seed in range(2):
        img = S.random_image(seed + 10, *shape, kind=kind)
        st, E, b, C, hid, msg, n = _roundtrip(O.EMR, img, seed)
        assert st == O.OK and 2 <= b <= 7
        Ef = E.ravel()
        assert ((Ef[0] & 1) << 2 | (Ef[1] & 1) << 1 | (Ef[2] & 1)) == b - 2        # header (Q14)
        k1, k2 = _keys(seed)
        st2, Em = hid
        if C < 32:
            assert st2 == O.E_CAPACITY and np.array_equal(Em, E)
            continue
        assert st2 == O.OK
        assert np.array_equal(Em & 1, E & 1)                 # the hider never touches the LSB map
        st3, out, nb = O.extract(O.EMR, Em, k2, S.msg_stride(*shape))
        assert st3 == O.OK and nb == n
        assert np.array_equal(_msg_bits(out, n), _msg_bits(msg, n))
        assert not _msg_bits(out, 32 * ((C - 32 + 31) // 32))[n:].any()
        assert not out[4 * ((C - 32 + 31) // 32):].any()       # region is whole 32-bit words
        st4, R = O.recover(O.EMR, Em, k1)
        assert st4 == O.OK
        assert np.array_equal(R >> 1, img >> 1)              # bits 1..7 exact


def test_emr_psnr_closed_form_and_expected_value():
    img = S.image(2, 0)                                       # 512 x 512, alpha = 2
    seed = S.image_seed(2, 0)
    k1, k2 = _keys(seed)
    st, E, b, C, (st2, Em), msg, n = _roundtrip(O.EMR, img, seed)
    M, N = img.shape
    # predicted mismatches: written LSB vs LSB of (I_r xor s), with I_r and s from the pinned pieces
    s = O.keystream(k1, 0, M * N).reshape(M, N)
    Ir = O.rotate_all(img, s, 1, False)
    n_mis = int(((E & 1) != ((Ir ^ s) & 1)).sum())
    st4, R = O.recover(O.EMR, Em, k1)
    sse = O.sse(img, R)
    assert sse == n_mis
    der, psnr = O.der_psnr(M, N, C, sse)
    assert psnr == pytest.approx(10 * math.log10(65025 * M * N / n_mis), rel=1e-12)
    assert abs(psnr - 51.1411) < 0.15
    assert der == C / (M * N)


def test_emr_capacity_boundary_and_empty_message():
    img = S.random_image(3, 64, 64, "smooth")
    k1, k2 = _keys(3)
    st, E, b, C = O.encode(O.EMR, img, k1)[0:4]
    msg = S.payload(3, S.msg_stride(64, 64))
    assert O.hide(O.EMR, E, k2, msg, C - 32)[0] == O.OK
    assert O.hide(O.EMR, E, k2, msg, C - 31)[0] == O.E_CAPACITY
    st2, Em = O.hide(O.EMR, E, k2, msg, 0)
    st3, out, nb = O.extract(O.EMR, Em, k2, S.msg_stride(64, 64))
    assert st2 == O.OK and st3 == O.OK and nb == 0
    # the capacity the receiver derives equals the encoder's
    assert O.capacity(O.EMR, Em) == (O.OK, b, C)


def test_emr_wrong_k2_is_integrity_or_self_consistent():
    img = S.random_image(4, 64, 64, "smooth")
    st, E, b, C, (st2, Em), msg, n = _roundtrip(O.EMR, img, 4)
    bad = bytes([x ^ 1 for x in S.key(4, 2)])
    st3, out, nb = O.extract(O.EMR, Em, bad, S.msg_stride(64, 64))
    assert (st3 == O.E_INTEGRITY and nb == -1 and not out.any()) or (st3 == O.OK and 0 <= nb <= C - 32)


def test_emr_constant_image():
    img = np.full((16, 16), 93, np.uint8)
    st, E, b, C = O.encode(O.EMR, img, S.key(0, 1))
    assert b == 7
    assert 7 * O.zero_counts(img)[7] / 256 == 6.5625            # pre-forcing DER 7(N-1)/N
    assert C % 7 == 0 and 7 * (240 - 3) <= C <= 7 * 240


def test_emr_monotone_safety_of_map_flips():
    """Flipping 0 -> 1 map bits (r >= 3) between encode and hide never breaks recovery."""
    img = S.random_image(6, 64, 64, "smooth")
    k1, k2 = _keys(6)
    st, E, b, C = O.encode(O.EMR, img, k1)
    rng = np.random.default_rng(6)
    flat = E.ravel().copy()
    zeros = np.flatnonzero((flat & 1) == 0)
    zeros = zeros[zeros >= 3]
    flip = rng.choice(zeros, size=len(zeros) // 5, replace=False)
    flat[flip] |= 1
    E2 = flat.reshape(E.shape)
    st2, C2 = O.capacity(O.EMR, E2)[0], O.capacity(O.EMR, E2)[2]
    msg = S.payload(6, S.msg_stride(64, 64))
    st3, Em = O.hide(O.EMR, E2, k2, msg, C2 - 32)
    assert st3 == O.OK
    st4, R = O.recover(O.EMR, Em, k1)
    assert np.array_equal(R >> 1, img >> 1)
    st5, out, nb = O.extract(O.EMR, Em, k2, S.msg_stride(64, 64))
    assert nb == C2 - 32 and np.array_equal(_msg_bits(out, nb), _msg_bits(msg, nb))


def test_emr_invalid_header_is_format():
    E = np.zeros((16, 16), np.uint8)
    E.ravel()[0] |= 1
    E.ravel()[1] |= 1                                            # b-field 6 > 5
    assert O.hide(O.EMR, E, S.key(0, 2), np.zeros(4, np.uint8), 0)[0] == O.E_FORMAT
    st, R = O.recover(O.EMR, E, S.key(0, 1))
    assert st == O.E_FORMAT and not R.any()


# ------------------------------------------------------------------------------ LMR
@pytest.mark.parametrize("shape", [(32, 32), (64, 64), (128, 128), (64, 256)])
@pytest.mark.parametrize("kind", ["smooth", "textured", "constant"])
def test_lmr_lossless_round_trip(shape, kind):
    img = S.random_image(20, *shape, kind=kind)
    st, E, b, C, hid, msg, n = _roundtrip(O.LMR, img, 20)
    k1, k2 = _keys(20)
    if st == O.E_BADCASE:
        assert O.hide(O.LMR, E, k2, msg, 0)[0] == O.E_BADCASE
        assert O.recover(O.LMR, E, k1)[0] == O.E_BADCASE
        return
    assert st == O.OK and 2 <= b <= 8
    z = O.zero_counts(img)
    assert C == (b - 1) * z[b]                                  # (b-1) bits per redundant pixel
    assert C * b == (b - 1) * (b * z[b])                        # = (b-1)/b of EMR's gross capacity
    st2, Em = hid
    if C < 32:
        assert st2 == O.E_CAPACITY
        return
    assert st2 == O.OK
    assert np.array_equal(Em >> 7, E >> 7)                      # MSB plane untouched
    st3, out, nb = O.extract(O.LMR, Em, k2, S.msg_stride(*shape))
    assert st3 == O.OK and nb == n and np.array_equal(_msg_bits(out, n), _msg_bits(msg, n))
    st4, R = O.recover(O.LMR, Em, k1)
    assert st4 == O.OK and np.array_equal(R, img)               # lossless
    assert O.der_psnr(*shape, C, O.sse(img, R))[1] == math.inf
    st5, R0 = O.recover(O.LMR, E, k1)                            # straight decode without hiding
    assert np.array_equal(R0, img)


def _parse_msb_header(E):
    bits = (E.ravel() >> 7).astype(np.int64)
    pos = [0]

    def rd(n):
        v = 0
        for _ in range(n):
            v = (v << 1) | int(bits[pos[0]])
            pos[0] += 1
        return v
    bfield, t = rd(3), rd(4)
    T = O.tile_count(*E.shape, t)
    sizes = [rd(16) for _ in range(2 * T)]
    streams = bytes(rd(8) for _ in range(sum(sizes)))
    return bfield, t, sizes, streams, pos[0]


def test_lmr_512_msb_plane_layout_and_eta():
    for j in (0, 1):
        img = S.image(3, j)
        seed = S.image_seed(3, j)
        k1, k2 = _keys(seed)
        st, E, b, C, (st2, Em), msg, n = _roundtrip(O.LMR, img, seed)
        assert st == O.OK and st2 == O.OK
        assert np.array_equal(O.recover(O.LMR, Em, k1)[1], img)
        bfield, t, sizes, streams, K = _parse_msb_header(Em)
        assert bfield == b - 2 and t == 7 and K <= 512 * 512
        s = O.keystream(k1, 0, 512 * 512).reshape(512, 512)
        Ir = O.rotate_all(img, s, 4, False)                  # LMR schedule {2^4..2^9}
        # MSB plane beyond the streams keeps the encrypted image's MSBs; bits 2..8 are I_r xor s
        assert np.array_equal((Em.ravel()[K:] >> 7), ((Ir ^ s).ravel()[K:] >> 7))
        assert np.array_equal(E & 0x7F, (Ir ^ s) & 0x7F)
        # the eta streams decode to the MSB plane of the rotated image (eq. MSB_map)
        T = len(sizes) // 2
        off = 0
        for k in range(T):
            ty, tx = divmod(k, 4)
            tile = O.tile_decode(streams[off:off + sizes[k]], 128, 128)
            off += sizes[k]
            assert np.array_equal(tile, Ir[ty * 128:(ty + 1) * 128, tx * 128:(tx + 1) * 128] >> 7)
        # the map streams decode to the rotated location map of the chosen b
        L = O.rotate_all(O.location_map(img, b), s, 4, False)
        for k in range(T):
            ty, tx = divmod(k, 4)
            tile = O.tile_decode(streams[off:off + sizes[T + k]], 128, 128)
            off += sizes[T + k]
            assert np.array_equal(tile, L[ty * 128:(ty + 1) * 128, tx * 128:(tx + 1) * 128])


def test_lmr_badcase_noise_and_tiny():
    for shape in [(4, 4), (8, 8), (64, 64)]:
        img = S.random_image(5, *shape, kind="noise")
        k1, k2 = _keys(5)
        st, E, b, C = O.encode(O.LMR, img, k1)
        assert st == O.E_BADCASE and b == 0 and C == 0
        assert O.hide(O.LMR, E, k2, np.zeros(4, np.uint8), 0)[0] == O.E_BADCASE
        st3, out, nb = O.extract(O.LMR, E, k2, 64)
        assert st3 == O.E_BADCASE and nb == -1
        st4, R = O.recover(O.LMR, E, k1)
        assert st4 == O.E_BADCASE and not R.any()


# ------------------------------------------------------------------------------ coder
def test_coder_exhaustive_4x4():
    for bits in itertools.product([0, 1], repeat=16):
        p = np.array(bits, np.uint8).reshape(4, 4)
        assert np.array_equal(O.tile_decode(O.tile_encode(p), 4, 4), p)


def _ideal_bits(plane, with_left2=False):
    """Sum of -log2 P(bit) under the adaptive model with the coder's own integer p0 (Q16's
    template; with_left2 adds the (0,-2) pixel, SURVEY O15's 10-pixel template, for contrast)."""
    h, w = plane.shape
    p0 = np.full(1024, 32768, np.int64)
    pad = np.zeros((h + 2, w + 4), np.int64)
    pad[2:, 2:w + 2] = plane
    total = 0.0
    for y in range(h):
        for x in range(w):
            Y, X = y + 2, x + 2
            nb = [pad[Y, X - 1]] + ([pad[Y, X - 2]] if with_left2 else []) + [
                pad[Y - 1, X - 2], pad[Y - 1, X - 1], pad[Y - 1, X], pad[Y - 1, X + 1], pad[Y - 1, X + 2],
                pad[Y - 2, X - 1], pad[Y - 2, X], pad[Y - 2, X + 1]]
            c = 0
            for v in nb:
                c = (c << 1) | int(v)
            bit = plane[y, x]
            q = p0[c] / 65536.0
            total += -math.log2(q if bit == 0 else 1 - q)
            p0[c] = p0[c] + ((65536 - p0[c]) >> 4) if bit == 0 else p0[c] - (p0[c] >> 4)
    return total


@pytest.mark.parametrize("density", [0.0, 0.02, 0.2, 0.5, 0.9])
def test_coder_round_trip_and_ideal_bound(density):
    rng = np.random.default_rng(int(density * 100))
    for shape in [(32, 32), (64, 48), (7, 13)]:
        p = (rng.random(shape) < density).astype(np.uint8)
        data = O.tile_encode(p)
        assert data == O.tile_encode(p)                            # deterministic
        assert np.array_equal(O.tile_decode(data, *shape), p)
        ideal = _ideal_bits(p)
        assert ideal - 8 <= 8 * len(data) <= ideal + 48, (shape, density, ideal, len(data))


def test_coder_template_has_no_left2_pixel():
    """Q16's 9-pixel template on a plane that tells the templates apart: rows repeating with period
    2 (constant or alternating, the type random per row) are predictable from the (0,-2) pixel,
    which the template leaves out.  The coded size matches the 9-pixel ideal within the coder's
    overhead and is far from the 10-pixel (with (0,-2)) ideal."""
    rng = np.random.default_rng(21)
    h, w = 64, 128
    rows = np.tile(rng.integers(0, 2, (h, 2)), (1, w // 2)).astype(np.uint8)     # b[y, x] = b[y, x - 2]
    coded = 8 * len(O.tile_encode(rows))
    i9, i10 = _ideal_bits(rows), _ideal_bits(rows, with_left2=True)
    assert i10 < 0.5 * i9                                               # the plane separates the templates
    assert i9 - 8 <= coded <= i9 + 48, (coded, i9, i10)


def test_coder_many_random_planes():
    rng = np.random.default_rng(11)
    for i in range(3000):
        h, w = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        kind = i % 3
        if kind == 0:
            p = (rng.random((h, w)) < rng.random()).astype(np.uint8)
        elif kind == 1:
            p = np.zeros((h, w), np.uint8)
            p[:, : w // 2] = 1
        else:
            p = ((np.arange(h)[:, None] + np.arange(w)[None, :]) % 2).astype(np.uint8)
        assert np.array_equal(O.tile_decode(O.tile_encode(p), h, w), p)


def test_coder_size_sanity():
    assert 8 * len(O.tile_encode(np.zeros((64, 64), np.uint8))) < 4096
    iid = (np.random.default_rng(0).random((64, 64)) < 0.5).astype(np.uint8)
    assert 8 * len(O.tile_encode(iid)) >= 3900
    cb = ((np.arange(512)[:, None] + np.arange(512)[None, :]) % 2).astype(np.uint8)
    assert len(O.tile_encode(cb)) < 0.02 * 512 * 512 / 8
    # worst-case expansion stays below the buffer bound (1.1 raw + 64 B)
    assert len(O.tile_encode((np.random.default_rng(1).random((128, 128)) < 0.5).astype(np.uint8))) < 2048 * 1.1 + 64


# ------------------------------------------------------------------------------ statistics
def test_statistics_closed_forms():
    a = np.zeros((512, 512), np.uint8)
    b = a.copy()
    b[100, 200] = 255
    assert O.sse(a, b) == 65025
    der, psnr = O.der_psnr(512, 512, 1000, O.sse(a, b))
    assert psnr == pytest.approx(54.1854, abs=5e-5)
    assert der == 1000 / 262144
    assert O.der_psnr(512, 512, 0, 0)[1] == math.inf
    # expected EMR PSNR, half of the LSBs wrong
    assert O.der_psnr(512, 512, 0, 512 * 512 // 2)[1] == pytest.approx(51.1411, abs=5e-5)


@pytest.mark.parametrize("emin", [1, 2, 3, 4])
def test_lmr_schedule_variants_round_trip(emin):
    """Tab. LMR_block_size: LMR with rotation blocks {2^e_min..2^e_max} stays lossless and
    separable for every schedule; e_min = 4 is the default."""
    for j, kind in enumerate(["smooth", "smooth", "textured"]):
        img = S.random_image(600 + j, 64, 64, kind)
        k1, k2 = S.key(600 + j, 1), S.key(600 + j, 2)
        st, E, b, C = O.encode(O.LMR, img, k1, lmr_emin=emin)
        if st != O.OK:
            continue
        if emin == 4:
            st0, E0, b0, C0 = O.encode(O.LMR, img, k1)
            assert (st0, b0, C0) == (st, b, C) and np.array_equal(E0, E)
        stride = S.msg_stride(64, 64)
        msg = S.payload(j, stride)
        _, Em = O.hide(O.LMR, E, k2, msg, C - 32)
        _, mo, nb = O.extract(O.LMR, Em, k2, stride)
        assert nb == C - 32
        assert np.array_equal(np.unpackbits(mo)[:nb], np.unpackbits(msg)[:nb])
        str_, R = O.recover(O.LMR, Em, k1, lmr_emin=emin)
        assert str_ == O.OK and np.array_equal(R, img)
        if emin != 4:            # the schedule is shared knowledge: the default schedule cannot decrypt it
            _, Rw = O.recover(O.LMR, Em, k1)
            assert not np.array_equal(Rw, img)
