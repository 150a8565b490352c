"""Pins for the reduced-round keystream option (P:656 asks only for "a
cryptographically secure stream cipher"; reading Q12 fixes ChaCha20, the option adds ChaCha12 and
ChaCha8 as a versioned format choice).

A ChaCha block is the input state plus r/2 double rounds of it (RFC 8439 §2.3).  The test's own
double round DR (RFC 8439 §2.1-2.2, written out below) is first pinned against an independent
ChaCha20 -- the `cryptography` package: its output minus the input state must be DR applied 10
times.  With DR pinned, the oracle's 12- and 8-round blocks must be the input plus DR^6 / DR^4:
a wrong round count, order or rotation fails.
"""
import numpy as np
import pytest

import oracle as O

M32 = 0xFFFFFFFF


def _rotl(v, c):
    return ((v << c) | (v >> (32 - c))) & M32


def _qr(x, a, b, c, d):
    x[a] = (x[a] + x[b]) & M32; x[d] = _rotl(x[d] ^ x[a], 16)
    x[c] = (x[c] + x[d]) & M32; x[b] = _rotl(x[b] ^ x[c], 12)
    x[a] = (x[a] + x[b]) & M32; x[d] = _rotl(x[d] ^ x[a], 8)
    x[c] = (x[c] + x[d]) & M32; x[b] = _rotl(x[b] ^ x[c], 7)


def _dr(x):                                   # column round, then diagonal round
    for q in ((0, 4, 8, 12), (1, 5, 9, 13), (2, 6, 10, 14), (3, 7, 11, 15),
              (0, 5, 10, 15), (1, 6, 11, 12), (2, 7, 8, 13), (3, 4, 9, 14)):
        _qr(x, *q)


def _state(key, counter, nonce=bytes(12)):
    w = lambda b, i: int.from_bytes(b[4 * i:4 * i + 4], "little")
    return ([0x61707865, 0x3320646E, 0x79622D32, 0x6B206574] + [w(key, i) for i in range(8)] + [counter & M32]
            + [w(nonce, i) for i in range(3)])


def _block_minus_input(out: bytes, st):
    return [(int.from_bytes(out[4 * i:4 * i + 4], "little") - st[i]) & M32 for i in range(16)]


def _dr_power(st, n):
    x = list(st)
    for _ in range(n):
        _dr(x)
    return x


def _keys():
    rng = np.random.default_rng(2024)
    return [(rng.integers(0, 256, 32, dtype=np.uint8).tobytes(), int(rng.integers(0, 2**32))) for _ in range(6)]


@pytest.mark.parametrize("key,counter", _keys())
def test_double_round_pinned_by_an_independent_chacha20(key, counter):
    pytest.importorskip("cryptography")
    from cryptography.hazmat.primitives.ciphers import Cipher, algorithms

    ref = Cipher(algorithms.ChaCha20(key, counter.to_bytes(4, "little") + bytes(12)), mode=None).encryptor().update(bytes(64))
    st = _state(key, counter)
    assert _block_minus_input(ref, st) == _dr_power(st, 10)


@pytest.mark.parametrize("key,counter", _keys())
@pytest.mark.parametrize("rounds", [8, 12, 20])
def test_reduced_round_blocks_are_the_double_round_powers(key, counter, rounds):
    st = _state(key, counter)
    assert _block_minus_input(O.chacha_block(key, counter, rounds), st) == _dr_power(st, rounds // 2)


def test_twenty_rounds_is_the_rfc_block_and_keystream_follows_the_setting():
    key = bytes(range(32))
    assert O.chacha_block(key, 3, 20) == O.chacha20_block(key, 3)
    assert O.cipher_rounds() == 20
    try:
        for r in (8, 12):
            O.set_cipher_rounds(r)
            assert O.cipher_rounds() == r
            ks = O.keystream(key, 100, 300).tobytes()
            ref = b"".join(O.chacha_block(key, c, r) for c in range(1, 7))[100 - 64:100 - 64 + 300]
            assert ks == ref
        O.set_cipher_rounds(7)                     # anything else: ChaCha20
        assert O.cipher_rounds() == 20
    finally:
        O.set_cipher_rounds(20)
