"""Pins for the oracle's keystream (reading Q12: ChaCha20 / RFC 8439).

Pinned against (a) the RFC 8439 A.1 test vector stored in tests/golden/ and (b) an
independent implementation: the `cryptography` package's ChaCha20.
"""
import os

import numpy as np
import pytest

import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "rfc8439_chacha20.txt")


def _golden(name):
    for line in open(GOLDEN):
        if line.startswith(name + " "):
            return bytes.fromhex(line.split()[1])
    raise KeyError(name)


def test_rfc8439_a1_tv1():
    assert O.chacha20_block(bytes(32), 0) == _golden("A1_TV1")
    assert O.keystream(bytes(32), 0, 64).tobytes() == _golden("A1_TV1")


def _crypto_stream(key: bytes, counter: int, n: int) -> bytes:
    pytest.importorskip("cryptography")
    from cryptography.hazmat.primitives.ciphers import Cipher, algorithms

    nonce16 = counter.to_bytes(4, "little") + bytes(12)   # RFC 8439 layout: LE counter || 96-bit nonce
    enc = Cipher(algorithms.ChaCha20(key, nonce16), mode=None).encryptor()
    return enc.update(bytes(n))


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_matches_cryptography_package(seed):
    key = np.random.default_rng(seed).integers(0, 256, 32, dtype=np.uint8).tobytes()
    n = 1 << 20 if seed == 0 else 70_000
    assert O.keystream(key, 0, n).tobytes() == _crypto_stream(key, 0, n)


def test_counter_jump_ahead_equals_slicing():
    key = bytes(range(32))
    full = O.keystream(key, 0, 64 * 40)
    rng = np.random.default_rng(7)
    for _ in range(20):
        off = int(rng.integers(0, 64 * 30))
        n = int(rng.integers(1, 64 * 9))
        assert np.array_equal(O.keystream(key, off, n), full[off:off + n])
    # block counter c starts at byte 64 c
    assert O.keystream(key, 64 * 5, 64).tobytes() == _crypto_stream(key, 5, 64)


def test_nonzero_nonce_block():
    key = bytes(range(32))
    nonce = bytes.fromhex("000000090000004a00000000")
    pytest.importorskip("cryptography")
    from cryptography.hazmat.primitives.ciphers import Cipher, algorithms

    ref = Cipher(algorithms.ChaCha20(key, (1).to_bytes(4, "little") + nonce), mode=None).encryptor().update(bytes(64))
    assert O.chacha20_block(key, 1, nonce) == ref
