"""CPU oracle of EMR-RDHEI / LMR-RDHEI (arXiv 2302.07992) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2302_07992_b200``) never imports it and shares no code with it.

The arithmetic lives in plain C (``mmsb_oracle.c``, single-threaded, every step cited
to PAPER.md); this module only builds it with gcc and marshals numpy arrays.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "mmsb_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

EMR, LMR = 0, 1
OK, E_INVAL, E_CAPACITY, E_INTEGRITY, E_BADCASE, E_FORMAT = 0, 2, 3, 4, 5, 8

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (building the checker is not using it)."""
    hdr = os.path.join(HERE, "mmsb_oracle.h")
    stale = (not os.path.exists(LIB)) or any(
        os.path.getmtime(p) > os.path.getmtime(LIB) for p in (SRC, hdr))
    if force or stale:
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-Wall", "-shared", "-fPIC",
                               "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(LIB)
            u8p, i32p, i64p = C.POINTER(C.c_uint8), C.POINTER(C.c_int32), C.POINTER(C.c_int64)
            sig = {
                "orc_chacha20_block": (None, [u8p, C.c_uint32, u8p, u8p]),
                "orc_chacha_block": (None, [u8p, C.c_uint32, u8p, C.c_int, u8p]),
                "orc_set_cipher_rounds": (None, [C.c_int]),
                "orc_cipher_rounds": (C.c_int, []),
                "orc_keystream": (None, [u8p, C.c_uint64, C.c_uint64, u8p]),
                "orc_location_map": (None, [u8p, C.c_int, C.c_int, C.c_int, u8p]),
                "orc_zero_counts": (None, [u8p, C.c_int, C.c_int, i64p]),
                "orc_select_b_emr": (C.c_int, [i64p]),
                "orc_lmr_candidates": (None, [i64p, C.POINTER(C.c_int)]),
                "orc_emax": (C.c_int, [C.c_int, C.c_int]),
                "orc_block_angles": (None, [u8p, C.c_int, C.c_int, C.c_int, u8p]),
                "orc_rotate_pass": (None, [u8p, C.c_int, C.c_int, C.c_int, u8p, C.c_int]),
                "orc_rotate_all": (None, [u8p, C.c_int, C.c_int, u8p, C.c_int, C.c_int]),
                "orc_tile_encode": (C.c_int, [u8p, C.c_int, C.c_int, u8p, C.c_int]),
                "orc_tile_decode": (None, [u8p, C.c_int, C.c_int, C.c_int, u8p]),
                "orc_tile_count": (C.c_int, [C.c_int, C.c_int, C.c_int]),
                "orc_encode": (C.c_int, [C.c_int, u8p, C.c_int, C.c_int, u8p, C.c_int, u8p, i32p, i64p]),
                "orc_hide": (C.c_int, [C.c_int, u8p, C.c_int, C.c_int, C.c_int, u8p, u8p, C.c_int64, u8p]),
                "orc_extract": (C.c_int, [C.c_int, u8p, C.c_int, C.c_int, C.c_int, u8p, u8p, C.c_int64, i64p]),
                "orc_recover": (C.c_int, [C.c_int, u8p, C.c_int, C.c_int, C.c_int, u8p, u8p]),
                "orc_encode_s": (C.c_int, [C.c_int, u8p, C.c_int, C.c_int, u8p, C.c_int, C.c_int, u8p, i32p, i64p]),
                "orc_recover_s": (C.c_int, [C.c_int, u8p, C.c_int, C.c_int, C.c_int, C.c_int, u8p, u8p]),
                "orc_capacity": (C.c_int, [C.c_int, u8p, C.c_int, C.c_int, C.c_int, i32p, i64p]),
                "orc_sse": (C.c_int64, [u8p, u8p, C.c_int64]),
                "orc_der_psnr": (None, [C.c_int, C.c_int, C.c_int64, C.c_int64,
                                        C.POINTER(C.c_double), C.POINTER(C.c_double)]),
                "orc_entropy": (C.c_double, [u8p, C.c_int64]),
                "orc_chi2": (C.c_double, [u8p, C.c_int64]),
                "orc_npcr_uaci": (None, [u8p, u8p, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
                "orc_ssim": (C.c_double, [u8p, u8p, C.c_int, C.c_int]),
            }
            for name, (res, args) in sig.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def _p(a: np.ndarray, ty=C.c_uint8):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(ty))


def _u8(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint8))


# ---------------------------------------------------------------- primitives
def chacha20_block(key: bytes, counter: int, nonce: bytes = bytes(12)) -> bytes:
    k, n, out = _u8(bytearray(key)), _u8(bytearray(nonce)), np.zeros(64, np.uint8)
    lib().orc_chacha20_block(_p(k), counter, _p(n), _p(out))
    return out.tobytes()


def chacha_block(key: bytes, counter: int, rounds: int, nonce: bytes = bytes(12)) -> bytes:
    """ChaCha block with an explicit round count (20 = RFC 8439; 12 / 8 = the reduced-round option)."""
    k, n, out = _u8(bytearray(key)), _u8(bytearray(nonce)), np.zeros(64, np.uint8)
    lib().orc_chacha_block(_p(k), counter, _p(n), rounds, _p(out))
    return out.tobytes()


def set_cipher_rounds(rounds: int) -> None:
    """Rounds of the keystream every oracle call uses (20 unless 8 or 12): process-wide."""
    lib().orc_set_cipher_rounds(int(rounds))


def cipher_rounds() -> int:
    return int(lib().orc_cipher_rounds())


def keystream(key: bytes, offset: int, n: int) -> np.ndarray:
    k, out = _u8(bytearray(key)), np.zeros(n, np.uint8)
    lib().orc_keystream(_p(k), offset, n, _p(out))
    return out


def location_map(img: np.ndarray, b: int) -> np.ndarray:
    img = _u8(img)
    out = np.zeros_like(img)
    lib().orc_location_map(_p(img), img.shape[0], img.shape[1], b, _p(out))
    return out


def zero_counts(img: np.ndarray) -> np.ndarray:
    img = _u8(img)
    z = np.zeros(9, np.int64)
    lib().orc_zero_counts(_p(img), img.shape[0], img.shape[1], _p(z, C.c_int64))
    return z


def select_b_emr(zeros) -> int:
    z = np.ascontiguousarray(np.asarray(zeros, np.int64))
    return lib().orc_select_b_emr(_p(z, C.c_int64))


def lmr_candidates(zeros) -> list[int]:
    z = np.ascontiguousarray(np.asarray(zeros, np.int64))
    o = (C.c_int * 7)()
    lib().orc_lmr_candidates(_p(z, C.c_int64), o)
    return list(o)


def emax(M: int, N: int) -> int:
    return lib().orc_emax(M, N)


def block_angles(s: np.ndarray, e: int) -> np.ndarray:
    s = _u8(s)
    M, N = s.shape
    n = 1 << e
    out = np.zeros((M // n) * (N // n) + 1, np.uint8)
    lib().orc_block_angles(_p(s), M, N, e, _p(out))
    return out[:-1].reshape(M // n, N // n)


def rotate_pass(grid: np.ndarray, e: int, ang: np.ndarray, inverse: bool) -> np.ndarray:
    g = _u8(grid).copy()
    a = _u8(ang).ravel().copy()
    lib().orc_rotate_pass(_p(g), g.shape[0], g.shape[1], e, _p(a), int(inverse))
    return g


def rotate_all(grid: np.ndarray, s: np.ndarray, emin: int, inverse: bool) -> np.ndarray:
    g = _u8(grid).copy()
    s = _u8(s)
    lib().orc_rotate_all(_p(g), g.shape[0], g.shape[1], _p(s), emin, int(inverse))
    return g


def tile_encode(bits: np.ndarray, cap: int | None = None) -> bytes:
    bits = _u8(bits)
    h, w = bits.shape
    cap = cap if cap is not None else h * w // 8 + h * w // 64 + 64
    out = np.zeros(cap, np.uint8)
    n = lib().orc_tile_encode(_p(bits), h, w, _p(out), cap)
    if n < 0:
        raise ValueError("tile stream exceeds cap")
    return out[:n].tobytes()


def tile_decode(data: bytes, h: int, w: int) -> np.ndarray:
    d = _u8(bytearray(data) if data else bytearray(1))
    out = np.zeros((h, w), np.uint8)
    lib().orc_tile_decode(_p(d), len(data), h, w, _p(out))
    return out


def tile_count(M: int, N: int, t: int) -> int:
    return lib().orc_tile_count(M, N, t)


# ---------------------------------------------------------------- the four calls
def encode(method: int, img: np.ndarray, k1: bytes, tile_log2: int = 7, lmr_emin: int = 0):
    img = _u8(img)
    M, N = img.shape
    E = np.zeros_like(img)
    b, cap = C.c_int32(0), C.c_int64(0)
    k = _u8(bytearray(k1))
    st = lib().orc_encode_s(method, _p(img), M, N, _p(k), tile_log2, lmr_emin, _p(E), C.byref(b), C.byref(cap))
    return st, E, b.value, cap.value


def hide(method: int, E: np.ndarray, k2: bytes, msg: np.ndarray, msg_bits: int, tile_log2: int = 7):
    E = _u8(E)
    M, N = E.shape
    out = np.zeros_like(E)
    m = _u8(msg) if len(msg) else np.zeros(1, np.uint8)
    k = _u8(bytearray(k2))
    st = lib().orc_hide(method, _p(E), M, N, tile_log2, _p(k), _p(m), msg_bits, _p(out))
    return st, out


def extract(method: int, marked: np.ndarray, k2: bytes, stride_bytes: int, fill: int = 0, tile_log2: int = 7):
    marked = _u8(marked)
    M, N = marked.shape
    out = np.full(stride_bytes, fill, np.uint8)
    nb = C.c_int64(0)
    k = _u8(bytearray(k2))
    st = lib().orc_extract(method, _p(marked), M, N, tile_log2, _p(k), _p(out), stride_bytes, C.byref(nb))
    return st, out, nb.value


def recover(method: int, marked: np.ndarray, k1: bytes, tile_log2: int = 7, lmr_emin: int = 0):
    marked = _u8(marked)
    M, N = marked.shape
    out = np.zeros_like(marked)
    k = _u8(bytearray(k1))
    st = lib().orc_recover_s(method, _p(marked), M, N, tile_log2, lmr_emin, _p(k), _p(out))
    return st, out


def capacity(method: int, marked: np.ndarray, tile_log2: int = 7):
    marked = _u8(marked)
    M, N = marked.shape
    b, cap = C.c_int32(0), C.c_int64(0)
    st = lib().orc_capacity(method, _p(marked), M, N, tile_log2, C.byref(b), C.byref(cap))
    return st, b.value, cap.value


def sse(a: np.ndarray, b: np.ndarray) -> int:
    a, b = _u8(a), _u8(b)
    assert a.shape == b.shape
    return lib().orc_sse(_p(a), _p(b), a.size)


def der_psnr(M: int, N: int, capacity_bits: int, sse_: int):
    d, p = C.c_double(0), C.c_double(0)
    lib().orc_der_psnr(M, N, capacity_bits, sse_, C.byref(d), C.byref(p))
    return d.value, p.value


def entropy(img: np.ndarray) -> float:
    img = _u8(img)
    return lib().orc_entropy(_p(img), img.size)


def chi2(img: np.ndarray) -> float:
    img = _u8(img)
    return lib().orc_chi2(_p(img), img.size)


def npcr_uaci(a: np.ndarray, b: np.ndarray):
    a, b = _u8(a), _u8(b)
    assert a.shape == b.shape
    n_, u_ = C.c_double(0), C.c_double(0)
    lib().orc_npcr_uaci(_p(a), _p(b), a.size, C.byref(n_), C.byref(u_))
    return n_.value, u_.value


def ssim(a: np.ndarray, b: np.ndarray) -> float:
    a, b = _u8(a), _u8(b)
    assert a.shape == b.shape
    return lib().orc_ssim(_p(a), _p(b), a.shape[0], a.shape[1])
