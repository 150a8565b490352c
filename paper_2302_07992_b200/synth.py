"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic: it only draws images, keys and payload
bytes.  Both sides (the CPU oracle and the CUDA path) read the bytes it produces.

Recipe; the paper's BOWS-2 corpus and the
classic test images are not in the container, so these fields stand in for them:
  * field: white Gaussian noise from ``numpy.random.default_rng(seed)`` (PCG64), FFT,
    amplitude spectrum multiplied by f**-alpha (f = sqrt(fx^2+fy^2) from ``fftfreq``, DC
    zeroed), inverse FFT, real part, standardised; pixel = clip(rint(128 + 48 x), 0, 255);
  * image j of config i uses seed = 1_000_000 * i + j;
  * K1 = 16 bytes from default_rng([seed, 1]), K2 from default_rng([seed, 2]), each passed
    as k || k (32-byte ChaCha20 keys for the configs' "128-bit" keys, reading Q13);
  * payload bytes from default_rng([seed, 3]); the bench embeds n = C - 32 bits (full
    capacity, reading Q17);
  * config 3: alpha = 2 for even j, 1 for odd j; config 4: alpha ~ U[1, 2.5] from
    default_rng([seed, 0]); config 5: alpha = 2 plus 5% of pixels (Bernoulli 0.05 from
    default_rng([seed, 4])) replaced by uniform bytes.
"""
from __future__ import annotations

import numpy as np

try:  # multithreaded FFT when scipy is present (it is in this image)
    import scipy.fft as _fft

    def _fft2(a):
        return _fft.fft2(a, workers=-1)

    def _ifft2(a):
        return _fft.ifft2(a, workers=-1)
except Exception:  # pragma: no cover
    _fft2, _ifft2 = np.fft.fft2, np.fft.ifft2

# BASELINE.json configs (1-based, as cited in SURVEY: BJ:configs[i])
CONFIGS = {
    1: dict(batch=1, H=512, W=512, method="emr"),
    2: dict(batch=1000, H=512, W=512, method="emr"),
    3: dict(batch=1000, H=512, W=512, method="lmr"),
    4: dict(batch=10000, H=512, W=512, method="emr+lmr"),
    5: dict(batch=64, H=4096, W=4096, method="emr+lmr"),
}


def image_seed(config: int, j: int) -> int:
    return 1_000_000 * config + j


def field(seed: int, alpha: float, H: int, W: int) -> np.ndarray:
    """1/f^alpha amplitude-spectrum Gaussian field mapped to uint8."""
    rng = np.random.default_rng(seed)
    noise = rng.standard_normal((H, W))
    fy = np.fft.fftfreq(H)[:, None]
    fx = np.fft.fftfreq(W)[None, :]
    f = np.sqrt(fx * fx + fy * fy)
    mult = np.zeros_like(f)
    nz = f > 0
    mult[nz] = f[nz] ** (-alpha)
    x = np.real(_ifft2(_fft2(noise) * mult))
    x = (x - x.mean()) / (x.std() + 1e-300)
    return np.clip(np.rint(128.0 + 48.0 * x), 0, 255).astype(np.uint8)


def alpha_for(config: int, j: int) -> float:
    if config == 3:
        return 2.0 if j % 2 == 0 else 1.0
    if config == 4:
        return float(np.random.default_rng([image_seed(config, j), 0]).uniform(1.0, 2.5))
    return 2.0


def image(config: int, j: int, H: int | None = None, W: int | None = None) -> np.ndarray:
    cfg = CONFIGS[config]
    H = H or cfg["H"]
    W = W or cfg["W"]
    seed = image_seed(config, j)
    img = field(seed, alpha_for(config, j), H, W)
    if config == 5:
        rng = np.random.default_rng([seed, 4])
        mask = rng.random((H, W)) < 0.05
        vals = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
        img = np.where(mask, vals, img).astype(np.uint8)
    return img


def key(seed: int, which: int) -> bytes:
    """which = 1 -> K1 (image encryption), 2 -> K2 (data hiding)."""
    k = np.random.default_rng([seed, which]).integers(0, 256, size=16, dtype=np.uint8).tobytes()
    return k + k


def payload(seed: int, nbytes: int) -> np.ndarray:
    return np.random.default_rng([seed, 3]).integers(0, 256, size=nbytes, dtype=np.uint8)


def msg_stride(H: int, W: int) -> int:
    """bytes per image of a message buffer that covers any capacity (<= 7 bits/px), 16-aligned."""
    n = (7 * H * W + 7) // 8
    return (n + 15) // 16 * 16


def batch(config: int, n: int | None = None, start: int = 0, H: int | None = None, W: int | None = None):
    """Images [start, start+n) of a config with their keys: (imgs[B,H,W], k1[B,32], k2[B,32])."""
    cfg = CONFIGS[config]
    n = cfg["batch"] if n is None else n
    imgs = np.stack([image(config, start + j, H, W) for j in range(n)])
    k1 = np.frombuffer(b"".join(key(image_seed(config, start + j), 1) for j in range(n)), np.uint8).reshape(n, 32)
    k2 = np.frombuffer(b"".join(key(image_seed(config, start + j), 2) for j in range(n)), np.uint8).reshape(n, 32)
    return imgs, k1.copy(), k2.copy()


def random_image(seed: int, H: int, W: int, kind: str = "smooth") -> np.ndarray:
    """Small test inputs: smooth / textured fields, uniform noise, constant, two-valued."""
    rng = np.random.default_rng([seed, 99])
    if kind == "smooth":
        return field(seed, 2.0, H, W)
    if kind == "textured":
        return field(seed, 1.0, H, W)
    if kind == "noise":
        return rng.integers(0, 256, size=(H, W), dtype=np.uint8)
    if kind == "constant":
        return np.full((H, W), int(rng.integers(0, 256)), np.uint8)
    if kind == "quantised":
        return (rng.integers(0, 4, size=(H, W)) * 64 + rng.integers(0, 2, size=(H, W))).astype(np.uint8)
    raise ValueError(kind)
