"""Thin Python binding of the C ABI in include/mmsb.h (argument marshalling only).

Every step of the method runs in libmmsb.so's sm_100a kernels; torch provides device
memory and the current stream.  There is no CPU fallback: if the library is missing the
first call raises.  Names follow the ABI (and the paper's three parties).
"""
from __future__ import annotations

import ctypes as C
import os

import torch

from . import build as _build

EMR, LMR = 0, 1
OK, E_INVAL, E_CAPACITY, E_INTEGRITY, E_BADCASE, E_CUDA, E_UNIMPLEMENTED, E_FORMAT = 0, 2, 3, 4, 5, 6, 7, 8

_lib = None


class _Shape(C.Structure):
    _fields_ = [("method", C.c_int32), ("batch", C.c_int32), ("height", C.c_int32), ("width", C.c_int32),
                ("tile_log2", C.c_int32), ("lmr_emin", C.c_int32), ("cipher_rounds", C.c_int32)]


class MmsbError(RuntimeError):
    pass


def lib():
    """Loads the in-tree libmmsb.so (never a CPU substitute)."""
    global _lib
    if _lib is None:
        path = os.environ.get("MMSB_LIB", _build.LIB)     # (tools/role_probe.py loads probe builds)
        if not os.path.exists(path):
            raise MmsbError(f"{path} is missing: run __graft_entry__.build() (nvcc sm_100a) first")
        L = C.CDLL(path)
        vp, sp = C.c_void_p, C.POINTER(_Shape)
        L.mmsb_workspace_bytes.restype = C.c_size_t
        L.mmsb_workspace_bytes.argtypes = [sp]
        L.mmsb_content_owner_encode.restype = C.c_int
        L.mmsb_content_owner_encode.argtypes = [sp, vp, vp, vp, vp, vp, vp, vp, C.c_size_t, vp]
        L.mmsb_hider_embed.restype = C.c_int
        L.mmsb_hider_embed.argtypes = [sp, vp, vp, vp, vp, C.c_int64, vp, vp, vp, C.c_size_t, vp]
        L.mmsb_receiver_extract.restype = C.c_int
        L.mmsb_receiver_extract.argtypes = [sp, vp, vp, vp, C.c_int64, vp, vp, vp, C.c_size_t, vp]
        L.mmsb_receiver_recover.restype = C.c_int
        L.mmsb_receiver_recover.argtypes = [sp, vp, vp, vp, vp, vp, C.c_size_t, vp]
        L.mmsb_receiver_recover_sse.restype = C.c_int
        L.mmsb_receiver_recover_sse.argtypes = [sp, vp, vp, vp, vp, vp, vp, vp, C.c_size_t, vp]
        L.mmsb_capacity.restype = C.c_int
        L.mmsb_capacity.argtypes = [sp, vp, vp, vp, vp, vp, C.c_size_t, vp]
        L.mmsb_receiver_both.restype = C.c_int
        L.mmsb_receiver_both.argtypes = [sp, vp, vp, vp, vp, C.c_int64, vp, vp, vp, vp, C.c_size_t, vp]
        L.mmsb_histogram.restype = C.c_int
        L.mmsb_histogram.argtypes = [sp, vp, vp, vp]
        L.mmsb_diff_stats.restype = C.c_int
        L.mmsb_diff_stats.argtypes = [sp, vp, vp, vp, vp, vp, vp]
        L.mmsb_ssim.restype = C.c_int
        L.mmsb_ssim.argtypes = [sp, vp, vp, vp, vp]
        L.mmsb_entropy_chi2_host.restype = None
        L.mmsb_entropy_chi2_host.argtypes = [C.c_int32, C.c_int32, C.c_int32, vp, vp, vp]
        L.mmsb_npcr_uaci_host.restype = None
        L.mmsb_npcr_uaci_host.argtypes = [C.c_int32, C.c_int32, C.c_int32, vp, vp, vp, vp]
        L.mmsb_stats.restype = C.c_int
        L.mmsb_stats.argtypes = [sp, vp, vp, vp, vp]
        L.mmsb_der_psnr_host.restype = None
        L.mmsb_der_psnr_host.argtypes = [C.c_int32, C.c_int32, C.c_int32, vp, vp, vp, vp]
        L.mmsb_status_string.restype = C.c_char_p
        L.mmsb_status_string.argtypes = [C.c_int]
        L.mmsb_kernel_launches.restype = C.c_uint64
        L.mmsb_kernel_launches.argtypes = []
        _lib = L
    return _lib


def _shape(method: int, B: int, H: int, W: int, tile_log2: int = 7, lmr_emin: int = 0, cipher_rounds: int = 0) -> _Shape:
    return _Shape(method, B, H, W, tile_log2, lmr_emin, cipher_rounds)


def _ptr(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda:
        raise MmsbError("mmsb: device tensors required (the product path has no CPU fallback)")
    if not t.is_contiguous():
        raise MmsbError("mmsb: contiguous tensors required")
    return C.c_void_p(t.data_ptr())


def _arg(t: torch.Tensor, name: str, dtype: torch.dtype, shape: tuple, device=None) -> torch.Tensor:
    """Checks one ABI argument before its raw pointer crosses the boundary: a wrong dtype, shape or
    device would otherwise be an out-of-bounds device read or write (the C side sees sizes only)."""
    if not isinstance(t, torch.Tensor):
        raise MmsbError(f"mmsb: {name} must be a torch tensor")
    if t.dtype != dtype:
        raise MmsbError(f"mmsb: {name} must be {dtype}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise MmsbError(f"mmsb: {name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if not t.is_cuda:
        raise MmsbError(f"mmsb: {name} must be a device tensor (the product path has no CPU fallback)")
    if device is not None and t.device != device:
        raise MmsbError(f"mmsb: {name} is on {t.device}, expected {device}")
    if not t.is_contiguous():
        raise MmsbError(f"mmsb: {name} must be contiguous")
    return t


def _images(t: torch.Tensor, name: str):
    if not isinstance(t, torch.Tensor) or t.dim() != 3:
        raise MmsbError(f"mmsb: {name} must be a [B, H, W] uint8 tensor")
    return _arg(t, name, torch.uint8, tuple(t.shape)).shape


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _check(rc: int, what: str):
    if rc != OK:
        raise MmsbError(f"{what}: {lib().mmsb_status_string(rc).decode()} ({rc})")


def kernel_launches() -> int:
    return int(lib().mmsb_kernel_launches())


class Workspace:
    """Caller-owned device scratch sized by mmsb_workspace_bytes (one per stream)."""

    def __init__(self, method: int, B: int, H: int, W: int, tile_log2: int = 7, device=None, lmr_emin: int = 0,
                 cipher_rounds: int = 0):
        self.shape = _shape(method, B, H, W, tile_log2, lmr_emin, cipher_rounds)
        n = lib().mmsb_workspace_bytes(C.byref(self.shape))
        if n == 0:
            raise MmsbError(f"unsupported shape method={method} B={B} H={H} W={W} t={tile_log2}")
        self.buf = torch.empty(n, dtype=torch.uint8, device=device or "cuda")
        self.nbytes = n


def _ws(ws: Workspace | None, method, B, H, W, tile_log2, device):
    if tile_log2 is None:                       # the workspace's coder tile size (default 2^7)
        tile_log2 = ws.shape.tile_log2 if ws is not None else 7
    if ws is None or (ws.shape.method, ws.shape.batch, ws.shape.height, ws.shape.width, ws.shape.tile_log2) != (
            method, B, H, W, tile_log2):
        ws = Workspace(method, B, H, W, tile_log2, device)
    return ws


def encode(method: int, images: torch.Tensor, k1: torch.Tensor, ws: Workspace | None = None, tile_log2: int | None = None,
           out: torch.Tensor | None = None):
    """Content owner: returns (encrypted, b, capacity_bits, status) -- mmsb_content_owner_encode."""
    B, H, W = _images(images, "images")
    _arg(k1, "k1", torch.uint8, (B, 32), images.device)
    if out is not None:
        _arg(out, "out", torch.uint8, (B, H, W), images.device)
    ws = _ws(ws, method, B, H, W, tile_log2, images.device)
    enc = out if out is not None else torch.empty_like(images)
    b = torch.empty(B, dtype=torch.int32, device=images.device)
    cap = torch.empty(B, dtype=torch.int64, device=images.device)
    st = torch.empty(B, dtype=torch.int32, device=images.device)
    rc = lib().mmsb_content_owner_encode(C.byref(ws.shape), _ptr(images), _ptr(k1), _ptr(enc), _ptr(b), _ptr(cap),
                                         _ptr(st), _ptr(ws.buf), ws.nbytes, _stream())
    _check(rc, "mmsb_content_owner_encode")
    return enc, b, cap, st


def embed(method: int, encrypted: torch.Tensor, k2: torch.Tensor, msg: torch.Tensor, msg_bits: torch.Tensor,
          ws: Workspace | None = None, tile_log2: int | None = None, out: torch.Tensor | None = None):
    """Data hider: returns (marked, status) -- mmsb_hider_embed."""
    B, H, W = _images(encrypted, "encrypted")
    dev = encrypted.device
    _arg(k2, "k2", torch.uint8, (B, 32), dev)
    if msg.dim() != 2:
        raise MmsbError("mmsb: msg must be a [B, stride_bytes] uint8 tensor")
    _arg(msg, "msg", torch.uint8, (B, msg.shape[1]), dev)
    if msg.shape[1] <= 0 or msg.shape[1] % 16:
        raise MmsbError(f"mmsb: msg stride {msg.shape[1]} must be a positive multiple of 16 bytes")
    _arg(msg_bits, "msg_bits", torch.int64, (B,), dev)
    if out is not None:
        _arg(out, "out", torch.uint8, (B, H, W), dev)
    ws = _ws(ws, method, B, H, W, tile_log2, encrypted.device)
    marked = out if out is not None else torch.empty_like(encrypted)
    st = torch.empty(B, dtype=torch.int32, device=encrypted.device)
    rc = lib().mmsb_hider_embed(C.byref(ws.shape), _ptr(encrypted), _ptr(k2), _ptr(msg), _ptr(msg_bits),
                                msg.shape[1], _ptr(marked), _ptr(st), _ptr(ws.buf), ws.nbytes, _stream())
    _check(rc, "mmsb_hider_embed")
    return marked, st


def extract(method: int, marked: torch.Tensor, k2: torch.Tensor, stride: int, ws: Workspace | None = None,
            tile_log2: int | None = None, out: torch.Tensor | None = None):
    """Receiver with K2: returns (msg_bytes, msg_bits, status) -- mmsb_receiver_extract."""
    B, H, W = _images(marked, "marked")
    _arg(k2, "k2", torch.uint8, (B, 32), marked.device)
    if stride <= 0 or stride % 16:
        raise MmsbError(f"mmsb: stride {stride} must be a positive multiple of 16 bytes")
    if out is not None:
        _arg(out, "out", torch.uint8, (B, stride), marked.device)
    ws = _ws(ws, method, B, H, W, tile_log2, marked.device)
    msg = out if out is not None else torch.zeros(B, stride, dtype=torch.uint8, device=marked.device)
    nb = torch.empty(B, dtype=torch.int64, device=marked.device)
    st = torch.empty(B, dtype=torch.int32, device=marked.device)
    rc = lib().mmsb_receiver_extract(C.byref(ws.shape), _ptr(marked), _ptr(k2), _ptr(msg), stride, _ptr(nb),
                                     _ptr(st), _ptr(ws.buf), ws.nbytes, _stream())
    _check(rc, "mmsb_receiver_extract")
    return msg, nb, st


def recover(method: int, marked: torch.Tensor, k1: torch.Tensor, ws: Workspace | None = None, tile_log2: int | None = None,
            out: torch.Tensor | None = None, original: torch.Tensor | None = None, sse_out: torch.Tensor | None = None):
    """Receiver with K1: returns (recovered, status) -- mmsb_receiver_recover.  With `original`
    (an evaluation harness's reference image) the SSE statistic is fused into the same pass and
    (recovered, status, sse) is returned -- mmsb_receiver_recover_sse."""
    B, H, W = _images(marked, "marked")
    _arg(k1, "k1", torch.uint8, (B, 32), marked.device)
    if out is not None:
        _arg(out, "out", torch.uint8, (B, H, W), marked.device)
    ws = _ws(ws, method, B, H, W, tile_log2, marked.device)
    rec = out if out is not None else torch.empty_like(marked)
    st = torch.empty(B, dtype=torch.int32, device=marked.device)
    if original is None:
        rc = lib().mmsb_receiver_recover(C.byref(ws.shape), _ptr(marked), _ptr(k1), _ptr(rec), _ptr(st),
                                         _ptr(ws.buf), ws.nbytes, _stream())
        _check(rc, "mmsb_receiver_recover")
        return rec, st
    _arg(original, "original", torch.uint8, (B, H, W), marked.device)
    sse = sse_out if sse_out is not None else torch.empty(B, dtype=torch.int64, device=marked.device)
    _arg(sse, "sse_out", torch.int64, (B,), marked.device)
    rc = lib().mmsb_receiver_recover_sse(C.byref(ws.shape), _ptr(marked), _ptr(k1), _ptr(original), _ptr(rec),
                                         _ptr(sse), _ptr(st), _ptr(ws.buf), ws.nbytes, _stream())
    _check(rc, "mmsb_receiver_recover_sse")
    return rec, st, sse


def receive_both(method: int, marked: torch.Tensor, k1: torch.Tensor, k2: torch.Tensor, stride: int,
                 ws: Workspace | None = None, tile_log2: int | None = None, msg_out: torch.Tensor | None = None,
                 rec_out: torch.Tensor | None = None):
    """Receiver with both keys: returns (msg_bytes, msg_bits, recovered, status) -- mmsb_receiver_both."""
    B, H, W = _images(marked, "marked")
    _arg(k1, "k1", torch.uint8, (B, 32), marked.device)
    _arg(k2, "k2", torch.uint8, (B, 32), marked.device)
    if stride <= 0 or stride % 16:
        raise MmsbError(f"mmsb: stride {stride} must be a positive multiple of 16 bytes")
    if msg_out is not None:
        _arg(msg_out, "msg_out", torch.uint8, (B, stride), marked.device)
    if rec_out is not None:
        _arg(rec_out, "rec_out", torch.uint8, (B, H, W), marked.device)
    ws = _ws(ws, method, B, H, W, tile_log2, marked.device)
    msg = msg_out if msg_out is not None else torch.zeros(B, stride, dtype=torch.uint8, device=marked.device)
    rec = rec_out if rec_out is not None else torch.empty_like(marked)
    nb = torch.empty(B, dtype=torch.int64, device=marked.device)
    st = torch.empty(B, dtype=torch.int32, device=marked.device)
    rc = lib().mmsb_receiver_both(C.byref(ws.shape), _ptr(marked), _ptr(k1), _ptr(k2), _ptr(msg), stride, _ptr(nb),
                                  _ptr(rec), _ptr(st), _ptr(ws.buf), ws.nbytes, _stream())
    _check(rc, "mmsb_receiver_both")
    return msg, nb, rec, st


def capacity(method: int, image: torch.Tensor, ws: Workspace | None = None, tile_log2: int | None = None):
    """Capacity of an encrypted / marked image: returns (b, capacity_bits, status) -- mmsb_capacity."""
    B, H, W = _images(image, "image")
    ws = _ws(ws, method, B, H, W, tile_log2, image.device)
    b = torch.empty(B, dtype=torch.int32, device=image.device)
    cap = torch.empty(B, dtype=torch.int64, device=image.device)
    st = torch.empty(B, dtype=torch.int32, device=image.device)
    rc = lib().mmsb_capacity(C.byref(ws.shape), _ptr(image), _ptr(b), _ptr(cap), _ptr(st), _ptr(ws.buf), ws.nbytes,
                             _stream())
    _check(rc, "mmsb_capacity")
    return b, cap, st


def stats(original: torch.Tensor, recovered: torch.Tensor, out: torch.Tensor | None = None):
    """Per-image SSE (int64) -- mmsb_stats."""
    B, H, W = _images(original, "original")
    _arg(recovered, "recovered", torch.uint8, (B, H, W), original.device)
    if out is not None:
        _arg(out, "out", torch.int64, (B,), original.device)
    sh = _shape(EMR, B, H, W)
    sse = out if out is not None else torch.empty(B, dtype=torch.int64, device=original.device)
    rc = lib().mmsb_stats(C.byref(sh), _ptr(original), _ptr(recovered), _ptr(sse), _stream())
    _check(rc, "mmsb_stats")
    return sse


def der_psnr(H: int, W: int, capacity_bits, sse):
    """Host DER / PSNR from integers (mmsb_der_psnr_host)."""
    import numpy as np

    cap = np.ascontiguousarray(np.asarray(capacity_bits, dtype=np.int64))
    s = np.ascontiguousarray(np.asarray(sse, dtype=np.int64))
    der = np.zeros(len(cap), np.float64)
    psnr = np.zeros(len(cap), np.float64)
    lib().mmsb_der_psnr_host(len(cap), H, W, cap.ctypes.data, s.ctypes.data, der.ctypes.data, psnr.ctypes.data)
    return der, psnr


# ---------------------------------------------------------------- the paper's statistics (NEXT 2)
def histogram(images: torch.Tensor, out: torch.Tensor | None = None):
    """[B, 256] int64 grey-level counts -- mmsb_histogram."""
    B, H, W = _images(images, "images")
    if out is not None:
        _arg(out, "out", torch.int64, (B, 256), images.device)
    h = out if out is not None else torch.empty(B, 256, dtype=torch.int64, device=images.device)
    _check(lib().mmsb_histogram(C.byref(_shape(EMR, B, H, W)), _ptr(images), _ptr(h), _stream()), "mmsb_histogram")
    return h


def diff_stats(a: torch.Tensor, b: torch.Tensor):
    """(sse, ndiff, absdiff) int64 per image -- mmsb_diff_stats."""
    B, H, W = _images(a, "a")
    _arg(b, "b", torch.uint8, (B, H, W), a.device)
    sse, nd, ad = (torch.empty(B, dtype=torch.int64, device=a.device) for _ in range(3))
    _check(lib().mmsb_diff_stats(C.byref(_shape(EMR, B, H, W)), _ptr(a), _ptr(b), _ptr(sse), _ptr(nd), _ptr(ad),
                                 _stream()), "mmsb_diff_stats")
    return sse, nd, ad


def ssim(a: torch.Tensor, b: torch.Tensor):
    """[B] float64 mean windowed SSIM -- mmsb_ssim."""
    B, H, W = _images(a, "a")
    _arg(b, "b", torch.uint8, (B, H, W), a.device)
    out = torch.empty(B, dtype=torch.float64, device=a.device)
    _check(lib().mmsb_ssim(C.byref(_shape(EMR, B, H, W)), _ptr(a), _ptr(b), _ptr(out), _stream()), "mmsb_ssim")
    return out


def entropy_chi2(H: int, W: int, hist):
    """Host entropy / chi^2 from [B, 256] counts (mmsb_entropy_chi2_host)."""
    import numpy as np

    h = np.ascontiguousarray(np.asarray(hist, dtype=np.int64))
    ent, chi = np.zeros(h.shape[0]), np.zeros(h.shape[0])
    lib().mmsb_entropy_chi2_host(h.shape[0], H, W, h.ctypes.data, ent.ctypes.data, chi.ctypes.data)
    return ent, chi


def npcr_uaci(H: int, W: int, ndiff, absdiff):
    """Host NPCR / UACI in percent (mmsb_npcr_uaci_host)."""
    import numpy as np

    nd = np.ascontiguousarray(np.asarray(ndiff, dtype=np.int64))
    ad = np.ascontiguousarray(np.asarray(absdiff, dtype=np.int64))
    npcr, uaci = np.zeros(len(nd)), np.zeros(len(nd))
    lib().mmsb_npcr_uaci_host(len(nd), H, W, nd.ctypes.data, ad.ctypes.data, npcr.ctypes.data, uaci.ctypes.data)
    return npcr, uaci
