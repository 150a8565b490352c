"""Data-parallel plumbing of the hot path over the GPUs of one box.

Images are independent (the paper processes each image alone), so the batch is cut into
contiguous shards, one per rank; every rank runs the four calls on its own shard and stream,
and the only exchange is one all-gather of small per-image int64 records after the statistics
step (NCCL on the GPUs; gloo in the CPU tests).  Rank 0 turns the gathered records into the
DER / PSNR aggregates in image-index order, so the result does not depend on the
number of ranks.
"""
from __future__ import annotations

import math

import torch
import torch.distributed as dist

# per-image record columns (int64)
REC_B, REC_CAP, REC_SSE, REC_STATUS = 0, 1, 2, 3
REC_COLS = 4


def shard(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [start, start + count) of `total` images for `rank` of `world`."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def _host_staged() -> bool:
    """gloo moves host tensors; it is the backend only when ranks share a GPU (bench.py) or in
    the CPU tests, so device tensors are staged through host memory for it."""
    return dist.get_backend() == "gloo"


def _all_gather(parts, t: torch.Tensor) -> None:
    if t.is_cuda and _host_staged():
        host = [torch.empty_like(p, device="cpu") for p in parts]
        dist.all_gather(host, t.cpu())
        for p, h in zip(parts, host):
            p.copy_(h)
        return
    dist.all_gather(parts, t)


def make_records(b, cap, sse, status) -> torch.Tensor:
    """[B, 4] int64 records on the device of `sse` (no host round trip)."""
    rec = torch.empty(sse.shape[0], REC_COLS, dtype=torch.int64, device=sse.device)
    rec[:, REC_B] = b
    rec[:, REC_CAP] = cap
    rec[:, REC_SSE] = sse
    rec[:, REC_STATUS] = status
    return rec


def gather_records(rec: torch.Tensor, world: int, counts=None) -> torch.Tensor:
    """All ranks' records concatenated in rank order (= image order with contiguous shards).
    `counts[r]` = images of rank r when the shards differ in size (padded exchange)."""
    if world == 1:
        return rec
    n = max(counts) if counts else rec.shape[0]
    pad = rec
    if rec.shape[0] < n:
        pad = torch.full((n, REC_COLS), -1, dtype=rec.dtype, device=rec.device)
        pad[: rec.shape[0]] = rec
    parts = [torch.empty_like(pad) for _ in range(world)]
    _all_gather(parts, pad.contiguous())
    if counts:
        parts = [p[:c] for p, c in zip(parts, counts)]
    return torch.cat(parts, 0)


def max_over_ranks(ms: float, device, world: int) -> float:
    """The slowest rank's device time (the step ends when every shard is done)."""
    if world == 1:
        return ms
    t = torch.tensor([ms], dtype=torch.float64, device="cpu" if _host_staged() else device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate(records: torch.Tensor, height: int, width: int) -> dict:
    """DER / PSNR aggregates over the good images, in image-index order (reading Q23):
    DER_i = C_i / (H W); PSNR_i = 10 log10(255^2 H W / SSE_i), +inf when SSE_i = 0."""
    r = records.detach().cpu().numpy()
    HW = float(height) * float(width)
    good = [i for i in range(r.shape[0]) if r[i, REC_STATUS] == 0]
    der = [r[i, REC_CAP] / HW for i in good]
    psnr_finite = [10.0 * math.log10(65025.0 * HW / r[i, REC_SSE]) for i in good if r[i, REC_SSE] > 0]
    n_inf = sum(1 for i in good if r[i, REC_SSE] == 0)
    out = {"images": int(r.shape[0]), "good": len(good), "bad": int(r.shape[0] - len(good)),
           "der_mean": sum(der) / len(der) if der else float("nan"),
           "der_min": min(der) if der else float("nan"), "der_max": max(der) if der else float("nan"),
           "capacity_bits_total": int(sum(int(r[i, REC_CAP]) for i in good)),
           "psnr_inf": n_inf, "psnr_mean_finite": sum(psnr_finite) / len(psnr_finite) if psnr_finite else None}
    return out


def gather_rows(rows: torch.Tensor, world: int, counts=None) -> torch.Tensor:
    """Per-image rows of any dtype / width (e.g. the float64 statistics of SURVEY §8(f) NEXT 2)
    from every rank, concatenated in rank order = image order (padded exchange when the shards
    differ in size)."""
    if world == 1:
        return rows
    n = max(counts) if counts else rows.shape[0]
    pad = rows
    if rows.shape[0] < n:
        pad = torch.zeros((n,) + tuple(rows.shape[1:]), dtype=rows.dtype, device=rows.device)
        pad[: rows.shape[0]] = rows
    parts = [torch.empty_like(pad) for _ in range(world)]
    _all_gather(parts, pad.contiguous())
    if counts:
        parts = [p[:c] for p, c in zip(parts, counts)]
    return torch.cat(parts, 0)
