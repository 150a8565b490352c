"""Multi-process (world_size 2, gloo on CPU) test of the data-parallel plumbing that bench.py runs
over NCCL: contiguous image shards, the all-gather of per-image records, the max-over-ranks time and
the rank-0 aggregates, which must not depend on the number of ranks.  The per-image records come
from the CPU oracle on small synthetic images (test infrastructure)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2302_07992_b200 import parallel as P
from paper_2302_07992_b200 import synth as S

H = W = 32
TOTAL = 7                                     # odd: shards of unequal size


def _records(j0, n, method):
    rows = []
    stride = S.msg_stride(H, W)
    for j in range(j0, j0 + n):
        kind = ["smooth", "textured", "noise", "constant"][j % 4]
        img = S.random_image(4000 + j, H, W, kind)
        k1, k2 = S.key(4000 + j, 1), S.key(4000 + j, 2)
        st, E, b, C = O.encode(method, img, k1)
        n_bits = max(C - 32, 0)
        _, Em = O.hide(method, E, k2, S.payload(j, stride), n_bits)
        st_r, R = O.recover(method, Em, k1)
        rows.append([b, C, O.sse(img, R), st_r])
    return torch.tensor(rows, dtype=torch.int64).reshape(n, P.REC_COLS)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, method, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        counts = [P.shard(TOTAL, r, world)[1] for r in range(world)]
        start, n = P.shard(TOTAL, rank, world)
        rec = _records(start, n, method)
        allrec = P.gather_records(rec, world, counts)
        t = P.max_over_ranks(float(rank + 1), torch.device("cpu"), world)
        out[rank] = (allrec.numpy().tolist(), t, P.aggregate(allrec, H, W))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("method", [O.EMR, O.LMR])
def test_two_rank_gather_equals_single_process(method):
    single = _records(0, TOTAL, method)
    ref = P.aggregate(single, H, W)
    with mp.Manager() as m:
        out = m.dict()
        mp.start_processes(_worker, args=(2, _free_port(), method, out), nprocs=2, start_method="spawn")
        res = dict(out)
    for rank in (0, 1):
        allrec, t, agg = res[rank]
        assert np.array_equal(np.array(allrec), single.numpy())          # image order preserved
        assert t == 2.0                                                   # max over ranks
        assert agg == ref


def test_shards_cover_the_batch():
    for total in (1, 7, 1000, 10000):
        for world in (1, 2, 4, 8):
            spans = [P.shard(total, r, world) for r in range(world)]
            assert sum(c for _, c in spans) == total
            assert all(spans[r][0] + spans[r][1] == spans[r + 1][0] for r in range(world - 1))
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1


def test_aggregate_closed_forms():
    rec = torch.tensor([[6, 1000, 65025, 0], [5, 262144, 0, 0], [0, 0, 0, 5]], dtype=torch.int64)
    agg = P.aggregate(rec, 512, 512)
    assert agg["good"] == 2 and agg["bad"] == 1 and agg["psnr_inf"] == 1
    assert agg["der_mean"] == (1000 / 262144 + 1.0) / 2
    assert abs(agg["psnr_mean_finite"] - 54.1854) < 5e-5      # one pixel off by 255
