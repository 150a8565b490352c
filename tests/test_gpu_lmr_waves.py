"""LMR candidate waves at batch sizes where they matter: wave 0 codes eta and
one candidate, later waves code several candidates of the still-undecided images at once and
abort a candidate's tiles once they cannot fit.  The walk's outcome must be the oracle's serial
walk exactly: b, capacity, status and the encrypted image (with its coded MSB plane) for every
image, plus the round trip on the decided ones."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2302_07992_b200 import mmsb as G
from paper_2302_07992_b200 import synth as S

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("t,B", [(5, 48), (6, 48)])
def test_lmr_waves_match_serial_walk(t, B):
    imgs, k1, k2 = S.batch(3, n=B)                    # alternating smooth / textured (alpha 2 / 1)
    H, W = imgs.shape[1:]
    ws = G.Workspace(G.LMR, B, H, W, tile_log2=t)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    enc, b, cap, st = G.encode(G.LMR, dev(imgs), dev(k1), ws, tile_log2=t)
    torch.cuda.synchronize()
    enc, b, cap, st = enc.cpu().numpy(), b.cpu().numpy(), cap.cpu().numpy(), st.cpu().numpy()
    outcomes, late = set(), 0
    for j in range(B):
        so, E, bo, Co = O.encode(O.LMR, imgs[j], k1[j].tobytes(), tile_log2=t)
        assert (int(st[j]), int(b[j]), int(cap[j])) == (so, bo, Co), (j, st[j], b[j], cap[j], so, bo, Co)
        assert np.array_equal(enc[j], E), (j, np.argwhere(enc[j] != E)[:5])
        outcomes.add((so, bo))
        if so == O.OK:
            late += O.lmr_candidates(O.zero_counts(imgs[j])).index(bo) >= 2
    assert len(outcomes) >= 2                          # several walk outcomes in the batch
    assert late > 0                                    # some images decided after candidate 1 (waves >= 1)
    # round trip through the GPU on the batch
    stride = S.msg_stride(H, W)
    msgs = np.stack([S.payload(S.image_seed(3, j), stride) for j in range(B)])
    nb = torch.from_numpy(np.maximum(cap.astype(np.int64) - 32, 0)).cuda()
    marked, st_h = G.embed(G.LMR, dev(enc), dev(k2), dev(msgs), nb, ws, tile_log2=t)
    rec, st_r = G.recover(G.LMR, marked, dev(k1), ws, tile_log2=t)
    torch.cuda.synchronize()
    ok = st == 0
    assert np.array_equal(rec.cpu().numpy()[ok], imgs[ok])
