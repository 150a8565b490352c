"""Round trip at the largest shapes the ABI accepts (16384^2 and 32768^2, one image; EMR and LMR):
statuses, payload and recovery.  python tools/big_shapes.py"""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2302_07992_b200 import mmsb as G
from paper_2302_07992_b200 import synth as S
for method in (G.EMR, G.LMR):
    for H in (16384, 32768):
        B = 1
        img = np.stack([S.random_image(5, 1024, 1024, "smooth")])
        img = np.tile(img, (1, H // 1024, H // 1024))    # cheap large image
        k1 = np.frombuffer(S.key(5, 1), np.uint8)[None]; k2 = np.frombuffer(S.key(5, 2), np.uint8)[None]
        I = torch.from_numpy(img).cuda(); K1 = torch.from_numpy(k1.copy()).cuda(); K2 = torch.from_numpy(k2.copy()).cuda()
        ws = G.Workspace(method, B, H, H)
        enc, b, cap, st = G.encode(method, I, K1, ws)
        n = min(max(int(cap[0]) - 32, 0), 2**32 - 1)      # the frame's length field is 32 bits (Q17)
        stride = ((n + 7) // 8 + 4 + 15) // 16 * 16
        msg = torch.randint(0, 256, (1, stride), dtype=torch.uint8, device='cuda')
        nb = torch.tensor([n], dtype=torch.int64, device='cuda')
        marked, sh = G.embed(method, enc, K2, msg, nb, ws)
        mo, nbo, sx = G.extract(method, marked, K2, stride, ws)
        rec, sr = G.recover(method, marked, K1, ws)
        torch.cuda.synchronize()
        ok_msg = torch.equal(mo[0, : n // 8], msg[0, : n // 8])
        lossless = torch.equal(rec, I) if method == G.LMR else torch.equal(rec >> 1, I >> 1)
        print(method, H, 'ws GB', round(ws.nbytes / 1e9, 2), 'b', int(b[0]), 'cap', int(cap[0]), 'st', int(st[0]), int(sh[0]), int(sx[0]), int(sr[0]), 'msg', ok_msg, 'rec', lossless, flush=True)
        del ws, enc, marked, rec, I
        torch.cuda.empty_cache()
