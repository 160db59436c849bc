import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import synth, kernel_model as km
import paper_1208_0277_b200 as sccg
A, B = synth.generate("tile", want_masks=True)
P = sccg.DeviceSet(*sccg.to_device(A.xy, A.offsets))
torch.cuda.synchronize()
ec = P._view("ecount", torch.int32, (P.n, 2)).cpu().numpy()
ed = P._view("edges", torch.int64, (P.nv,)).cpu().numpy().view(np.uint32)
mb = P.mbr.cpu().numpy()
nr = bad = 0
for i in range(P.n):
    if not (ec[i, 1] & (1 << 30)):
        continue
    nr += 1
    x0, y0, m = A.masks[i]
    H, W = m.shape
    base = 2 * (int(A.offsets[i]) + int(ec[i, 0]))
    rows = ed[base: base + H]
    got = np.array([[(int(rows[r]) >> x) & 1 for x in range(W)] for r in range(H)])
    if not (got == m).all():
        bad += 1
        if bad < 3:
            print("poly", i, "W H", W, H, "nv", ec[i, 0], "V", A.offsets[i + 1] - A.offsets[i], "mbr", mb[i], (x0, y0))
            print(got.astype(int)); print(m.astype(int))
print("rasters", nr, "bad", bad, "of", P.n)
