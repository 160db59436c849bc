import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, oracle
import paper_1208_0277_b200 as sccg
A, B = synth.generate("tile")
P = sccg.DeviceSet(*sccg.to_device(A.xy, A.offsets))
Q = sccg.DeviceSet(*sccg.to_device(B.xy, B.offsets))
pairs = sccg.filter_pairs(P, Q)
i1, u1, s1 = sccg.pixelbox(P, Q, pairs, raster=True)
i0, u0, s0 = sccg.pixelbox(P, Q, pairs, raster=False)
pn = pairs.cpu().numpy(); a = i1.cpu().numpy(); b = i0.cpu().numpy()
ei, _ = oracle.pair_areas(A, B, pn)
print("edge path ok:", (b == ei).all(), "raster mismatches:", (a != ei).sum(), "of", len(pn))
_, mp = oracle.set_props(A); _, mq = oracle.set_props(B)
ecp = P._view("ecount", torch.int32, (P.n, 2)).cpu().numpy()
ecq = Q._view("ecount", torch.int32, (Q.n, 2)).cpu().numpy()
for k in np.nonzero(a != ei)[0][:12]:
    p, q = pn[k]
    m1, m2 = mp[p], mq[q]
    bx0, by0 = max(m1[0], m2[0]), max(m1[1], m2[1])
    W, H = min(m1[2], m2[2]) - bx0, min(m1[3], m2[3]) - by0
    print(k, "gpu", a[k], "oracle", ei[k], "W H", W, H, "dxp dyp", m1[0] - bx0, m1[1] - by0, "dxq dyq", m2[0] - bx0,
          m2[1] - by0, "raster", bool(ecp[p, 1] >> 30), bool(ecq[q, 1] >> 30), "k%32", k % 32)
