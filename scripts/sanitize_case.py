"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck):
tile + a skewed window with glands, counting and non-counting builds, all T."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1208_0277_b200 as sccg
import synth

for cfg, kw in [("tile", {}), ("skewed", dict(width=4096, height=4096))]:
    A, B = synth.generate(cfg, **kw)
    P = sccg.DeviceSet(*sccg.to_device(A.xy, A.offsets))
    Q = sccg.DeviceSet(*sccg.to_device(B.xy, B.offsets))
    pairs = sccg.filter_pairs(P, Q)
    for T in (16, 2048):
        c = torch.zeros(8, dtype=torch.int64, device="cuda")
        sccg.pixelbox(P, Q, pairs, threshold=T, counters=c)
        sccg.pixelbox(P, Q, pairs, threshold=T)
    sccg.pixelbox(P, Q, pairs, mode=1)
torch.cuda.synchronize()
print("sanitize case ok")
