"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck):
tile + a skewed window with glands, counting and non-counting builds, all T,
the bench's pipeline step, comb pairs (dense splits / Alg. 1's split order) and
the packed transfer decode."""
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
    sccg.pixelbox(P, Q, pairs, threshold=2048, paper_split=True)
    # the bench's step: prep of both sets in one launch, async join + PixelBox, read-back kernel
    rb = [torch.zeros(len(sccg.SUMS_FIELDS), dtype=torch.int64).pin_memory()]
    pipe = sccg.Pipeline(P, Q, graph=False, readback=rb)
    pipe.run()
    torch.cuda.synchronize()
    pipe.check()
# combs: dense splits pixelized whole, and Alg. 1's split order
from synth import combs
A, B = combs.generate(n_pairs=24)
P = sccg.DeviceSet(*sccg.to_device(A.xy, A.offsets))
Q = sccg.DeviceSet(*sccg.to_device(B.xy, B.offsets))
pairs = sccg.filter_pairs(P, Q)
for ps in (False, True):
    sccg.pixelbox(P, Q, pairs, threshold=2048, paper_split=ps)
torch.cuda.synchronize()
# the packed transfer encoding's decode (offsets rebuilt on the device, staged vertices), a partial last block
A, B = synth.generate("tile")
for S in (A, B):
    enc = sccg.encode_rect_packed(S.xy, S.offsets)
    xy, off = sccg.decode_rect_packed({k: torch.from_numpy(v).cuda() for k, v in enc.items()}, int(S.offsets[-1]))
    torch.cuda.synchronize()
    assert torch.equal(xy.cpu(), torch.from_numpy(S.xy.astype("int32")))
if os.environ.get("SANITIZE_INDEX"):
    # enough comb pairs that the large path builds per-pair edge indexes (first items >= 4 x the item
    # kernel's warps), with and without the pool
    A, B = combs.generate(n_pairs=12000)
    P = sccg.DeviceSet(*sccg.to_device(A.xy, A.offsets))
    Q = sccg.DeviceSet(*sccg.to_device(B.xy, B.offsets))
    pairs = sccg.filter_pairs(P, Q)
    i1, u1, s1 = sccg.pixelbox(P, Q, pairs, threshold=2048)
    i2, u2, s2 = sccg.pixelbox(P, Q, pairs, threshold=2048, index=False)
    torch.cuda.synchronize()
    assert torch.equal(i1, i2) and torch.equal(s1, s2)
torch.cuda.synchronize()
print("sanitize case ok")
