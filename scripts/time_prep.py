"""Time sccg_prep_sets alone on the C2 slide (CUDA events, median of reps): for prep experiments."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, ctypes
import paper_1208_0277_b200 as sccg
import synth
A, B = synth.generate("slide")
P = sccg.DeviceSet(*sccg.to_device(A.xy, A.offsets), prep=False)
Q = sccg.DeviceSet(*sccg.to_device(B.xy, B.offsets), prep=False)
lib = sccg.load()
sets = (sccg.PolySet * 2)(P.c, Q.c)
ts = []
for r in range(60):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    lib.sccg_prep_sets(sets, 2, 1, None)
    e1.record()
    torch.cuda.synchronize()
    if r >= 10:
        ts.append(e0.elapsed_time(e1))
print(os.environ.get("SCCG_LIB", "main"), "prep median %.1f us" % (1e3 * statistics.median(ts)))
