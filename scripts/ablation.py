"""The paper's PixelBox ablations on B200.

Fig. 8 analog (§5.2): ~16k nucleus pairs (16 tiles of configs[0]),
coordinates scaled by SF = 1..5 (areas x SF^2), PixelOnly (mode 1) vs
PixelBox-NoSep (mode 2) vs PixelBox (mode 0).  Fig. 10 analog (§5.4):
the T sweep {n/2, n, n^2/8, n^2/2, n^2, 4n^2, 16n^2} at n = 64 for each SF.
Every run is also a property check at full size: I(SF) = SF^2 I(1) pair by
pair (the scale law of rectilinear grid dilation) and all modes agree.

    python scripts/ablation.py [--out profiles/r01/ablation.json] [--reps 5]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1208_0277_b200 as sccg
    import synth

    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01", "ablation.json"))
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--tiles", type=int, default=4, help="tiles per side")
    args = ap.parse_args()
    A, B = synth.generate("tile", width=4096 * args.tiles, height=4096 * args.tiles)
    n = 64
    Ts = [n // 2, n, n * n // 8, n * n // 2, n * n, 4 * n * n, 16 * n * n]
    rows = []
    base_inter = None
    for sf in range(1, 6):
        P = sccg.DeviceSet(*sccg.to_device(A.xy * sf, A.offsets))
        Q = sccg.DeviceSet(*sccg.to_device(B.xy * sf, B.offsets))
        pairs = sccg.filter_pairs(P, Q)
        ref = None

        def timed(mode, T):
            ts = []
            for r in range(args.reps + 1):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                out = sccg.pixelbox(P, Q, pairs, mode=mode, threshold=T, paper_split=True)
                e1.record()
                torch.cuda.synchronize()
                if r:
                    ts.append(e0.elapsed_time(e1))
            return float(np.median(ts)), out

        for mode, name in ((1, "PixelOnly"), (2, "PixelBox-NoSep"), (0, "PixelBox")):
            for T in (Ts if mode != 1 else [0]):
                ms, (inter, uni, sums) = timed(mode, T)
                if ref is None:
                    ref = (inter.clone(), uni.clone())
                    if sf == 1:
                        base_inter = inter.clone()
                    else:
                        assert torch.equal(inter, base_inter * sf * sf), "scale law I(s) = s^2 I(1) violated"
                else:
                    assert torch.equal(inter, ref[0]) and torch.equal(uni, ref[1]), (name, T)
                rows.append({"sf": sf, "mode": name, "T": T, "ms": ms, "pairs": int(pairs.shape[0]),
                             "pairs_per_s": pairs.shape[0] / (ms / 1e3)})
                print(json.dumps(rows[-1]), flush=True)
    best = {}
    for r in rows:
        k = (r["sf"], r["mode"])
        if k not in best or r["ms"] < best[k]["ms"]:
            best[k] = r
    summary = {f"SF{sf}": {m: {"ms": best[(sf, m)]["ms"], "T": best[(sf, m)]["T"]}
                            for m in ("PixelOnly", "PixelBox-NoSep", "PixelBox")} for sf in range(1, 6)}
    with open(args.out, "w") as f:
        json.dump({"workload": f"{args.tiles}x{args.tiles} tiles of configs[0], ~{rows[0]['pairs']} pairs, "
                               "coordinates x SF", "rows": rows, "best": summary}, f, indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
