"""Fig. 9 analog on B200 (§5.3).

The paper switches its implementation optimizations on one at a time (shared-
memory vertex staging, a bank-conflict-free sampling-box stack, loop
unrolling) on 15,724 nucleus pairs at scale factors 1, 3 and 5, and reports
the time of each variant normalized to the unoptimized one (PixelBox-NoOpt).
The B200 counterparts, switched on cumulatively:

  V0 NoOpt        every optimization below off (Alg. 1's split order as written)
  V1 +DenseSplit  a split whose sub-boxes are all < T and mostly hover is
                  pixelized whole            runtime flag
  V2 +Raster      memoized per-polygon rasters (PIXELINPOLY once per polygon,
                  DESIGN.md §9)                             runtime flag
  V3 +TMA         prep stages its tiles with cp.async.bulk + L2 prefetch
                  instead of LSU copies                     build SCCG_PREP_NO_TMA
  V4 +PDL         programmatic dependent launch between the step's kernels
                  (all optimizations = the shipped build)   build SCCG_NO_PDL

Workload: 4 x 4 tiles of configs[0] (~16k nucleus pairs), coordinates x SF.
One process per library build (the library is loaded once per process):

    python scripts/fig9.py --lib libsccg_noopt.so --variants V0,V1,V2 --out a.json
    python scripts/fig9.py --lib libsccg_nopdl.so --variants V3 --out b.json
    python scripts/fig9.py --variants V4 --out c.json
    python scripts/fig9.py --merge a.json b.json c.json --out profiles/r02/fig9.json

Each row: per-stage device times (CUDA events, median of --reps graph-free
passes) and the whole step as one CUDA graph replay (median).  Every variant
must produce the same sums at a given SF (checked at --merge), and the areas
obey I(SF) = SF^2 I(1) (checked per process).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

VARIANTS = {  # name -> (raster, dense split, build)
    "V0": dict(name="NoOpt", raster=False, dense=False, build="noopt"),
    "V1": dict(name="+DenseSplit", raster=False, dense=True, build="noopt"),
    "V2": dict(name="+Raster", raster=True, dense=True, build="noopt"),
    "V3": dict(name="+TMA", raster=True, dense=True, build="nopdl"),
    "V4": dict(name="+PDL (all)", raster=True, dense=True, build="main"),
}


def run(args):
    import numpy as np
    import torch

    if args.lib:
        os.environ["SCCG_LIB"] = args.lib
    import paper_1208_0277_b200 as sccg
    import synth

    A, B = synth.generate("tile", width=4096 * args.tiles, height=4096 * args.tiles)
    rows = []
    base = None
    for sf in (1, 3, 5):
        P = sccg.DeviceSet(*sccg.to_device(A.xy * sf, A.offsets), prep=False)
        Q = sccg.DeviceSet(*sccg.to_device(B.xy * sf, B.offsets), prep=False)
        for v in args.variants.split(","):
            cfg = VARIANTS[v]
            pipe = sccg.Pipeline(P, Q, threshold=args.threshold, graph=True, raster=cfg["raster"],
                                 paper_split=not cfg["dense"])
            stage, step = [], []
            for r in range(args.reps + 2):
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
                torch.cuda.synchronize()
                pipe.run(ev)
                torch.cuda.synchronize()
                if r >= 2:
                    stage.append([ev[k].elapsed_time(ev[k + 1]) for k in range(3)])
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                pipe.run()
                e1.record()
                torch.cuda.synchronize()
                if r >= 2:
                    step.append(e0.elapsed_time(e1))
            n = pipe.check()
            sums = [int(x) for x in pipe.sums.tolist()]
            inter = pipe.inter[:n].cpu().numpy().copy()
            if sf == 1 and base is None:
                base = inter
            elif sf > 1 and not np.array_equal(inter, base * sf * sf):
                raise RuntimeError(f"scale law I(SF) = SF^2 I(1) fails at SF {sf} ({v})")
            med = np.median(np.array(stage), axis=0)
            rows.append({"variant": v, "name": cfg["name"], "build": cfg["build"], "sf": sf, "pairs": n,
                         "prep_ms": float(med[0]), "join_ms": float(med[1]), "pixelbox_ms": float(med[2]),
                         "step_ms": float(np.median(step)), "sums": sums, "lib": args.lib or "libsccg.so"})
            print(json.dumps(rows[-1]), flush=True)
            del pipe
    with open(args.out, "w") as f:
        json.dump(rows, f, indent=1)


def merge(args):
    rows = []
    for p in args.merge:
        with open(p) as f:
            rows += json.load(f)
    out = {"what": "Fig. 9 analog (PAPER.md §5.3, P:350-360): B200 implementation optimizations switched on "
                   "cumulatively, times normalized to V0 (NoOpt); ~16k nucleus pairs (4 x 4 tiles of configs[0]) "
                   "x SF", "variants": {k: v["name"] for k, v in VARIANTS.items()}, "by_sf": {}}
    for sf in (1, 3, 5):
        rs = sorted((r for r in rows if r["sf"] == sf), key=lambda r: r["variant"])
        if not rs:
            continue
        if any(r["sums"] != rs[0]["sums"] for r in rs):
            raise RuntimeError(f"variants disagree on the sums at SF {sf}")
        v0 = next(r for r in rs if r["variant"] == "V0")
        out["by_sf"][str(sf)] = [{"variant": r["variant"], "name": r["name"], "pixelbox_ms": r["pixelbox_ms"],
                                  "step_ms": r["step_ms"], "prep_ms": r["prep_ms"], "join_ms": r["join_ms"],
                                  "pixelbox_speedup_vs_noopt": v0["pixelbox_ms"] / r["pixelbox_ms"],
                                  "step_speedup_vs_noopt": v0["step_ms"] / r["step_ms"]} for r in rs]
    sp = {sf: out["by_sf"][sf][-1]["step_speedup_vs_noopt"] for sf in out["by_sf"]}
    out["trend"] = {"paper": "all optimizations: 1.14x at SF 1 rising to 1.30x at SF 5 (P:357)",
                    "b200_step_speedup_all_vs_noopt": sp,
                    "rises_with_sf": all(sp[a] <= sp[b] for a, b in zip(sorted(sp), sorted(sp)[1:]))}
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out["trend"]))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=None)
    ap.add_argument("--variants", default="V4")
    ap.add_argument("--tiles", type=int, default=4)
    ap.add_argument("--threshold", type=int, default=0)
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--out", default="fig9.json")
    ap.add_argument("--merge", nargs="*")
    a = ap.parse_args()
    merge(a) if a.merge else run(a)
