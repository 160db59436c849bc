#!/usr/bin/env python
"""Benchmark of the B200 PixelBox hot path (SCCG, arXiv 1208.0277).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config slide]

One step = one pass of the whole hot path over one
whole-slide image pair resident in HBM: prep of both sets (MBR, shoelace area,
edge records), the grid-hash MBR join, PixelBox over every candidate pair, the
deterministic integer sums, (N > 1: one NCCL all_reduce of the int64 sums) and
J' on the host.  Workload: BASELINE.json configs[1] ("slide"), synthetic,
~500k nucleus polygons per set, ~670k MBR-overlapping pairs.  At N GPUs each
rank processes its own slide image (weak scaling, sharded by image as in
configs[3]); the only collective is the sums all_reduce.

Prints ONE JSON line (rank 0).  value = pairs/s over all ranks (max-over-ranks
device time).  e2e = the same metric through the public API with host inputs
(pinned H2D copies + D2H of the sums inside the timed region).  roofline =
the dominant kernel, prep (about half the step): its algorithmic HBM bytes per
launch over its live CUDA-event time inside the timed
region, against the measured HBM copy bandwidth (MEASURED_PEAKS.json).
cpu_baseline = the oracle (oracle/) on this box's cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "polygon pairs/sec (and pixels tested/sec) at 1/2/4/8 B200 vs int-issue peak"
SMS_B200 = 148
ISSUE_LANES_PER_CLK_SM = 128  # 4 SMSPs x 1 warp-instruction x 32 lanes (nominal dispatch)
ALU_LANES_PER_CLK_SM = 64  # measured: ALU pipe 2 warp-inst/clk/SM (profiles/int_peak.json, scripts/int_peak.cu)
STAGE_EVERY = 5  # per-stage CUDA events on every 5th timed step (from the third: the first steps ramp up)
# our kernels per step besides the read-back (one GPU) or the sums pack + unpack around the all-reduce (N > 1):
# sums reset, prep init, prep, join (grid selection, Q insert, probe, compaction), PixelBox (counter reset, small,
# item)
LAUNCHES_PER_STEP = 10
OPS_PER_ROWTEST = 3  # sub, unsigned compare, predicated xor
OPS_PER_BOXEDGE = 8  # one lane classifying one edge against all sub-boxes of a split (minimum)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="slide", choices=["slide", "tile", "skewed", "combs", "study"])
    ap.add_argument("--images", type=int, default=100, help="study: whole-slide image pairs in the study (configs[3])")
    ap.add_argument("--bases", type=int, default=2, help="study: distinct generated slides the images are instanced from")
    ap.add_argument("--threshold", type=int, default=0)
    ap.add_argument("--shard", default="image", choices=["image", "tile"],
                    help="N > 1: image = one slide image per rank (weak scaling, configs[3]); tile = ONE slide cut "
                         "into y bands of P with their Q halo (strong scaling, SURVEY 8(e))")
    ap.add_argument("--e2e-steps", type=int, default=30)
    ap.add_argument("--e2e-unfused", action="store_true",
                    help="e2e: decode the packed rings with sccg_decode_rect_packed before the step graph "
                         "instead of inside prep (sccg_prep_sets_packed)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the skewed / combs lines added to the slide run")
    ap.add_argument("--json-out", default=None)
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
    }

    def __init__(self, index: int):
        self.index = index
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover - NVML missing
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in self.REASONS.items():
                    if r & bit and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------- workloads
def prep_algorithmic_bytes(sccg, S) -> int:
    """Bytes prep must move for set S: read the vertices (8 B)
    and offsets (8 B); write MBR (16 B), area (8 B), ecount (8 B) per polygon,
    one 8-byte record per vertical edge and one 4-byte word per raster row."""
    ec = S.ecount.long()
    m = S.mbr.long()
    rast = (ec[:, 0] & sccg.RASTER_FLAG) != 0
    nv = ec[:, 0] & (sccg.RASTER_FLAG - 1)
    rows = int(((m[:, 3] - m[:, 1]) * rast).sum())
    return 8 * S.nv + 8 * (S.n + 1) + 32 * S.n + 8 * int(nv.sum()) + 4 * rows


def lib_digest() -> str:
    """sha256 prefix of the library's SOURCES (csrc/*, include/sccg.h without
    comments and blank space, the nvcc flags of build.py; nvcc output is not
    byte-reproducible): static profile numbers
    (profiles/prep_traffic.json, issue_counts.json) apply only to the code they
    were taken on.  An experiment variant (SCCG_LIB) gets its own tag."""
    import glob
    import hashlib

    from paper_1208_0277_b200 import build as sbuild

    h = hashlib.sha256()
    pkg = os.path.join(ROOT, "paper_1208_0277_b200")
    import re

    for f in sorted(glob.glob(os.path.join(pkg, "csrc", "*"))) + [os.path.join(ROOT, "include", "sccg.h")]:
        with open(f, encoding="utf-8") as fh:
            code = fh.read()
        # comments and blank space do not change the code: drop them before hashing
        code = re.sub(r"/\*.*?\*/", "", code, flags=re.S)
        code = re.sub(r"//[^\n]*", "", code)
        code = "\n".join(line.strip() for line in code.splitlines() if line.strip())
        h.update(os.path.basename(f).encode() + b"\0" + code.encode())
    h.update(" ".join(sbuild.ARCH + sbuild.FLAGS).encode())  # the compile flags, not build.py's other logic
    h.update((os.environ.get("SCCG_LIB") or "").encode())
    return h.hexdigest()[:16]


def pixelbox_issue(key, pix_s, sms, clocks):
    """PixelBox warp-instruction issue rate against the measured integer-issue
    peak: ncu's instruction count of the small kernel for this
    exact workload key (config/shard/world; profiles/issue_counts.json, taken on
    the same library build -- otherwise None) over the live PixelBox stage time
    (CUDA events; includes the item kernel and the graph launch, so the rate is
    a lower bound).  Peak = the best integer mix of the microbenchmark
    (profiles/int_peak.json, LOP3 + IMAD on the ALU and FMA pipes) x SMs x the
    SM clock sampled during the run."""
    try:
        with open(os.path.join(ROOT, "profiles", "issue_counts.json")) as f:
            counts = json.load(f).get(key)
        with open(os.path.join(ROOT, "profiles", "int_peak.json")) as f:
            ip = json.load(f)
    except Exception:
        return None
    if not counts or "small_kernel" not in counts or counts.get("lib") != lib_digest():
        return None
    best = max(r["warp_inst_per_clk_per_sm"] for r in ip["results"])
    alu = max(r["warp_inst_per_clk_per_sm"] for r in ip["results"] if r["pipe"] == "alu")
    mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0
    achieved = counts["small_kernel"] / pix_s
    peak = best * sms * mhz * 1e6
    return {"achieved": achieved, "peak": peak, "unit": "warp-inst/s", "frac": achieved / peak,
            "frac_of_nominal_issue": achieved / (4 * sms * mhz * 1e6),
            "warp_inst_per_launch": counts["small_kernel"], "kernel": "small_kernel", "key": key,
            "peak_source": f"measured integer mix {best:.3f} warp-inst/clk/SM (ALU pipe alone {alu:.3f}; "
                           f"profiles/int_peak.json) x {sms} SMs x {mhz:.0f} MHz",
            "count_source": "ncu smsp__inst_executed.sum (profiles/issue_counts.json, same library) / live stage time"}


def pixelbox_algorithmic_bytes(sccg, P, Q, pairs) -> int:
    """Bytes the PixelBox stage must move for this pair list:
    per pair its index pair (8 B) and outputs (16 B), both polygons' MBR (16 B),
    area (8 B), ecount (8 B) and offset (8 B), and -- when both rings carry a
    raster -- the box's rows of both rasters (4 B each), else both rings'
    vertical-edge data (8 B per vertex slot used).  Computed with torch on the
    device, untimed."""
    import torch

    pr = pairs.long()
    p, q = pr[:, 0], pr[:, 1]
    mp, mq = P.mbr.long()[p], Q.mbr.long()[q]
    H = (torch.minimum(mp[:, 3], mq[:, 3]) - torch.maximum(mp[:, 1], mq[:, 1])).clamp(min=0)
    ep, eq = P.ecount.long()[p], Q.ecount.long()[q]
    rast = ((ep[:, 0] & sccg.RASTER_FLAG) != 0) & ((eq[:, 0] & sccg.RASTER_FLAG) != 0)
    edge = 8 * ((ep[:, 0] & (sccg.RASTER_FLAG - 1)) + (eq[:, 0] & (sccg.RASTER_FLAG - 1)))
    per = 24 + 2 * 40 + torch.where(rast, 8 * H, edge)
    return int(per.sum())


def hbm_peak():
    """Measured HBM copy bandwidth (MEASURED_PEAKS.json), else the profiling
    guide's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            v = float(json.load(f)["hbm_gbs"])
        return v, "MEASURED_PEAKS.json hbm_gbs (copy bandwidth, read+write)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def make_workload(config: str, image: int):
    import synth

    return synth.generate(config, image=image)


def synth_set(xy, offsets):
    import synth

    return synth.PolygonSet(xy, offsets)


def config_desc(config):
    return {
        "slide": "configs[1]: one 100k x 100k whole-slide image, two synthetic result sets of ~500k nucleus polygons",
        "tile": "configs[0]: one 4096x4096 tile, ~1,000 nucleus polygons per set",
        "skewed": "configs[2]: 4x4 tiles, nuclei + 16 glands per tile (MBR side up to 512)",
        "combs": "configs[4] analog: 16,384 independent highly concave comb pairs, 500-2000 vertices",
        "study": "configs[3]: a multi-image study of whole-slide image pairs (100k x 100k, ~500k nuclei per set), "
                 "sharded by image over the GPUs, one all-reduce of the integer sums",
    }[config]


# -------------------------------------------------------------- our arm
def self_check(args, A, B, pipe, n_local, local_sums, threads):
    """The benched step checks itself (rank-local, before any all-reduce): the
    pair list, EVERY pair's (I, U) written by the step, the integer sums, the
    exact ratio limbs and J' must equal the oracle's on the same workload
    (oracle/, all host threads; the combs workload -- too slow for a full
    oracle pass -- on a seeded 32-pair sample plus the size-free identities).
    Raises on any mismatch.  Returns (summary, the oracle pass or None)."""
    import numpy as np

    import oracle

    if local_sums[10] != 0:
        raise RuntimeError(f"self-check: sums status bits {local_sums[10]:#x}")
    pairs = pipe.pairs[:n_local].cpu().numpy()
    gi = pipe.inter[:n_local].cpu().numpy()
    gu = pipe.uni[:n_local].cpu().numpy()
    units = sum(int(v) << (30 * k) for k, v in enumerate(local_sums[6:10]))
    if args.config == "combs":
        idx = np.sort(np.random.default_rng(7).choice(n_local, size=min(32, n_local), replace=False))
        ei, eu = oracle.pair_areas(A, B, pairs[idx], threads=threads)
        if not ((ei == gi[idx]).all() and (eu == gu[idx]).all()):
            raise RuntimeError("self-check: sampled pairs differ from the oracle")
        ap, _ = oracle.set_props(A)
        aq, _ = oracle.set_props(B)
        if not (gi + gu == ap[pairs[:, 0]] + aq[pairs[:, 1]]).all() or local_sums[2] != int(gi.sum()):
            raise RuntimeError("self-check: size-free identities fail")
        return {"oracle": "32 sampled pairs + identities", "pairs_checked": int(len(idx))}, None
    ref = oracle_pass(A, B, threads)
    if pairs.shape != ref["pairs"].shape or not (pairs == ref["pairs"]).all():
        raise RuntimeError("self-check: pair list differs from the oracle's join")
    bad = np.nonzero((gi != ref["inter"]) | (gu != ref["uni"]))[0]
    if len(bad):
        raise RuntimeError(f"self-check: {len(bad)} pairs differ from the oracle, first {bad[:5].tolist()}")
    o = ref["sums"]
    want = [o["n_pairs"], o["n_nonzero"], o["sum_inter"], o["sum_union"], o["sum_area_p"], o["sum_area_q"]]
    if local_sums[:6] != want or units != ref["units"]:
        raise RuntimeError(f"self-check: sums {local_sums} differ from the oracle's {want} / units")
    rel = None
    if ref["jprime_exact"] is not None:
        import paper_1208_0277_b200 as sccg

        j, _ = sccg.jaccard(local_sums)
        ex = float(ref["jprime_exact"])
        rel = abs(j - ex) / ex
        if rel > 1e-12:
            raise RuntimeError(f"self-check: J' {j} vs exact {ex}")
    return {"oracle": "full pass (join, all pairs' I and U, sums, limbs, J')", "pairs_checked": int(n_local),
            "jprime_rel_err_vs_exact": rel, "oracle_seconds": ref["seconds"], "oracle_threads": threads}, ref


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1208_0277_b200 as sccg
    from paper_1208_0277_b200 import dist as sdist

    local_rank = local_rank % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if rank == 0:
        sccg.load(build=True)  # rebuild only if stale; other ranks wait, then load
    if world > 1:
        dist.barrier()
    sccg.load(build=False)
    if args.shard == "tile":
        # one slide for all ranks: this rank's P band and the Q that can meet it
        A, B = make_workload(args.config, image=0)
        pl, ph = sdist.ring_bounds(A.xy, A.offsets)
        ql, qh = sdist.ring_bounds(B.xy, B.offsets)
        pi, qi = sdist.band_shards(pl, ph, ql, qh, world)[rank]
        A = synth_set(*sdist.subset_rings(A.xy, A.offsets, pi))
        B = synth_set(*sdist.subset_rings(B.xy, B.offsets, qi))
    else:
        A, B = make_workload(args.config, image=rank)
    xy_p = torch.from_numpy(A.xy).pin_memory()
    off_p = torch.from_numpy(A.offsets).pin_memory()
    xy_q = torch.from_numpy(B.xy).pin_memory()
    off_q = torch.from_numpy(B.offsets).pin_memory()
    d_xy_p, d_off_p = xy_p.to(dev), off_p.to(dev)
    d_xy_q, d_off_q = xy_q.to(dev), off_q.to(dev)
    torch.cuda.synchronize()
    P = sccg.DeviceSet(d_xy_p, d_off_p, prep=False)
    Q = sccg.DeviceSet(d_xy_q, d_off_q, prep=False)
    stream = torch.cuda.current_stream()
    # The whole step (prep x2, join, PixelBox with the per-pair outputs) is
    # device-resident with no host sync until the sums are read, replayed as
    # ONE CUDA graph.  Steps are pipelined on the host: step i+1 is enqueued
    # before step i's sums are read (the read-back is in-stream into one of two
    # pinned buffers), so the GPU never idles on the host's per-step read-back;
    # every step's result is still read and checked.  One GPU: the PixelBox
    # graph ends with sccg_sums_copy into the pinned buffer (the GPU writes it,
    # no copy-engine transfer).  N > 1: all_reduce first, then the copy.
    host_bufs = [torch.zeros(len(sccg.SUMS_FIELDS), dtype=torch.int64).pin_memory() for _ in range(2)]
    done_ev = [torch.cuda.Event() for _ in range(2)]
    cap = 3 * max(P.n, Q.n) + 1024
    # N > 1 over NCCL: the all-reduce is captured in the step graph (before the
    # read-back); gloo (several ranks sharing one GPU, tests) runs it after the graph
    in_graph = world > 1 and dist.get_backend() == "nccl"
    pipe = sccg.Pipeline(P, Q, cap=cap, threshold=args.threshold, graph=True,
                         readback=host_bufs if world == 1 or in_graph else ())
    threads = max(1, (os.cpu_count() or 1) // world)

    # ---- self-check of the benched step against the oracle (rank-local, before any all-reduce)
    pipe.run(slot=0)
    torch.cuda.synchronize()
    n_local = pipe.check()  # raises on a pair-buffer overflow or any device status bit
    local = [int(v) for v in pipe.sums.tolist()]
    check, ref_pass = self_check(args, A, B, pipe, n_local, local, threads)
    collective = "eager after the graph" if world > 1 else None
    if in_graph:  # recapture with the collective inside (the self-check needed the rank-local sums)
        try:
            pipe = sccg.Pipeline(P, Q, cap=cap, threshold=args.threshold, graph=True, readback=host_bufs,
                                 allreduce=sdist.allreduce_sums)
            collective = "NCCL, captured in the step graph"
        except Exception as exc:  # keep the run: the same collective, launched after each replay
            print(f"[bench] NCCL capture failed ({exc!r}); all-reduce after the graph", file=sys.stderr)
            in_graph = False
            pipe = sccg.Pipeline(P, Q, cap=cap, threshold=args.threshold, graph=True, readback=())

    def enqueue(i, events=None):
        sums = pipe.run(events, slot=i % 2)
        if world > 1 and not in_graph:
            sdist.allreduce_sums(sums)  # row a9: the only collective (int64 SUM of the packed vector)
            host_bufs[i % 2].copy_(sums, non_blocking=True)
        done_ev[i % 2].record()

    def collect(i):
        done_ev[i % 2].synchronize()
        return sccg.sums_to_host(host_bufs[i % 2])

    for i in range(max(args.warmup, 3)):
        enqueue(i)
        first = collect(i)
    if world == 1 and [getattr(first, f) for f in sccg.SUMS_FIELDS] != local:
        raise RuntimeError("warm-up sums differ from the checked step's")
    # one untimed counting run for the algorithmic work per launch
    counters = torch.zeros(8, dtype=torch.int64, device=dev)
    sccg.pixelbox(P, Q, pipe.pairs[:n_local], threshold=args.threshold, counters=counters, want_inter=False,
                  want_union=False)
    cnt = counters.cpu().tolist()
    pix_alg = pixelbox_algorithmic_bytes(sccg, P, Q, pipe.pairs[:n_local])

    # ---- timed region: K steps, barrier + synchronize on both sides
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # prep | join | PixelBox: live CUDA events on the launch stream, recorded
    # around the stages of every STAGE_EVERY-th timed step (each event record
    # between graphs costs the step ~2.5 us, so sampling keeps the step honest)
    sampled = list(range(min(2, args.steps - 1), args.steps, STAGE_EVERY))
    stage_ev = {i: [torch.cuda.Event(enable_timing=True) for _ in range(4)] for i in sampled}
    results = []
    with ClockSampler(local_rank) as clk:
        t0.record(stream)
        wall0 = time.perf_counter()
        for i in range(args.steps):
            enqueue(i, stage_ev.get(i))
            if i > 0:
                results.append(collect(i - 1))
        results.append(collect(args.steps - 1))
        t1.record(stream)
        torch.cuda.synchronize()
        wall1 = time.perf_counter()
    stage_ms = [sum(ev[k].elapsed_time(ev[k + 1]) for ev in stage_ev.values()) for k in range(3)]
    host = results[-1]
    if any(bytes(r) != bytes(first) for r in results):
        raise RuntimeError("a timed step's sums differ from the warm-up's (nondeterminism)")
    if any(int(r.status) for r in results):
        raise RuntimeError("a timed step's sums carry device status bits")
    if world > 1:
        dist.barrier()
    if pipe.check() != n_local:
        raise RuntimeError("pair count changed between steps")
    ms = t0.elapsed_time(t1)
    times = torch.tensor([ms] + [t / len(sampled) for t in stage_ms] + [float(n_local)], dtype=torch.float64,
                         device=dev)
    if world > 1:
        mx = times.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        tot = times.clone()
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    else:
        mx, tot = times, times
    ms_max, prep_ms_max, join_ms_max, pix_ms_max = (float(v) for v in mx[:4])
    total_pairs = int(round(float(tot[4])))
    jprime, pooled = sccg.jaccard(host)

    # ---- e2e: public API from pinned host buffers, H2D + D2H inside the timed region
    e2e_steps = max(1, min(args.e2e_steps, args.steps))
    h2d = xy_p.numel() * 4 + off_p.numel() * 8 + xy_q.numel() * 4 + off_q.numel() * 8
    d2h = len(sccg.SUMS_FIELDS) * 8

    def e2e_step():
        a = xy_p.to(dev, non_blocking=True)
        b = off_p.to(dev, non_blocking=True)
        c = xy_q.to(dev, non_blocking=True)
        d = off_q.to(dev, non_blocking=True)
        Pe = sccg.DeviceSet(a, b)
        Qe = sccg.DeviceSet(c, d)
        pr = sccg.filter_pairs(Pe, Qe, cap=cap)
        s = sccg.new_sums(dev)
        sccg.pixelbox(Pe, Qe, pr, threshold=args.threshold, sums=s, want_inter=False, want_union=False, check=False)
        if world > 1:
            sdist.allreduce_sums(s)
        return sccg.jaccard(s.cpu())  # raises on device status bits

    e2e_step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        je, _ = e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    if not (je == jprime or (math.isnan(je) and math.isnan(jprime))):
        raise RuntimeError("e2e J' differs from the device-resident step's")
    e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
    e2e_value = total_pairs * e2e_steps / (float(e_ms[0]) / 1e3)
    e2e = {"value": e2e_value, "unit": "pairs/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
           "steps": e2e_steps, "encoding": "plain int32 vertices"}

    # the same through the packed rectilinear encoding (sccg_decode_rect_packed):
    # the host holds each ring as a 16-bit head (vertex count, move width, first
    # axis), its start as an int16 delta and its axis-alternating moves at 4, 8
    # or 16 bits -- ~0.8 bytes per vertex over PCIe instead of 8, no offsets --
    # decoded exactly on the GPU (offsets rebuilt by a block scan)
    enc = [sccg.encode_rect_packed(S.xy, S.offsets) for S in (A, B)]
    e2e_plain = None
    if all(e is not None for e in enc):
        cp = [sccg.pin_packed(e) for e in enc]
        h2d_c = sum(t.numel() * t.element_size() for e in cp for t in e.values())

        def e2e_compact_step():
            sets = []
            for e, S in zip(cp, (A, B)):
                xy, o = sccg.decode_rect_packed({k: t.to(dev, non_blocking=True) for k, t in e.items()},
                                                int(S.offsets[-1]))
                sets.append(sccg.DeviceSet(xy, o))
            pr = sccg.filter_pairs(sets[0], sets[1], cap=cap)
            s = sccg.new_sums(dev)
            sccg.pixelbox(sets[0], sets[1], pr, threshold=args.threshold, sums=s, want_inter=False, want_union=False,
                          check=False)
            if world > 1:
                sdist.allreduce_sums(s)
            return sccg.jaccard(s.cpu())

        st = None
        if world == 1:  # (N > 1: eager steps with the eager collective -- Streamer(allreduce=...) exists but the
            # multi-GPU NCCL capture of three slot graphs is unexercised on hardware here)
            # streamed: step i + 1's host -> device copy (copy stream) overlaps step i's decode and compute
            # three slots: the host reads step i - 2's result while steps i - 1 and i are in flight, so
            # enqueueing (Python) never delays the next copy
            step = sccg.PackedStep(enc[0], enc[1])  # both sets in one pinned buffer: one copy per step
            # fused: the step graph's prep decodes the packed rings itself (sccg_prep_sets_packed); N > 1: the
            # NCCL all-reduce inside each slot's graph
            try:
                st = sccg.Streamer(A.n, int(A.offsets[-1]), B.n, int(B.offsets[-1]), cap=cap,
                                   threshold=args.threshold, depth=3, fused=None if args.e2e_unfused else step,
                                   allreduce=sdist.allreduce_sums if world > 1 else None)
            except Exception as exc:
                if world == 1:
                    raise
                print(f"[bench] e2e: NCCL capture in the Streamer failed ({exc!r}); eager steps", file=sys.stderr)
                st = None
        if st is not None:
            h2d_c = step.nbytes
            for _ in range(st.depth):  # warm-up: every slot once (each slot's graph was captured at construction)
                st.result(st.submit_step(step))
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0.record(stream)
            st.copy_stream.wait_event(e0)  # the first copy starts inside the timed region
            inflight = []
            for _ in range(e2e_steps):
                inflight.append(st.submit_step(step))
                if len(inflight) == st.depth:
                    jc, _ = sccg.jaccard(st.result(inflight.pop(0)))
            for t in inflight:
                jc, _ = sccg.jaccard(st.result(t))
            e1.record(stream)
            torch.cuda.synchronize()
        else:
            e2e_compact_step()
            dist.barrier()
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(e2e_steps):
                jc, _ = e2e_compact_step()
            e1.record(stream)
            torch.cuda.synchronize()
        if not (jc == jprime or (math.isnan(jc) and math.isnan(jprime))):
            raise RuntimeError("compact e2e J' differs from the device-resident step's")
        c_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(c_ms, op=dist.ReduceOp.MAX)
        e2e_plain = e2e
        e2e = {"value": total_pairs * e2e_steps / (float(c_ms[0]) / 1e3), "unit": "pairs/s",
               "h2d_bytes_per_step": int(h2d_c), "d2h_bytes_per_step": int(d2h), "steps": e2e_steps,
               "encoding": ("packed rectilinear rings (16-bit head, int16 start delta, variable-length or 4/8/16-bit "
                            "axis-alternating moves; no offsets), decoded "
                            + ("inside prep (sccg_prep_sets_packed)" if st is not None and not args.e2e_unfused
                               else "by sccg_decode_rect_packed")),
               "pipelining": ("sccg.Streamer, three slots: each step's host -> device copy (one pinned buffer) on a "
                              "copy stream overlaps the previous step's graph (" +
                              ("decode kernels on a decode stream, then the step graph" if args.e2e_unfused
                               else "prep decoding the packed rings, join, PixelBox") +
                              ")" + (", the NCCL all-reduce in the graph" if world > 1 else "") +
                              "; every step's sums read back" if st is not None else None)}

    if rank != 0:
        return None, None
    value = total_pairs * args.steps / (ms_max / 1e3)
    clocks = clk.summary()
    # roofline of the dominant kernel: prep (HBM-bound; one launch preps both
    # sets), rank 0's algorithmic bytes per launch (inputs read once + outputs
    # written once) over its live time (CUDA events around the
    # prep graph on the launch stream)
    alg = prep_algorithmic_bytes(sccg, P) + prep_algorithmic_bytes(sccg, Q)
    prep_launch_s = prep_ms_max / 1e3
    achieved = alg / prep_launch_s / 1e9
    peak, peak_src = hbm_peak()
    traffic = None
    prof = os.path.join(ROOT, "profiles", "prep_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                pj = json.load(f)
            if pj.get("config") == args.config and pj.get("lib") == lib_digest() and world == 1:
                traffic = pj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    # PixelBox (second kernel group): integer lane-op rate vs the issue peak, context only
    ops = OPS_PER_ROWTEST * cnt[sccg.CNT_ROWTESTS] + OPS_PER_BOXEDGE * cnt[sccg.CNT_BOXEDGES]
    pix_s = pix_ms_max / 1e3
    peak_mhz = clocks["sm_max_mhz"] or 1965.0
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    alu_peak = sms * ALU_LANES_PER_CLK_SM * peak_mhz * 1e6 / 1e9
    issue = pixelbox_issue(f"{args.config}/{args.shard if world > 1 else 'image'}/{world}", pix_s, sms, clocks)
    # our kernels per step (profiles/<round>/launches_slide_summary.txt)
    launches_per_step = LAUNCHES_PER_STEP + (1 if world == 1 else 2)
    cfg = workload_config(args.config, A, B, n_local, world, args.shard)
    cfg.update({"pairs_total": total_pairs, "threshold_T": args.threshold or 2048, "allreduce": collective,
                "l2": "inputs larger than L2 (vertex arrays ~%d MB per rank > 126 MB)" % ((P.nv + Q.nv) * 8 // 2**20)})
    out = {
        "metric": METRIC,
        "value": value,
        "unit": "pairs/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(args.warmup, 3),
        "ms_per_step": ms_max / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if args.shard == "tile" and world > 1 else "weak",
        "vs_baseline": None,
        "dtype": "int32",
        "data": "synthetic (seeded generator synth/, nucleus polygons per PAPER.md §5.1)",
        "impl": "ours",
        "config": cfg,
        "pixels_tested_per_s": cnt[sccg.CNT_PIXELS] * world / pix_s,
        "stage_ms": {"prep": prep_ms_max, "join": join_ms_max, "pixelbox": pix_ms_max,
                     "sampled_steps": len(sampled), "every": STAGE_EVERY},
        "jprime": jprime,
        "pooled_jaccard": pooled,
        "self_check": check,
        "counters": {"pixels": cnt[0], "rowtests": cnt[1], "boxes": cnt[2], "boxedges": cnt[3], "splits": cnt[4],
                     "pixboxes": cnt[5], "rootpx": cnt[6]},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": "prep_kernel (P and Q in one launch)", "algorithmic_bytes_per_launch": alg,
                     "peak_source": peak_src},
        "pixelbox_hbm": {"achieved": pix_alg / pix_s / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": pix_alg / pix_s / 1e9 / peak, "algorithmic_bytes_per_step": pix_alg,
                         "note": "PixelBox stage (small + item kernels): pair list, per-polygon metadata, raster rows "
                                 "or edge records, per-pair outputs (bench.py pixelbox_algorithmic_bytes)"},
        "pixelbox_alu": {"achieved": ops / pix_s / 1e9, "peak": alu_peak, "unit": "Gop/s",
                         "frac": ops / pix_s / 1e9 / alu_peak,
                         "peak_source": f"{sms} SMs x 64 ALU-pipe lanes/clk (measured, profiles/int_peak.json) x "
                                        f"{peak_mhz:.0f} MHz"},
        "pixelbox_issue": issue,
        "e2e": e2e,
        "e2e_plain": e2e_plain,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks,
        "wall_s": wall1 - wall0,
    }
    return out, (A, B, ref_pass)


# ------------------------------------------------- extra configs (N = 1)
def extra_configs(args, dev, names=("skewed", "combs"), steps: int = 20):
    """Short device-resident runs of the sampling-box configs beside the
    headline line (configs[2] glands and the configs[4] comb analog: the
    large-pair path the slide hardly enters), each self-checked against the
    oracle like the main step, timed as whole-step graph replays (CUDA events,
    inputs resident) plus one stage-event pass."""
    import torch

    import paper_1208_0277_b200 as sccg

    out = {}
    threads = os.cpu_count() or 1
    for name in names:
        A, B = make_workload(name, 0)
        P = sccg.DeviceSet(*sccg.to_device(A.xy, A.offsets, dev), prep=False)
        Q = sccg.DeviceSet(*sccg.to_device(B.xy, B.offsets, dev), prep=False)
        pipe = sccg.Pipeline(P, Q, cap=3 * max(P.n, Q.n) + 1024, threshold=args.threshold, graph=True)
        pipe.run()
        torch.cuda.synchronize()
        n = pipe.check()
        local = [int(v) for v in pipe.sums.tolist()]
        sub = argparse.Namespace(**{**vars(args), "config": name})
        chk, _ = self_check(sub, A, B, pipe, n, local, threads)
        for _ in range(3):
            pipe.run()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        pipe.run(ev)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0.record()
        for _ in range(steps):
            pipe.run()
        t1.record()
        torch.cuda.synchronize()
        if [int(v) for v in pipe.sums.tolist()] != local:
            raise RuntimeError(f"{name}: timed sums differ from the checked step's")
        ms = t0.elapsed_time(t1) / steps
        out[name] = {"description": config_desc(name), "pairs": n, "ms_per_step": ms, "value": n / (ms / 1e3),
                     "unit": "pairs/s", "steps": steps,
                     "stage_ms": {"prep": ev[0].elapsed_time(ev[1]), "join": ev[1].elapsed_time(ev[2]),
                                  "pixelbox": ev[2].elapsed_time(ev[3])},
                     "self_check": chk}
        del pipe, P, Q
    return out


# ----------------------------------------------------------- configs[3]
def study_images(n_images: int, n_bases: int):
    """The study's image list: image i is base slide i % n_bases under grid
    symmetry (i // n_bases) % 8 (transpose, then mirror x / y) and an integer
    translation.  A symmetry of the pixel lattice maps pixel cells to pixel
    cells, so every pair's |p n q| and |p u q| -- and the MBR pair list -- are
    the base's (pinned by the oracle's symmetry invariants, tests/test_oracle.py);
    the coordinates, ring orientation (mirrors make rings clockwise) and raster
    shapes (transposes) differ per image."""
    out = []
    for i in range(n_images):
        sym = (i // n_bases) % 8
        out.append({"image": i, "base": i % n_bases, "sym": sym,
                    "dx": 200_000 + 131_072 * (i % 64), "dy": 200_000 + 131_072 * (i // 64)})
    return out


def instance_xy(xy, sym: int, dx: int, dy: int):
    """Device-side instancing of one image from its base (torch on the GPU;
    input synthesis, not a step of the path): (x, y) -> symmetry -> + (dx, dy)."""
    import torch

    x, y = xy[:, 0], xy[:, 1]
    if sym & 4:
        x, y = y, x
    if sym & 1:
        x = -x
    if sym & 2:
        y = -y
    return torch.stack([x + dx, y + dy], 1).to(torch.int32).contiguous()


def run_study(args, rank, world, local_rank):
    """configs[3]: the study's images sharded over the ranks by LPT (equal
    costs per base: round robin), each rank's images resident in HBM and run
    back to back as ONE graph (sccg.Study: prep, join, PixelBox per image, all
    adding into one device sums vector), then ONE all-reduce of the packed
    int64 sums (NCCL, captured in the same graph; gloo: after it).  A step =
    one pass over all images of the study.  The rank-local sums must equal
    the sum of the oracle's sums of each image's base (self-check)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1208_0277_b200 as sccg
    from paper_1208_0277_b200 import dist as sdist

    local_rank = local_rank % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if rank == 0:
        sccg.load(build=True)
    if world > 1:
        dist.barrier()
    sccg.load(build=False)
    plan = study_images(args.images, args.bases)
    mine = [plan[i] for i in sdist.shard_for_rank(len(plan), world, rank)]
    bases_needed = sorted({im["base"] for im in mine})
    threads = max(1, (os.cpu_count() or 1) // world)
    host, dbase, ref = {}, {}, {}
    for b in bases_needed:
        A, B = make_workload("slide", image=b)
        t = [torch.from_numpy(v).pin_memory() for v in (A.xy, A.offsets, B.xy, B.offsets)]
        host[b] = t
        dbase[b] = [v.to(dev) for v in t]
        r = oracle_pass(A, B, threads)  # the self-check's expected sums for every image of this base
        o = r["sums"]
        ref[b] = {"sums": [o["n_pairs"], o["n_nonzero"], o["sum_inter"], o["sum_union"], o["sum_area_p"],
                           o["sum_area_q"]], "units": r["units"], "seconds": r["seconds"], "A": A, "B": B}
    images = []
    for im in mine:
        xp, op, xq, oq = dbase[im["base"]]
        images.append((instance_xy(xp, im["sym"], im["dx"], im["dy"]), op,
                       instance_xy(xq, im["sym"], im["dx"], im["dy"]), oq))
    torch.cuda.synchronize()
    backend = dist.get_backend() if world > 1 else None
    host_bufs = [torch.zeros(len(sccg.SUMS_FIELDS), dtype=torch.int64).pin_memory() for _ in range(2)]
    done_ev = [torch.cuda.Event() for _ in range(2)]
    # the all-reduce inside the step graph when NCCL (graph-capturable); gloo runs it after the graph
    in_graph = world > 1 and backend == "nccl"
    try:
        study = sccg.Study(images, threshold=args.threshold, graph=True,
                           readback=host_bufs if world == 1 or in_graph else (),
                           allreduce=sdist.allreduce_sums if in_graph else None)
    except Exception as exc:  # keep the run: the same collective, launched after each replay
        if not in_graph:
            raise
        print(f"[bench] NCCL capture failed ({exc!r}); all-reduce after the graph", file=sys.stderr)
        in_graph = False
        study = sccg.Study(images, threshold=args.threshold, graph=True, readback=())
    # the self-check needs the rank-local sums: one eager pass without the all-reduce
    study.allreduce = None
    study.run(events=[[torch.cuda.Event() for _ in range(4)] for _ in images])
    torch.cuda.synchronize()
    study.check()
    local = [int(v) for v in study.sums.tolist()]
    want = [sum(ref[im["base"]]["sums"][f] for im in mine) for f in range(6)]
    units = sum(int(v) << (30 * k) for k, v in enumerate(local[6:10]))
    if local[:6] != want or units != sum(ref[im["base"]]["units"] for im in mine):
        raise RuntimeError(f"study self-check: rank sums {local[:6]} != the oracle's {want} (or ratio units)")
    study.allreduce = sdist.allreduce_sums if in_graph else None
    check = {"oracle": f"full oracle pass of each base slide; every image's sums = its base's (lattice symmetry), "
                       f"rank-local sums == sum over its {len(mine)} images", "images_checked": len(mine),
             "oracle_seconds": sum(ref[b]["seconds"] for b in bases_needed)}

    def enqueue(i, events=None):
        sums = study.run(events, slot=i % 2)
        if world > 1 and not in_graph:
            sdist.allreduce_sums(sums)
            host_bufs[i % 2].copy_(sums, non_blocking=True)
        done_ev[i % 2].record()

    def collect(i):
        done_ev[i % 2].synchronize()
        return sccg.sums_to_host(host_bufs[i % 2])

    for i in range(max(args.warmup, 3)):
        enqueue(i)
        first = collect(i)
    if world == 1 and [getattr(first, f) for f in sccg.SUMS_FIELDS] != local:
        raise RuntimeError("study warm-up sums differ from the checked pass's")
    # algorithmic prep bytes of every image (untimed: each image prepped once on its own)
    alg = 0
    for xp, op, xq, oq in images:
        for xy, off in ((xp, op), (xq, oq)):
            S = sccg.DeviceSet(xy, off)
            alg += prep_algorithmic_bytes(sccg, S)
            del S
    stream = torch.cuda.current_stream()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # (the study's sampled passes run eagerly: one in ten)
    sampled = list(range(min(2, args.steps - 1), args.steps, 2 * STAGE_EVERY))
    stage_ev = {i: [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in images] for i in sampled}
    results = []
    with ClockSampler(local_rank) as clk:
        t0.record(stream)
        wall0 = time.perf_counter()
        for i in range(args.steps):
            enqueue(i, stage_ev.get(i))
            if i > 0:
                results.append(collect(i - 1))
        results.append(collect(args.steps - 1))
        t1.record(stream)
        torch.cuda.synchronize()
        wall1 = time.perf_counter()
    stage_ms = [sum(ev[k].elapsed_time(ev[k + 1]) for evs in stage_ev.values() for ev in evs) for k in range(3)]
    final = results[-1]
    if any(bytes(r) != bytes(first) for r in results):
        raise RuntimeError("a timed study step's sums differ from the warm-up's (nondeterminism)")
    if any(int(r.status) for r in results):
        raise RuntimeError("a timed study step's sums carry device status bits")
    if world > 1:
        dist.barrier()
    ms = t0.elapsed_time(t1)
    times = torch.tensor([ms] + [t / len(sampled) for t in stage_ms] + [float(local[0]), float(alg)],
                         dtype=torch.float64, device=dev)
    if world > 1:
        mx = times.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        tot = times.clone()
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    else:
        mx, tot = times, times
    ms_max, prep_ms_max, join_ms_max, pix_ms_max = (float(v) for v in mx[:4])
    total_pairs = int(round(float(tot[4])))
    if int(final.n_pairs) != total_pairs:
        raise RuntimeError("all-reduced pair count differs from the ranks' total")
    jprime, pooled = sccg.jaccard(final)

    # e2e: each image through the public API from pinned host memory (H2D of its inputs -- the base slide's
    # buffers: an image differs from its base only by an exact lattice symmetry, so the bytes moved and the
    # areas are the same), join, PixelBox, all-reduce, D2H of the sums
    # (the packed rectilinear encoding when both sets of the base encode: ~0.8 bytes per vertex, no offsets)
    e2e_steps = 1
    compact = {}
    for b in bases_needed:
        ea, eb = (sccg.encode_rect_packed(S.xy, S.offsets) for S in (ref[b]["A"], ref[b]["B"]))
        if ea is not None and eb is not None:
            compact[b] = [sccg.pin_packed(e) for e in (ea, eb)]
    h2d = 0
    for im in mine:
        b = im["base"]
        if b in compact:
            h2d += sum(t.numel() * t.element_size() for e in compact[b] for t in e.values())
        else:
            h2d += sum(t.numel() * t.element_size() for t in host[b])

    def upload(b):
        if b not in compact:
            a, o1, c, o2 = (t.to(dev, non_blocking=True) for t in host[b])
            return sccg.DeviceSet(a, o1), sccg.DeviceSet(c, o2)
        sets = []
        for e, S in zip(compact[b], (ref[b]["A"], ref[b]["B"])):
            xy, o = sccg.decode_rect_packed({k: t.to(dev, non_blocking=True) for k, t in e.items()},
                                            int(S.offsets[-1]))
            sets.append(sccg.DeviceSet(xy, o))
        return sets

    def e2e_step():
        s = sccg.new_sums(dev)
        for im in mine:
            Pe, Qe = upload(im["base"])
            pr = sccg.filter_pairs(Pe, Qe, cap=study.cap)
            sccg.pixelbox(Pe, Qe, pr, threshold=args.threshold, sums=s, want_inter=False, want_union=False,
                          check=False)
        if world > 1:
            sdist.allreduce_sums(s)
        return sccg.jaccard(s.cpu())

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    je, _ = e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    if not (je == jprime or (math.isnan(je) and math.isnan(jprime))):
        raise RuntimeError("study e2e J' differs from the device-resident step's")
    e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
    e2e_value = total_pairs * e2e_steps / (float(e_ms[0]) / 1e3)
    if rank != 0:
        return None, None
    clocks = clk.summary()
    alg_rank0 = float(times[5])
    achieved = alg_rank0 / (prep_ms_max / 1e3) / 1e9
    peak, peak_src = hbm_peak()
    cfg = {"workload": "study", "description": config_desc("study"), "images": args.images, "bases": args.bases,
           "images_per_gpu": len(mine), "pairs_total": total_pairs, "pairs_per_image": ref[bases_needed[0]]["sums"][0],
           "instancing": "image i = base slide i % bases under lattice symmetry (i // bases) % 8 + translation, "
                         "instanced on the device before the timed region",
           "parallelism": f"image-sharded x{world} (LPT)" if world > 1 else "1 GPU",
           "allreduce": ("NCCL, in the step graph" if in_graph else "gloo, after the graph") if world > 1 else None,
           "threshold_T": args.threshold or 2048,
           "l2": "inputs larger than L2 (~%d MB of vertices per image)" % ((images[0][0].numel() + images[0][2].numel()) * 4 // 2**20)}
    out = {
        "metric": METRIC, "value": total_pairs * args.steps / (ms_max / 1e3), "unit": "pairs/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_max / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic (seeded generator synth/, instanced per image on the device)", "impl": "ours",
        "config": cfg,
        "stage_ms": {"prep": prep_ms_max, "join": join_ms_max, "pixelbox": pix_ms_max, "sampled_steps": len(sampled),
                     "every": 2 * STAGE_EVERY, "note": "summed over the rank's images (sampled steps run eagerly)"},
        "jprime": jprime, "pooled_jaccard": pooled, "self_check": check,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "kernel": "prep_kernel (P and Q in one launch per image)",
                     "algorithmic_bytes_per_launch": alg_rank0 / max(1, len(mine)), "peak_source": peak_src},
        "e2e": {"value": e2e_value, "unit": "pairs/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": len(sccg.SUMS_FIELDS) * 8, "steps": e2e_steps,
                "encoding": "packed rectilinear rings (sccg_decode_rect_packed)" if compact else "plain int32 vertices"},
        "gpu_launches": (LAUNCHES_PER_STEP - 1) * len(mine) * args.steps + (2 if world == 1 else 4) * args.steps,
        "clocks": clocks, "wall_s": wall1 - wall0,
    }
    return out, None


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_pass(A, B, threads: int) -> dict:
    """One full pass of the oracle (oracle/, as it stands) over a workload:
    shoelace areas + MBRs of both sets, the sweep join, per-pair I and U by
    pixel counting, the integer sums, the exact ratio units and J' (Eq. 1).
    Returns the results and the seconds it took."""
    import oracle

    t0 = time.perf_counter()
    oracle.set_props(A)
    oracle.set_props(B)
    pairs = oracle.join(A, B)
    inter, uni = oracle.pair_areas(A, B, pairs, threads=threads)
    sums = oracle.sums(A, B, pairs, inter, uni)
    j = oracle.jaccard(inter, uni)
    sec = time.perf_counter() - t0
    units = sum(oracle.ratio_units(i, u) for i, u in zip(inter.tolist(), uni.tolist()) if i)
    return {"pairs": pairs, "inter": inter, "uni": uni, "sums": sums, "units": units, "jprime": j,
            "jprime_exact": oracle.jaccard_exact(inter, uni), "seconds": sec}


def oracle_sample(A, B, threads: int, budget_s: float) -> dict:
    """The oracle on whole 4096 x 4096 tiles of the image (polygons by MBR
    corner) in a seeded random order until ~budget_s seconds are spent: a
    bounded sample of the same workload for slow settings (1 thread)."""
    import numpy as np

    import oracle

    _, ma = oracle.set_props(A)
    _, mb = oracle.set_props(B)
    tile = 4096
    ta = (ma[:, 0] // tile) * 100000 + ma[:, 1] // tile
    tb = (mb[:, 0] // tile) * 100000 + mb[:, 1] // tile
    tiles = sorted(set(ta.tolist()))
    np.random.default_rng(0).shuffle(tiles)
    done_pairs, spent, ntiles = 0, 0.0, 0
    for t in tiles:
        Ai = A.subset(np.nonzero(ta == t)[0])
        Bi = B.subset(np.nonzero(tb == t)[0])
        t0 = time.perf_counter()
        oracle.set_props(Ai)
        oracle.set_props(Bi)
        pr = oracle.join(Ai, Bi)
        I, U = oracle.pair_areas(Ai, Bi, pr, threads=threads)
        oracle.jaccard(I, U)
        spent += time.perf_counter() - t0
        done_pairs += len(pr)
        ntiles += 1
        if spent > budget_s:
            break
    return {"pairs": done_pairs, "seconds": spent, "tiles": ntiles, "of_tiles": len(tiles)}


def cpu_baseline(config: str, A, B, full=None) -> dict:
    """The oracle, as it stands, on this host's cores (rank 0, N = 1): all
    threads over the whole workload (`full`, the pass bench.py also checks the
    GPU against), and one thread over a bounded sample of whole tiles."""
    threads = os.cpu_count() or 1
    if full is None:
        full = oracle_pass(A, B, threads)
    one = oracle_sample(A, B, 1, budget_s=4.0)
    n = len(full["pairs"])
    return {"value": n / full["seconds"], "unit": "pairs/s", "cores": threads, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"the whole {config} workload ({n} pairs): shoelace areas, sweep join, pixel-count I/U, "
                      f"integer sums, J' -- all {threads} threads",
            "seconds": full["seconds"],
            "one_thread": {"value": one["pairs"] / one["seconds"], "unit": "pairs/s", "cores": 1,
                           "sample": f"{one['tiles']} of {one['of_tiles']} 4096 x 4096 tiles ({one['pairs']} pairs), "
                                     f"same path, 1 thread", "seconds": one["seconds"]}}


def run_reference(args):
    """--impl reference: the oracle is this tier's reference arm.  Every step
    is one full oracle pass over the same workload (all host threads), so the
    line's steps / ms_per_step are what ran; warm-up passes untimed."""
    A, B = make_workload(args.config, 0)
    threads = os.cpu_count() or 1
    # warm-up passes (at least one: it also sizes the steps)
    for _ in range(max(args.warmup, 1)):
        r0 = oracle_pass(A, B, threads)
    # every step is a full pass unless that would run past ~3 minutes; then each
    # step is a bounded sample: whole 4096 x 4096 tiles of the same image until
    # its share of the budget is spent (oracle_sample)
    per_step = 180.0 / max(args.steps, 1)
    full = r0["seconds"] <= per_step
    secs, npairs, tiles = [], 0, 0
    for _ in range(args.steps):
        if full:
            r = oracle_pass(A, B, threads)
            secs.append(r["seconds"])
            npairs += len(r["pairs"])
        else:
            r = oracle_sample(A, B, threads, per_step)
            secs.append(r["seconds"])
            npairs += r["pairs"]
            tiles += r["tiles"]
    tot = sum(secs)
    value = npairs / tot
    out = {
        "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic", "impl": "reference",
        "config": workload_config(args.config, A, B, len(r0["pairs"])),
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": threads, "kind": "oracle",
                         "cpu_model": cpu_model(),
                         "sample": (f"each step: the whole {args.config} workload ({len(r0['pairs'])} pairs), full "
                                    f"oracle path, all {threads} threads" if full else
                                    f"each step: whole 4096 x 4096 tiles of the {args.config} workload for ~{per_step:.1f} s "
                                    f"({tiles} tiles, {npairs} pairs over {args.steps} steps), full oracle path, "
                                    f"all {threads} threads")},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    return out


def workload_config(config, A, B, n_pairs, world=1, shard="image"):
    return {"workload": config, "description": config_desc(config), "pairs_per_gpu": n_pairs,
            "polygons_p": A.n, "polygons_q": B.n, "vertices_p": int(A.offsets[-1]), "vertices_q": int(B.offsets[-1]),
            "parallelism": (f"{shard}-sharded x{world}" if world > 1 else "1 GPU")}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            out = run_reference(args)
            print(json.dumps(out))
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        # NCCL over NVLink/NVSwitch; SCCG_DIST_BACKEND=gloo lets several ranks share one
        # GPU for testing the multi-rank path (NCCL refuses two ranks on one device)
        backend = os.environ.get("SCCG_DIST_BACKEND", "nccl")
        if backend == "nccl":
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    out, extra = (run_study if args.config == "study" else run_ours)(args, rank, world, local_rank)
    if rank == 0:
        if not args.no_cpu_baseline and world == 1 and args.config not in ("combs", "study"):  # rank 0, N = 1
            A, B, ref_pass = extra
            out["cpu_baseline"] = cpu_baseline(args.config, A, B, ref_pass)
        if not args.no_extras and world == 1 and args.config == "slide":
            import torch

            out["other_configs"] = extra_configs(args, torch.device("cuda", 0))
        line = json.dumps(out)
        print(line)
        if args.json_out:
            with open(args.json_out, "w") as f:
                f.write(line + "\n")
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
