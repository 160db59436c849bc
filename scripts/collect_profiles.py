"""Turn a round's raw GPU outputs (scripts/gpu_profile.sh) into the tracked
summaries under profiles/<round>/: bench lines, the launch list and its per-step
summary, and key ncu metrics of each captured kernel.

    python scripts/collect_profiles.py gpurun_out/round_r01 profiles/r01
"""
import csv
import json
import os
import shutil
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
    "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "sm__cycles_elapsed.avg.per_second",
]


def ncu_summary(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    lines = []
    for vals in rows[2:]:
        lines += ncu_one(rows[0], rows[1], vals)
    return "\n".join(lines) + "\n"


def ncu_one(h, units, vals):
    d = {h[i]: (vals[i], units[i]) for i in range(len(h))}
    lines = [f"kernel: {d.get('Kernel Name', ('?', ''))[0]}"]
    for k in KEYS:
        if k in d:
            lines.append(f"{k:70s} {d[k][0]} {d[k][1]}")
    st = []
    for k, (v, _) in d.items():
        if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
            try:
                st.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    lines.append("stalls (warps per issue): " + ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)[:8]))
    return lines


def launch_summary(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    seq = [(r[ki], float(r[vi].replace(",", ""))) for r in data]
    idx = [i for i, s in enumerate(seq) if s[0].startswith("sccg::prep_init")] + [len(seq)]
    # the last timed Pipeline step: a prep_init .. next prep_init window holding
    # the join (grid_select) right after another such window -- an e2e step is
    # a P-only prep window followed by the Q prep + join + PixelBox window
    wins = [seq[a:b] for a, b in zip(idx, idx[1:])]
    has_join = [any("grid_select" in n for n, _ in w) for w in wins]
    # a timed step: only our kernels (no torch kernels of the untimed bookkeeping, no e2e decode), the join in it
    clean = [not any(n.startswith("at::") or "decode" in n or "small_kernel<1>" in n or "void at::" in n or
                     "prep_kernel<1>" in n  # the e2e step's prep from packed rings
                     for n, _ in w) for w in wins]
    full = [wins[i] for i in range(1, len(wins)) if has_join[i] and has_join[i - 1] and clean[i]]
    step = full[-1] if full else seq
    out = ["one bench step (timed Pipeline), ncu --metrics gpu__time_duration.sum --clock-control none",
           "(cold caches, serialised: compare shares, not absolute times)", ""]
    tot = sum(t for _, t in step)
    for name, t in step:
        out.append(f"{t / 1000:9.1f} us  {100 * t / tot:5.1f} %  {name[:90]}")
    out.append(f"total {tot / 1000:.1f} us over {len(step)} launches")
    return "\n".join(out) + "\n"


def ncu_rows(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    return [dict(zip(rows[0], r)) for r in rows[2:]]


def num(v):
    return float(str(v).replace(",", ""))


def static_profiles(src, dst):
    """profiles/prep_traffic.json (DRAM bytes of one prep launch) and
    profiles/issue_counts.json (the small kernel's warp instructions per launch),
    keyed by the library digest the bench checks before using them."""
    dig = open(os.path.join(src, "lib_digest.txt")).read().strip()
    root = os.path.dirname(os.path.abspath(dst.rstrip("/")))
    prep = os.path.join(src, "ncu_prep_kernel.ncu-rep")
    if os.path.exists(prep):
        d = ncu_rows(prep)[0]
        mb = {"MB": 1e6, "Mbyte": 1e6, "GB": 1e9, "Gbyte": 1e9, "KB": 1e3, "Kbyte": 1e3, "byte": 1}
        raw = subprocess.run(["ncu", "-i", prep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(raw.splitlines()))
        units = dict(zip(rows[0], rows[1]))
        rd = num(d["dram__bytes_read.sum"]) * mb.get(units["dram__bytes_read.sum"], 1)
        wr = num(d["dram__bytes_write.sum"]) * mb.get(units["dram__bytes_write.sum"], 1)
        with open(os.path.join(root, "prep_traffic.json"), "w") as f:
            json.dump({"config": "slide", "kernel": "prep_kernel (P and Q in one launch)", "lib": dig,
                       "source": f"ncu --set full --clock-control none, {dst}/ncu_prep_kernel.txt (one launch)",
                       "dram_bytes_read": int(rd), "dram_bytes_write": int(wr), "dram_bytes_per_launch": int(rd + wr)},
                      f, indent=1)
    small = os.path.join(src, "ncu_small_kernel.ncu-rep")
    if os.path.exists(small):
        d = ncu_rows(small)[0]
        with open(os.path.join(root, "issue_counts.json"), "w") as f:
            json.dump({"source": "ncu --set full --clock-control none, smsp__inst_executed.sum of one launch "
                                 "(bench.py --config slide); fixed by the workload and the library build",
                       "slide/image/1": {"small_kernel": int(num(d["smsp__inst_executed.sum"])), "lib": dig}},
                      f, indent=1)


def main(src, dst):
    os.makedirs(dst, exist_ok=True)
    if os.path.exists(os.path.join(src, "lib_digest.txt")):
        static_profiles(src, dst)
    for name in sorted(os.listdir(src)):
        p = os.path.join(src, name)
        if name.startswith("bench_") and name.endswith(".json"):
            with open(p) as f:
                line = f.read().strip().splitlines()[-1]
            json.loads(line)
            with open(os.path.join(dst, name), "w") as f:
                f.write(line + "\n")
        elif name == "launches_slide.csv":
            shutil.copy(p, os.path.join(dst, name))
            with open(os.path.join(dst, "launches_slide_summary.txt"), "w") as f:
                f.write(launch_summary(p))
        elif name.endswith(".ncu-rep"):
            with open(os.path.join(dst, name.replace(".ncu-rep", ".txt")), "w") as f:
                f.write(ncu_summary(p))
        elif name == "sanitize_summary.txt":
            shutil.copy(p, os.path.join(dst, "sanitize.txt"))
        elif name == "sanitize_summary_index.txt":
            shutil.copy(p, os.path.join(dst, "sanitize_index.txt"))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
