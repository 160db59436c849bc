"""Instruction / stall-sample breakdown by SASS region of one kernel in an ncu report."""
import csv, subprocess, sys
rep = sys.argv[1]; B = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source=sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]; data = rows[2:]
ie = h.index('Instructions Executed'); src = h.index('Source'); samp = h.index('Warp Stall Sampling (All Samples)')
te = h.index('Thread Instructions Executed')
vals = [(int(r[ie]) if r[ie].isdigit() else 0, r[src].strip(), int(r[samp]) if r[samp].isdigit() else 0,
         int(r[te]) if r[te].isdigit() else 0) for r in data]
tot = sum(v[0] for v in vals); ts = sum(v[2] for v in vals)
print('total warp inst', tot)
for b in range(0, len(vals), B):
    blk = vals[b:b + B]
    s = sum(v[0] for v in blk); sm = sum(v[2] for v in blk); th = sum(v[3] for v in blk)
    if s / tot > 0.01 or sm / ts > 0.01:
        ops = {}
        for v in blk:
            t = v[1].split()
            if not t: continue
            op = t[1] if t[0].startswith('@') and len(t) > 1 else t[0]
            op = op.split('.')[0]
            ops[op] = ops.get(op, 0) + v[0]
        top = sorted(ops.items(), key=lambda x: -x[1])[:7]
        print(f'{b:5d}-{b + B:5d} inst {s / tot * 100:5.1f}% samp {sm / ts * 100:5.1f}% lanes {th / max(s, 1):4.1f} ', ' '.join(f'{k}:{v / max(s, 1) * 100:.0f}' for k, v in top))
