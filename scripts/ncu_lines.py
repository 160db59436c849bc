"""Per-CUDA-source-line totals (instructions executed, warp-stall samples) of one
kernel in an ncu report (needs -lineinfo).  Usage: ncu_lines.py REP KERNEL_REGEX [N]"""
import csv, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(['ncu', '-i', rep, '-k', 'regex:' + kre, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
def num(x):
    try: return float(x.replace(',', ''))
    except ValueError: return 0.0
agg, cur, path, hdr = {}, None, '', None
for r in rows:
    if not r: continue
    if r[0] == 'File Path': path = r[1].split('/')[-1]; continue
    if r[0] == 'Line No': hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    if r[0]:  # a source line row (metrics aggregated over its SASS)
        ie = hdr.index('Instructions Executed'); iw = hdr.index('Warp Stall Sampling (All Samples)')
        key = (path, int(r[0]))
        a = agg.setdefault(key, [0.0, 0.0, r[1]])
        a[0] += num(r[ie]); a[1] += num(r[iw])
ti = sum(v[0] for v in agg.values()) or 1; ts = sum(v[1] for v in agg.values()) or 1
print(f'total warp-inst {ti:.3e}')
for (p, l), (i, w, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f'{p}:{l:<5} {100*i/ti:5.1f}% inst {100*w/ts:5.1f}% stall  {src.strip()[:90]}')
