"""Per-CUDA-source-line shared-memory wavefronts (actual vs ideal) of one kernel
in an ncu report (needs -lineinfo).  Usage: ncu_smem_lines.py REP KERNEL_REGEX [N]"""
import csv, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(['ncu', '-i', rep, '-k', 'regex:' + kre, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
def num(x):
    try: return float(x.replace(',', ''))
    except ValueError: return 0.0
agg, path, hdr = {}, '', None
for r in rows:
    if not r: continue
    if r[0] == 'File Path': path = r[1].split('/')[-1]; continue
    if r[0] == 'Line No': hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    if r[0]:
        w, wi = hdr.index('L1 Wavefronts Shared'), hdr.index('L1 Wavefronts Shared Ideal')
        a = agg.setdefault((path, int(r[0])), [0.0, 0.0, r[1]])
        a[0] += num(r[w]); a[1] += num(r[wi])
tw = sum(v[0] for v in agg.values()) or 1
print(f'total shared wavefronts {tw:.3e} (ideal {sum(v[1] for v in agg.values()):.3e})')
for (p, l), (w, wi, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f'{p}:{l:<5} {100*w/tw:5.1f}%  x{w/max(wi,1):4.2f} of ideal  {src.strip()[:90]}')
