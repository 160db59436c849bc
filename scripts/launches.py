"""Summarise an ncu launch-list CSV: per-kernel time of the last full step."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; data = rows[hi + 1:]
ki = h.index('Kernel Name'); vi = h.index('Metric Value')
seq = [(r[ki][:60], float(r[vi].replace(',', ''))) for r in data]
idx = [i for i, s in enumerate(seq) if s[0].startswith('sccg::prep_init')]
last = seq[idx[-2]:] if len(idx) >= 2 else seq
tot = 0
for s in last:
    print(f'{s[1]/1000:9.1f} us  {s[0]}'); tot += s[1]
print(f'total {tot/1000:.1f} us, {len(last)} launches')
