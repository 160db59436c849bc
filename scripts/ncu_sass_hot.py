"""Hottest SASS instructions of each matching kernel in an ncu report
(share of instructions executed, share of warp-stall samples)."""
import csv, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25


def num(x):
    try:
        return float(x.replace(',', ''))
    except ValueError:
        return 0.0


raw = subprocess.run(['ncu', '-i', rep, '-k', 'regex:' + kre, '--page', 'source', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
sections, cur = [], None
for r in rows:
    if r and r[0] == 'Kernel Name':
        cur = [r[1], None, []]
        sections.append(cur)
    elif r and r[0] == 'Address' and cur is not None:
        cur[1] = r
    elif cur is not None and cur[1] is not None and len(r) == len(cur[1]):
        cur[2].append(r)
for name, h, data in sections:
    ia, isrc, iex, ist = h.index('Address'), h.index('Source'), h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)')
    tot = sum(num(r[iex]) for r in data) or 1; tst = sum(num(r[ist]) for r in data) or 1
    print(f'=== {name[:100]}\n total warp-inst {tot:.3e}, stall samples {tst:.0f}')
    print(' --- by instructions executed')
    for r in sorted(data, key=lambda r: -num(r[iex]))[:n]:
        print(f' {r[ia][-5:]:>6} {num(r[iex])/tot*100:5.1f}% {num(r[ist])/tst*100:5.1f}%s  {r[isrc][:80]}')
    print(' --- by stall samples')
    for r in sorted(data, key=lambda r: -num(r[ist]))[:n]:
        print(f' {r[ia][-5:]:>6} {num(r[iex])/tot*100:5.1f}% {num(r[ist])/tst*100:5.1f}%s  {r[isrc][:80]}')
