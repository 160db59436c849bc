"""Brief per-kernel metrics of an ncu report (all captured launches)."""
import csv, subprocess, sys
raw = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h = r[0]
keys = ['gpu__time_duration.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sector_hit_rate.pct',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'launch__grid_size', 'launch__registers_per_thread']
for row in r[2:]:
    d = dict(zip(h, row))
    print(d['Kernel Name'][:90])
    print('   ' + '  '.join(f"{k.split('.')[0].split('__')[1][:22]}={d.get(k)}" for k in keys))
    st = []
    for k, v in d.items():
        if k.startswith('smsp__average_warps_issue_stalled') and k.endswith('per_issue_active.ratio'):
            try: st.append((float(v), k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]))
            except ValueError: pass
    print('   stalls: ' + ', '.join(f'{n}={v:.2f}' for v, n in sorted(st, reverse=True)[:6]))
