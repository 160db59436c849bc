"""Key metrics from an ncu --set full report (one kernel)."""
import csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, units, vals = r[0], r[1], r[2]
d = {h[i]: (vals[i], units[i]) for i in range(len(h))}
keys = ['Kernel Name', 'gpu__time_duration.sum', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'smsp__thread_inst_executed_per_inst_executed.ratio',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__t_bytes.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem', 'sm__maximum_warps_per_active_cycle_pct',
        'achieved_occupancy', 'sm__cycles_elapsed.avg.per_second']
for k in keys:
    if k in d: print(f'{k:70s} {d[k][0]} {d[k][1]}')
st = []
for k, (v, u) in d.items():
    if k.startswith('smsp__average_warps_issue_stalled') and k.endswith('per_issue_active.ratio'):
        try: st.append((float(v), k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')))
        except ValueError: pass
print('stalls (cycles per issue):', ', '.join(f'{n}={v:.2f}' for v, n in sorted(st, reverse=True)[:8]))
