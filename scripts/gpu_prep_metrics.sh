#!/bin/bash
# Shared-memory metrics of one prep launch for each library variant (main + $VARIANTS).
set -u
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active
for v in main ${VARIANTS:-}; do
  lib=""; [ "$v" != main ] && lib=libsccg_$v.so
  SCCG_LIB=$lib timeout 600 ncu --metrics $M --clock-control none -k regex:${K:-prep_kernel} -s 2 -c 1 --csv python bench.py --config ${CFG:-slide} --steps 1 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 1 > gpurun_out/pm_$v.csv 2>/dev/null
  echo "== $v"; grep -E '"(gpu__|l1tex|smsp)' gpurun_out/pm_$v.csv | awk -F'","' '{print $(NF-2), $NF}' | sed 's/"//g'
done
