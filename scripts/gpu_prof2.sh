#!/bin/bash
# ncu --set full of the kernels matching a regex (one launch each) from a short bench run of a config.
# Usage: TAG=x KREGEX='probe|insert' CFG=slide COUNT=2 bash scripts/gpu_prof2.sh
set -u
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py > gpurun_out/build_check.txt 2>&1 || { echo "BUILD FAILED"; tail -20 gpurun_out/build_check.txt; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${KREGEX}" -s ${SKIP:-0} -c ${COUNT:-1} \
  -o gpurun_out/prof_${TAG} -f python bench.py --config ${CFG:-slide} --steps 1 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 1 > gpurun_out/ncu_full_${TAG}.txt 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_full_${TAG}.txt
