#!/bin/bash
# ncu --set full capture of one kernel (regex) from a short bench run.
set -u
mkdir -p gpurun_out
TAG=${1:-v}; KREGEX=${2:-small_kernel}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -s 2 -c 1 \
  -o gpurun_out/prof_${TAG} -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 1 > gpurun_out/ncu_full_${TAG}.txt 2>&1
echo "full $KREGEX rc=$?"
