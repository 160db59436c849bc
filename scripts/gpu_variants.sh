#!/bin/bash
# Bench each library variant (libsccg_<name>.so built by build.py --variant) on the given configs.
# Usage: VARIANTS="spec1 hb0" CFG="slide skewed" TAG=x bash scripts/gpu_variants.sh
set -u
mkdir -p gpurun_out
TAG=${TAG:-v}
timeout 300 python __graft_entry__.py > gpurun_out/build_check.txt 2>&1 || { echo "BUILD FAILED"; tail -20 gpurun_out/build_check.txt; exit 1; }
for v in main ${VARIANTS:-}; do
  lib=""; [ "$v" != main ] && lib=libsccg_$v.so
  for c in ${CFG:-slide}; do
    SCCG_LIB=$lib timeout 600 python bench.py --config $c --steps ${STEPS:-30} --warmup 5 --no-cpu-baseline --no-extras --e2e-steps 1 --json-out gpurun_out/bench_${TAG}_${v}_$c.json > gpurun_out/bench_${TAG}_${v}_$c.txt 2>&1
    rc=$?; python -c "
import json; d=json.load(open('gpurun_out/bench_${TAG}_${v}_$c.json')); s=d['stage_ms']; print('%-8s %-7s rc=$rc ms/step %.4f prep %.4f join %.4f pix %.4f frac %.3f' % ('$v', '$c', d['ms_per_step'], s['prep'], s['join'], s['pixelbox'], d['roofline']['frac']))" 2>&1 | tail -1
  done
done
