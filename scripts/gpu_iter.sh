#!/bin/bash
# Iteration round: build, GPU tests, bench for each lib variant given, launch list.
set -u
mkdir -p gpurun_out
TAG=${TAG:-it}
timeout 300 python __graft_entry__.py > gpurun_out/build.txt 2>&1; echo "build rc=$?" >> gpurun_out/build.txt
timeout 1500 python -m pytest tests -m gpu -q -rf -x --timeout 240 > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_${TAG}.txt
tail -4 gpurun_out/pytest_gpu_${TAG}.txt
if [ -n "${SANITIZE:-}" ]; then
  for tool in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_case.py > gpurun_out/sanitize_${tool}_${TAG}.txt 2>&1
    echo "sanitizer $tool rc=$?"; tail -2 gpurun_out/sanitize_${tool}_${TAG}.txt
  done
fi
for v in "" "$@"; do
  name=${v:-main}
  SCCG_LIB=$v timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-extras --json-out gpurun_out/bench_${TAG}_${name}.json > gpurun_out/bench_${TAG}_${name}.txt 2>&1
  echo "bench $name rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_${TAG}_${name}.json')); print('$name', 'value %.3e'%d['value'], 'ms/step %.3f'%d['ms_per_step'], 'stages', d['stage_ms'], 'frac %.3f'%d['roofline']['frac'], 'e2e %.3e'%d['e2e']['value'], d['clocks'])" 2>&1 | tail -1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 1 > /dev/null 2>&1
echo "ncu rc=$?"
