#!/bin/bash
# Quick iteration on the GPU box: build, selected GPU tests, one short bench.
# Usage: K="filter or slide" CFG=slide bash scripts/gpu_quick.sh
set -u
mkdir -p gpurun_out
TAG=${TAG:-q}
timeout 300 python __graft_entry__.py > gpurun_out/build_${TAG}.txt 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests -m gpu -q -x -rf --timeout 300 -k "${K:-.}" > gpurun_out/pytest_${TAG}.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_${TAG}.txt
for c in ${CFG:-slide}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-30} --warmup 5 --no-cpu-baseline --no-extras --json-out gpurun_out/bench_${TAG}_$c.json > gpurun_out/bench_${TAG}_$c.txt 2>&1
  echo "bench $c rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_${TAG}_$c.json')); print('$c', 'value %.3e'%d['value'], 'ms/step %.4f'%d['ms_per_step'], 'stages', {k: round(v,4) if isinstance(v,float) else v for k,v in d['stage_ms'].items()}, 'frac %.3f'%d['roofline']['frac'], d['clocks']['sm_mhz'])" 2>&1 | tail -1
done
if [ -n "${NCU:-}" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --config ${NCU} --steps 2 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 1 > /dev/null 2>&1
  echo "ncu rc=$?"; python scripts/launches.py gpurun_out/launches_${TAG}.csv 2>&1 | tail -20
fi
if [ -n "${PROF:-}" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${PROF}" -c ${PCOUNT:-2} \
    -o gpurun_out/prof_${TAG} -f python bench.py --config ${PCFG:-slide} --steps 1 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 1 > gpurun_out/ncu_full_${TAG}.txt 2>&1
  echo "ncu full rc=$?"
fi
