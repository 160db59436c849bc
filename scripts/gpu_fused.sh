#!/bin/bash
# Fused packed prep: tests, bench (fused e2e and unfused), launch list of the e2e kernels.
set -u
mkdir -p gpurun_out
TAG=${TAG:-fz}
python __graft_entry__.py > gpurun_out/build_${TAG}.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -rf --timeout 300 -k "${K:-packed or streamer or decode}" > gpurun_out/pytest_${TAG}.txt 2>&1; tail -3 gpurun_out/pytest_${TAG}.txt
for mode in fused unfused; do
  flag=""; [ $mode = unfused ] && flag="--e2e-unfused"
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 20 $flag --json-out gpurun_out/bench_${TAG}_$mode.json > gpurun_out/bench_${TAG}_$mode.txt 2>&1; echo "bench $mode rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_${TAG}_$mode.json')); print('$mode value %.4g ms %.4f e2e %.4g h2d %d' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['h2d_bytes_per_step']))"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 1 > /dev/null 2>&1
python scripts/launches.py gpurun_out/launches_${TAG}.csv | grep -E "prep_kernel|decode" | head -12
