#!/bin/bash
# Decode / e2e iteration: build, decode + streamer GPU tests, bench (e2e), launch list of decode kernels.
set -u
mkdir -p gpurun_out
TAG=${TAG:-e2e}
python __graft_entry__.py > gpurun_out/build_${TAG}.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -rf --timeout 300 -k "${K:-decode or streamer}" > gpurun_out/pytest_${TAG}.txt 2>&1; tail -2 gpurun_out/pytest_${TAG}.txt
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --json-out gpurun_out/bench_${TAG}.json > gpurun_out/bench_${TAG}.txt 2>&1; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_${TAG}.json')); print('value %.4g ms %.4f e2e %.4g h2d %d' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['h2d_bytes_per_step']), d['stage_ms'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 1 > /dev/null 2>&1
python scripts/launches.py gpurun_out/launches_${TAG}.csv | grep -i "decode" | head -4
