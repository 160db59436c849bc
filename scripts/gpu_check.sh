#!/bin/bash
# One gpurun round: build check, GPU parity tests, smoke, short bench, ncu launch list.
# Usage (from repo root, on the GPU box): bash scripts/gpu_check.sh [pytest-args]
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
timeout 300 python __graft_entry__.py > gpurun_out/build.txt 2>&1; echo "build rc=$?" >> gpurun_out/build.txt
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 240 "$@" > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench.json > gpurun_out/bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/bench.txt
tail -5 gpurun_out/pytest_gpu.txt; tail -2 gpurun_out/smoke.txt; tail -3 gpurun_out/bench.txt
