#!/bin/bash
# Profile round: ncu launch list of a short bench + one full capture of the PixelBox kernel.
set -u
mkdir -p gpurun_out
TAG=${1:-v}
timeout 300 python __graft_entry__.py > gpurun_out/build.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch_bench_${TAG}.txt 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pixelbox_kernel -s 3 -c 1 \
  -o gpurun_out/prof_${TAG} -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full_${TAG}.txt 2>&1
echo "full rc=$?"
tail -3 gpurun_out/ncu_full_${TAG}.txt
