#!/bin/bash
# Round profile (one gpurun call): the default bench line, the bench's launch
# list (ncu gpu__time_duration, --clock-control none), one ncu --set full
# capture per hot kernel, compute-sanitizer runs, and one bench line per other
# config.  Outputs land in gpurun_out/round_${TAG}/; scripts/collect_profiles.py
# turns them into profiles/<round>/ (+ profiles/prep_traffic.json, issue_counts.json).
set -u
TAG=${1:-r02}
OUT=gpurun_out/round_${TAG}
mkdir -p $OUT
timeout 300 python __graft_entry__.py > $OUT/build.txt 2>&1
echo "build rc=$?"
python -c "import bench; print(bench.lib_digest())" > $OUT/lib_digest.txt
timeout 900 python bench.py > $OUT/bench_slide.json 2> $OUT/bench_slide.err
echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_slide.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 1 > $OUT/launches_bench.txt 2>&1
echo "launch list rc=$?"
for k in prep_kernel grid_insert_kernel small_kernel decode_rect_packed_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
    -o $OUT/ncu_$k -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 1 > $OUT/ncu_$k.txt 2>&1
  echo "ncu $k rc=$?"
done
# both probe passes (bucket pass, compaction)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:probe_kernel -s 2 -c 2 \
  -o $OUT/ncu_probe_kernel -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 1 > $OUT/ncu_probe.txt 2>&1
echo "ncu probe rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:item_kernel -s 1 -c 1 \
  -o $OUT/ncu_item_kernel_combs -f python bench.py --config combs --steps 1 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 1 > $OUT/ncu_item.txt 2>&1
echo "ncu item rc=$?"
# compute-sanitizer runs (memcheck, racecheck, synccheck; SANITIZE_INDEX=1 for the indexed large path):
# the sanitizer is closed on this pool since round 2's last sessions, so the committed
# profiles/r02/sanitize*.txt are from the earlier library; run by hand where it is available:
#   compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_case.py
for c in tile skewed combs; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  echo "bench $c rc=$?"
done
timeout 900 python bench.py --config study --steps 10 --warmup 3 > $OUT/bench_study.json 2> $OUT/bench_study.err
echo "bench study rc=$?"
