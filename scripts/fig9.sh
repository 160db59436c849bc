#!/bin/bash
# Fig. 9 analog: build variants must exist (python paper_1208_0277_b200/build.py --variant noopt -DSCCG_NO_PDL
# -DSCCG_PREP_NO_TMA; --variant nopdl -DSCCG_NO_PDL).  Usage on the GPU box: bash scripts/fig9.sh [outdir]
set -u
OUT=${1:-gpurun_out}
mkdir -p $OUT
timeout 300 python __graft_entry__.py > gpurun_out/build_check.txt 2>&1 || { echo "BUILD FAILED"; tail -20 gpurun_out/build_check.txt; exit 1; }
timeout 900 python scripts/fig9.py --lib libsccg_noopt.so --variants V0,V1,V2 --out $OUT/fig9_a.json > $OUT/fig9_a.txt 2>&1; echo "a rc=$?"
timeout 900 python scripts/fig9.py --lib libsccg_nopdl.so --variants V3 --out $OUT/fig9_b.json > $OUT/fig9_b.txt 2>&1; echo "b rc=$?"
timeout 900 python scripts/fig9.py --variants V4 --out $OUT/fig9_c.json > $OUT/fig9_c.txt 2>&1; echo "c rc=$?"
python scripts/fig9.py --merge $OUT/fig9_a.json $OUT/fig9_b.json $OUT/fig9_c.json --out $OUT/fig9.json
