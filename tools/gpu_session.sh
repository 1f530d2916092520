#!/usr/bin/env bash
# One GPU call: GPU tests, A/B of variant builds, the default bench line.
#   bash tools/gpu_session.sh TAG "cfgs for A/B" "variants"
tag=${1:-s}; cfgs=${2:-cfg2}; variants=${3:-base}
out=gpurun_out/$tag
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:randomly > $out/pytest_gpu.log 2>&1; tail -3 $out/pytest_gpu.log
cp gpurun_out/fullsize_paths.json $out/ 2>/dev/null
for c in $cfgs; do timeout 900 python tools/ab_variants.py bench $c 2 $variants 2>&1 | tee -a $out/ab.txt; done
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; tail -c 3000 $out/bench.json
