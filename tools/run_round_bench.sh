#!/usr/bin/env bash
# One GPU call's worth of measurements for profiles/: the default bench line (cfg2 + cfg4 SDF +
# hybrid + CPU baseline), the other configs, and the reference arm. Usage (on the GPU box):
#   bash tools/run_round_bench.sh gpurun_out/rNN
set -u
out=${1:-gpurun_out/bench}
mkdir -p "$out"
timeout 900 python bench.py > "$out/bench_cfg2.json" 2> "$out/bench_cfg2.err"
for c in cfg1 cfg3 cfg5; do
  timeout 900 python bench.py --config $c --steps 60 --warmup 5 --no-cpu-baseline --no-sdf-batch \
    > "$out/bench_$c.json" 2> "$out/bench_$c.err"
done
timeout 900 python bench.py --impl reference > "$out/bench_reference_cfg2.json" 2> "$out/bench_reference.err"
