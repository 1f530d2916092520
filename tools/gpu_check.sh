#!/usr/bin/env bash
# One GPU call: the GPU test suite, a warm (no cache flush) launch list of 20 config-2 steps and
# quick bench lines. Usage (on the box): bash tools/gpu_check.sh TAG [configs...]
tag=${1:-chk}; shift
mkdir -p gpurun_out/$tag
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/$tag/pytest_gpu.log 2>&1; tail -2 gpurun_out/$tag/pytest_gpu.log
python tools/ncu_targets.py step 20 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/$tag/warm_cfg2.csv python tools/ncu_targets.py step 20 > /dev/null 2>&1; python tools/launch_table.py gpurun_out/$tag/warm_cfg2.csv 20
bash tools/quick_bench.sh $tag "${@:-cfg2}"
