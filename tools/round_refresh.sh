#!/usr/bin/env bash
# Everything profiles/ records, in one GPU call (run on the box from the repo root):
#   bash tools/round_refresh.sh gpurun_out/r01 r01
# 1. pytest -m gpu; 2. ncu launch list of 5 config-2 steps; 3. ncu --set full of the config-2
# grid SDF kernel and of the config-4 pairs kernel (summaries written to profiles/ first, so
# the bench lines below read the fresh traffic / pipe figures); 4. the bench lines.
# Every ncu run follows the same command run plainly (exit 0) in this call.
set -u
out=${1:-gpurun_out/r01}
tag=${2:-r01}
mkdir -p "$out"
timeout 1200 python -m pytest tests -m gpu -q > "$out/pytest_gpu.log" 2>&1
tail -1 "$out/pytest_gpu.log"
python tools/ncu_targets.py step 5 > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file "$out/launches_step_cfg2.csv" python tools/ncu_targets.py step 5 > /dev/null 2>&1
# the same with warm caches (no flush between kernels): the in-step durations
python tools/ncu_targets.py step 20 > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
      --log-file "$out/launches_step_cfg2_warm.csv" python tools/ncu_targets.py step 20 > /dev/null 2>&1
# a steady-state step (the 25th: the nominal has converged, as in the bench's timed steps)
python tools/ncu_targets.py step 26 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
      -k regex:"10k_sdf_gridI" -s 25 -c 1 -f -o "$out/ncu_sdf_grid_cfg2" \
      python tools/ncu_targets.py step 26 > /dev/null 2>&1 && \
  python tools/ncu_summary.py "$out/ncu_sdf_grid_cfg2.ncu-rep" > "profiles/${tag}_ncu_sdf_grid_cfg2.json"
python tools/ncu_targets.py pairs 2 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
      -k regex:"k_sdf_pairs" -s 1 -c 1 -f -o "$out/ncu_sdf_pairs_cfg4" \
      python tools/ncu_targets.py pairs 2 > /dev/null 2>&1 && \
  python tools/ncu_summary.py "$out/ncu_sdf_pairs_cfg4.ncu-rep" > "profiles/${tag}_ncu_sdf_pairs_cfg4.json"
cp "profiles/${tag}_ncu_sdf_grid_cfg2.json" "profiles/${tag}_ncu_sdf_pairs_cfg4.json" "$out/" 2>/dev/null
bash tools/run_round_bench.sh "$out"
