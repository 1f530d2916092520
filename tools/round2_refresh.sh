#!/usr/bin/env bash
# Everything profiles/ records for round 2, in one GPU call (run on the box from the repo root):
#   bash tools/round2_refresh.sh gpurun_out/r02 r02
set -u
out=${1:-gpurun_out/r02}
tag=${2:-r02}
mkdir -p "$out"
timeout 1500 python -m pytest tests -m gpu -q -rs > "$out/pytest_gpu.log" 2>&1
tail -2 "$out/pytest_gpu.log"
cp gpurun_out/fullsize_paths.json "$out/" 2>/dev/null
timeout 900 python bench.py > "$out/bench_cfg2.json" 2> "$out/bench_cfg2.err"
for c in cfg1 cfg3 cfg5; do
  timeout 900 python bench.py --config $c --steps 60 --warmup 10 --no-cpu-baseline --no-sdf-batch \
    > "$out/bench_$c.json" 2> "$out/bench_$c.err"
done
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > "$out/bench_reference_cfg2.json" 2> "$out/bench_reference.err"
python tools/ncu_targets.py step 30 > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
      --log-file "$out/launches_step_cfg2_warm.csv" python tools/ncu_targets.py step 30 > /dev/null 2>&1
python tools/launch_table.py "$out/launches_step_cfg2_warm.csv" 30 > "$out/launches_step_cfg2_warm.txt"
python tools/ncu_targets.py cfg3 20 > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
      --log-file "$out/launches_step_cfg3_warm.csv" python tools/ncu_targets.py cfg3 20 > /dev/null 2>&1
python tools/launch_table.py "$out/launches_step_cfg3_warm.csv" 20 > "$out/launches_step_cfg3_warm.txt"
python tools/ncu_targets.py step 26 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
      -k regex:"10k_sdf_gridI" -s 25 -c 1 -f -o "$out/ncu_sdf_grid_cfg2" \
      python tools/ncu_targets.py step 26 > /dev/null 2>&1 && \
  python tools/ncu_summary.py "$out/ncu_sdf_grid_cfg2.ncu-rep" > "$out/${tag}_ncu_sdf_grid_cfg2.json"
python tools/ncu_targets.py pairs 2 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
      -k regex:"k_sdf_pairs" -s 1 -c 1 -f -o "$out/ncu_sdf_pairs_cfg4" \
      python tools/ncu_targets.py pairs 2 > /dev/null 2>&1 && \
  python tools/ncu_summary.py "$out/ncu_sdf_pairs_cfg4.ncu-rep" > "$out/${tag}_ncu_sdf_pairs_cfg4.json"
[ -f "$out/ncu_sdf_grid_cfg2.ncu-rep" ] && \
  ncu -i "$out/ncu_sdf_grid_cfg2.ncu-rep" --page source --csv --print-source cuda,sass > "$out/sdf_grid_src.csv" 2>/dev/null && \
  python tools/ncu_lines.py "$out/sdf_grid_src.csv" 40 > "$out/${tag}_ncu_lines_sdf_grid_cfg2.txt" && rm -f "$out/sdf_grid_src.csv"
rm -f "$out"/*.ncu-rep
