set -u
out=gpurun_out/s6; mkdir -p $out
# steady-state step 26 (after tuning and warm-up) of config 2: full ncu set with source
python tools/ncu_targets.py step 26 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:"10k_sdf_gridI" -s 25 -c 1 -f -o $out/ncu_sdf_grid_cfg2 python tools/ncu_targets.py step 26 > /dev/null 2>&1
ncu -i $out/ncu_sdf_grid_cfg2.ncu-rep --page source --csv --print-source cuda,sass > $out/mix_cfg2.csv 2>/dev/null
python tools/ncu_lines.py $out/mix_cfg2.csv 45
python tools/ncu_summary.py $out/ncu_sdf_grid_cfg2.ncu-rep > $out/summary_cfg2.json; cat $out/summary_cfg2.json
