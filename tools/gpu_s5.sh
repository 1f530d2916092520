set -u
out=gpurun_out/s5; mkdir -p $out
python tools/ncu_targets.py step 30 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file $out/warm_cfg2.csv python tools/ncu_targets.py step 30 > /dev/null 2>&1; python tools/launch_table.py $out/warm_cfg2.csv 30
python tools/ncu_targets.py cfg3 30 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file $out/warm_cfg3.csv python tools/ncu_targets.py cfg3 30 > /dev/null 2>&1; python tools/launch_table.py $out/warm_cfg3.csv 30
