#!/usr/bin/env bash
# Warm launch-list A/B: for each "ENV=VAL ..." argument, the per-kernel mean of 20 config-2
# steps under that environment. Usage (on the box): bash tools/ab_launch.sh "" "EXM_X=1" ...
cfg=${AB_CFG:-step}
for envs in "$@"; do
  echo "== [$envs]"
  env $envs python tools/ncu_targets.py $cfg 20 > /dev/null 2>&1 && \
  env $envs ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
      --log-file gpurun_out/ab.csv python tools/ncu_targets.py $cfg 20 > /dev/null 2>&1
  python tools/launch_table.py gpurun_out/ab.csv 20 | grep -v "^kernel"
done
