#!/usr/bin/env bash
# Interleaved bench A/B (device ms/step and SDF ms of one config, R rounds):
#   bash tools/ab_bench.sh CFG ROUNDS "ENV=1" "ENV=2" ...
cfg=$1; rounds=$2; shift 2
mkdir -p gpurun_out/ab
for r in $(seq 1 $rounds); do
  i=0
  for envs in "$@"; do
    i=$((i+1))
    env $envs timeout 300 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline --no-sdf-batch > gpurun_out/ab/$i.json 2>/dev/null
    python - "$envs" gpurun_out/ab/$i.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
print(f"[{sys.argv[1]:40s}] step {d['ms_per_step']:.4f} p50 {d['ms_per_step_p50']:.4f} sdf {d['roofline']['sdf_kernel_ms']:.4f} e2e {d['e2e']['value']:.0f}")
PY
  done
done
