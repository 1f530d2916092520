#!/usr/bin/env bash
# A/B timing of compile-time variants (tools/ab_variants.py build NAME=-DFLAG ...), interleaved:
#   bash tools/gpu_ab.sh OUTDIR "cfg2 cfg3 cfg5" base quad single ...
set -u
out=$1; cfgs=$2; shift 2
mkdir -p $out
for r in 1 2; do for lib in "$@"; do
  EXM_LIB_PATH=$(python -c "import tools.ab_variants as a;print(a.lib_of('$lib'))") timeout 600 \
    python tools/sdf_counters.py $cfgs 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print('$lib', d['cfg'], 'sdf', d['sdf_ms'], 'step', d.get('step_ms'))
    else: print(l.strip())
" | tee -a $out/ab.txt
done; done
