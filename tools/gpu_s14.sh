set -u
out=gpurun_out/s14; mkdir -p $out
for lib in base minb10 minb12 t64; do EXM_LIB_PATH=$(python -c "import tools.ab_variants as a;print(a.lib_of('$lib'))") timeout 600 python tools/sdf_counters.py cfg2 cfg3 cfg5 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print('$lib', d['cfg'], d['sdf_ms'], d['lane_eff_points'])
    else: print(l.strip())
" | tee -a $out/ab.txt; done
