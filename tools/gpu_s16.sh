set -u
out=gpurun_out/s16; mkdir -p $out
EXM_LIB_PATH=$(python -c "import tools.ab_variants as a;print(a.lib_of('pair'))") timeout 900 python -m pytest tests/test_gpu_cull_exact.py -q -x > $out/pytest_pair.log 2>&1; tail -2 $out/pytest_pair.log
for r in 1 2; do for lib in base pair; do EXM_LIB_PATH=$(python -c "import tools.ab_variants as a;print(a.lib_of('$lib'))") timeout 600 python tools/sdf_counters.py cfg2 cfg3 cfg5 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print('$lib', d['cfg'], d['sdf_ms'])
    else: print(l.strip())
" | tee -a $out/ab.txt; done; done
