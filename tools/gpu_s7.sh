set -u
out=gpurun_out/s7; mkdir -p $out
for lib in base chunk4 chunk8 chunk16; do EXM_LIB_PATH=$(python -c "import tools.ab_variants as a;print(a.lib_of('$lib'))") timeout 600 python tools/sdf_counters.py cfg2 cfg3 cfg5 2>&1 | tee -a $out/counters.txt; done
timeout 900 python bench.py --steps 50 --warmup 10 > $out/bench.json 2> $out/bench.err; python -c "
import json;d=json.loads(open('$out/bench.json').read().strip().splitlines()[-1]);print(json.dumps(d['hybrid_cfg5']), json.dumps(d['hybrid']))"
