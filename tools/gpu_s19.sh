set -u
out=gpurun_out/s19; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_threshold.py tests/test_gpu_parity.py tests/test_hybrid.py tests/test_gpu_sharding.py tests/test_gpu_fullsize.py -q -x > $out/pytest.log 2>&1; tail -3 $out/pytest.log
timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > $out/bench_cfg2.json 2> $out/bench_cfg2.err; python -c "
import json; d=json.load(open('$out/bench_cfg2.json')); print('cfg2', d['ms_per_step'], d['value'], d['e2e']['value'], d['roofline'].get('sdf_ms'), d['roofline']['frac'])"
for c in cfg1 cfg3 cfg5; do timeout 600 python bench.py --config $c --steps 40 --warmup 10 --no-cpu-baseline --no-sdf-batch > $out/bench_$c.json 2> $out/bench_$c.err; python -c "
import json; d=json.load(open('$out/bench_$c.json')); print('$c', d['ms_per_step'], d['value'], d['e2e']['value'])"; done
