set -u
out=gpurun_out/s4; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -x > $out/pytest_gpu.log 2>&1; tail -3 $out/pytest_gpu.log
grep -E "criterion 3|tuned mapping|cycles:" $out/pytest_gpu.log | head
timeout 600 python tools/sdf_counters.py cfg2 cfg3 cfg5 2>&1 | tee $out/counters.txt
for c in cfg1 cfg3 cfg5; do timeout 600 python bench.py --config $c --steps 60 --warmup 10 --no-cpu-baseline --no-sdf-batch > $out/bench_$c.json 2>&1; python -c "
import json;d=json.loads(open('$out/bench_$c.json').read().strip().splitlines()[-1]);print('$c',d['ms_per_step'],d['roofline']['sdf_kernel_ms'],d['e2e']['value'],d['roofline']['sdf_path'])"; done
timeout 900 python bench.py > $out/bench.json 2> $out/bench.err; python -c "
import json;d=json.loads(open('$out/bench.json').read().strip().splitlines()[-1]);print('cfg2',d['ms_per_step'],d['roofline']['sdf_kernel_ms'],d['e2e']['value'],d['roofline']['frac'],d['roofline']['sdf_path'],d['cpu_baseline'])"
timeout 900 python bench.py --impl reference > $out/bench_ref.json 2> $out/bench_ref.err; tail -c 1500 $out/bench_ref.json
