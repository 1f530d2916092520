set -u
out=gpurun_out/s11; mkdir -p $out
timeout 900 python -m pytest tests/test_sense.py tests/test_gpu_parity.py -q -x > $out/pytest.log 2>&1; tail -3 $out/pytest.log
timeout 600 python -c "
import sys, json; sys.path.insert(0, '.')
import bench, argparse
a = argparse.Namespace(steps=200)
print(json.dumps(bench.bench_sense(a, True)))
"
