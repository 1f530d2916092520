set -u
out=gpurun_out/s8; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharding.py tests/test_hybrid.py -q -x > $out/pytest.log 2>&1; tail -2 $out/pytest.log
timeout 300 python tools/host_timing.py
for c in cfg2 cfg1; do timeout 900 python tools/ab_variants.py bench $c 3 base nofuse 2>&1 | tee -a $out/ab.txt; done
