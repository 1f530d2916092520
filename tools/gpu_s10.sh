set -u
out=gpurun_out/s10; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharding.py -q -x > $out/pytest.log 2>&1; tail -2 $out/pytest.log
for lib in base oldio; do EXM_LIB_PATH=$(python -c "import tools.ab_variants as a;print(a.lib_of('$lib'))") timeout 300 python tools/host_timing.py; done
EXM_LIB_PATH=$(python -c "import tools.ab_variants as a;print(a.lib_of('smem'))") timeout 900 python -m pytest tests/test_gpu_cull_exact.py -q -x -k "thread or persist" > $out/pytest_smem.log 2>&1; tail -2 $out/pytest_smem.log
for c in cfg2 cfg3; do timeout 900 python tools/ab_variants.py bench $c 2 base oldio smem 2>&1 | tee -a $out/ab.txt; done
timeout 900 python tools/ab_variants.py bench cfg5 1 base smem 2>&1 | tee -a $out/ab.txt
