set -u
out=gpurun_out/s3; mkdir -p $out
for lib in base hm_allslots rmajor rm_allslots rm_persist; do EXM_LIB_PATH=$(python -c "import tools.ab_variants as a;print(a.lib_of('$lib'))") timeout 600 python tools/sdf_counters.py cfg2 cfg3 cfg5 2>&1 | tee -a $out/counters.txt; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cull_exact.py -q -x -k "sdf or batch or culled" > $out/pytest.log 2>&1; tail -2 $out/pytest.log
timeout 900 python tools/scaling_benchmark.py --trials 30 --cpu-max 1000 > $out/scaling.csv 2> $out/scaling.err; grep -E "100000,|1000000," $out/scaling.csv | grep -E "call|dropin"
