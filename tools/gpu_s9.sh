set -u
out=gpurun_out/s9; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -x > $out/pytest.log 2>&1; tail -2 $out/pytest.log
for lib in base oldio; do EXM_LIB_PATH=$(python -c "import tools.ab_variants as a;print(a.lib_of('$lib'))") timeout 300 python tools/host_timing.py; done
for c in cfg2 cfg5; do timeout 900 python tools/ab_variants.py bench $c 2 base oldio 2>&1 | tee -a $out/ab.txt; done
