set -u
out=gpurun_out/s2; mkdir -p $out
for lib in base rmajor; do EXM_LIB_PATH=$(python -c "import tools.ab_variants as a;print(a.lib_of('$lib'))") timeout 600 python tools/sdf_counters.py cfg2 cfg3 cfg5 2>&1 | tee -a $out/counters.txt; done
timeout 900 python tools/scaling_benchmark.py --trials 30 --cpu-max 100000 > $out/scaling.csv 2> $out/scaling.err; tail -40 $out/scaling.csv
