for cm in 0.5 1 2 4; do for ppc in 32 64; do
EXM_CELL_MAX_R=$cm EXM_PTS_PER_CELL=$ppc bash tools/quick_bench.sh cm${cm}_p${ppc} cfg1 cfg2 cfg3 cfg5
done; done
EXM_WARP_MAX=40000 bash tools/quick_bench.sh warp40k cfg1
EXM_WARP_MAX=40000 EXM_CELL_MAX_R=2 bash tools/quick_bench.sh warp40k_cm2 cfg1
