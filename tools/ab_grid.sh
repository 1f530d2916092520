# A/B of the grid-kernel options on every config (EXM_GRID_CHUNKS=0|1); results in gpurun_out/ab3
mkdir -p gpurun_out/ab3
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab3/pytest.log 2>&1; tail -2 gpurun_out/ab3/pytest.log
for v in 1 0; do
EXM_GRID_CHUNKS=$v python tools/grid_stats.py cfg1 cfg2 cfg3
for c in cfg1 cfg2 cfg3 cfg5; do
EXM_GRID_CHUNKS=$v timeout 300 python bench.py --config $c --steps 60 --warmup 5 --no-cpu-baseline --no-sdf-batch > gpurun_out/ab3/v${v}_$c.json 2>gpurun_out/ab3/v${v}_$c.err
python - <<PY
import json; d=json.loads(open("gpurun_out/ab3/v${v}_$c.json").read().strip().splitlines()[-1])
print("chunks=$v $c", round(d["ms_per_step"],4), "sdf", round(d["roofline"]["sdf_kernel_ms"],4), "e2e", round(d["e2e"]["value"],1))
PY
done; done
