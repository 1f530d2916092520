# quick per-config bench summary: bash tools/quick_bench.sh tag [configs...]
tag=$1; shift
mkdir -p gpurun_out/qb
for c in "$@"; do
timeout 300 python bench.py --config $c --steps 60 --warmup 5 --no-cpu-baseline --no-sdf-batch > gpurun_out/qb/${tag}_$c.json 2>gpurun_out/qb/${tag}_$c.err
python - <<PY
import json; d=json.loads(open("gpurun_out/qb/${tag}_$c.json").read().strip().splitlines()[-1])
print("$tag $c", round(d["ms_per_step"],4), "sdf", round(d["roofline"]["sdf_kernel_ms"],4), "e2e", round(d["e2e"]["value"],1))
PY
done
