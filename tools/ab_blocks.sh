#!/usr/bin/env bash
# A/B of the config-3 block-product kernel shapes (QOC_BF_BLOCK_SHAPE) on one GPU.
out=gpurun_out/${1:-ab_blocks}; mkdir -p "$out"
for shape in default 1 3 8 9; do
  if [ "$shape" = default ]; then unset QOC_BF_BLOCK_SHAPE; else export QOC_BF_BLOCK_SHAPE=$shape; fi
  timeout 600 python bench.py --workload ising10 --blocks 8 --steps 3 --warmup 1 --no-cpu-baseline --no-ttf \
    > "$out/bench_$shape.json" 2> "$out/bench_$shape.err"
  python - "$out/bench_$shape.json" "$shape" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k = d["roofline"]["kernels"]
print(sys.argv[2], "ms/iter %.2f" % d["ms_per_step"], "block products %.2f ms" % k["block products"]["ms_per_iteration"])
PY
done
