set -u
o=gpurun_out/r03b; mkdir -p $o
timeout 1500 python -m pytest tests/test_gpu_blocked.py tests/test_gpu_bitflip.py -q > $o/pytest.log 2>&1; echo "pytest rc=$?"
tail -15 $o/pytest.log
for spec in "b8:--blocks 8" "b8s8:--blocks 8" "b256:--blocks 256" "direct:"; do
  tag=${spec%%:*}; a=${spec#*:}
  if [ $tag = b8s8 ]; then export QOC_BF_BLOCK_SHAPE=8; else unset QOC_BF_BLOCK_SHAPE; fi
  timeout 600 python bench.py --workload ising10 $a --steps 5 --warmup 3 --no-cpu-baseline > $o/bench_$tag.json 2> $o/bench_$tag.err
  echo "$tag rc=$?"; python -c "import json,sys; d=json.load(open('$o/bench_$tag.json')); print(d['value'], d['ms_per_step'], {k:(round(v['ms_per_iteration'],3)) for k,v in d['roofline']['kernels'].items()}, d['roofline']['frac'])" 2>&1 | tail -1
done
unset QOC_BF_BLOCK_SHAPE
timeout 1200 python tools/config4_drift.py 1e-15 > $o/drift.log 2>&1; echo "drift rc=$?"; tail -4 $o/drift.log
