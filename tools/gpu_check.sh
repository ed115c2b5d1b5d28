#!/usr/bin/env bash
# One gpurun call of the build -> measure loop (run from the repo root under gpurun):
#   gpu_check.sh TAG [pytest-args...]
# runs the fp64 / DMMA peak probes, `pytest -m gpu` (args forwarded), smoke(), and the default
# bench line.  Outputs land in gpurun_out/TAG/.
set -u
tag=$1; shift
out=gpurun_out/$tag
mkdir -p "$out"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$out/gpu.txt" 2>&1
nproc > "$out/nproc.txt"
if [ -x tools/dmma_peak ]; then timeout 120 tools/dmma_peak > "$out/dmma_peak.json" 2>&1; fi
if [ -x tools/fp64_peak ]; then timeout 120 tools/fp64_peak > "$out/fp64_peak.json" 2>&1; fi
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 2400 python -m pytest tests -m gpu -q "$@" > "$out/pytest_gpu.log" 2>&1; echo "pytest rc=$?"
  tail -5 "$out/pytest_gpu.log"
  timeout 300 python __graft_entry__.py > "$out/smoke.log" 2>&1; echo "smoke rc=$?"
fi
if [ "${SKIP_BENCH:-0}" != 1 ]; then
  timeout 1200 python bench.py ${BENCH_ARGS:-} > "$out/bench.json" 2> "$out/bench.err"; echo "bench rc=$?"
  tail -c 3000 "$out/bench.json"
fi
