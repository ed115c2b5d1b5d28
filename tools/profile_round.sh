#!/usr/bin/env bash
# GPU-box measurement recipe (run under gpurun from the repo root):
#   bench lines per workload, the ncu launch list of each bench command (cold, serialised
#   per-launch times; B200_PROFILING.md), and one `ncu --set full` capture of the dominant
#   kernel.  Outputs land in gpurun_out/; summaries are copied into profiles/ by hand.
#   usage: tools/profile_round.sh TAG WORKLOAD[:KERNEL_REGEX] ...
set -u
tag=$1; shift
out=gpurun_out/$tag
mkdir -p "$out"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$out/gpu.txt" 2>&1
for spec in "$@"; do
  wl=${spec%%:*}
  kre=${spec#*:}
  [ "$kre" = "$spec" ] && kre=""
  timeout 900 python bench.py --workload "$wl" --steps 10 --warmup 3 --no-cpu-baseline \
    > "$out/bench_$wl.json" 2> "$out/bench_$wl.err"
  echo "bench $wl rc=$?"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "$out/launches_$wl.csv" python bench.py --workload "$wl" --steps 2 --warmup 3 \
    --no-cpu-baseline > "$out/ncu_launch_$wl.log" 2>&1
  echo "launches $wl rc=$?"
  if [ -n "$kre" ]; then
    timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$kre" -c 1 \
      -o "$out/full_$wl" python bench.py --workload "$wl" --steps 1 --warmup 3 --no-cpu-baseline \
      > "$out/ncu_full_$wl.log" 2>&1
    echo "full $wl rc=$?"
  fi
done
