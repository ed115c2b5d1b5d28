#!/usr/bin/env bash
# ncu --set full captures of the density-kind task kernel (5-spin preset) and the split-step task
# kernel after the kinetic merge / FFT rewrite.  usage: tools/ncu_extra.sh TAG
out=gpurun_out/${1:-ncu_extra}; mkdir -p "$out"
cap() {
  local name=$1 re=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$re" --launch-skip "$skip" -c 1 \
    -o "$out/full_$name" python bench.py "$@" --steps 2 --warmup 3 --no-cpu-baseline --no-ttf > "$out/ncu_full_$name.log" 2>&1
  echo "full $name rc=$?"
}
cap spins_task density_task_kernel 2 --workload spins
cap gpe1024_task strang_task_kernel 3 --workload gpe1024
for f in "$out"/full_*.ncu-rep; do python tools/ncu_brief.py "$f" >> "$out/ncu_brief.txt" 2>&1; done
cat "$out/ncu_brief.txt"
