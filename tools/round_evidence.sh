#!/usr/bin/env bash
# Round-end evidence on one GPU (run under gpurun from the repo root): default bench line
# (with cpu_baseline), the reference arm, every workload's bench line, the ncu launch list of
# the default bench command and one --set full capture of its dominant kernel.
set -u
out=gpurun_out/${1:-evidence}
mkdir -p "$out"
nproc > "$out/nproc.txt"; lscpu > "$out/lscpu.txt" 2>&1
timeout 900 python bench.py > "$out/bench_default.json" 2> "$out/bench_default.err"; echo "default rc=$?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > "$out/bench_reference.json" 2> "$out/bench_reference.err"; echo "reference rc=$?"
for wl in spin2 batch4096 ising10 gpe1024; do
  timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline > "$out/bench_$wl.json" 2> "$out/bench_$wl.err"; echo "$wl rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file "$out/launches_default.csv" \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > "$out/ncu_launch.log" 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:tri_pc_assemble|pc_eval|chain_small" -c 3 \
  -o "$out/full_default" python bench.py --steps 1 --warmup 3 --no-cpu-baseline > "$out/ncu_full.log" 2>&1; echo "full rc=$?"
