#!/usr/bin/env bash
# Round evidence on one GPU (run under gpurun from the repo root):
#   * the default bench line (config 5, with cpu_baseline) and the reference arm;
#   * every other workload's bench line with its cpu_baseline;
#   * the ncu launch list of the default bench command (cold, serialised per-launch times);
#   * one `ncu --set full` capture of each workload's dominant kernel(s);
#   * compute-sanitizer memcheck and racecheck on the smoke workloads (one tool per run).
# usage: tools/round_evidence.sh TAG [SECTION...]   sections: bench ncu sanitize (default: all)
set -u
out=gpurun_out/${1:-evidence}
shift || true
sections=${*:-"bench ncu sanitize"}
# (gpurun copies back at most 64 MiB of gpurun_out/: run the ncu section in its own call)
mkdir -p "$out"
nproc > "$out/nproc.txt"; lscpu > "$out/lscpu.txt" 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$out/gpu.txt" 2>&1
if [[ " $sections " == *" bench "* ]]; then
  timeout 900 python bench.py > "$out/bench_default.json" 2> "$out/bench_default.err"; echo "default rc=$?"
  timeout 900 python bench.py --impl reference > "$out/bench_reference.json" 2> "$out/bench_reference.err"; echo "reference rc=$?"
  for wl in spin2 rotor21 ising10 gpe1024 spins; do
    timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 > "$out/bench_$wl.json" 2> "$out/bench_$wl.err"
    echo "$wl rc=$?"
  done
  # config 3 sharded into 8 subinterval blocks (the 8-GPU layout on one GPU)
  timeout 900 python bench.py --workload ising10 --blocks 8 --steps 5 --warmup 3 --no-cpu-baseline \
    > "$out/bench_ising10_b8.json" 2> "$out/bench_ising10_b8.err"; echo "ising10 b8 rc=$?"
fi
if [[ " $sections " == *" ncu "* ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file "$out/launches_default.csv" \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ttf > "$out/ncu_launch.log" 2>&1; echo "launches rc=$?"
  # one --set full capture per dominant kernel, taken inside the outer iterations (the bootstrap's
  # launches of the same kernels are skipped)
  cap() {  # cap NAME REGEX SKIP bench-args...
    local name=$1 re=$2 skip=$3; shift 3
    timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$re" --launch-skip "$skip" -c 1 \
      -o "$out/full_$name" python bench.py "$@" --steps 2 --warmup 3 --no-cpu-baseline --no-ttf > "$out/ncu_full_$name.log" 2>&1
    echo "full $name rc=$?"
  }
  cap batch4096_assembly dense_nm_assemble 2
  cap batch4096_evaluation dense_pc_eval16 2
  cap ising10_node_sweeps bitflip_horizon_cluster 2 --workload ising10
  cap ising10_block_products bitflip_block_kernel 1 --workload ising10 --blocks 8
  cap gpe1024_task strang_task 2 --workload gpe1024
  cap rotor21_assembly tri_pc_assemble 2 --workload rotor21
  for f in "$out"/full_*.ncu-rep; do
    [ -f "$f" ] && python tools/ncu_brief.py "$f" >> "$out/ncu_brief.txt" 2>&1
  done
fi
if [[ " $sections " == *" sanitize "* ]]; then
  timeout 1200 compute-sanitizer --tool memcheck --leak-check full python __graft_entry__.py > "$out/memcheck.log" 2>&1
  echo "memcheck rc=$?"
  timeout 1500 compute-sanitizer --tool racecheck python __graft_entry__.py > "$out/racecheck.log" 2>&1
  echo "racecheck rc=$?"
fi
