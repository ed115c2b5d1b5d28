#!/usr/bin/env python
"""bench.py -- ISM hot path (arXiv 1603.01237) on B200: propagation steps/s.

One "step" is one ISM outer iteration over the whole workload: every subinterval task's
forward sweep, adjoint sweep with the fused gradient + control update, residual sweeps and
propagator assembly, then the boundary chain and waypoint rebuild (ism.cpp:396-592).
metric = 2 * K * B * iterations / seconds: one forward and one adjoint
single-state step per grid step, B independent problems.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload NAME]

Default workload = BASELINE.json configs[4], the largest configuration and the one that fits one
GPU: 4096 independent 4-qubit problems (d = 16, dense), K = 2000, L = 128 (80 x 16 + 48 x 15
steps), rho = 0.1/dt.  N > 1 shards the 4096 problems over N ranks (one process per GPU, no
data-path collective; controls gathered once at the end); without torchrun in the environment
``--gpus N`` spawns the N ranks itself.  The single-problem configs (rotor21, spin2, gpe1024)
run N replicas ("replicas only").  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "propagation steps/s (fwd+adjoint, all subintervals); time-to-fidelity 0.999"
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2: every timed iteration starts cold
# --blocks G (config 3): the blocked boundary refresh with G subinterval blocks; None keeps the
# direct node sweeps on one GPU and one block per rank under torchrun (SURVEY §8(e) option A)
BLOCKS = None


def ising_blocked(world: int) -> bool:
    return BLOCKS is not None or world > 1


def flops_per_iteration(name: str, w) -> float:
    """Algorithmic fp64 flops of one outer iteration (SURVEY.md §8(d) model, '+err' variant:
    forward + adjoint/gradient + assembly + residual forward/adjoint per grid step)."""
    p = w.problem
    d, C, K, B = p.model.state_dim(), p.model.channels(), p.grid.steps, p.batch
    if name == "rotor21":  # tridiagonal: W_tri = 64d, W_g = 24d, W_asm = 41d^2 + 23d
        per = 4 * 64 * d + 2 * 24 * d + 41 * d * d + 23 * d
    elif name in ("spin2", "batch4096"):  # dense Cayley
        w_cay = (8 / 3) * d ** 3 + (4 * C + 20) * d ** 2
        w_bg = w_cay + 4 * d + C * (8 * d ** 2 + 8 * d)
        w_asm = (56 / 3) * d ** 3 + (4 * C + 4) * d ** 2
        per = 2 * w_cay + 2 * w_bg + w_asm
    elif name == "ising10":
        cay = ising_cayley_flops(w)  # summed over the K grid steps
        n = p.model.nspins
        # direct plan: entry, forward, adjoint, residual forward + adjoint in the tasks and the two
        # node sweeps = 7 Cayley steps per grid step, and 2 gradient evaluations (C channels x n
        # flips x 16 flop per amplitude)
        total = 7 * cay + 2 * C * n * 16 * d * K
        if w.config.plan == "assembled":
            total += d * cay  # blocked plan: the block products carry d columns per grid step
        return total * B
    elif name == "spins":
        # density-matrix conjugation kind (dm x dm matrix states): per grid step and sweep one
        # dm x dm inverse (8/3 dm^3 + build) and complex dm^3 products (8 dm^3 flop each):
        # forward rho' = A rho A^dag 2 products, adjoint + gradient 5 products (r1, r2, M = r2 r1^dag,
        # X' and its half) + C dm^2 contractions, assembly 1 product.  Entry, gradient (fwd + bwd),
        # residual (fwd + bwd), assembly = 3 forward + 2 backward + 1 assembly sweeps.
        dm = d  # state_dim() is the matrix edge of the dm x dm states
        inv = (8 / 3) * dm ** 3 + (4 * C + 4) * dm ** 2
        fwd, bwd, asm = inv + 2 * 8 * dm ** 3, inv + 5 * 8 * dm ** 3 + C * 8 * dm ** 2, inv + 8 * dm ** 3
        per = 3 * fwd + 2 * bwd + asm
    elif name == "gpe1024":
        # split variant: entry, gradient (fwd + bwd), residual (fwd + bwd), lagged refresh
        # (fwd + bwd) = 4 forward + 3 backward stages per grid step; FFT = 5 n log2 n
        n = d
        fft = 5 * n * np.log2(n)
        w_s, w_sb = 4 * fft + 32 * n, 6 * fft + 84 * n
        per = 4 * w_s + 3 * w_sb
    else:
        return float("nan")
    return per * K * B


def ising_cayley_flops(w) -> float:
    """Flops of one bit-flip Cayley step summed over the grid steps: s_j Jacobi sweeps of
    z <- (1 + sD)^-1 (x - s V z), each n complex FMAs per amplitude for V z (8n flop) plus 12 flop
    of diagonal work, with s_j the kernel's a-priori count ceil(54 ln 2 / -ln q_j),
    q_j = dt/2 sum_i |(ax_i, ay_i)| at u_j (bitflip_kernels.cu begin_step)."""
    p = w.problem
    d, C, K, n = p.model.state_dim(), p.model.channels(), p.grid.steps, p.model.nspins
    u = np.asarray(w.u0).reshape(C, K)
    q = 0.5 * p.grid.dt * 0.5 * n * np.sqrt(u[0] ** 2 + u[1] ** 2)
    sweeps = np.where(q > 0, np.ceil(54 * np.log(2) / -np.log(np.maximum(q, 1e-300))), 0.0)
    return float(np.sum(sweeps) * (8 * n + 12) * d)


def dmma_peak():
    f = ROOT / "profiles" / "dmma_peak.json"
    if f.exists():
        return json.loads(f.read_text())["fp64_mma_tflops"], "measured (tools/dmma_peak.cu, profiles/dmma_peak.json)"
    return 37.2, "nominal fp64 tensor rate (no measurement found)"


def fp64_peak():
    f = ROOT / "profiles" / "fp64_peak.json"
    if f.exists():
        j = json.loads(f.read_text())
        return j["fp64_fma_tflops"], "measured (tools/fp64_peak.cu, profiles/fp64_peak.json)"
    return 37.2, "nominal 148 SM x 64 DFMA x 2 x 1.965 GHz (no measurement found)"


def ncu_traffic(name: str):
    f = ROOT / "profiles" / f"ncu_{name}.json"
    if f.exists():
        j = json.loads(f.read_text())
        return j.get("dram_bytes_per_launch")
    return None


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.tmp = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.tmp, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        self.tmp.seek(0)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.tmp.read().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def build_workload(name: str, iterations: int, rank: int, world: int, rho_fast: bool = True):
    from paper_1603_01237_b200 import problems
    from paper_1603_01237_b200.partition import shard
    if name == "rotor21":
        w = problems.rotor21(subintervals=128, iterations=iterations)
    elif name == "spin2":
        w = problems.spin2(iterations=iterations)
    elif name == "batch4096":
        first, count = shard(4096, world, rank)
        w = problems.batch4096(batch=count, iterations=iterations, first=first)
    elif name == "ising10":
        w = problems.ising10(iterations=iterations)
        if ising_blocked(world):
            w.config.plan, w.config.blocks = "assembled", BLOCKS or 0
    elif name == "spins":
        # the reference's `spins` preset at full size (5 spins, 32 x 32 density matrices, 10 x/y
        # controls, 2^15 steps, rho = 1e4; config.cpp:132-146) -- the paper's 5-spin case -- on 256
        # subintervals; rho of the preset kept (rho_fast would be 0.1/dt = 234)
        w = problems.spins_preset(quick=False, subintervals=256, iterations=iterations)
        w.rho_fast = w.solver.step_size
    elif name == "gpe1024":
        w = problems.gpe1024(iterations=iterations)
        # the exact-payoff instrumentation (a serial K-step sweep per iteration) is outside the
        # reference's critical path (ism.cpp:580-584); time-to-fidelity runs switch it back on
        w.config.log_exact_objective = False
    else:
        raise SystemExit(f"unknown workload {name}")
    if rho_fast:
        w.solver.step_size = w.rho_fast
    return w


def workload_config(name: str, world: int) -> dict:
    """The `config` echo shared by both arms (same keys and values for the same N)."""
    from paper_1603_01237_b200 import problems
    w = build_workload(name, 1, 0, world)
    desc = problems.describe(w)
    total = 4096 if name == "batch4096" else 1
    return {"workload": name, "dim": desc["dim"], "channels": desc["channels"], "grid_steps": desc["steps"],
            "subintervals": desc["subintervals"], "partition": desc["partition"], "problems": total,
            "problems_per_gpu": w.problem.batch, "step_size": w.solver.step_size, "variant": desc["variant"],
            "plan": desc["plan"],
            "parallelism": (f"problem blocks x{world}" if name == "batch4096" else
                            f"subinterval blocks: {BLOCKS or world} blocks over {world} rank(s), one all-gather "
                            "per outer iteration" if name == "ising10" and ising_blocked(world) else
                            f"replicas x{world}"),
            "l2": "flushed between timed iterations (256 MiB memset outside the event brackets)"}


def problem_bytes(w) -> int:
    from paper_1603_01237_b200 import ism as I
    packed = I.pack_problem(w.problem)
    return int(sum(a.nbytes for a in packed.keep)) + int(np.asarray(w.u0).nbytes)


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    return world, rank, local, dist


def spawn_ranks(nproc: int) -> int:
    """`bench.py --gpus N` outside torchrun: launch the N ranks (one process per GPU) through
    torch.distributed.run on 127.0.0.1 and pass rank 0's JSON line through."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def _t(dist, v: float):
    import torch
    dev = "cuda" if (torch.cuda.is_available() and dist.get_backend() == "nccl") else "cpu"
    return torch.tensor([v], dtype=torch.float64, device=dev)


def allmax(dist, v: float) -> float:
    if dist is None:
        return v
    t = _t(dist, v)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allsum(dist, v: float) -> float:
    if dist is None:
        return v
    t = _t(dist, v)
    dist.all_reduce(t)
    return float(t.item())


def barrier_sync(dist):
    try:
        import torch
        if torch.cuda.is_available():
            torch.cuda.synchronize()
    except ImportError:
        pass
    if dist is not None:
        dist.barrier()


# sample of the CPU path per workload: problems of the batch timed (the rest scale linearly)
CPU_SAMPLE_PROBLEMS = {"batch4096": 256}


def cpu_reference(name: str, warmup: int, steps: int, world: int = 1):
    """The reference's CPU path: the oracle restatement with reference arithmetic (dense
    partial-pivot LU per step, like Eigen::PartialPivLU in propagation.cpp:85-106) on all host
    threads, as WorkerPool does (runtime.cpp:72-90).  Test infrastructure: only this leg and the
    --impl reference arm execute oracle/ code, after (or instead of) the timed device region."""
    from tests import oracle_api as O
    from paper_1603_01237_b200 import problems
    threads = os.cpu_count() or 1
    if name == "batch4096":
        sample_b = CPU_SAMPLE_PROBLEMS[name]
        w = problems.batch4096(batch=sample_b, iterations=warmup + steps)
        desc = f"{sample_b} of the 4096 problems (d=16, K=2000, L=128); steps/s of the sample"
    elif name == "spins":
        # 1/16 of the horizon: 2048 of the 2^15 grid steps on 16 subintervals (the same 128 steps
        # per task); the work per grid step does not depend on the step's position or size
        w = problems.spins_preset(quick=False, subintervals=16, steps=2048, iterations=warmup + steps)
        w.rho_fast = w.solver.step_size
        steps, warmup = min(steps, 2), 0
        desc = "2048 of the 32768 grid steps of the 5-spin preset on 16 subintervals (128 steps per task)"
    else:
        w = build_workload(name, warmup + steps, 0, 1)
        desc = f"full {name} workload"
    arith = O.REFERENCE
    if name == "ising10":  # dense LU at d = 1024 is ~1.4e14 flop per iteration: structured solve
        arith = O.STRUCTURED
        w.config.plan, w.config.blocks = "direct", 0  # the oracle's plan (agrees to rounding)
        steps = min(steps, 2)
        warmup = 0
    if name == "rotor21":  # the reference builds the rotor as a dense model (models.cpp:361-380)
        from paper_1603_01237_b200.models import TridiagonalModel
        assert isinstance(w.problem.model, TridiagonalModel)
        w.problem.model = w.problem.model.to_dense()
    w.solver.step_size = w.rho_fast
    w.config.max_outer = warmup + steps
    p = w.problem
    work = 2.0 * p.grid.steps * p.batch * steps
    # The reference ITSELF where it was compiled (oracle/_ref/libqocref.so: /root/reference's own
    # run_ism and everything under it, built from source against oracle/eigen_shim; it travels
    # with the snapshot): its WorkerPool runs the L tasks on `workers` threads, problems of the
    # batch one after another.  Config 3 stays on the oracle port: the reference's dense LU at
    # d = 1024 is ~1.4e14 flop per iteration.
    if arith == O.REFERENCE and O.REF_LIBPATH.exists() and not os.environ.get("QOC_BENCH_PORT"):
        w.config.partition = "balanced"
        if p.grid.steps % w.config.subintervals:  # Decomposition::uniform throws (ism.cpp:234): largest divisor
            w.config.subintervals = max(L for L in range(1, w.config.subintervals + 1) if p.grid.steps % L == 0)
        # the reference's own WorkerPool (runtime.cpp:72-90) over the L tasks, the sample's problems
        # one after another (one run_ism per host thread with workers = 1 measured slower here:
        # 1.7e5 vs 2.05e5 steps/s on 8 cores)
        w.config.workers = threads
        t0 = time.perf_counter()
        runs = O.ref_ism_run(p, w.u0, w.config, w.solver)
        wall = time.perf_counter() - t0
        secs = sum(it.device_seconds for r in runs for it in r.record.iterations[warmup + 1:warmup + steps + 1])
        how = f"WorkerPool of {threads} threads, problems in sequence"
        return {"value": work / secs, "unit": "steps/s", "cores": threads, "kind": "reference",
                "sample": f"{desc}; the reference's own run_ism compiled from /root/reference (Eigen-subset shim), "
                          f"L = {w.config.subintervals}, {steps} timed outer iterations after {warmup} warm-up, {how}",
                "seconds": secs, "wall": wall, "seconds_per_iteration": secs / steps, "sample_problems": p.batch,
                "horizon_scale": (32768.0 / p.grid.steps) if name == "spins" else 1.0}
    t0 = time.perf_counter()
    runs = O.ism_run(w.problem, w.u0, w.config, w.solver, arith, threads=threads)
    wall = time.perf_counter() - t0
    its = runs[0].record.iterations
    secs = sum(it.device_seconds for it in its[warmup + 1:warmup + steps + 1])
    if p.batch > 1:  # problems run concurrently on the threads: the sample's wall clock, not one problem's
        secs = wall * steps / float(warmup + steps)
    return {"value": work / secs, "unit": "steps/s", "cores": threads, "kind": "port",
            "sample": f"{desc}; {steps} timed outer iterations after {warmup} warm-up, "
                      f"{'dense-LU reference' if arith == O.REFERENCE else 'structured (Neumann) Cayley'} "
                      f"arithmetic, {threads} threads",
            "seconds": secs, "wall": wall, "seconds_per_iteration": secs / steps,
            "sample_problems": p.batch}


def full_batch(name: str) -> int:
    return 4096 if name == "batch4096" else 1


def run_reference_arm(args, world, rank, dist):
    if rank != 0:
        return 0
    ref = cpu_reference(args.workload, args.warmup, args.steps)
    line = {"metric": METRIC, "value": ref["value"], "unit": "steps/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            # one outer iteration of the whole workload at the sample's rate
            "ms_per_step": 1e3 * ref["seconds_per_iteration"] * full_batch(args.workload) / ref["sample_problems"]
                           * ref.get("horizon_scale", 1.0),
            "higher_is_better": True,
            "scaling": "strong" if args.workload == "batch4096" else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded, SURVEY §8(d))",
            "config": workload_config(args.workload, max(args.gpus, world)),
            "cpu_baseline": {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": ref["value"], "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def label_flops(name: str, label: str, w, world: int = 1) -> float:
    """Algorithmic fp64 flops of one launch of the kernel behind a launch label (SURVEY §8(d)
    per-grid-step model x K x B).  'assembly' = the d-column propagator product sweep
    (assemble_propagator, propagation.cpp:236-249); 'gradient'/'residual' = a forward sweep +
    an adjoint/gradient sweep (objective.cpp:38-89); 'task'/'node sweeps' = the whole
    iteration's task work (flops_per_iteration)."""
    p = w.problem
    d, C, K, B = p.model.state_dim(), p.model.channels(), p.grid.steps, p.batch
    if name == "batch4096" and label == "assembly":
        # executed by the Neumann/tensor-core sweep (dense_nm.cu): the d x d complex product
        # P_{j+1}^T = P_j^T C_j^T on DMMA = 4 real d^3 GEMMs per grid step
        return 8 * d ** 3 * K * B
    if name in ("spin2", "batch4096"):
        w_cay = (8 / 3) * d ** 3 + (4 * C + 20) * d ** 2
        w_bg = w_cay + 4 * d + C * (8 * d ** 2 + 8 * d)
        per = {"assembly": (56 / 3) * d ** 3 + (4 * C + 4) * d ** 2, "gradient": w_cay + w_bg,
               "residual": w_cay + w_bg}.get(label)
    elif name == "rotor21":
        per = {"assembly": 41 * d * d + 23 * d, "gradient": 64 * d + 64 * d + 24 * d,
               "residual": 64 * d + 64 * d + 24 * d}.get(label)
    elif name == "ising10":
        n = p.model.nspins
        cay = ising_cayley_flops(w)  # summed over the K grid steps
        tot = {"node sweeps": 2 * cay,  # forward + adjoint full-horizon sweeps
               "task": 5 * cay + 2 * C * n * 16 * d * K,
               # blocked plan: d basis columns through this rank's K / W steps
               "block products": d * cay / world}.get(label)
        if tot is not None:
            return tot * B
        per = None
    else:
        per = None
    if per is None:
        return flops_per_iteration(name, w)
    return per * K * B


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="batch4096",
                    choices=["batch4096", "rotor21", "spin2", "ising10", "gpe1024", "spins"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ttf", action="store_true", help="skip the time-to-fidelity run")
    ap.add_argument("--blocks", type=int, default=None,
                    help="ising10: subinterval blocks of the blocked boundary refresh (default: direct "
                         "node sweeps on one GPU, one block per rank on N GPUs)")
    args = ap.parse_args()
    global BLOCKS
    BLOCKS = args.blocks
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    world, rank, local, dist = dist_setup()
    if args.impl == "reference":
        return run_reference_arm(args, world, rank, dist)

    from paper_1603_01237_b200 import _native, abi
    from paper_1603_01237_b200 import ism as I
    from paper_1603_01237_b200 import problems

    K_, W_ = args.steps, args.warmup
    ctx = _native.default_context(local)
    blocked = args.workload == "ising10" and ising_blocked(world)
    if blocked and world > 1:  # one NCCL communicator inside libqoc_b200.so per rank
        obj = [_native.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx.init_comm(rank, world, obj[0])
    w = build_workload(args.workload, W_ + K_, rank, world)
    p = w.problem
    # untimed first call (context, module load)
    w1 = build_workload(args.workload, 1, rank, world)
    I.run_ism_batch(w1.problem, w1.u0, w1.config, w1.solver, ctx)

    # ---- timed: W warm-up + K timed outer iterations inside one run; per-iteration CUDA events
    # (no per-launch event brackets here: they would add their own gaps to the timed stream)
    ctx.set_option(abi.OPT_PROFILE, 0)
    ctx.set_option(abi.OPT_FLUSH_L2_BYTES, L2_FLUSH_BYTES)
    ctx.profile(reset=True)
    barrier_sync(dist)
    with Clocks(local) as clk:
        runs = I.run_ism_batch(p, w.u0, w.config, w.solver, ctx)
        barrier_sync(dist)
    prof_main = ctx.profile(reset=True)
    # ---- a separate short profiled run: per-launch CUDA events on the launching stream
    wp = build_workload(args.workload, W_ + 2, rank, world)
    ctx.set_option(abi.OPT_PROFILE, 1)
    I.run_ism_batch(wp.problem, wp.u0, wp.config, wp.solver, ctx)
    prof = ctx.profile()
    kprof = ctx.kernel_profile()
    ctx.profile(reset=True)
    ctx.set_option(abi.OPT_PROFILE, 0)
    its = runs[0].record.iterations
    timed = its[W_ + 1:W_ + K_ + 1]
    assert len(timed) == K_, "run stopped early"
    t_rank = sum(it.device_seconds for it in timed)
    t_max = allmax(dist, t_rank)
    work_rank = 2.0 * p.grid.steps * p.batch * K_
    # a sharded config-3 run is ONE problem over all ranks: its steps are counted once
    work = work_rank if blocked else allsum(dist, work_rank)
    value = work / t_max
    launches_per_iter = prof_main["iteration_launches"] / max(prof_main["iterations"], 1)

    # ---- roofline of the dominant kernel: the launch site with the most device time in the
    # profiled run (its launches bracketed by CUDA events on the launching stream)
    n_iter = max(prof["iterations"], 1)
    iter_ms = prof["iteration_ms"] / n_iter
    dom, (dom_ms, dom_n) = max(kprof.items(), key=lambda kv: kv[1][0]) if kprof else ("task", (float("nan"), 1))
    per_launch_ms = dom_ms / max(dom_n, 1)
    fl_launch = label_flops(args.workload, dom, wp, world)
    tensor = args.workload == "batch4096" and dom == "assembly"
    peak, peak_src = dmma_peak() if tensor else fp64_peak()
    achieved = fl_launch / (per_launch_ms * 1e-3) / 1e12
    # the same kernel counted with the reference algorithm's flops (SURVEY §8(d) per-unit figure,
    # LU + d-column solve per step) -- exceeds the fp64 roof because the Neumann formulation
    # does far less work than the reference per unit
    ref_count = None
    if tensor:
        p_ = wp.problem
        d_, C_, K_p, B_ = p_.model.state_dim(), p_.model.channels(), p_.grid.steps, p_.batch
        ref_count = ((56 / 3) * d_ ** 3 + (4 * C_ + 4) * d_ ** 2) * K_p * B_ / (per_launch_ms * 1e-3) / 1e12
    fl_iter = flops_per_iteration(args.workload, w)
    kernels = {k: {"ms_per_iteration": v[0] / n_iter, "launches_per_iteration": v[1] / n_iter,
                   "share": v[0] / max(sum(x[0] for x in kprof.values()), 1e-12)} for k, v in kprof.items()}

    # ---- end to end through the public API: host buffers in, host results out
    ctx.set_option(abi.OPT_FLUSH_L2_BYTES, 0)
    we = build_workload(args.workload, K_, rank, world)
    sharded = args.workload == "batch4096" and world > 1
    walls = []
    for _ in range(3):  # median of three whole calls (host-side jitter is ms-scale)
        barrier_sync(dist)
        t0 = time.perf_counter()
        if sharded:  # this rank's problem block, then the one all-gather of every control
            from paper_1603_01237_b200 import partition as PT
            res = PT.run_batch_sharded(lambda f, c: (we.problem, we.u0, we.config, we.solver),
                                       lambda p_, u_, c_, s_: I.run_ism_batch(p_, u_, c_, s_, ctx), 4096, dist)
            e2e_runs = [None] * res.count
            assert res.controls.shape[0] == 4096
        else:
            e2e_runs = I.run_ism_batch(we.problem, we.u0, we.config, we.solver, ctx)
        barrier_sync(dist)
        walls.append(time.perf_counter() - t0)
    e2e_wall = allmax(dist, statistics.median(walls))
    e2e_work = 2.0 * we.problem.grid.steps * we.problem.batch * K_
    e2e_value = (e2e_work if blocked else allsum(dist, e2e_work)) / e2e_wall
    h2d = problem_bytes(we)
    nb = we.problem.batch
    d2h = int(8 * we.problem.model.channels() * we.problem.grid.steps * nb
              + (K_ + 1) * (abi.REC_DTYPE.itemsize + 8 * we.config.subintervals) * nb)

    # ---- time to fidelity 0.999 (rho = 0.1/dt): device time and wall clock of a run_ism call
    ttf = None
    if not args.no_ttf and args.workload in ("rotor21", "spin2", "batch4096") and rank == 0:
        ttf = time_to_fidelity(args.workload, ctx, I, problems)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ref = cpu_reference(args.workload, 0, 3)
        cpu = {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample")}
        if ttf and ttf.get("iterations"):
            scale = 1.0 / ref["sample_problems"] if args.workload == "batch4096" else 1.0
            ttf["cpu_seconds_est"] = ttf["iterations"] * ref["seconds_per_iteration"] * scale * ttf.get("problems", 1)

    if rank != 0:
        return 0
    line = {
        "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": K_, "warmup": W_,
        "ms_per_step": 1e3 * t_max / K_, "higher_is_better": True,
        "scaling": "strong" if args.workload == "batch4096" or blocked else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded, SURVEY §8(d))", "config": workload_config(args.workload, world),
        "e2e": {"value": e2e_value, "unit": "steps/s", "h2d_bytes_per_step": h2d // K_,
                "d2h_bytes_per_step": d2h // K_, "note": "one run_ism_batch call of K outer iterations from host "
                "arrays (median of 3 calls), wall clock incl. packing, upload, bootstrap, trailing "
                "evaluation and download"},
        "gpu_launches": int(round(launches_per_iter * K_)),
        "roofline": {"bound": "tensor" if tensor else "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "reference_count_tflops": ref_count,
                     "frac": achieved / peak, "traffic": ncu_traffic(args.workload),
                     "kernel": dom, "kernel_ms_per_launch": per_launch_ms, "flops_per_launch": fl_launch,
                     "share_of_step": dom_ms / max(prof["iteration_ms"], 1e-12), "peak_source": peak_src,
                     "iteration": {"flops": fl_iter, "ms": iter_ms,
                                   "tflops": fl_iter / (iter_ms * 1e-3) / 1e12 if iter_ms > 0 else None},
                     "kernels": kernels},
        "time_to_fidelity": ttf,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    return 0


def time_to_fidelity(name, ctx, I, problems):
    """Iterations, device seconds and wall-clock seconds until F = 1 + objective >= 0.999
    (rho = 0.1/dt).  Batch: 64 problems, the first one that reaches it counts."""
    if name == "batch4096":
        wt = problems.batch4096(batch=64, iterations=400)
    else:
        wt = build_workload(name, 4000 if name == "rotor21" else 300, 0, 1)
    wt.solver.step_size = wt.rho_fast
    rr = I.run_ism_batch(wt.problem, wt.u0, wt.config, wt.solver, ctx)
    hits = []
    for b, r in enumerate(rr):
        h = np.nonzero(1.0 + r.record.objectives() >= 0.999)[0]
        if len(h):
            hits.append((int(h[0]), b))
    best = [float(np.nanmax(1.0 + r.record.objectives())) for r in rr]
    out = {"target": 0.999, "rho": wt.solver.step_size, "problems": wt.problem.batch,
           "reached": len(hits), "best_fidelity_max": max(best)}
    if not hits:
        out["iterations"] = None
        return out
    k = max(h for h, _ in hits)  # iterations until every reaching problem got there
    r0 = rr[hits[0][1]]
    out["iterations"] = k
    out["device_seconds"] = float(sum(it.device_seconds for it in rr[0].record.iterations[:k + 1]))
    # wall clock: the same call stopped at k iterations (host arrays in and out)
    wt.config.max_outer = k
    t0 = time.perf_counter()
    I.run_ism_batch(wt.problem, wt.u0, wt.config, wt.solver, ctx)
    out["wall_seconds"] = time.perf_counter() - t0
    out["first_problem_iterations"] = int(min(h for h, _ in hits))
    del r0
    return out


if __name__ == "__main__":
    sys.exit(main())
