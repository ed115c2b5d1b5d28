"""Multi-GPU partitioner of the ISM path: one process per GPU over
torch.distributed (NCCL on the GPU box, gloo in the CPU tests).

* Batched problems (BASELINE config 5): contiguous problem blocks per rank, no data-path
  collective; controls and run records are gathered once at the end (``run_batch_sharded``).
* Subinterval blocks (config 3 layout): rank g owns a contiguous block of subintervals.  The
  one exchange step per outer iteration is an all-gather of the block products
  P_g = M_{last} ... M_{first} (``block_boundaries``); every rank then forms its own boundary
  states psi_n, chi_n exactly as ``compose_from_propagators`` (ism.cpp:298-312) would, using
  psi_start(g) = P_{g-1} ... P_0 psi_i and chi_end(g) = (P_{G-1} ... P_{g+1})^dag target.
  This matches the serial chain to rounding (< 1e-11).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def balanced_blocks(total: int, world: int) -> list[tuple[int, int]]:
    """Contiguous (first, count) blocks; the first total % world ranks get one extra item."""
    if world < 1:
        raise ValueError("world size must be positive")
    base, extra = divmod(total, world)
    out, first = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((first, n))
        first += n
    return out


def shard(total: int, world: int, rank: int) -> tuple[int, int]:
    return balanced_blocks(total, world)[rank]


@dataclass
class ShardedRun:
    controls: np.ndarray     # (B, C, K), all problems, on every rank
    objectives: np.ndarray   # (B, max_outer + 1), NaN-padded
    first: int
    count: int


def _collective_device(dist):
    """Device of the collective buffers: the current CUDA device under NCCL (which rejects host
    tensors), the host under gloo."""
    import torch
    if dist is not None and dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def all_gather_blocks(dist, local: np.ndarray, counts: list[int]) -> np.ndarray:
    """One all-gather of ragged contiguous row blocks (rank r contributes counts[r] rows of equal
    trailing shape): rows are padded to the largest block, gathered as one float64 tensor on the
    collective device (NVLink under NCCL), then un-padded in rank order."""
    import torch
    world = len(counts)
    mx = max(counts)
    dev = _collective_device(dist)
    flat = np.ascontiguousarray(local, dtype=np.float64)
    if np.iscomplexobj(local):
        flat = np.ascontiguousarray(local).view(np.float64)
    tail = flat.shape[1:]
    buf = torch.zeros((mx,) + tuple(tail), dtype=torch.float64, device=dev)
    buf[:flat.shape[0]] = torch.from_numpy(flat).to(dev)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    out = np.concatenate([parts[r][:counts[r]].cpu().numpy() for r in range(world)])
    return out.view(np.complex128) if np.iscomplexobj(local) else out


def run_batch_sharded(problem_builder, solve, total: int, dist=None) -> ShardedRun:
    """Config-5 partition: this rank solves problems [first, first + count) with ``solve``
    (the device ``ism.run_ism_batch`` in production) and all ranks gather the results once --
    one all-gather of the controls and one of the objective histories.

    problem_builder(first, count) -> (ControlProblem, u0, IsmConfig, SolverSpec)
    solve(problem, u0, cfg, solver) -> list[IsmRun]
    """
    world = dist.get_world_size() if dist is not None else 1
    rank = dist.get_rank() if dist is not None else 0
    first, count = shard(total, world, rank)
    p, u0, cfg, sv = problem_builder(first, count)
    runs = solve(p, u0, cfg, sv)
    C, K = p.model.channels(), p.grid.steps
    cap = cfg.max_outer + 1
    ctl = np.stack([r.control for r in runs]).reshape(count, C, K)
    obj = np.full((count, cap), np.nan)
    for i, r in enumerate(runs):
        o = r.record.objectives()
        obj[i, :len(o)] = o
    if dist is None or world == 1:
        return ShardedRun(ctl, obj, first, count)
    counts = [n for _, n in balanced_blocks(total, world)]
    return ShardedRun(all_gather_blocks(dist, ctl, counts), all_gather_blocks(dist, obj, counts), first, count)


def block_product(props: np.ndarray) -> np.ndarray:
    """P = M_{n-1} ... M_0 for a rank's contiguous propagators props[n] (d x d)."""
    d = props.shape[-1]
    P = np.eye(d, dtype=np.complex128)
    for M in props:
        P = M @ P
    return P


def block_boundaries(local_props: np.ndarray, initial: np.ndarray, target: np.ndarray, dist=None):
    """Boundary states of this rank's subintervals after the one all-gather of block products.

    local_props: (n_local, d, d) propagators M_n of this rank's contiguous subinterval block.
    Returns (psi, chi): (n_local + 1, d) each -- psi_n at the block's nodes (forward chain,
    psi_{n+1} = M_n psi_n) and chi_n (chi_n = M_n^dag chi_{n+1}, seeded with the target at the
    final node), i.e. the rank's slice of compose_from_propagators (ism.cpp:298-312).
    """
    world = dist.get_world_size() if dist is not None else 1
    rank = dist.get_rank() if dist is not None else 0
    Pg = block_product(local_props)
    if dist is None or world == 1:
        blocks = [Pg]
    else:  # the per-iteration exchange: G block products (complex128 as float64 pairs)
        blocks = list(all_gather_blocks(dist, Pg[None], [1] * world))
    psi = np.asarray(initial, dtype=np.complex128)
    for g in range(rank):
        psi = blocks[g] @ psi
    chi = np.asarray(target, dtype=np.complex128)
    for g in range(world - 1, rank, -1):
        chi = blocks[g].conj().T @ chi
    n = len(local_props)
    psis = [psi]
    for m in range(n):
        psis.append(local_props[m] @ psis[-1])
    chis = [chi]
    for m in range(n - 1, -1, -1):
        chis.append(local_props[m].conj().T @ chis[-1])
    return np.stack(psis), np.stack(chis[::-1])
