"""Multi-GPU partitioner of the ISM path: one process per GPU over
torch.distributed (NCCL on the GPU box, gloo in the CPU tests).

* Batched problems (BASELINE config 5): contiguous problem blocks per rank, no data-path
  collective; controls and run records are gathered once at the end (``run_batch_sharded``).
* Subinterval blocks (config 3 layout): rank r owns a contiguous run of subinterval blocks.
  The one exchange step per outer iteration is an all-gather of the block products
  P_g = M_{last} ... M_{first} (``block_boundaries``); every rank then forms its own boundary
  states psi_n, chi_n exactly as ``compose_from_propagators`` (ism.cpp:298-312) would, using
  psi_start(g) = P_{g-1} ... P_0 psi_i and chi_end(g) = (P_{G-1} ... P_{g+1})^dag target.
  This matches the serial chain to rounding (< 1e-11).  On the GPU box the same exchange runs
  inside libqoc_b200.so (one in-place ncclAllGather of per-rank slabs per outer iteration,
  driver.cu); ``init_device_comm`` binds a device context to the torch.distributed world.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def init_device_comm(ctx, dist) -> None:
    """Bind a libqoc_b200 context to this process's rank of the torch.distributed world: rank 0
    draws the NCCL unique id, one broadcast hands it to every rank (qoc_ctx_init_comm)."""
    from . import _native
    world = dist.get_world_size() if dist is not None else 1
    rank = dist.get_rank() if dist is not None else 0
    if world == 1:
        ctx.init_comm(0, 1)
        return
    obj = [_native.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx.init_comm(rank, world, obj[0])


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


def block_nodes(L: int, G: int) -> list[int]:
    """Balanced contiguous split of L subintervals into G blocks (the first L mod G blocks get one
    more), as boundary indices [G+1] -- the split the device driver uses (driver.cu block_nodes)."""
    if not 1 <= G <= L:
        raise ValueError("blocks must lie in [1, subintervals]")
    out = [0]
    for g in range(G):
        out.append(out[-1] + L // G + (1 if g < L % G else 0))
    return out


def block_boundaries(local_props: np.ndarray, initial: np.ndarray, target: np.ndarray, dist=None,
                     blocks_per_rank: int = 1):
    """Boundary states of this rank's subintervals after the one all-gather of block products
    (the host-side statement of the device's blocked refresh, driver.cu / blocks.cu).

    local_props: (n_local, d, d) propagators M_n of this rank's contiguous subintervals, which
    form `blocks_per_rank` contiguous blocks (balanced split).  Every rank contributes the same
    number of blocks; one all-gather exchanges the G = world * blocks_per_rank block products
    P_g = M_{last} ... M_{first}.  Then every rank chains them into the block-boundary nodes,
    psi_{b[g+1]} = P_g psi_{b[g]} from psi_0 = initial and chi_{b[g]} = P_g^dag chi_{b[g+1]} from
    chi_L = target (compose_from_propagators, ism.cpp:298-312, over blocks), and fills its blocks'
    interior nodes from their chain-formed ends (the device runs node sweeps there).
    Returns (psi, chi): (n_local + 1, d) each, the rank's slice of the serial chain's nodes.
    """
    world = dist.get_world_size() if dist is not None else 1
    rank = dist.get_rank() if dist is not None else 0
    n = len(local_props)
    inner = block_nodes(n, blocks_per_rank)
    mine = np.stack([block_product(local_props[inner[q]:inner[q + 1]]) for q in range(blocks_per_rank)])
    if dist is None or world == 1:
        blocks = list(mine)
    else:  # the per-iteration exchange: G block products (complex128 as float64 pairs)
        blocks = list(all_gather_blocks(dist, mine, [blocks_per_rank] * world))
    G = len(blocks)
    # chain over all G blocks (every rank forms every block-boundary node)
    psi_b = [np.asarray(initial, dtype=np.complex128)]
    for g in range(G):
        psi_b.append(blocks[g] @ psi_b[-1])
    chi_b = [np.asarray(target, dtype=np.complex128)]
    for g in range(G - 1, -1, -1):
        chi_b.append(blocks[g].conj().T @ chi_b[-1])
    chi_b = chi_b[::-1]
    psis, chis = [None] * (n + 1), [None] * (n + 1)
    for q in range(blocks_per_rank):
        g = rank * blocks_per_rank + q
        a, z = inner[q], inner[q + 1]
        psis[a], psis[z] = psi_b[g], psi_b[g + 1]
        chis[a], chis[z] = chi_b[g], chi_b[g + 1]
        for m in range(a, z - 1):  # interior nodes from the block's chain-formed ends
            psis[m + 1] = local_props[m] @ psis[m]
        for m in range(z - 1, a, -1):
            chis[m] = local_props[m].conj().T @ chis[m + 1]
    return np.stack(psis), np.stack(chis)
