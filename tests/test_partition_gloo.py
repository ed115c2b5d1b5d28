"""Multi-rank partitioner on CPU: world_size-2 gloo process groups (no GPU).

The per-rank compute is the CPU oracle here (the checker); on the GPU box the same
partitioner drives the device library, one process per GPU over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1603_01237_b200 import ism as I
from paper_1603_01237_b200 import partition as PT
from paper_1603_01237_b200 import problems


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    finally:
        dist.destroy_process_group()


def run_ranks(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    return [out[r] for r in range(world)]


def test_balanced_blocks():
    assert PT.balanced_blocks(4096, 8) == [(512 * r, 512) for r in range(8)]
    assert PT.balanced_blocks(10, 4) == [(0, 3), (3, 3), (6, 2), (8, 2)]
    assert sum(n for _, n in PT.balanced_blocks(257, 3)) == 257


def _batch_job(rank, world):
    from tests import oracle_api as O

    def build(first, count):
        w = problems.batch4096(batch=count, iterations=2, first=first)
        w.config.subintervals = 4
        return w.problem, w.u0, w.config, w.solver

    r = PT.run_batch_sharded(build, lambda p, u, c, s: O.ism_run(p, u, c, s, O.REFERENCE, threads=1), 6, dist)
    return r.controls, r.objectives, r.first, r.count


def test_batch_sharding_gathers_every_problem():
    from tests import oracle_api as O
    res = run_ranks(_batch_job)
    (c0, o0, f0, n0), (c1, o1, f1, n1) = res
    assert (f0, n0, f1, n1) == (0, 3, 3, 3)
    assert np.array_equal(c0, c1) and np.array_equal(o0, o1, equal_nan=True)
    w = problems.batch4096(batch=6, iterations=2)
    w.config.subintervals = 4
    serial = O.ism_run(w.problem, w.u0, w.config, w.solver, O.REFERENCE, threads=1)
    assert np.array_equal(c0, np.stack([r.control for r in serial]))


def _block_job(rank, world):
    from tests import oracle_api as O
    p, u = O.dense_fixture(4242, dim=5, steps=48, channels=1)
    nodes = I.balanced_nodes(48, 8)
    first, count = PT.shard(8, world, rank)
    props = []
    for n in range(first, first + count):
        a, b = nodes[n], nodes[n + 1]
        sub = I.ControlProblem(p.model, I.TimeGrid(p.grid.node(a), p.grid.dt, b - a), p.initial, p.target,
                               None)
        props.append(O.assemble_propagator(sub, u[:, a:b], O.REFERENCE)[0])
    psi, chi = PT.block_boundaries(np.stack(props), p.initial, p.target, dist)
    return first, psi, chi


def test_block_boundaries_match_serial_chain():
    from tests import oracle_api as O
    res = run_ranks(_block_job)
    p, u = O.dense_fixture(4242, dim=5, steps=48, channels=1)
    psi_ref, chi_ref = O.boundary_sweep(p, u, I.balanced_nodes(48, 8), O.REFERENCE)
    for first, psi, chi in res:
        n = len(psi) - 1
        assert np.max(np.abs(psi - psi_ref[first:first + n + 1])) < 1e-11
        assert np.max(np.abs(chi - chi_ref[first:first + n + 1])) < 1e-11


def test_block_nodes_split():
    assert PT.block_nodes(256, 8) == [32 * g for g in range(9)]
    assert PT.block_nodes(7, 3) == [0, 3, 5, 7]
    assert PT.block_nodes(5, 5) == list(range(6))
    with pytest.raises(ValueError):
        PT.block_nodes(4, 5)


def _multi_block_job(rank, world):
    # 12 subintervals, 2 ranks x 3 blocks each (G = 6): the device layout of a 2-GPU run with
    # blocks = 6 (driver.cu: rank r owns blocks [3r, 3r + 3), subintervals [6r, 6r + 6))
    from tests import oracle_api as O
    p, u = O.dense_fixture(4243, dim=4, steps=60, channels=2)
    nodes = I.balanced_nodes(60, 12)
    bn = PT.block_nodes(12, 6)
    first, last = bn[3 * rank], bn[3 * rank + 3]
    props = []
    for n in range(first, last):
        a, b = nodes[n], nodes[n + 1]
        sub = I.ControlProblem(p.model, I.TimeGrid(p.grid.node(a), p.grid.dt, b - a), p.initial, p.target, None)
        props.append(O.assemble_propagator(sub, u[:, a:b], O.REFERENCE)[0])
    psi, chi = PT.block_boundaries(np.stack(props), p.initial, p.target, dist, blocks_per_rank=3)
    return first, psi, chi


def test_multi_block_exchange_matches_serial_chain():
    from tests import oracle_api as O
    res = run_ranks(_multi_block_job)
    p, u = O.dense_fixture(4243, dim=4, steps=60, channels=2)
    psi_ref, chi_ref = O.boundary_sweep(p, u, I.balanced_nodes(60, 12), O.REFERENCE)
    assert [r[0] for r in res] == [0, 6]
    for first, psi, chi in res:
        n = len(psi) - 1
        assert np.max(np.abs(psi - psi_ref[first:first + n + 1])) < 1e-11
        assert np.max(np.abs(chi - chi_ref[first:first + n + 1])) < 1e-11
