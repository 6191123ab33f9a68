"""World-size-2 (and 3) CPU test of the multi-GPU host logic over gloo: the
contiguous weighted Morton partition (ifgf_partition, host-only), the per-rank
source restriction (exact by linearity of eq. field1)
and the one exchange step, a sum of the ranks' partial fields over all N targets
(in the product an in-library ncclAllReduce; here a gloo all_reduce of the same
arrays).  Partial fields come from oracle plans that own each rank's Morton
range of leaves."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def morton3(i, j, k, bits=21):
    key = 0
    for b in range(bits):
        key |= ((int(i) >> b) & 1) << (3 * b + 2) | ((int(j) >> b) & 1) << (3 * b + 1) | ((int(k) >> b) & 1) << (3 * b)
    return key


def _worker(rank, world, port, n, D, result_q):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    from paper_2010_02857_b200 import ifgf, inputs
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    k = 4 * math.pi
    pts = inputs.fibonacci_sphere(n)
    a = inputs.densities(n)
    plan = oracle.OraclePlan(pts, k, D, 3, 5)
    leaves = plan.level_boxes(D)
    keys = np.array([morton3(*b[:3]) for b in leaves], dtype=np.uint64)
    order = np.argsort(keys, kind="stable")
    w = leaves[order, 3].astype(np.float64)  # any non-negative weights: points per leaf
    bounds = ifgf.partition(w, world)
    lo = int(keys[order[bounds[rank]]]) if bounds[rank] < len(keys) else 2 ** 64 - 1
    hi = int(keys[order[bounds[rank + 1]]]) if bounds[rank + 1] < len(keys) else 2 ** 64 - 1
    if bounds[rank] == 0:
        lo = 0
    part = oracle.OraclePlan(pts, k, D, 3, 5, owned_morton=(lo, hi)).apply(a)
    info = plan.level_info(D)
    q = np.clip(np.floor((pts - info["x0"]) / info["H"]).astype(np.int64), 0, 2 ** (D - 1) - 1)
    qk = np.array([morton3(*x) for x in q], dtype=np.uint64)
    mine = (qk >= np.uint64(lo)) & (qk < np.uint64(hi))
    field = torch.from_numpy(part.copy())
    dist.all_reduce(torch.view_as_real(field), op=dist.ReduceOp.SUM)
    full = plan.apply(a)
    cover = torch.tensor([int(mine.sum())])
    dist.all_reduce(cover)
    result_q.put((rank, oracle.rel_l2(field.numpy(), full), int(cover.item()), list(bounds)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_sum_equals_full(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n, D = 3000, 4
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, D, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, cover, bounds in res:
        assert err < 1e-13
        assert cover == n  # every source owned by exactly one rank
        assert bounds[0] == 0 and all(bounds[i] <= bounds[i + 1] for i in range(world))
