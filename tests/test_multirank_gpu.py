"""Multi-GPU boundary on one B200, through the C ABI.

- An nranks = 1 NCCL communicator made by the library (ifgf_nccl_comm_create)
  and borrowed by a plan: ifgf_apply's in-library ncclAllReduce leaves the field
  unchanged.
- Two processes sharing cuda:0, each with its REAL CUDA rank plan (nranks = 2,
  work-weighted Morton leaf ranges): the partial fields, summed over gloo (two
  ranks on one GPU cannot form an NCCL communicator), equal the one-rank field
  and match the oracle.  The kernels of the two processes never wait on each
  other.
- The captured CUDA graph of an apply replays bitwise the eager launches.
"""
import math
import os
import socket

import numpy as np
import pytest

import oracle
from paper_2010_02857_b200 import inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ifgf():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2010_02857_b200 import ifgf as m
    return m


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda:0")


def test_nccl_comm_one_rank(ifgf):
    c = inputs.CONFIGS["cfg1"]
    pts, a = c.points(), c.densities()
    comm = ifgf.NcclComm(1, 0, 0, ifgf.NcclComm.unique_id())
    with_comm = ifgf.Plan(dev(pts), c.k, c.levels, c.Ps, c.Pang, comm=comm)
    plain = ifgf.Plan(dev(pts), c.k, c.levels, c.Ps, c.Pang)
    got = with_comm.apply(dev(a)).cpu().numpy()
    ref = plain.apply(dev(a)).cpu().numpy()
    assert np.array_equal(got, ref)
    with_comm.stats()
    del with_comm
    comm.close()


def test_comm_rank_mismatch_rejected(ifgf):
    pts = inputs.fibonacci_sphere(1000)
    comm = ifgf.NcclComm(1, 0, 0, ifgf.NcclComm.unique_id())
    with pytest.raises(ifgf.IfgfError) as e:
        ifgf.Plan(dev(pts), 5.0, 4, 3, 5, rank=1, nranks=2, comm=comm)
    assert e.value.code == 1
    comm.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_2010_02857_b200 import ifgf, inputs
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    n, k, D = 60_000, 8 * math.pi, 6
    pts = inputs.fibonacci_sphere(n)
    a = inputs.densities(n, seed=7)
    plan = ifgf.Plan(torch.from_numpy(pts).cuda(), k, D, 3, 5, rank=rank, nranks=world)
    st = plan.stats()
    part = plan.apply(torch.from_numpy(a).cuda()).cpu()
    plan.stats()
    dist.all_reduce(torch.view_as_real(part), op=dist.ReduceOp.SUM)
    q.put((rank, part.numpy(), st["owned_leaf_range"], st["partition_weight"], st["upward_kernel"][D]))
    dist.destroy_process_group()


def test_two_processes_real_rank_plans(ifgf):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n, k, D = 60_000, 8 * math.pi, 6
    pts = inputs.fibonacci_sphere(n)
    a = inputs.densities(n, seed=7)
    full = ifgf.Plan(dev(pts), k, D, 3, 5).apply(dev(a)).cpu().numpy()
    ref = oracle.OraclePlan(pts, k, D, 3, 5).apply(a)
    (_, f0, r0, w0, k0), (_, f1, r1, w1, k1) = res
    assert np.array_equal(f0, f1)  # both ranks hold the summed field
    assert r0[0] == 0 and r0[1] == r1[0] and r1[1] > r1[0]  # contiguous, complete leaf ranges
    assert k0 == 1 and k1 == 1  # the tensor-core K7 on the finest level of both rank plans
    assert abs(w0[0] + w1[0] - w0[1]) <= 1e-9 * w0[1] and max(w0[0], w1[0]) <= 0.6 * w0[1]  # balanced weights
    assert oracle.rel_l2(f0, full) < 1e-13
    assert oracle.rel_l2(f0, ref) <= 1e-11


def test_graph_replay_equals_eager(ifgf):
    n, k, D = 30_000, 6 * math.pi, 5
    pts = inputs.fibonacci_sphere(n)
    a = dev(inputs.densities(n, seed=3))
    b = dev(inputs.densities(n, seed=4))
    g = ifgf.Plan(dev(pts), k, D, 3, 5)
    e = ifgf.Plan(dev(pts), k, D, 3, 5, graph=False)
    out1 = torch.empty(n, dtype=torch.complex128, device="cuda:0")
    out2 = torch.empty_like(out1)
    for _ in range(2):
        g.apply(a, out1)
    g.apply(b, out2)  # new (densities, out) pair: captured again
    g.apply(a, out1)
    torch.cuda.synchronize()
    assert g.stats()["graph_applies"] == 4 and e.stats()["graph_applies"] == 0
    assert torch.equal(out1, e.apply(a))
    assert torch.equal(out2, e.apply(b))
    # profiling switches to eager launches (events around each kernel)
    g.profile_enable(True)
    assert torch.equal(g.apply(a), out1)
    prof = g.profile_read()
    g.profile_enable(False)
    assert g.stats()["graph_applies"] == 4 and prof["upward"][1] > 0
