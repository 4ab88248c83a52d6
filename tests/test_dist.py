"""World-size-2 gloo tests (CPU) of the multi-GPU data path (paper_2601_22137_b200.dist).

The partition is the native LPT partitioner; the per-rank solve is the fp64
oracle here (the CUDA library on a GPU); the exchange is the real
all_gather_into_tensor.  The sharded result must equal solving the whole
batch in one process, matrix by matrix, with the same global sketch ids.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import prism
from paper_2601_22137_b200 import dist as D
from paper_2601_22137_b200 import workloads as W


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


SHAPES = [(40, 24), (24, 56), (64, 32), (32, 32), (48, 16), (20, 60), (36, 36)]


def _oracle_solve(mats, idx):
    return [torch.tensor(prism.polar(m.double().numpy(), d=2, p=8, tol=1e-10, seed=42, b=i)[0]) for m, i in zip(mats, idx)]


def _oracle_sqrt(mats, idx):
    out = [prism.sqrt_invsqrt(m.double().numpy(), d=2, p=8, tol=1e-10, seed=42, b=i) for m, i in zip(mats, idx)]
    return [torch.tensor(o[0]) for o in out], [torch.tensor(o[1]) for o in out]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mats = [torch.tensor(W.gaussian(m, n, seed=i)) for i, (m, n) in enumerate(SHAPES)]
        outs = D.polar_sharded(mats, solve=_oracle_solve)
        spd = [torch.tensor(W.spd_logspaced(n, 50.0, seed=i)) for i, n in enumerate([16, 24, 20])]
        sq, isq = D.sqrt_invsqrt_sharded(spd, solve=_oracle_sqrt)
        q.put((rank, [o.numpy() for o in outs], [x.numpy() for x in sq], [y.numpy() for y in isq],
               D.lpt_plan([tuple(t.shape) for t in mats], world)))
    finally:
        dist.destroy_process_group()


def test_sharded_polar_and_sqrt_equal_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    # every rank holds every output, identical across ranks
    for a, b in zip(res[0][1], res[1][1]):
        assert np.array_equal(a, b)
    # the plan is deterministic and actually splits the batch
    assert res[0][4] == res[1][4] and set(res[0][4]) == {0, 1}
    # equal to solving the batch in one process with the same global sketch ids
    for i, (m, n) in enumerate(SHAPES):
        ref = prism.polar(W.gaussian(m, n, seed=i), d=2, p=8, tol=1e-10, seed=42, b=i)[0]
        assert np.array_equal(res[0][1][i], ref)
    for i, n in enumerate([16, 24, 20]):
        rs, ri, _ = prism.sqrt_invsqrt(W.spd_logspaced(n, 50.0, seed=i), d=2, p=8, tol=1e-10, seed=42, b=i)
        assert np.array_equal(res[1][2][i], rs) and np.array_equal(res[1][3][i], ri)


def test_lpt_plan_balances_the_1b_muon_batch():
    shapes = W.gpt_1b_shapes()
    for world in (2, 4, 8):
        owner = D.lpt_plan(shapes, world)
        loads = [0.0] * world
        for (m, n), o in zip(shapes, owner):
            loads[o] += __import__("paper_2601_22137_b200").polar_flops_per_iter(m, n, 5, 8)
        assert max(loads) / (sum(loads) / world) < 1.05
