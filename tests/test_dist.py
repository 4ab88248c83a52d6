"""World-size-2 gloo tests (CPU) of the multi-GPU path's host logic.

The library's multi-GPU entry points (prism_polar_sharded, prism_polar_rowblock) need a
GPU; on CPU these tests check what they are built on, with the fp64 oracle as the per-rank
solver and gloo as the exchange:

* sharded batch: prism_shard_plan is identical on every rank, covers every matrix once and
  balances the load; solving each rank's share with global sketch ids and broadcasting
  bucket by bucket from the owners (the library's protocol) reproduces the single-process
  solve of the whole batch bit for bit.
* row block: with the library's packed Gram layout (prism_rowblock_layout), partial Grams
  of the ranks' row blocks summed by all-reduce give X^T X; one alpha fit per iteration on
  that R (identical on every rank) and the per-rank update Y_r = X_r R,
  X_r + Y_r/2 + a Y_r R (no R^2) reproduce the oracle's polar iteration.
"""

import math
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import prism
from oracle.philox import gaussian_sketch
from paper_2601_22137_b200 import dist as D
from paper_2601_22137_b200 import workloads as W


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


SHAPES = [(40, 24), (24, 56), (64, 32), (32, 32), (48, 16), (20, 60), (36, 36), (72, 24)]


def _run(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=fn, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        r, v = q.get(timeout=600)
        res[r] = v
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _sharded_worker(rank, world, port, q):
    _init(rank, world, port)
    try:
        own, bk = D.shard_plan(SHAPES, world, nbuckets=2)
        plans = [None] * world
        dist.all_gather_object(plans, (own, bk))
        mats = [W.gaussian(m, n, seed=i) for i, (m, n) in enumerate(SHAPES)]
        outs = [torch.zeros(m, n, dtype=torch.float64) for (m, n) in SHAPES]
        for i, A in enumerate(mats):
            if own[i] == rank:   # this rank's share, global index i as the sketch id
                outs[i] = torch.tensor(prism.polar(A, d=2, p=8, tol=1e-10, seed=42, b=i)[0])
        for j in range(2):       # owners broadcast each bucket (prism_polar_sharded_tr's order)
            for i in range(len(SHAPES)):
                if bk[i] == j:
                    dist.broadcast(outs[i], src=own[i])
        q.put((rank, (plans, [o.numpy() for o in outs])))
    finally:
        dist.destroy_process_group()


def test_sharded_plan_and_exchange_equal_single_process():
    res = _run(_sharded_worker)
    plans0, outs0 = res[0]
    plans1, outs1 = res[1]
    assert plans0[0] == plans0[1] == plans1[0]          # identical plan on every rank
    own, bk = plans0[0]
    assert sorted(set(own)) == [0, 1] and set(bk) <= {0, 1}
    cost = [D.B.polar_flops_per_iter(m, n) for (m, n) in SHAPES]
    loads = [sum(c for c, o in zip(cost, own) if o == r) for r in range(2)]
    assert max(loads) - min(loads) <= max(cost)          # LPT bound
    for i, (m, n) in enumerate(SHAPES):
        ref = prism.polar(W.gaussian(m, n, seed=i), d=2, p=8, tol=1e-10, seed=42, b=i)[0]
        assert np.array_equal(outs0[i], ref) and np.array_equal(outs1[i], ref)


def _pack(G, off):
    n = G.shape[0]
    buf = np.zeros(off[-1])
    for t in range(len(off) - 1):
        r0 = 256 * t
        h, w = min(256, n - r0), n - r0
        buf[off[t]:off[t] + h * w] = np.triu(G[r0:r0 + h, r0:], k=0).reshape(-1) if h == w else \
            np.where(np.arange(w)[None, :] >= np.arange(h)[:, None], G[r0:r0 + h, r0:], 0.0).reshape(-1)
    return buf


def _unpack(buf, off, n):
    G = np.zeros((n, n))
    for t in range(len(off) - 1):
        r0 = 256 * t
        h, w = min(256, n - r0), n - r0
        G[r0:r0 + h, r0:] = buf[off[t]:off[t] + h * w].reshape(h, w)
    U = np.triu(G)
    return U + np.triu(G, 1).T


M_RB, N_RB = 640, 300   # two 256-row panels (256 x 300, 44 x 44)


def _rowblock_worker(rank, world, port, q):
    _init(rank, world, port)
    try:
        A = W.gaussian(M_RB, N_RB, seed=5)
        rows = np.array_split(np.arange(M_RB), world)[rank]
        X = A[rows].copy()
        fro2 = torch.tensor([float(np.sum(X * X))], dtype=torch.float64)
        dist.all_reduce(fro2)
        X /= math.sqrt(float(fro2))
        off, ge = D.rowblock_layout(N_RB, 2)
        lo, hi, aT = prism.interval(2)
        I = np.eye(N_RB)
        alphas, k = [], 0
        while True:
            buf = torch.tensor(_pack(X.T @ X, off))
            dist.all_reduce(buf)                          # summed packed partial Grams
            R = I - _unpack(buf.numpy(), off, N_RB)
            if np.linalg.norm(R) <= 1e-10 * math.sqrt(N_RB) or k == 30:
                break
            S = gaussian_sketch(42, 0, k, 8, N_RB)        # matrix id 0: the same S_k on every rank
            a, _ = prism.fit_alpha(R, 2, prism.FIT_SKETCHED, S, lo, hi, aT)
            alphas.append(a)
            Y = X @ R                                     # no R^2, no second collective
            X = (X + 0.5 * Y) + a * (Y @ R)
            k += 1
        q.put((rank, (rows, X, alphas, k, off, ge)))
    finally:
        dist.destroy_process_group()


def test_rowblock_algorithm_and_packed_layout_reproduce_oracle():
    res = _run(_rowblock_worker)
    off, ge = res[0][4], res[0][5]
    assert off[1] == 256 * N_RB and off[2] == off[1] + 44 * 44 and ge == [1, 2]
    assert res[0][2] == res[1][2] and res[0][3] == res[1][3]      # identical alphas and iteration counts
    Q = np.zeros((M_RB, N_RB))
    for r in range(2):
        Q[res[r][0]] = res[r][1]
    Qo, ro = prism.polar(W.gaussian(M_RB, N_RB, seed=5), d=2, p=8, tol=1e-10, max_iters=30, seed=42, b=0)
    assert res[0][3] == ro.iters
    # alpha_k agree to rounding; the last fit sees ||R|| ~ 1e-6, where the quartic's
    # coefficients are ~1e-30 and the fp64 rounding of R (summation order) moves alpha ~1e-9
    assert np.allclose(res[0][2][:-1], ro.alphas[:-1], rtol=1e-12, atol=1e-14)
    assert abs(res[0][2][-1] - ro.alphas[-1]) <= 1e-6
    assert np.linalg.norm(Q - Qo) / np.linalg.norm(Qo) <= 1e-12


def test_layout_groups_balance_tiles():
    off, ge = D.rowblock_layout(8192, 4)
    T = 32
    assert len(off) == T + 1 and off[-1] == sum(256 * (8192 - 256 * t) for t in range(T))
    tiles = [T - t for t in range(T)]
    starts = [0] + ge[:-1]
    sums = [sum(tiles[a:b]) for a, b in zip(starts, ge)]
    assert ge[-1] == T and max(sums) - min(sums) <= T
