"""The multi-GPU C ABI on one B200.

* NCCL transport with a 1-rank communicator (prism_nccl_comm_init through the library's
  run-time NCCL): the sharded batch and the row-block solve run their real collectives.
* Several ranks emulated as host threads on the one GPU through the library's real
  multi-GPU code, with a host transport (dist.HostTransport: stream synchronised, copies,
  fixed-order host sum) — no kernel ever waits on another rank's kernel.

Bars (north_star): FP32 <= 1e-5, BF16 <= 2e-2 relative Frobenius error against the fp64
oracle, iterations +-1; sharded outputs bit-identical to the single-GPU batch solve; the
row-block ranks agree on every alpha_k bit for bit (one R, one sketch, one fit).
"""

import threading

import numpy as np
import pytest
import torch

import paper_2601_22137_b200 as P
from oracle import prism
from paper_2601_22137_b200 import dist as D
from paper_2601_22137_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


SHAPES = [(300, 200), (128, 256), (256, 256), (520, 136), (96, 96), (640, 384), (200, 600)]


def _batch(prec):
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    return [torch.tensor(W.gaussian(m, n, seed=60 + i)).to(dt).cuda() for i, (m, n) in enumerate(SHAPES)]


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_sharded_nccl_one_rank_equals_batch(prec):
    mats = _batch(prec)
    tol = 1e-5 if prec == "fp32" else 3e-2
    ref, rref = P.polar(mats, degree=5, tol=tol, precision=prec, matrix_ids=list(range(len(mats))))
    comm = D.Comm()
    try:
        out, rep = D.polar_sharded(mats, comm, nbuckets=3, degree=5, tol=tol, precision=prec)
        torch.cuda.synchronize()
    finally:
        comm.close()
    for a, b in zip(out, ref):
        assert torch.equal(a, b)
    for k in ("iters", "status", "resid"):
        assert torch.equal(rep[k], rref[k])
    assert torch.equal(torch.nan_to_num(rep["alphas"]), torch.nan_to_num(rref["alphas"]))


def test_sharded_three_thread_ranks_equal_batch_and_oracle():
    world = 3
    base = _batch("fp32")
    ref, rref = P.polar(base, degree=5, tol=1e-5, precision="fp32", matrix_ids=list(range(len(base))))
    torch.cuda.synchronize()
    g = D.HostGroup(world)
    res = [None] * world

    def run(r):
        torch.cuda.set_device(0)
        mats = [t.clone() for t in base]          # each rank holds the full batch
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            res[r] = D.polar_sharded(mats, D.HostTransport(g, r), nbuckets=2, handle=P.Handle(), stream=st,
                                     degree=5, tol=1e-5, precision="fp32")
        st.synchronize()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    own, _ = D.shard_plan(SHAPES, world, nbuckets=2)
    assert sorted(set(own)) == list(range(world))
    for r in range(world):
        out, rep = res[r]
        for a, b in zip(out, ref):
            assert torch.equal(a, b)                  # every rank holds every output, bit-identical
        assert torch.equal(rep["iters"], rref["iters"]) and torch.equal(rep["status"], rref["status"])
    for i in (0, 3, 6):
        Qo, ro = prism.polar(base[i].double().cpu().numpy(), d=2, p=8, tol=1e-5, seed=42, b=i)
        assert _rel(res[1][0][i].double().cpu().numpy(), Qo) <= 1e-5


SPD_SIZES = [200, 96, 384, 256, 130, 512]


def _spd_batch():
    return [torch.tensor(W.spd_logspaced(n, 1e2, seed=70 + i)).float().cuda() for i, n in enumerate(SPD_SIZES)]


def test_sqrt_sharded_nccl_one_rank_equals_batch():
    mats = _spd_batch()
    rs, ri, rref = P.sqrt_invsqrt(mats, degree=5, tol=1e-5, precision="fp32", matrix_ids=list(range(len(mats))))
    comm = D.Comm()
    try:
        s, si, rep = D.sqrt_invsqrt_sharded(mats, comm, nbuckets=2, degree=5, tol=1e-5, precision="fp32")
        # one output only: the other array is NULL through the C ABI
        _, si2, _ = D.sqrt_invsqrt_sharded(mats, comm, want_sqrt=False, nbuckets=3, degree=5, tol=1e-5,
                                           precision="fp32")
        torch.cuda.synchronize()
    finally:
        comm.close()
    for a, b, c, d, e in zip(s, rs, si, ri, si2):
        assert torch.equal(a, b) and torch.equal(c, d) and torch.equal(e, d)
    for k in ("iters", "status", "resid"):
        assert torch.equal(rep[k], rref[k])


def test_sqrt_sharded_two_thread_ranks_equal_batch_and_oracle():
    world = 2
    base = _spd_batch()
    rs, ri, rref = P.sqrt_invsqrt(base, degree=5, tol=1e-5, precision="fp32", matrix_ids=list(range(len(base))))
    torch.cuda.synchronize()
    g = D.HostGroup(world)
    res = [None] * world

    def run(r):
        torch.cuda.set_device(0)
        mats = [t.clone() for t in base]
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            res[r] = D.sqrt_invsqrt_sharded(mats, D.HostTransport(g, r), nbuckets=2, handle=P.Handle(), stream=st,
                                            degree=5, tol=1e-5, precision="fp32")
        st.synchronize()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for r in range(world):
        s, si, rep = res[r]
        for a, b, c, d in zip(s, rs, si, ri):
            assert torch.equal(a, b) and torch.equal(c, d)
        assert torch.equal(rep["iters"], rref["iters"])
    for i in (0, 2):
        Xo, Yo, ro = prism.sqrt_invsqrt(base[i].double().cpu().numpy(), d=2, p=8, tol=1e-5, seed=42, b=i)
        assert _rel(res[1][0][i].double().cpu().numpy(), Xo) <= 1e-5
        assert _rel(res[0][1][i].double().cpu().numpy(), Yo) <= 1e-5


@pytest.mark.parametrize("shape,prec,tol,bound", [((1000, 384), "fp32", 1e-5, 1e-5), ((1536, 768), "bf16", 3e-2, 2e-2),
                                                  ((600, 300), "tf32", 1e-2, 5e-3)])
@pytest.mark.parametrize("deg", [3, 5])
def test_rowblock_nccl_one_rank_parity(shape, prec, tol, bound, deg):
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    A = torch.tensor(W.gaussian(*shape, seed=31)).to(dt).cuda()
    comm = D.Comm()
    try:
        Q, rep = D.polar_rowblock(A, comm, m_global=shape[0], row0=0, degree=deg, tol=tol, max_iters=30,
                                  precision=prec)
        torch.cuda.synchronize()
    finally:
        comm.close()
    Qo, ro = prism.polar(A.double().cpu().numpy(), d=1 if deg == 3 else 2, p=8, tol=tol, max_iters=30, seed=42, b=0)
    assert int(rep["status"][0]) == prism.CONVERGED
    assert abs(int(rep["iters"][0]) - ro.iters) <= 1
    assert _rel(Q.double().cpu().numpy(), Qo) <= bound


def _rowblock_threads(A, splits, **opts):
    world = len(splits) - 1
    g = D.HostGroup(world)
    res = [None] * world

    def run(r):
        torch.cuda.set_device(0)
        part = A[splits[r]:splits[r + 1]].contiguous()
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            res[r] = D.polar_rowblock(part, D.HostTransport(g, r), m_global=A.shape[0], row0=splits[r], stream=st,
                                      **opts)
        st.synchronize()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return res


@pytest.mark.parametrize("deg", [3, 5])
def test_rowblock_two_thread_ranks_fp32_parity(deg):
    # n = 640: three 256-row panels in two all-reduced groups; ragged row blocks 600 / 424
    A = torch.tensor(W.gaussian(1024, 640, seed=21)).float().cuda()
    res = _rowblock_threads(A, [0, 600, 1024], degree=deg, tol=1e-5, max_iters=30, precision="fp32")
    Q = torch.cat([res[0][0], res[1][0]]).double().cpu().numpy()
    r0, r1 = res[0][1], res[1][1]
    assert int(r0["iters"][0]) == int(r1["iters"][0])
    it = int(r0["iters"][0])
    assert torch.equal(r0["alphas"][0, :it], r1["alphas"][0, :it])      # one R, one fit: identical alphas
    Qo, ro = prism.polar(A.double().cpu().numpy(), d=1 if deg == 3 else 2, p=8, tol=1e-5, max_iters=30, seed=42, b=0)
    assert abs(it - ro.iters) <= 1
    assert _rel(Q, Qo) <= 1e-5


@pytest.mark.parametrize("prec,tol,bound", [("bf16", 3e-2, 2e-2), ("tf32", 1e-2, 5e-3)])
def test_rowblock_four_thread_ranks_ragged(prec, tol, bound):
    # four ranks, ragged cuts (one rank holds fewer rows than a 256-row tile), n = 768:
    # three panels, pipelined panel groups, every rank's alphas bit-identical
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    A = torch.tensor(W.gaussian(1100, 768, seed=23)).to(dt).cuda()
    cuts = [0, 300, 555, 700, 1100]
    res = _rowblock_threads(A, cuts, degree=5, tol=tol, max_iters=30, precision=prec)
    it = [int(res[r][1]["iters"][0]) for r in range(4)]
    assert len(set(it)) == 1
    for r in range(1, 4):
        assert torch.equal(res[r][1]["alphas"][0, :it[0]], res[0][1]["alphas"][0, :it[0]])
    Q = torch.cat([res[r][0] for r in range(4)]).double().cpu().numpy()
    Qo, ro = prism.polar(A.double().cpu().numpy(), d=2, p=8, tol=tol, max_iters=30, seed=42, b=0)
    assert abs(it[0] - ro.iters) <= 1
    assert _rel(Q, Qo) <= bound


def test_sharded_four_thread_ranks_three_buckets_reports():
    world = 4
    base = _batch("bf16")
    ref, rref = P.polar(base, degree=5, tol=3e-2, precision="bf16", matrix_ids=list(range(len(base))))
    torch.cuda.synchronize()
    g = D.HostGroup(world)
    res = [None] * world

    def run(r):
        torch.cuda.set_device(0)
        mats = [t.clone() for t in base]
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            res[r] = D.polar_sharded(mats, D.HostTransport(g, r), nbuckets=3, handle=P.Handle(), stream=st,
                                     degree=5, tol=3e-2, precision="bf16")
        st.synchronize()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for r in range(world):
        out, rep = res[r]
        for a, b in zip(out, ref):
            assert torch.equal(a, b)
        for k in ("iters", "status", "resid"):
            assert torch.equal(rep[k], rref[k])
        assert torch.equal(torch.nan_to_num(rep["alphas"]), torch.nan_to_num(rref["alphas"]))


@pytest.mark.slow
def test_config3_8192_rowblock_two_ranks_vs_oracle():
    """configs[3] at full size: 8192^2 BF16 split by rows over 2 emulated ranks, against one
    fp64 oracle solve of the whole matrix (minutes of host BLAS)."""
    m = n = 8192
    A = torch.tensor(W.gaussian(m, n, seed=3000)).to(torch.bfloat16).cuda()
    res = _rowblock_threads(A, [0, m // 2, m], degree=5, tol=3e-2, max_iters=25, precision="bf16")
    it = [int(res[r][1]["iters"][0]) for r in range(2)]
    assert it[0] == it[1] and int(res[0][1]["status"][0]) == prism.CONVERGED
    assert torch.equal(res[0][1]["alphas"][0, :it[0]], res[1][1]["alphas"][0, :it[0]])
    Q = torch.cat([res[0][0], res[1][0]]).double().cpu().numpy()
    Qo, ro = prism.polar(A.double().cpu().numpy(), d=2, p=8, tol=3e-2, max_iters=25, seed=42, b=0)
    assert abs(it[0] - ro.iters) <= 1
    assert _rel(Q, Qo) <= 2e-2
