"""End-to-end parity of the CUDA path (through the C ABI) with the fp64 oracle.

Bounds (BASELINE.json north_star, refined per input class in SURVEY §8(c)):
relative Frobenius error <= 1e-5 in FP32 (3xTF32) mode and <= 2e-2 in BF16
mode, iteration count to tolerance within +-1.  Inputs are the exact values
stored in the device dtype, read back as fp64 for the oracle.
"""

import numpy as np
import pytest
import torch

import paper_2601_22137_b200 as P
from oracle import prism
from paper_2601_22137_b200 import workloads as W

pytestmark = pytest.mark.gpu

DT = {"bf16": torch.bfloat16, "fp32": torch.float32, "tf32": torch.float32}


def _dev(A, prec):
    t = torch.tensor(A).to(DT[prec]).cuda()
    return t, t.double().cpu().numpy()


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _polar_pair(A, prec, deg, tol, max_iters=30, seed=42, warmup=0, fit="sketched"):
    At, Aq = _dev(A, prec)
    Q, rep = P.polar([At], degree=deg, max_iters=max_iters, tol=tol, seed=seed, precision=prec,
                     warmup_iters=warmup, fit=fit)
    torch.cuda.synchronize()
    Qo, ro = prism.polar(Aq, d=1 if deg == 3 else 2, p=8, tol=tol, max_iters=max_iters, seed=seed,
                         warmup=warmup, fit=fit)
    return Q[0].double().cpu().numpy(), {k: v[0].cpu().numpy() for k, v in rep.items()}, Qo, ro


@pytest.mark.parametrize("shape", [(256, 128), (128, 256), (300, 200), (1000, 700), (520, 520)])
@pytest.mark.parametrize("deg", [3, 5])
def test_polar_fp32_parity(shape, deg):
    A = W.gaussian(*shape, seed=shape[0] + deg)
    Q, rep, Qo, ro = _polar_pair(A, "fp32", deg, tol=1e-5)
    assert int(rep["status"]) == prism.CONVERGED and ro.status == prism.CONVERGED
    assert abs(int(rep["iters"]) - ro.iters) <= 1
    assert _rel(Q, Qo) <= 1e-5
    n = min(len(ro.alphas), int(rep["iters"]))
    assert np.max(np.abs(rep["alphas"][:n] - np.array(ro.alphas[:n]))) <= 1e-3


@pytest.mark.parametrize("kind", ["htmp", "logspaced"])
def test_polar_fp32_parity_spectra(kind):
    A = W.htmp(600, 384, 0.5, seed=3) if kind == "htmp" else W.logspaced(600, 384, 1e-3, seed=3)
    Q, rep, Qo, ro = _polar_pair(A, "fp32", 5, tol=1e-5, max_iters=40)
    assert abs(int(rep["iters"]) - ro.iters) <= 1
    assert _rel(Q, Qo) <= (1e-5 if kind == "htmp" else 5e-5)   # SURVEY §8(c) log-uniform row


@pytest.mark.parametrize("shape,deg", [((768, 768), 5), ((3072, 768), 5), ((768, 2304), 3), ((768, 3072), 5)])
def test_polar_bf16_parity_gpt2_shapes(shape, deg):
    A = W.gaussian(*shape, seed=7)
    Q, rep, Qo, ro = _polar_pair(A, "bf16", deg, tol=3e-2)
    assert int(rep["status"]) == prism.CONVERGED
    assert abs(int(rep["iters"]) - ro.iters) <= 1
    assert _rel(Q, Qo) <= 2e-2


def test_polar_tf32_parity():
    A = W.gaussian(300, 200, seed=5)
    Q, rep, Qo, ro = _polar_pair(A, "tf32", 5, tol=1e-2)
    assert abs(int(rep["iters"]) - ro.iters) <= 1
    assert _rel(Q, Qo) <= 5e-3


def test_polar_taylor_and_warmup_modes():
    A = W.gaussian(200, 136, seed=9)
    Q, rep, Qo, ro = _polar_pair(A, "fp32", 5, tol=1e-5, fit="taylor")
    assert int(rep["iters"]) == ro.iters and _rel(Q, Qo) <= 1e-5
    assert np.all(rep["alphas"][: ro.iters] == 0.375)
    Q, rep, Qo, ro = _polar_pair(A, "fp32", 3, tol=1e-5, warmup=3)
    assert np.all(rep["alphas"][:3] == 1.0) and abs(int(rep["iters"]) - ro.iters) <= 1
    assert _rel(Q, Qo) <= 1e-5


def test_polar_equal_sigma_closed_form():
    # A = c Q: R_k = l_k I, closed-form trajectory (tests/test_oracle_prism.py); d=2, s=256 -> 5 iterations
    A = W.equal_sigma(512, 256, 2.5, seed=4)
    Q, rep, Qo, ro = _polar_pair(A, "fp32", 5, tol=1e-6)
    assert int(rep["iters"]) == ro.iters
    assert _rel(Q, A / 2.5) <= 1e-5


@pytest.mark.parametrize("n,kappa,deg", [(256, 1e2, 5), (200, 1e2, 3), (640, 1e2, 5), (384, 1e4, 5)])
def test_sqrt_fp32_parity(n, kappa, deg):
    A = W.spd_logspaced(n, kappa, seed=n)
    At, Aq = _dev(A, "fp32")
    tol = 1e-5 if kappa <= 1e2 else 3e-5
    X, Y, rep = P.sqrt_invsqrt([At], degree=deg, max_iters=40, tol=tol, seed=42, precision="fp32")
    torch.cuda.synchronize()
    Xo, Yo, ro = prism.sqrt_invsqrt(Aq, d=1 if deg == 3 else 2, p=8, tol=tol, max_iters=40, seed=42)
    assert int(rep["status"][0]) == prism.CONVERGED
    assert abs(int(rep["iters"][0]) - ro.iters) <= 1
    assert _rel(X[0].double().cpu().numpy(), Xo) <= 1e-5
    # inverse root: cond(A^{-1/2}) ~ kappa^{1/2} amplifies; SURVEY §8(c) rows
    assert _rel(Y[0].double().cpu().numpy(), Yo) <= (1e-5 if kappa <= 1e2 else 3e-4)


def test_batch_mixed_shapes_equals_single_solves():
    shapes = [(300, 200), (128, 256), (256, 256), (520, 136)]
    mats = [torch.tensor(W.gaussian(m, n, seed=i)).float().cuda() for i, (m, n) in enumerate(shapes)]
    Qb, rb = P.polar(mats, degree=5, tol=1e-5, precision="fp32")
    torch.cuda.synchronize()
    for i, t in enumerate(mats):
        Qs, rs = P.polar([t], degree=5, tol=1e-5, precision="fp32", matrix_ids=[i])
        torch.cuda.synchronize()
        assert torch.equal(Qs[0], Qb[i])                      # same kernels, same sketch stream -> same bits
        assert int(rs["iters"][0]) == int(rb["iters"][i])
        Qo, ro = prism.polar(t.double().cpu().numpy(), d=2, p=8, tol=1e-5, seed=42, b=i)
        assert _rel(Qb[i].double().cpu().numpy(), Qo) <= 1e-5


def test_split_chain_parity_and_batch_bits():
    # s >= 1024 takes the N = 32 chain with K split over a CTA cluster (split factor s/512,
    # capped at 4); smaller s the transposed chain.  One batch mixes factors 4, 2 and the
    # transposed form: each matrix must come out bit-identical to its single solve (the
    # launch cluster is the batch maximum; smaller factors leave empty slices), and the
    # s = 1024 one within the FP32 bound of the oracle.
    shapes = [(2048, 2048), (1536, 1024), (300, 200)]
    mats = [torch.tensor(W.gaussian(m, n, seed=10 + i)).float().cuda() for i, (m, n) in enumerate(shapes)]
    Qb, rb = P.polar(mats, degree=5, tol=1e-5, precision="fp32")
    torch.cuda.synchronize()
    for i, t in enumerate(mats):
        Qs, rs = P.polar([t], degree=5, tol=1e-5, precision="fp32", matrix_ids=[i])
        torch.cuda.synchronize()
        assert torch.equal(Qs[0], Qb[i])
        assert int(rs["iters"][0]) == int(rb["iters"][i])
    Qo, ro = prism.polar(mats[1].double().cpu().numpy(), d=2, p=8, tol=1e-5, seed=42, b=1)
    assert _rel(Qb[1].double().cpu().numpy(), Qo) <= 1e-5
    assert abs(int(rb["iters"][1]) - ro.iters) <= 1


def test_chain_slices_sequential_equals_cluster_split():
    # A matrix's chain K-slices (s >= 1024) are either spread over a CTA cluster (the
    # batch has fewer row tiles than SMs) or run in order by one CTA (it has enough):
    # both sum the slices in the same order, so the results must be bit-identical.
    big = torch.tensor(W.gaussian(2048, 2048, seed=77)).float().cuda()
    small = [torch.tensor(W.gaussian(256, 256, seed=100 + i)).float().cuda() for i in range(150)]
    Qa, ra = P.polar([big], degree=5, tol=1e-5, precision="fp32", matrix_ids=[0])   # 8 tiles: cluster of 4
    Qb, rb = P.polar([big] + small, degree=5, tol=1e-5, precision="fp32")          # 158 tiles: one CTA
    torch.cuda.synchronize()
    assert int(ra["iters"][0]) == int(rb["iters"][0])
    assert torch.equal(Qa[0], Qb[0])


def test_host_path_pipelined_equals_device_path():
    # prism_polar_host: three different batches submitted back to back (two staging
    # slots, so the third reuses the first slot while the pipeline is busy); each result
    # must be bit-identical to the device-path solve of the same inputs
    shapes = [(300, 200), (128, 256), (520, 136)]
    batches = [[torch.tensor(W.gaussian(m, n, seed=100 * c + i)).to(torch.bfloat16).pin_memory()
                for i, (m, n) in enumerate(shapes)] for c in range(3)]
    h = P.Handle()
    outs = [P.polar_host(b, degree=5, tol=3e-2, precision="bf16", handle=h)[0] for b in batches]
    torch.cuda.synchronize()
    for b, o in zip(batches, outs):
        ref, _ = P.polar([t.cuda() for t in b], degree=5, tol=3e-2, precision="bf16")
        torch.cuda.synchronize()
        for x, y in zip(o, ref):
            assert torch.equal(x, y.cpu())
    A = [torch.tensor(W.spd_logspaced(96, 1e2, seed=7)).float().pin_memory()]
    sq, isq, _ = P.sqrt_invsqrt_host(A, degree=5, tol=1e-5, precision="fp32", handle=h)
    torch.cuda.synchronize()
    rs, ri, _ = P.sqrt_invsqrt([A[0].cuda()], degree=5, tol=1e-5, precision="fp32")
    torch.cuda.synchronize()
    assert torch.equal(sq[0], rs[0].cpu()) and torch.equal(isq[0], ri[0].cpu())


def test_edge_cases():
    # zero input, single column, p = s, max_iters stop, NaN input
    z = torch.zeros(64, 32, device="cuda")
    one = torch.tensor(W.gaussian(40, 1, seed=1)).float().cuda()
    small = torch.tensor(W.gaussian(16, 8, seed=2)).float().cuda()
    nan = torch.tensor(W.gaussian(48, 24, seed=3)).float().cuda()
    nan[3, 5] = float("nan")
    Q, rep = P.polar([z, small, nan], degree=5, tol=1e-5, precision="fp32", sketch_size=8)
    Q1, rep1 = P.polar([one], degree=5, tol=1e-5, precision="fp32", sketch_size=1)
    torch.cuda.synchronize()
    st = rep["status"].cpu().tolist()
    assert st[0] == prism.ZERO_INPUT and torch.all(Q[0] == 0)
    assert st[1] == prism.CONVERGED
    assert st[2] == prism.NONFINITE
    assert int(rep1["status"][0]) == prism.CONVERGED
    v = one.double().cpu().numpy()
    assert _rel(Q1[0].double().cpu().numpy(), v / np.linalg.norm(v)) <= 1e-6
    Qo, ro = prism.polar(small.double().cpu().numpy(), d=2, p=8, tol=1e-5, seed=42, b=1)
    assert _rel(Q[1].double().cpu().numpy(), Qo) <= 1e-5
    A = torch.tensor(W.logspaced(96, 64, 1e-4, seed=4)).float().cuda()
    Q, rep = P.polar([A], degree=5, tol=1e-9, max_iters=3, precision="fp32")
    torch.cuda.synchronize()
    assert int(rep["status"][0]) == prism.MAX_ITERS and int(rep["iters"][0]) == 3


def test_gpt2_mixed_batch_exactly_as_benchmarked():
    """configs[1] at full size, the exact batch bench.py times (muon_batch(seed=1,
    kind="mixed"): even members Gaussian MP, odd members HTMP-like kappa = 0.5), in one BF16
    call with the bench's options: every one of the 48 matrices against the fp64 oracle.
    MP members: <= 2e-2 and +-1 iteration (north_star).  HTMP members: SURVEY §8(c) gives the
    kappa = 0.5 class no separate row; they are held to the same bar (measured 5.4e-3 -
    9.4e-3, iterations equal) and the maximum is reported by bench.py (sampled rel_err)."""
    shapes = W.gpt2_small_shapes()
    mats_np = W.muon_batch(shapes, seed=1, kind="mixed")
    mats = [torch.tensor(a).to(torch.bfloat16).cuda() for a in mats_np]
    Q, rep = P.polar(mats, degree=5, max_iters=20, tol=3e-2, sketch_size=8, seed=42, precision="bf16",
                     matrix_ids=list(range(48)))
    torch.cuda.synchronize()
    assert torch.all(rep["status"] == prism.CONVERGED)
    errs = {"mp": [], "htmp": []}
    for i in range(48):
        Qo, ro = prism.polar(mats[i].double().cpu().numpy(), d=2, p=8, tol=3e-2, max_iters=20, seed=42, b=i)
        assert abs(int(rep["iters"][i]) - ro.iters) <= 1, (i, int(rep["iters"][i]), ro.iters)
        e = _rel(Q[i].double().cpu().numpy(), Qo)
        errs["mp" if i % 2 == 0 else "htmp"].append(e)
        assert e <= 2e-2, (i, e)
    print("gpt2 mixed batch: max rel err MP %.3e, HTMP %.3e" % (max(errs["mp"]), max(errs["htmp"])))


@pytest.mark.gpu
def test_sqrt_caller_outputs_equal_fresh_outputs():
    mats = [torch.tensor(W.spd_logspaced(s, 1e2, seed=900 + s)).float().cuda() for s in (96, 300)]
    X, Y, _ = P.sqrt_invsqrt(mats, degree=5, tol=1e-5, max_iters=30, precision="fp32")
    osq = [torch.full_like(m, float("nan")) for m in mats]
    oisq = [torch.full_like(m, float("nan")) for m in mats]
    X2, Y2, _ = P.sqrt_invsqrt(mats, degree=5, tol=1e-5, max_iters=30, precision="fp32", out_sqrt=osq,
                               out_invsqrt=oisq)
    torch.cuda.synchronize()
    assert X2[1] is osq[1] and Y2[0] is oisq[0]
    for a, b in zip(X + Y, X2 + Y2):
        assert torch.equal(a, b)


@pytest.mark.gpu
def test_early_square_gemm_is_bit_identical():
    """The square GEMM whose mainloop runs under k_alpha (bf16 polar batches <= 16 matrices:
    only its epilogue waits for alpha) computes exactly what the waiting launch of a larger
    batch computes: the same three matrices solved alone (early) and inside a batch of 17
    (waiting) come out bit for bit equal."""
    shapes = [(1024, 1024), (768, 2304), (3072, 768)]
    mats = [torch.tensor(W.gaussian(m, n, seed=7 + i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
    filler = [torch.tensor(W.gaussian(256, 128, seed=50 + i)).to(torch.bfloat16).cuda() for i in range(14)]
    Qe, re_ = P.polar(mats, degree=5, tol=3e-2, max_iters=20, matrix_ids=[0, 1, 2])
    Qw, rw = P.polar(mats + filler, degree=5, tol=3e-2, max_iters=20, matrix_ids=list(range(17)))
    torch.cuda.synchronize()
    assert torch.equal(re_["iters"], rw["iters"][:3])
    for a, b in zip(Qe, Qw[:3]):
        assert torch.equal(a, b)


@pytest.mark.parametrize("p", [5, 16, 32])
@pytest.mark.parametrize("deg", [3, 5])
def test_polar_sketch_sizes_beyond_8(p, deg):
    """Sketch sizes other than the default 8 ("as small as 5"; Theorem 2, asks
    for more): p > 8 runs the chain in column chunks of 8 whose <Va, Vb> partials k_alpha sums
    — the same quartic as one wide chain (the products R^i S^T are column-separable)."""
    A = W.gaussian(600, 300, seed=40 + p)
    At, Aq = _dev(A, "fp32")
    Q, rep = P.polar([At], degree=deg, max_iters=30, tol=1e-5, seed=42, precision="fp32", sketch_size=p)
    torch.cuda.synchronize()
    Qo, ro = prism.polar(Aq, d=1 if deg == 3 else 2, p=p, tol=1e-5, max_iters=30, seed=42)
    assert int(rep["status"][0]) == prism.CONVERGED
    assert abs(int(rep["iters"][0]) - ro.iters) <= 1
    assert _rel(Q[0].double().cpu().numpy(), Qo) <= 1e-5
    n = min(len(ro.alphas), int(rep["iters"][0]))
    assert np.max(np.abs(rep["alphas"][0, :n].cpu().numpy() - np.array(ro.alphas[:n]))) <= 1e-3


@pytest.mark.parametrize("p", [16, 32])
def test_sqrt_and_bf16_sketch_16_32(p):
    A = W.spd_logspaced(384, 1e2, seed=p)
    At, Aq = _dev(A, "fp32")
    X, Y, rep = P.sqrt_invsqrt([At], degree=5, max_iters=40, tol=1e-5, seed=42, precision="fp32", sketch_size=p)
    torch.cuda.synchronize()
    Xo, Yo, ro = prism.sqrt_invsqrt(Aq, d=2, p=p, tol=1e-5, max_iters=40, seed=42)
    assert abs(int(rep["iters"][0]) - ro.iters) <= 1
    assert _rel(X[0].double().cpu().numpy(), Xo) <= 1e-5 and _rel(Y[0].double().cpu().numpy(), Yo) <= 1e-5
    G = W.gaussian(768, 2304, seed=p)
    Gt, Gq = _dev(G, "bf16")
    Q, rq = P.polar([Gt], degree=5, max_iters=20, tol=3e-2, seed=42, precision="bf16", sketch_size=p)
    torch.cuda.synchronize()
    Qo, ro = prism.polar(Gq, d=2, p=p, tol=3e-2, max_iters=20, seed=42)
    assert abs(int(rq["iters"][0]) - ro.iters) <= 1
    assert _rel(Q[0].double().cpu().numpy(), Qo) <= 2e-2


def test_folded_normalisation_edge_cases():
    """BF16 / TF32 polar fold the normalisation X_0 = A/||A||_F into iteration 0's Gram and
    apply when A and Q are TMA-legal, with X[0] = Q.  Checked here: a batch
    mixing folded and unfolded matrices (misaligned leading dimension) against the oracle and
    against single solves bit for bit; in place (Q = A); a solve that stops at k = 0 (one
    column: X_0 is already orthonormal); a zero matrix into a non-zeroed output."""
    # mixed: 300 columns bf16 with lda 300 (600 B: not a 16-B multiple -> unfolded) + aligned
    base = torch.tensor(W.gaussian(256, 300, seed=91)).to(torch.bfloat16).cuda()
    aligned = [torch.tensor(W.gaussian(m, n, seed=92 + i)).to(torch.bfloat16).cuda()
               for i, (m, n) in enumerate([(512, 256), (256, 640)])]
    mats = [base] + aligned
    Q, rep = P.polar(mats, degree=5, tol=3e-2, max_iters=20, precision="bf16")
    torch.cuda.synchronize()
    for i, t in enumerate(mats):
        Qs, rs = P.polar([t], degree=5, tol=3e-2, max_iters=20, precision="bf16", matrix_ids=[i])
        torch.cuda.synchronize()
        assert torch.equal(Qs[0], Q[i]) and int(rs["iters"][0]) == int(rep["iters"][i])
        Qo, ro = prism.polar(t.double().cpu().numpy(), d=2, p=8, tol=3e-2, max_iters=20, seed=42, b=i)
        assert abs(int(rep["iters"][i]) - ro.iters) <= 1 and _rel(Q[i].double().cpu().numpy(), Qo) <= 2e-2
    # in place: Q aliases A
    A = torch.tensor(W.gaussian(768, 384, seed=95)).to(torch.bfloat16).cuda()
    A0 = A.clone()
    Qn, rn = P.polar([A0], degree=5, tol=3e-2, max_iters=20, precision="bf16")
    Qi, ri = P.polar([A], out=[A], degree=5, tol=3e-2, max_iters=20, precision="bf16")
    torch.cuda.synchronize()
    assert Qi[0] is A and torch.equal(A, Qn[0])
    # stop at k = 0: one column (lda 8 elements = 16 B through a strided view) and a zero matrix
    buf = torch.zeros(40, 8, dtype=torch.bfloat16, device="cuda")
    buf[:, 0] = torch.tensor(W.gaussian(40, 1, seed=96)[:, 0]).to(torch.bfloat16)
    col = buf[:, :1]
    obuf = torch.full((40, 8), float("nan"), dtype=torch.bfloat16, device="cuda")
    zero = torch.zeros(64, 32, dtype=torch.bfloat16, device="cuda")
    ozero = torch.full((64, 32), float("nan"), dtype=torch.bfloat16, device="cuda")
    Qc, rc = P.polar([col, zero], out=[obuf[:, :1], ozero], degree=5, tol=3e-2, max_iters=20, precision="bf16",
                     sketch_size=1)
    torch.cuda.synchronize()
    assert int(rc["iters"][0]) == 0 and int(rc["status"][0]) == prism.CONVERGED
    v = col.double().cpu().numpy()
    assert _rel(Qc[0].double().cpu().numpy(), v / np.linalg.norm(v)) <= 1e-2
    assert int(rc["status"][1]) == prism.ZERO_INPUT and torch.all(Qc[1] == 0)
    # TF32 folds too
    T = torch.tensor(W.gaussian(300, 200, seed=97)).float().cuda()
    Qt, rt = P.polar([T], degree=5, tol=1e-2, max_iters=30, precision="tf32")
    torch.cuda.synchronize()
    Qo, ro = prism.polar(T.double().cpu().numpy(), d=2, p=8, tol=1e-2, max_iters=30, seed=42)
    assert abs(int(rt["iters"][0]) - ro.iters) <= 1 and _rel(Qt[0].double().cpu().numpy(), Qo) <= 5e-3


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["sqrt", "db_newton"])
def test_single_output_requests_device_and_host(kind):
    """Either output of the coupled kinds may be omitted (NULL in the C-ABI): the requested one
    must equal the two-output solve bit for bit, through the device and the host entry points."""
    mats = [torch.tensor(W.spd_logspaced(s, 1e2, seed=950 + s)).float().cuda() for s in (96, 260)]
    host = [m.cpu().pin_memory() for m in mats]
    dev_f, host_f = (P.sqrt_invsqrt, P.sqrt_invsqrt_host) if kind == "sqrt" else (P.db_newton, P.db_newton_host)
    kw = dict(tol=1e-5, max_iters=40)
    X, Y, _ = dev_f(mats, **kw)
    X1, Y1, _ = dev_f(mats, want_invsqrt=False, **kw)
    X2, Y2, _ = dev_f(mats, want_sqrt=False, **kw)
    Xh1, Yh1, _ = host_f(host, want_invsqrt=False, **kw)
    Xh2, Yh2, _ = host_f(host, want_sqrt=False, **kw)
    torch.cuda.synchronize()
    assert not Y1 and not X2 and not Yh1 and not Xh2
    for i in range(len(mats)):
        assert torch.equal(X1[i], X[i]) and torch.equal(Y2[i], Y[i])
        assert torch.equal(Xh1[i], X[i].cpu()) and torch.equal(Yh2[i], Y[i].cpu())


@pytest.mark.gpu
def test_sqrt_divergence_status_and_residual_history():
    """DIVERGED on the device (5 consecutive increases of ||R_k||_F): PRISM-3 with the
    Taylor coefficient on a 64 x 64 diagonal with a negative eigenvalue, whose iterates are a
    scalar recurrence per eigenvalue (tests/test_oracle_prism.py pins the same case): the
    residuals fall, then grow from k = 5, and the solve stops at k = 9."""
    lam = [1.0, 0.5, -0.03, 0.2] * 16
    c = float(np.sqrt(np.sum(np.square(lam))))
    x, y = np.array(lam) / c, np.ones(64)
    hist = []
    for _ in range(10):
        r = 1.0 - y * x
        hist.append(float(np.linalg.norm(r)) / 8.0)
        x, y = x * (1.0 + 0.5 * r), (1.0 + 0.5 * r) * y
    A = torch.diag(torch.tensor(lam, dtype=torch.float32)).cuda()
    X, Y, rep = P.sqrt_invsqrt([A], degree=3, fit="taylor", tol=1e-6, max_iters=40, precision="fp32")
    torch.cuda.synchronize()
    assert int(rep["status"][0]) == prism.DIVERGED and int(rep["iters"][0]) == 9
    np.testing.assert_allclose(rep["resid_hist"][0, :10].double().cpu().numpy(), hist, rtol=1e-3)


@pytest.mark.gpu
def test_folded_parity_flip_across_solves():
    """Folded BF16 polar: the caller's Q holds the even iterates on a plan's first solve and,
    per matrix, the odd ones once a solve ended after an odd number of updates (k_init_state
    flips the ping-pong tables).  Repeats, flips back and mispredictions (new
    values in the same buffers) must all give the bits of a fresh solve."""
    shapes = [(300, 200), (200, 520), (768, 768), (130, 66), (256, 640)]
    mats = [torch.tensor(W.gaussian(m, n, seed=70 + i)).to(torch.bfloat16).cuda() for i, (m, n) in enumerate(shapes)]
    outs = [torch.empty_like(t) for t in mats]
    kw = dict(degree=5, tol=3e-2, max_iters=20, precision="bf16", matrix_ids=list(range(len(shapes))))
    h = P.Handle()

    def fresh():
        Q, rep = P.polar(mats, handle=P.Handle(), **kw)
        torch.cuda.synchronize()
        return [q.clone() for q in Q], rep["iters"].cpu().tolist()

    seen = set()
    for spectrum in range(3):
        if spectrum:
            for i, t in enumerate(mats):   # new values in the same buffers: the same plan, other counts
                m, n = shapes[i]
                a = W.logspaced(m, n, 10.0 ** (-2 * spectrum), seed=170 + 10 * spectrum + i)
                t.copy_(torch.tensor(a).to(torch.bfloat16))
        ref, iters = fresh()
        seen |= {k & 1 for k in iters}
        for _ in range(3):
            Q, rep = P.polar(mats, out=outs, handle=h, **kw)
            torch.cuda.synchronize()
            assert rep["iters"].cpu().tolist() == iters
            for q, r in zip(Q, ref):
                assert torch.equal(q, r)
        if spectrum == 0:   # Gaussian inputs: the oracle agrees (bf16 bar of the GPT-2 shapes)
            for i in (1, 2):
                Qo, _ = prism.polar(mats[i].double().cpu().numpy(), d=2, p=8, tol=3e-2, max_iters=20, seed=42, b=i)
                assert _rel(outs[i].double().cpu().numpy(), Qo) <= 2e-2
    assert seen == {0, 1}


@pytest.mark.gpu
@pytest.mark.parametrize("B", [300, 1100])
def test_large_bf16_batches_equal_single_solves(B):
    """Large BF16 batches of small matrices with spread-out iteration counts: the per-iteration
    tile compaction (k_alpha's compaction blocks; lists of more than 1024 runs keep the full
    list) must not change any matrix's bits, iterations or status against its single solve."""
    g = np.random.default_rng(B)
    shapes = [(int(g.integers(16, 160)), int(g.integers(16, 160))) for _ in range(B)]
    mats = []
    for i, (m, n) in enumerate(shapes):   # a third ill-conditioned: more iterations, later stops
        a = W.logspaced(m, n, 1e-3, seed=5000 + i) if i % 3 == 0 else W.gaussian(m, n, seed=5000 + i)
        mats.append(torch.tensor(a).to(torch.bfloat16).cuda())
    kw = dict(degree=5, tol=3e-2, max_iters=25, precision="bf16")
    Qb, rb = P.polar(mats, matrix_ids=list(range(B)), **kw)
    torch.cuda.synchronize()
    iters = rb["iters"].cpu().tolist()
    assert len(set(iters)) >= 3
    assert all(int(s) == prism.CONVERGED for s in rb["status"].cpu().tolist())
    for i in list(range(0, B, max(1, B // 12))) + [B - 1]:
        Qs, rs = P.polar([mats[i]], matrix_ids=[i], **kw)
        torch.cuda.synchronize()
        assert torch.equal(Qs[0], Qb[i]), i
        assert int(rs["iters"][0]) == iters[i]


@pytest.mark.gpu
def test_flip_compaction_early_square_together():
    """A 12-matrix BF16 batch takes every scheduling path at once: folded parity flip (repeat
    solves), per-iteration tile compaction (>= 8 matrices) and the early square (<= 16):
    three repeats must give the bits and iteration counts of the single solves."""
    shapes = [(256, 192), (192, 640), (512, 512), (130, 66), (320, 320), (96, 400)] * 2
    mats = []
    for i, (m, n) in enumerate(shapes):
        a = W.logspaced(m, n, 1e-3, seed=880 + i) if i % 2 else W.gaussian(m, n, seed=880 + i)
        mats.append(torch.tensor(a).to(torch.bfloat16).cuda())
    kw = dict(degree=5, tol=3e-2, max_iters=25, precision="bf16")
    ids = list(range(len(mats)))
    single = []
    for i, t in enumerate(mats):
        Q, rep = P.polar([t], matrix_ids=[i], **kw)
        torch.cuda.synchronize()
        single.append((Q[0].clone(), int(rep["iters"][0])))
    assert len({k for _, k in single}) >= 2
    h = P.Handle()
    outs = [torch.empty_like(t) for t in mats]
    for _ in range(3):
        Q, rep = P.polar(mats, out=outs, matrix_ids=ids, handle=h, **kw)
        torch.cuda.synchronize()
        for i, (q, k) in enumerate(single):
            assert torch.equal(Q[i], q), i
            assert int(rep["iters"][i]) == k


@pytest.mark.gpu
def test_launch_ledger_counts_every_solve_since_the_last_read():
    mats = [torch.tensor(W.gaussian(300, 200, seed=960)).to(torch.bfloat16).cuda()]
    kw = dict(degree=5, tol=3e-2, max_iters=20, precision="bf16")
    h = P.Handle()
    P.polar(mats, handle=h, **kw)
    one = h.launch_count()
    assert one > 10
    assert h.launch_count() == 0                       # the read resets the ledger
    for _ in range(3):
        P.polar(mats, handle=h, **kw)
    assert h.launch_count() == 3 * one                 # same plan, same iterations


@pytest.mark.gpu
def test_gpt2_batch_host_path_equals_device_path():
    """The e2e entry point on the benchmarked GPT-2 batch (48 matrices: tile compaction, parity
    flip, three staging slots in rotation): every call's outputs equal the device path's bits."""
    shapes = W.gpt2_small_shapes()
    mats_np = W.muon_batch(shapes, seed=1, kind="mixed")
    host = [torch.tensor(a).to(torch.bfloat16).pin_memory() for a in mats_np]
    kw = dict(degree=5, tol=3e-2, max_iters=20, precision="bf16", matrix_ids=list(range(len(host))))
    ref, _ = P.polar([t.cuda() for t in host], **kw)
    torch.cuda.synchronize()
    ref = [r.cpu() for r in ref]
    h = P.Handle()
    outs = [[torch.empty_like(t).pin_memory() for t in host] for _ in range(4)]
    for o in outs:
        P.polar_host(host, out=o, handle=h, **kw)
    torch.cuda.synchronize()
    for o in outs:
        for x, y in zip(o, ref):
            assert torch.equal(x, y)
