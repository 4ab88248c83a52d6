"""Multi-GPU PRISM: a Muon/Shampoo step's batch sharded across ranks.

One process per GPU with torch.distributed (NCCL over NVLink / NVSwitch on B200).

* Partition: whole matrices are assigned to ranks by the native LPT
  partitioner (prism_lpt_partition): cost = F_min(m, n) x expected iterations,
  largest first to the least-loaded rank; identical on every rank.
* Solve: each rank runs prism_polar / prism_sqrt_invsqrt on its matrices with
  their *global* indices as sketch stream ids, so S_k — and therefore every
  result bit — equals the single-GPU solve of the whole batch.
* Exchange (the one collective on the path): every rank packs its outputs
  into one flat buffer, the buffers are all-gathered (padded to the largest
  rank's size, one NCCL all_gather_into_tensor), and each rank unpacks every
  owner's matrices into place.

`solve` is the CUDA library by default; the parameter exists so the
world-size-2 gloo test on CPU can check the partition / pack / exchange /
unpack logic without a GPU (tests/test_dist.py).

Row-block split (one matrix too large for one GPU, BASELINE configs[3]):
polar_rowblock runs the library's row-block steps with a sum all-reduce of the
fp32 partial Gram X_r^T X_r between them every iteration (the one exchange of
that path), so every rank forms the same R, alpha_k and P and updates its rows.
"""

from __future__ import annotations

from typing import Callable, List, Sequence

import torch
import torch.distributed as dist

from . import binding as B


def lpt_plan(shapes: Sequence[tuple], world: int, degree: int = 5, iters_est: Sequence[int] | None = None) -> List[int]:
    """Owner rank of each matrix (deterministic; same on every rank)."""
    costs = []
    for i, (m, n) in enumerate(shapes):
        f = B.polar_flops_per_iter(m, n, degree, 8)
        costs.append(f * (iters_est[i] if iters_est is not None else 1))
    return B.lpt_partition(costs, world)


def _pack(ts: Sequence[torch.Tensor], numel: int, dtype, device) -> torch.Tensor:
    buf = torch.zeros(numel, dtype=dtype, device=device)
    off = 0
    for t in ts:
        n = t.numel()
        buf[off:off + n].copy_(t.reshape(-1))
        off += n
    return buf


def all_gather_owned(outs: List[torch.Tensor | None], owner: List[int], group=None) -> List[torch.Tensor]:
    """Give every rank every output: owners' tensors are packed, all-gathered, unpacked.

    outs[i] must be set on rank owner[i] (shape/dtype known to all ranks through
    `outs_like`), and is filled in on the other ranks.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = [0] * world
    for i, t in enumerate(outs):
        sizes[owner[i]] += t.numel()
    width = max(sizes) if sizes else 0
    mine = [outs[i] for i in range(len(outs)) if owner[i] == rank]
    ref = outs[0]
    send = _pack(mine, width, ref.dtype, ref.device)
    recv = torch.empty(world * width, dtype=ref.dtype, device=ref.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    cursor = [r * width for r in range(world)]
    for i, t in enumerate(outs):
        r = owner[i]
        n = t.numel()
        if r != rank:
            t.copy_(recv[cursor[r]:cursor[r] + n].view_as(t))
        cursor[r] += n
    return outs


def polar_sharded(mats: Sequence[torch.Tensor], group=None, iters_est=None,
                  solve: Callable | None = None, **opts) -> List[torch.Tensor]:
    """Polar factors of the whole batch on every rank; each rank solves its LPT share.

    `mats` is the full batch (replicated on every rank, as the gradients of a
    data-parallel step after their all-reduce).  Returns outputs for all matrices.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    shapes = [tuple(t.shape) for t in mats]
    owner = lpt_plan(shapes, world, opts.get("degree", 5), iters_est)
    idx = [i for i in range(len(mats)) if owner[i] == rank]
    outs: List[torch.Tensor] = [torch.empty_like(t) for t in mats]
    if idx:
        if solve is None:
            mine, _ = B.polar([mats[i] for i in idx], matrix_ids=idx, **opts)
        else:
            mine = solve([mats[i] for i in idx], idx)
        for i, q in zip(idx, mine):
            outs[i] = q
    return all_gather_owned(outs, owner, group)


def sqrt_invsqrt_sharded(mats: Sequence[torch.Tensor], group=None, iters_est=None,
                         solve: Callable | None = None, **opts):
    """A^{1/2}, A^{-1/2} of the whole batch on every rank (Shampoo blocks), LPT-sharded."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    shapes = [tuple(t.shape) for t in mats]
    owner = lpt_plan(shapes, world, opts.get("degree", 5), iters_est)
    idx = [i for i in range(len(mats)) if owner[i] == rank]
    sq: List[torch.Tensor] = [torch.empty_like(t) for t in mats]
    isq: List[torch.Tensor] = [torch.empty_like(t) for t in mats]
    if idx:
        if solve is None:
            a, b, _ = B.sqrt_invsqrt([mats[i] for i in idx], matrix_ids=idx, **opts)
        else:
            a, b = solve([mats[i] for i in idx], idx)
        for i, x, y in zip(idx, a, b):
            sq[i] = x
            isq[i] = y
    all_gather_owned(sq, owner, group)
    all_gather_owned(isq, owner, group)
    return sq, isq


def polar_rowblock(A_rows: torch.Tensor, group=None, allreduce: Callable | None = None, steps=None, **opts):
    """Polar factor of a tall matrix split by rows across ranks; returns (Q_rows, report).

    Per iteration: partial Gram -> all-reduce(sum) -> identical R / alpha / P on
    every rank -> local update.  The host checks the device stop flag after each
    iteration (one 4-byte read; the exchange already synchronises the ranks).
    """
    if allreduce is None:
        def allreduce(t):
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    st = steps if steps is not None else B.RowBlockSolver(A_rows, **opts)
    st.begin()
    allreduce(st.fro2)
    for k in range(st.max_iters + 1):
        st.gram(k)
        allreduce(st.G)
        st.update(k)
        if int(st.done.item()):
            break
    return st.end()
