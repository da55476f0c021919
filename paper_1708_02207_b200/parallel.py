"""Z-batch sharding over GPUs: one process per GPU, one NCCL all-gather.

Each rank evaluates a contiguous block of Z rows with its own device plan
(no data-path collective: samples are independent); the only
exchange is the all-gather of the per-sample log-likelihoods, after which
every rank computes the same global posterior weights and argmax
(the reusable piece of posterior_grid, bayes.py:325-330).  Per-sample
arithmetic never depends on the shard, so results are bitwise identical for
any world size.
"""
from __future__ import annotations

import ctypes as C

import numpy as np


def shard_rows(n_rows: int, world: int, rank: int):
    """Contiguous [lo, hi) block of rows owned by `rank` (balanced, remainder first)."""
    base, rem = divmod(n_rows, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def gather_log_likelihood(ll_local, world: int, group=None):
    """All-gather equal-length ll shards (torch tensors) into the global vector."""
    if world == 1:
        return ll_local
    import torch
    import torch.distributed as dist
    out = torch.empty(world * ll_local.numel(), dtype=ll_local.dtype, device=ll_local.device)
    dist.all_gather_into_tensor(out, ll_local.contiguous(), group=group)
    return out


def gather_ragged(x_local, counts, group=None):
    """All-gather shards of unequal length (counts[r] rows on rank r)."""
    import torch
    import torch.distributed as dist
    world = len(counts)
    if world == 1:
        return x_local
    mx = max(counts)
    pad = torch.zeros((mx,) + tuple(x_local.shape[1:]), dtype=x_local.dtype, device=x_local.device)
    pad[: x_local.shape[0]] = x_local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)])


def posterior_weights_device(ll_all, log_prior=None):
    """(weights, argmax, logsumexp) on the device — one launch of the native
    posterior kernel (hdd_posterior_weights) on ll's device and current stream;
    argmax follows numpy (first NaN if any, else the first maximal index).  CPU
    tensors (gloo tests) use the same formulas in torch."""
    import torch
    if not ll_all.is_cuda:
        joint = ll_all if log_prior is None else ll_all + log_prior
        lse = torch.logsumexp(joint, dim=0)
        return torch.exp(joint - lse), torch.argmax(joint), lse
    from . import _lib
    from .errors import UsageError
    ll = ll_all.to(torch.float64).reshape(-1).contiguous()
    n = int(ll.numel())
    lp = None if log_prior is None else torch.as_tensor(log_prior, dtype=torch.float64, device=ll.device).reshape(-1).contiguous()
    if lp is not None and int(lp.numel()) != n:
        raise UsageError(f"log_prior has {int(lp.numel())} entries for {n} log-likelihoods")
    if n == 0:
        raise UsageError("posterior weights of an empty batch")
    with torch.cuda.device(ll.device):
        w = torch.empty_like(ll)
        idx = torch.empty((), dtype=torch.int64, device=ll.device)
        lse = torch.empty((), dtype=torch.float64, device=ll.device)
        rc = _lib.lib().hdd_posterior_weights(
            C.c_void_p(ll.data_ptr()), None if lp is None else C.c_void_p(lp.data_ptr()), n,
            C.c_void_p(w.data_ptr()), C.c_void_p(idx.data_ptr()), C.c_void_p(lse.data_ptr()),
            C.c_void_p(torch.cuda.current_stream(ll.device).cuda_stream))
    _lib.raise_for(rc)
    return w, idx, lse


def sharded_log_likelihood(problem, Z_global, group=None, forward=None):
    """Evaluate ll for all rows of Z_global across the process group.

    Each rank evaluates its contiguous block with `forward(problem, Z_block)`
    (default: the device path `log_likelihood_batch`) and the blocks are
    all-gathered, so every rank returns the full ll vector and the global
    posterior weights / argmax."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = int(Z_global.shape[0])
    lo, hi = shard_rows(n, world, rank)
    if forward is None:
        from .bayes import log_likelihood_batch as forward
    ll_local = forward(problem, Z_global[lo:hi])
    if not isinstance(ll_local, torch.Tensor):
        ll_local = torch.as_tensor(np.asarray(ll_local, dtype=np.float64))
    counts = [shard_rows(n, world, r)[1] - shard_rows(n, world, r)[0] for r in range(world)]
    ll_all = gather_ragged(ll_local, counts, group)
    w, idx, lse = posterior_weights_device(ll_all)
    return ll_all, w, int(idx), float(lse)
