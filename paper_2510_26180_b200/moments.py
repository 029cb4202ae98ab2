"""Monte Carlo moments of the solution fields, sharded by sample.

The reference computes no moments; the BASELINE north
star asks for the mean and variance of the final fields over the samples,
with NCCL used only to allreduce them. Protocol (two-pass variance, ddof=0,
i.e. ``np.mean`` / ``np.var`` over the sample axis):

    S  = allreduce(sum_s u_s)             mean = S / M_total
    M2 = allreduce(sum_s (u_s - mean)^2)  var  = M2 / M_total

Local column sums are deterministic device reductions (``kle_col_sum_f64``);
the combination step is backend agnostic (NCCL on B200, gloo in the CPU
tests of the sharding logic).
"""
from __future__ import annotations

from . import _lib


def shard_bounds(M: int, rank: int, world: int) -> tuple:
    """Contiguous block of sample ids owned by ``rank``: ids are global, so a
    sharded run reproduces the single-GPU sample set exactly."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    lo = (M * rank) // world
    hi = (M * (rank + 1)) // world
    return lo, hi


def device_col_sum(U2, center=None):
    """U2: (M_local, L) device tensor -> (L,) sums (of squares about center)."""
    from .device import empty, ptr, stream_ptr, torch

    M, L = U2.shape
    out = empty(L)
    nbytes = int(_lib.query("kle_col_sum_scratch_bytes", M, L))
    scratch = torch.empty(max(nbytes, 8), dtype=torch.uint8, device="cuda")
    _lib.call("kle_col_sum_f64", ptr(U2.contiguous()), M, L, ptr(center), ptr(out), ptr(scratch), stream_ptr())
    return out


def device_scale(x, a):
    from .device import empty, ptr, stream_ptr

    out = empty(*x.shape)
    _lib.call("kle_axpby_f64", ptr(x), ptr(x), ptr(out), float(a), 0.0, x.numel(), stream_ptr())
    return out


def two_pass_moments(U_local, M_total: int, group=None, col_sum=device_col_sum, scale=device_scale):
    """Mean and variance over all ranks' samples of U_local (M_local, ...).

    ``group``: a torch.distributed process group (or None for one process).
    Returns (mean, var) shaped like one sample."""
    import torch.distributed as dist

    shape = tuple(U_local.shape[1:])
    U2 = U_local.reshape(U_local.shape[0], -1)
    use_dist = dist.is_available() and dist.is_initialized()
    s = col_sum(U2, None)
    if use_dist:
        dist.all_reduce(s, op=dist.ReduceOp.SUM, group=group)
    mean = scale(s, 1.0 / M_total)
    m2 = col_sum(U2, mean)
    if use_dist:
        dist.all_reduce(m2, op=dist.ReduceOp.SUM, group=group)
    var = scale(m2, 1.0 / M_total)
    return mean.reshape(shape), var.reshape(shape)
