"""Multi-process (gloo, world size 2, CPU) tests of the sharding and moment
combination logic used by the multi-GPU path (NCCL on B200)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_26180_b200.moments import shard_bounds, two_pass_moments


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _np_col_sum(U2, center=None):
    a = U2.numpy()
    out = a.sum(axis=0) if center is None else ((a - center.numpy()[None]) ** 2).sum(axis=0)
    return torch.from_numpy(np.ascontiguousarray(out))


def _np_scale(x, a):
    return x * a


def _worker(rank, world, port, M, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(7)
        U = rng.normal(1.0, 0.3, size=(M, 4, 5))
        lo, hi = shard_bounds(M, rank, world)
        mean, var = two_pass_moments(torch.from_numpy(U[lo:hi].copy()), M, col_sum=_np_col_sum, scale=_np_scale)
        if rank == 0:
            q.put((mean.numpy(), var.numpy(), U.mean(axis=0), U.var(axis=0)))
    finally:
        dist.destroy_process_group()


def test_shard_bounds_partition():
    for M in (1, 7, 256, 1048576):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(M, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == M
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def test_two_pass_moments_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    M = 101
    procs = [ctx.Process(target=_worker, args=(r, 2, port, M, q)) for r in range(2)]
    for p in procs:
        p.start()
    mean, var, want_mean, want_var = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    np.testing.assert_allclose(mean, want_mean, rtol=1e-13)
    np.testing.assert_allclose(var, want_var, rtol=1e-12)
