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


def _bench_worker(rank, world, port, q):
    """One rank of the bench's multi-GPU plan, with the oracle standing in for
    the device solve: shard the global ids, receive the surrogate from rank 0,
    solve the shard, combine the moments over gloo."""
    import argparse

    import bench
    from oracle import batched
    from paper_2510_26180_b200 import RngStream
    from paper_2510_26180_b200.engine import gauss_hermite_grid  # noqa: F401  (bench's c1 training grid)

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        args = argparse.Namespace(config="c1", samples=24)
        c = bench.CONFIGS["c1"]
        _, eval_rng, _ = RngStream(bench.SEED).split(3)
        M_total, lo, hi, xi_all = bench.shard_inputs(args, c, eval_rng, rank, world)
        gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "c1.npz"))
        sur = bench.share_from_rank0(lambda: {k: gold[k] for k in ("mean_field", "eigenvalues", "modes", "coeffs")},
                                     rank, True)
        from paper_2510_26180_b200 import LogNormalKL1D

        model = LogNormalKL1D(nx=127, d=4)
        xi = xi_all[lo:hi]
        dia, off = batched.tridiag_from_xi(xi, model.kl_table, model.h)
        U0 = batched.hermite_predict(sur["mean_field"], sur["eigenvalues"], sur["modes"], sur["coeffs"], 2, xi)
        out = batched.pcgc(dia, off, model.initial_condition(), U0, 16, 32, 1.0, 1e-3, 1e-8, 60)
        mean, var = two_pass_moments(torch.from_numpy(out["states"]), M_total, col_sum=_np_col_sum,
                                     scale=_np_scale)
        its = [None] * world
        dist.all_gather_object(its, (lo, hi, out["iters"].tolist()))
        if rank == 0:
            q.put((M_total, xi_all, its, mean.numpy(), var.numpy()))
    finally:
        dist.destroy_process_group()


def test_bench_sharding_gloo_world2(golden):
    """bench.py's strong-scaling plan at world size 2: the shards tile the
    global ids, the broadcast surrogate is rank 0's, and the sharded solve +
    two-pass allreduce reproduces the single-process iteration counts and
    moments of the same global samples."""
    from oracle import batched
    from paper_2510_26180_b200 import LogNormalKL1D

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    M_total, xi_all, parts, mean, var = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert M_total == 24 and parts[0][0] == 0 and parts[0][1] == parts[1][0] and parts[1][1] == 24
    g = golden("c1")
    model = LogNormalKL1D(nx=127, d=4)
    dia, off = batched.tridiag_from_xi(xi_all, model.kl_table, model.h)
    U0 = batched.hermite_predict(g["mean_field"], g["eigenvalues"], g["modes"], g["coeffs"], 2, xi_all)
    one = batched.pcgc(dia, off, model.initial_condition(), U0, 16, 32, 1.0, 1e-3, 1e-8, 60)
    np.testing.assert_array_equal(np.array(parts[0][2] + parts[1][2]), one["iters"])
    np.testing.assert_allclose(mean, one["states"].mean(axis=0), rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(var, one["states"].var(axis=0), rtol=1e-11, atol=1e-15)
    # the bench draws its eval samples exactly like the harness (RngStream(seed).split(3)[1])
    np.testing.assert_array_equal(xi_all[:16], g["xi_all"][:16])


def test_bench_launcher_world2(tmp_path):
    """`bench.py --gpus 2` outside torchrun re-launches itself under
    torch.distributed.run with two ranks; the reference arm runs on rank 0
    only and prints exactly one JSON line with n_gpus = 2."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--impl", "reference",
                          "--config", "c1", "--samples", "16", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["impl"] == "reference" and rec["n_gpus"] == 2 and rec["config"]["n_ranks"] == 2
    assert rec["unit"] == rec["e2e"]["unit"] == "KLE-CGC solves/s"
    assert rec["config"]["global_samples"] == 16 and rec["cpu_baseline"]["subset_size"] == 16
