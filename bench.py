#!/usr/bin/env python
"""Benchmark: KLE-CGC solves/s (and fine-step DOF-updates/s) at fixed tol,
one process per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config c4|c2|c1|c3|c5|burgers|allen-cahn]

Default workload: BASELINE configs[3] (c4), the metric's own "1/2/4/8 B200"
sweep: the config-1 problem (nx 127, N 16, J 32, d 4, Hermite p 2 on the 3^4
Gauss-Hermite grid) over M = 1,048,576 seeded samples, STRONG-scaled: the
global sample ids are sharded in contiguous blocks across ranks
(moments.shard_bounds), each rank solves its block, and the mean/variance
are combined by the two-pass NCCL allreduce. ``--config c2`` runs configs[1]
(nx 511, N 64, J 64, d 8, p 3 on 2,048 points, M = 65,536) the same way.

``--gpus N`` with N > 1 outside torchrun re-launches this script under
``torch.distributed.run`` with N ranks (127.0.0.1 rendezvous).

A step = one complete batched KLE-CGC solve of the rank's shard with the
inputs resident in HBM: coefficient field, factorisation, Hermite-gPC
surrogate U0 (DMMA GEMM), the PCGC outer loop to tol with per-sample
freezing, and the two-pass mean/variance. The surrogate is built once on
rank 0 (device snapshots, untimed) and broadcast.

``--impl reference`` times the CPU reference path (oracle/ref_port: the
per-sample restatement of pintuq, scipy SuperLU/LAPACK/pocketfft,
bit-identical to the reference's goldens) on a fixed subset of the same
config's sample ids over all host cores (one BLAS thread per worker) and
reports it in the same metric, unit and config.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # BASELINE.json configs[3]: scaling sweep of config 1 (the metric's 1/2/4/8 B200 workload)
    "c4": dict(index=3, nx=127, d=4, N=16, J=32, M=1048576, degree=2, train="gh3", alpha=1e-3, tol=1e-8,
               cpu_subset=4096),
    # configs[1]: config 1 scaled up, one B200
    "c2": dict(index=1, nx=511, d=8, N=64, J=64, M=65536, degree=3, train="gauss2048", alpha=1e-3, tol=1e-8,
               cpu_subset=512),
    # configs[0]: the CPU oracle config
    "c1": dict(index=0, nx=127, d=4, N=16, J=32, M=256, degree=2, train="gh3", alpha=1e-3, tol=1e-8,
               cpu_subset=256),
}
METRIC = "fine-step DOF-updates/s and KLE-CGC solves/s at fixed tol, 1/2/4/8 B200"
UNIT = "KLE-CGC solves/s"
FLOPS_PER_DOF = 6.0   # rhs add 1, forward FMA 2, diagonal scale 1, back-substitution FMA 2
SEED = 2718


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", default="c4", choices=sorted(CONFIGS) + ["c3", "c5", "burgers", "allen-cahn"])
    p.add_argument("--samples", type=int, default=0,
                   help="total samples (default: the config's M; c3: evaluation samples, default 4096)")
    p.add_argument("--train", type=int, default=1024, help="c3: surrogate training samples (config: 1024)")
    p.add_argument("--solver", default="direct", choices=["direct", "krylov"],
                   help="c3: banded direct factors or matrix-free PCG/COCG")
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def maybe_relaunch(args):
    """--gpus N > 1 outside torchrun: re-run this script under
    torch.distributed.run with N ranks on this node (one process per GPU)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    sys.exit(subprocess.call(cmd, env=env))


def problem(cfgname):
    from paper_2510_26180_b200 import LogNormalKL1D, RngStream, SolverConfig, make_time_grid

    c = CONFIGS[cfgname]
    model = LogNormalKL1D(nx=c["nx"], d=c["d"], sigma=0.5, ell=0.3)
    grid = make_time_grid(1.0, c["N"], c["J"])
    cfg = SolverConfig(alpha=c["alpha"], tol=c["tol"], max_outer_iters=60, seed=SEED)
    train_rng, eval_rng, _ = RngStream(SEED).split(3)
    if c["train"] == "gh3":
        from paper_2510_26180_b200.engine import gauss_hermite_grid

        train = gauss_hermite_grid(c["d"], 3)
    else:
        train = train_rng.normal(0.0, 1.0, size=(2048, c["d"]))
    return c, model, grid, cfg, train, eval_rng


def total_samples(args, c):
    return args.samples or c["M"]


def eval_samples(eval_rng, M_total, d):
    """Eval xi = eval_rng.normal(0, 1, (M_total, d)) row-major; sample id =
    row (pintuq/experiments.py:271-272 stream split)."""
    return eval_rng.normal(0.0, 1.0, size=(M_total, d))


def config_dict(args, c, world):
    """The `config` object, identical in both arms for the same invocation."""
    M = total_samples(args, c)
    return {"workload": f"BASELINE configs[{c['index']}] ({args.config}): nx={c['nx']}, N={c['N']}, J={c['J']}, "
                        f"d={c['d']}, Hermite p={c['degree']}, alpha={c['alpha']}, tol={c['tol']}, M={M}",
            "global_samples": M, "n_ranks": world, "parallelism": f"sample-sharded x{world} (strong)",
            "l2": "inputs larger than L2 (state 8*M*N*nx bytes)"}


def cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        try:
            proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                     "--format=csv,noheader,nounits", "-lms", "100"],
                                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            return
        while not self._stop.is_set():
            line = proc.stdout.readline()
            if not line:
                break
            self.rows.append([x.strip() for x in line.split(",")])
        proc.terminate()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        time.sleep(0.3)
        self._stop.set()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 6 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 6 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 6 for i in range(4) if r[2 + i] == "Active"})
        loaded = [v for v in sm if v > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": float(np.median(loaded)) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
def share_from_rank0(builder, rank, use_dist):
    """Rank 0 runs ``builder()``; the result is broadcast to every rank."""
    import torch.distributed as dist

    box = [builder() if rank == 0 else None]
    if use_dist:
        dist.broadcast_object_list(box, src=0)
    return box[0]


def build_and_share_surrogate(model, grid, cfg, train, degree, rank, use_dist):
    """Rank 0 builds the surrogate (device snapshots + KL + Hermite fit) and
    broadcasts it; every rank evaluates the identical tables."""
    from paper_2510_26180_b200.core import ParameterSample
    from paper_2510_26180_b200.surrogate import build_surrogate

    def build():
        training = [ParameterSample(x, id=i) for i, x in enumerate(train)]
        return build_surrogate(model, grid, cfg, training, eps_kl=1e-10, degree=degree, family="hermite")

    t0 = time.time()
    sur = share_from_rank0(build, rank, use_dist)
    return sur, time.time() - t0


def shard_inputs(args, c, eval_rng, rank, world):
    """This rank's contiguous block of global sample ids and its xi rows
    (all ranks draw the same global xi from the seed, then slice)."""
    from paper_2510_26180_b200.moments import shard_bounds

    M_total = total_samples(args, c)
    lo, hi = shard_bounds(M_total, rank, world)
    xi_all = eval_samples(eval_rng, M_total, c["d"])
    return M_total, lo, hi, xi_all


def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2510_26180_b200 import _lib
    from paper_2510_26180_b200.device import DeviceOperator, empty, ptr, stream_ptr
    from paper_2510_26180_b200.engine import KleCgcSolver

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    # under torchrun (even with one rank) the moments go through the NCCL allreduce path
    use_dist = world > 1 or "TORCHELASTIC_RUN_ID" in os.environ
    if use_dist:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c, model, grid, cfg, train, eval_rng = problem(args.config)
    M_total, lo, hi, xi_all = shard_inputs(args, c, eval_rng, rank, world)
    M = hi - lo
    sur, t_build = build_and_share_surrogate(model, grid, cfg, train, c["degree"], rank, use_dist)
    solver = KleCgcSolver(model, grid, cfg, sur)
    xi_host = np.ascontiguousarray(xi_all[lo:hi])
    xi_d = torch.as_tensor(xi_host, device="cuda")
    stream = torch.cuda.current_stream()

    def step(x):
        res = solver.solve(x)
        mean, var = solver.moments(res, M_total=M_total)
        return res, mean, var

    def barrier():
        torch.cuda.synchronize()
        if use_dist:
            dist.barrier()

    for _ in range(args.warmup):
        res, mean, var = step(xi_d)
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            res, mean, var = step(xi_d)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    it = res.batch.iters
    n_sub = min(c["cpu_subset"], M_total)
    stats = torch.tensor([ms, float(it.sum().item()), float(it.max().item()),
                          float((res.batch.status != 1).sum().item()),
                          float(it[:max(0, min(n_sub - lo, M))].sum().item())], device="cuda", dtype=torch.float64)
    if use_dist:
        mx = stats[[0, 2]].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = stats[[1, 3, 4]].clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        stats = torch.stack([mx[0], sm[0], mx[1], sm[1], sm[2]])
    ms_max, total_iters, kmax, n_bad, sub_iters = [float(v) for v in stats.tolist()]
    dof_per_iter = grid.n_coarse * grid.n_fine_per_coarse * model.nx
    solves_per_s = M_total / (ms_max * 1e-3)
    dof_per_s = total_iters * dof_per_iter / (ms_max * 1e-3)

    # ---- kernel-level timing of the hot kernels on this rank's shard (all samples active) ----
    op = DeviceOperator.from_model(model, xi_d)
    U = solver.surrogate.predict(xi_d)
    blob = op.blob(grid.deltat)
    tables = solver.tables
    R = empty(M, grid.n_coarse, model.nx)
    st_ptr = stream_ptr()

    def fgr():
        _lib.call("kle_fgr_f64", ptr(U), ptr(op.u0), None, None, ptr(R), ptr(blob), ptr(op.dia), ptr(op.off),
                  ptr(tables.scaling), None, M, grid.n_coarse, model.nx, grid.n_fine_per_coarse, grid.deltat,
                  grid.deltaT, op.g0, cfg.alpha, st_ptr)

    from paper_2510_26180_b200.pcgc import shift_factors

    sfac = shift_factors(op, tables, grid.n_coarse, grid.deltaT)
    nbytes = 16 * M if sfac is not None else int(_lib.query("kle_cgc_scratch_bytes", M, grid.n_coarse, model.nx))
    scratch = torch.zeros(max(nbytes, 8), dtype=torch.uint8, device="cuda")

    def cgc():
        _lib.call("kle_cgc_update_f64", ptr(R), ptr(U), ptr(tables.inv_scaling), ptr(tables.lam), ptr(op.dia),
                  ptr(op.off), ptr(sfac), M, grid.n_coarse, model.nx, grid.deltaT, 1, 1, -1.0, None, None, None,
                  None, None, ptr(scratch), nbytes, st_ptr)

    def timed(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    fgr_ms = timed(fgr)
    cgc_ms = timed(cgc)
    gemm_ms = timed(lambda: solver.surrogate.predict(xi_d, out=U))
    peaks = load_peaks()
    fgr_flops = FLOPS_PER_DOF * M * dof_per_iter
    fgr_tflops = fgr_flops / (fgr_ms * 1e-3) / 1e12
    cgc_bytes = 24.0 * M * grid.n_coarse * model.nx   # read R, read U, write U (compulsory)
    cgc_gbs = cgc_bytes / (cgc_ms * 1e-3) / 1e9
    fgr_bytes = 16.0 * M * grid.n_coarse * model.nx   # read U, write R
    K_g = solver.surrogate.inner_dim
    gemm_tflops = 2.0 * M * K_g * grid.n_coarse * model.nx / (gemm_ms * 1e-3) / 1e12
    avg_iters = total_iters / M_total
    local_ms = ms   # this rank's own step (the shares are of its own step)
    share_fgr = float(it.double().mean().item()) * fgr_ms / local_ms
    share_cgc = float(it.double().mean().item()) * cgc_ms / local_ms
    del R, scratch, sfac, U, op

    # ---- end to end through the public API: pinned host xi -> device -> host moments + counts ----
    pinned = torch.from_numpy(xi_host).pin_memory()
    host_mean = torch.empty(mean.numel(), dtype=torch.float64).pin_memory()
    host_var = torch.empty_like(host_mean).pin_memory()
    host_it = torch.empty(M, dtype=torch.int32).pin_memory()
    host_st = torch.empty(M, dtype=torch.int32).pin_memory()

    def e2e_step():
        xd = pinned.to("cuda", non_blocking=True)
        r2, m2, v2 = step(xd)
        host_mean.copy_(m2.reshape(-1), non_blocking=True)
        host_var.copy_(v2.reshape(-1), non_blocking=True)
        host_it.copy_(r2.batch.iters, non_blocking=True)
        host_st.copy_(r2.batch.status, non_blocking=True)

    e2e_step()  # warm-up of the host-buffer path (untimed)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    nrep = max(1, args.steps)
    for _ in range(nrep):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / nrep], device="cuda", dtype=torch.float64)
    if use_dist:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e = {"value": M_total / (float(e2e_ms.item()) * 1e-3), "unit": UNIT,
           "h2d_bytes_per_step": int(xi_host.nbytes) * world,
           "d2h_bytes_per_step": int(host_mean.numel() * 16 * world + M_total * 8),
           "ms_per_step": float(e2e_ms.item())}

    # per step: kl_tridiag, fine_factor, gpc basis + 1-2 GEMMs, shift_factor, then per outer iteration and
    # sample pipeline (two when the batch is large, kle_capi.cu) one fgr and one CGC launch (an upper bound:
    # a pipeline stops as soon as its own samples have converged), and 2 x (2 col-sum + 1 scale) for the moments
    tw_small = 64 < c["nx"] <= 128 and c["N"] <= 16 and os.environ.get("KLE_FGR_TW", "1") != "0"
    pipes = int(os.environ.get("KLE_PCGC_PIPES", "1" if tw_small else "2")) if M >= 8192 else 1
    # the twisted two-lane fine sweep (kle_fine_tw.cu, 64 < nx <= 128) adds its table kernel and the count of the
    # samples flagged as having no scaled form (none here, so the partitioned fallback kernel is never launched)
    tw_path = 64 < c["nx"] <= 128 and os.environ.get("KLE_FGR_TW", "1") != "0"
    pw_path = 128 < c["nx"] <= 512 and os.environ.get("KLE_FGR_PW", "1") != "0"
    launches_per_step = (1 + 1 + (1 + (1 if solver.surrogate.mode == "direct" else 2)) + 1
                         + 2 * pipes * int(kmax) + 6 + (2 if (tw_path or pw_path) else 0))
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, c, model, grid, cfg, sur, xi_all[:n_sub])
    if rank == 0:
        fp64_peak = peaks.get("fp64_tflops")
        # small blocks take the row-FFT kernel (kle_cgc_row.cu), the others the cluster kernel
        row_path = c["N"] <= 16 and c["nx"] <= 128 and os.environ.get("KLE_CGC_ROW", "1") != "0"
        cgc_path = "row (one CTA per sample, register FFTs)" if row_path else "cluster"
        cgc_kernel_name = "cgc_row_kernel" if row_path else "cgc_cluster_kernel"
        line = {
            "metric": METRIC,
            "value": solves_per_s,
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_max,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded N(0,1) KL coordinates, BASELINE configs; no dataset exists)",
            "config": config_dict(args, c, world),
            "samples_per_rank": M,
            "fine_dof_updates_per_s": dof_per_s,
            "avg_outer_iters": avg_iters,
            "avg_outer_iters_cpu_subset": sub_iters / n_sub,
            "cpu_subset_ids": [0, n_sub],
            "max_outer_iters": int(kmax),
            "all_converged": n_bad == 0,
            "surrogate_build_s": t_build,
            "surrogate": {"m_q": sur.m_q, "P": solver.surrogate.P, "K_g": K_g, "mode": solver.surrogate.mode,
                          "built_on": "rank 0 (device snapshots), broadcast"},
            "roofline": {
                "kernel": ("fgr_tw_kernel (twisted two-lane J-step fine sweep + CGC rhs)" if tw_path
                           else "fgr_pw_kernel (eight-lane scaled J-step fine sweep + CGC rhs)" if pw_path
                           else "fgr_kernel (fused J-step fine sweep + CGC rhs)"),
                "bound": "fp64",
                "achieved": fgr_tflops,
                "peak": fp64_peak,
                "unit": "TFLOP/s",
                "frac": (fgr_tflops / fp64_peak) if fp64_peak else None,
                "traffic": traffic_of(peaks, args.config,
                                      "fgr_tw_kernel" if tw_path else "fgr_pw_kernel" if pw_path else "fgr_kernel", M),
                "traffic_source": "ncu --set full dram__bytes_read.sum + dram__bytes_write.sum per sample-iteration "
                                  "(profiles/traffic.json) x samples per launch",
                "peak_source": peaks.get("fp64_source"),
                "algorithmic": f"{FLOPS_PER_DOF:g} flop per fine DOF-update x M*N*J*nx per launch (M = rank shard)",
                "executed_flop_per_dof_update": 4 if tw_path else 7 if pw_path else 10,
                # the twisted / eight-lane sweeps read their factor rows as shared-memory broadcasts: ncu's
                # shared-memory wavefront utilisation of the kernel (profiles/traffic.json), the resource that
                # binds them beside the FP64 pipe
                "shared_wavefronts_pct_ncu": ncu_field(peaks, args.config,
                                                       "fgr_tw_kernel" if tw_path else "fgr_pw_kernel" if pw_path
                                                       else "fgr_kernel", "shared_wavefronts_pct"),
                "fp64_pipe_pct_ncu": ncu_field(peaks, args.config,
                                               "fgr_tw_kernel" if tw_path else "fgr_pw_kernel" if pw_path
                                               else "fgr_kernel", "fp64_pipe_pct"),
                "hbm_frac": (fgr_bytes / (fgr_ms * 1e-3) / 1e9) / peaks["hbm_gbs"],
                "ms_per_launch": fgr_ms,
            },
            "kernels": {
                "cgc_kernel": {"bound": "hbm", "achieved": cgc_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                               "frac": cgc_gbs / peaks["hbm_gbs"], "ms_per_launch": cgc_ms,
                               "algorithmic": "24 B per (n, i) per sample: read R, read U, write U "
                                              "(+ pivots 16 (N/2+1)/N B not counted)",
                               "path": cgc_path,
                               "traffic": traffic_of(peaks, args.config, cgc_kernel_name, M)},
                "gemm_bias_kernel": {"bound": "tensor(dmma)", "achieved": gemm_tflops,
                                     "peak": peaks.get("dmma_tflops"), "unit": "TFLOP/s",
                                     "frac": gemm_tflops / peaks["dmma_tflops"] if peaks.get("dmma_tflops") else None,
                                     "ms_per_launch": gemm_ms},
                "step_share": {"fgr": share_fgr, "cgc": share_cgc},
            },
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()


def ncu_field(peaks, config, kernel, field):
    return peaks.get("traffic", {}).get(config, {}).get(kernel, {}).get(field)


def traffic_of(peaks, config, kernel, M):
    t = peaks.get("traffic", {}).get(config, {}).get(kernel)
    return t["bytes_per_sample_iteration"] * M if t else None


def load_peaks():
    out = {"hbm_gbs": 6537.0}
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        out["hbm_gbs"] = float(json.loads(p.read_text()).get("hbm_gbs", 6537.0))
        out["hbm_source"] = "MEASURED_PEAKS.json"
    else:
        out["hbm_gbs"] = 6650.0
        out["hbm_source"] = "fallback (B200_PROFILING.md)"
    f = ROOT / "profiles" / "r01_fp64_peaks.jsonl"
    if f.exists():
        for line in f.read_text().splitlines():
            try:
                d = json.loads(line)
            except ValueError:
                continue
            if d.get("what") == "dfma_tflops":
                out["fp64_tflops"] = d["value"]
                out["fp64_source"] = "measured DFMA peak, profiles/r01_fp64_peaks.jsonl (tools/fp64_peaks.cu)"
            if d.get("what") == "dmma_tflops":
                out["dmma_tflops"] = d["value"]
    t = ROOT / "profiles" / "traffic.json"
    if t.exists():  # DRAM bytes per sample-iteration from one ncu --set full capture, per config
        out["traffic"] = json.loads(t.read_text())
    return out


# ---------------------------------------------------------------------------
# CPU reference path (oracle/ref_port: bit-identical restatement of pintuq)
# ---------------------------------------------------------------------------
_W = {}


def _cpu_init(payload):
    _W.update(payload)
    try:  # one BLAS/OpenMP thread per worker process (cores x cores threads thrash)
        from threadpoolctl import threadpool_limits

        _W["_tp"] = threadpool_limits(1)
    except ImportError:
        pass


def _cpu_solve(i):
    from oracle import ref_port

    w = _W
    xi = w["xi"][i]
    a = np.exp(xi @ w["kl_table"])
    dia = (a[:-1] + a[1:]) * w["inv_h2"]
    off = -a[1:-1] * w["inv_h2"]
    op = ref_port.SampleOperator(dia, off, np.full(len(dia), 1.0))
    U0 = ref_port.surrogate_predict(w["mean"], w["lam"], w["modes"], w["coeffs"], w["degree"], xi)
    out = ref_port.pcgc(op, w["u0"], U0, w["N"], w["J"], 1.0, w["alpha"], w["tol"], 60)
    return out["iters"]


def _cpu_pool(payload, cores):
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor

    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    # fork: workers inherit the surrogate tables without pickling them
    return ProcessPoolExecutor(cores, mp_context=mp.get_context("fork"), initializer=_cpu_init,
                               initargs=(payload,))


def _cpu_payload(c, model, grid, sur, xi_sub):
    return dict(xi=xi_sub, kl_table=model.kl_table, inv_h2=1.0 / (model.h * model.h), u0=model.initial_condition(),
                mean=sur.mean_field, lam=sur.eigenvalues, modes=sur.modes, coeffs=sur.coeffs, degree=sur.degree,
                N=grid.n_coarse, J=grid.n_fine_per_coarse, alpha=c["alpha"], tol=c["tol"])


def _cpu_record(n, wall, its, cores, c, model, grid, M_total, steps=None):
    dof = float(np.sum(its)) * grid.n_coarse * grid.n_fine_per_coarse * model.nx
    v = n / wall
    return {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "cpu_model": cpu_model(),
            "blas_threads_per_worker": 1,
            "sample": f"sample ids 0..{n - 1} of the {M_total} config samples"
                      + (f" ({steps} timed chunks)" if steps else "")
                      + ", surrogate_predict + pcgc_solve per sample (oracle/ref_port = pintuq arithmetic, scipy "
                        f"SuperLU/LAPACK/pocketfft), {cores} processes x 1 BLAS thread, {wall:.1f} s wall",
            "extrapolated": True,
            "extrapolation": f"linear: the full M = {M_total} would take {M_total / v:.0f} s at this rate",
            "subset_size": n, "avg_outer_iters_subset": float(np.mean(its)),
            "fine_dof_updates_per_s": dof / wall}


def cpu_baseline(args, c, model, grid, cfg, sur, xi_sub):
    """The reference CPU path on the fixed subset of sample ids 0..n-1 over
    all host cores (ProcessPool, one sample per task)."""
    cores = os.cpu_count() or 1
    n = len(xi_sub)
    with _cpu_pool(_cpu_payload(c, model, grid, sur, xi_sub), cores) as ex:
        list(ex.map(_cpu_solve, range(min(cores, n))))  # warm the workers
        t0 = time.time()
        its = list(ex.map(_cpu_solve, range(n), chunksize=max(1, n // (8 * cores))))
        wall = time.time() - t0
    return _cpu_record(n, wall, its, cores, c, model, grid, total_samples(args, c))


def run_reference(args):
    """--impl reference: the reference's CPU path on the box's host cores, on
    this arm's config/metric/unit; rank 0 only (other ranks exit 0)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    c, model, grid, cfg, train, eval_rng = problem(args.config)
    M_total = total_samples(args, c)
    # the reference builds its surrogate on the CPU too (collect_snapshots ->
    # kl_build -> gpc_fit); training solves run over all cores
    t0 = time.time()
    cores = os.cpu_count() or 1
    sur = _cpu_build_surrogate(model, grid, cfg, train, c["degree"], cores)
    t_build = time.time() - t0
    n_sub = min(c["cpu_subset"], M_total)
    xi_sub = eval_samples(eval_rng, M_total, c["d"])[:n_sub]
    steps = max(1, args.steps)
    bounds = [(n_sub * s) // steps for s in range(steps + 1)]
    its, walls = [], []
    with _cpu_pool(_cpu_payload(c, model, grid, sur, xi_sub), cores) as ex:
        for _ in range(args.warmup):  # warm-up steps only spin the workers up (a few samples)
            list(ex.map(_cpu_solve, range(min(cores, n_sub))))
        for s in range(steps):  # each timed step = one contiguous chunk of the fixed id subset
            ids = range(bounds[s], bounds[s + 1])
            t1 = time.time()
            its += list(ex.map(_cpu_solve, ids, chunksize=max(1, len(ids) // (8 * cores))))
            walls.append(time.time() - t1)
    wall = float(np.sum(walls))
    rec = _cpu_record(n_sub, wall, its, cores, c, model, grid, M_total, steps)
    line = {"impl": "reference", "metric": METRIC, "value": rec["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded N(0,1) KL coordinates, BASELINE configs; no dataset exists)",
            "config": config_dict(args, c, world), "avg_outer_iters_cpu_subset": rec["avg_outer_iters_subset"],
            "cpu_subset_ids": [0, n_sub], "cpu_baseline": rec, "surrogate_build_s": t_build,
            "e2e": {"value": rec["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _snap_one(args):
    from oracle import ref_port

    xi, kl_table, inv_h2, u0, N, J, alpha, tol = args
    a = np.exp(xi @ kl_table)
    dia = (a[:-1] + a[1:]) * inv_h2
    off = -a[1:-1] * inv_h2
    op = ref_port.SampleOperator(dia, off, np.full(len(dia), 1.0))
    init = ref_port.coarse_sweep(op, u0, N, 1.0 / N)
    return ref_port.pcgc(op, u0, init, N, J, 1.0, alpha, tol, 60)["states"]


def _cpu_build_surrogate(model, grid, cfg, train, degree, cores):
    from oracle import ref_port
    from paper_2510_26180_b200.models import ParameterMap
    from paper_2510_26180_b200.surrogate import KLGpcSurrogate

    jobs = [(x, model.kl_table, 1.0 / (model.h * model.h), model.initial_condition(), grid.n_coarse,
             grid.n_fine_per_coarse, cfg.alpha, cfg.tol) for x in train]
    with _cpu_pool({}, cores) as ex:
        fields = np.array(list(ex.map(_snap_one, jobs, chunksize=4)))
    w = model.cell_volume * grid.deltaT
    mean, lam, modes, X = ref_port.kl_build(fields, w, 1e-10)
    zeta = ref_port.kl_coefficients(X, modes, lam, w)
    coeffs = ref_port.gpc_fit(train, zeta, degree)
    return KLGpcSurrogate(mean, lam, modes, coeffs, degree,
                          [ParameterMap("identity", -np.inf, np.inf)] * len(train[0]), family="hermite")


def run_c5(args):
    """BASELINE configs[4]: diagonalised-CGC stress. nx = 4095, N = 1024, J = 8,
    alpha in {1e-1, 1e-2, 1e-4}, 4096 samples (coarse-sweep initial guess),
    processed in sample chunks (one state copy is 137 GB at M = 4096).
    Reports iteration counts per alpha, end-to-end solves/s and the CGC
    throughput (sample-iterations/s and compulsory GB/s of one CGC launch)."""
    import torch

    from paper_2510_26180_b200 import LogNormalKL1D, RngStream, SolverConfig, make_time_grid
    from paper_2510_26180_b200 import _lib
    from paper_2510_26180_b200.device import AlphaTables, DeviceOperator, empty, ptr, stream_ptr
    from paper_2510_26180_b200.pcgc import build_alpha_circulant, pcgc_solve_device, shift_factors
    from paper_2510_26180_b200.propagators import coarse_sweep_init_batched

    nx, N, J, M, chunk = 4095, 1024, 8, int(os.environ.get("KLE_C5_M", "4096")), 256
    model = LogNormalKL1D(nx=nx, d=4)
    grid = make_time_grid(1.0, N, J)
    _, eval_rng, _ = RngStream(SEED).split(3)
    xi = eval_rng.normal(0.0, 1.0, size=(M, 4))
    out = {"metric": "c5 CGC stress: iterations per alpha, CGC throughput", "config": {
        "workload": "BASELINE configs[4]: nx=4095, N=1024, J=8, d=4, coarse-sweep init, tol=1e-8",
        "samples": M, "chunk": chunk}, "alphas": {}}
    # warm-up (untimed): one small chunk through the whole path (kernel attributes, allocator)
    op = DeviceOperator.from_model(model, xi[:8])
    U = coarse_sweep_init_batched(op, grid).contiguous()
    pcgc_solve_device(op, U, grid, SolverConfig(alpha=1e-1, tol=1e-8, max_outer_iters=60, seed=SEED))
    torch.cuda.synchronize()
    del U, op
    for alpha in (1e-1, 1e-2, 1e-4):
        cfg = SolverConfig(alpha=alpha, tol=1e-8, max_outer_iters=60, seed=SEED)
        tables = AlphaTables(build_alpha_circulant(N, alpha))
        iters = []
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ev0.record()
        for c0 in range(0, M, chunk):
            op = DeviceOperator.from_model(model, xi[c0:c0 + chunk])
            U = coarse_sweep_init_batched(op, grid).contiguous()
            res = pcgc_solve_device(op, U, grid, cfg, tables)
            iters.append(res.iters.cpu().numpy())
            del U, res, op
        ev1.record()
        torch.cuda.synchronize()
        wall_ms = ev0.elapsed_time(ev1)
        it = np.concatenate(iters)
        # one CGC launch on a full chunk (all samples active)
        op = DeviceOperator.from_model(model, xi[:chunk])
        U = coarse_sweep_init_batched(op, grid).contiguous()
        R = empty(chunk, N, nx)
        blob = op.blob(grid.deltat)
        fa, fb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fa.record()
        _lib.call("kle_fgr_f64", ptr(U), ptr(op.u0), None, None, ptr(R), ptr(blob), ptr(op.dia),
                  ptr(op.off), ptr(tables.scaling), None, chunk, N, nx, J, grid.deltat, grid.deltaT, op.g0, alpha,
                  stream_ptr())
        fb.record()
        torch.cuda.synchronize()
        fgr_ms = fa.elapsed_time(fb)
        sfac = shift_factors(op, tables, N, grid.deltaT)
        nb = 16 * chunk if sfac is not None else int(_lib.query("kle_cgc_scratch_bytes", chunk, N, nx))
        scratch = torch.zeros(max(nb, 8), dtype=torch.uint8, device="cuda")
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.call("kle_cgc_update_f64", ptr(R), ptr(U), ptr(tables.inv_scaling), ptr(tables.lam), ptr(op.dia),
                  ptr(op.off), ptr(sfac), chunk, N, nx, grid.deltaT, 1, 1, -1.0, None, None, None, None, None,
                  ptr(scratch), nb, stream_ptr())
        b.record()
        torch.cuda.synchronize()
        cgc_ms = a.elapsed_time(b)
        hist = {int(k): int(v) for k, v in zip(*np.unique(it, return_counts=True))}
        out["alphas"][f"{alpha:g}"] = {
            "iters_mean": float(it.mean()), "iters_hist": hist, "solves_per_s": M / (wall_ms * 1e-3),
            "wall_s": wall_ms * 1e-3, "cgc_ms_per_launch": cgc_ms,
            "cgc_sample_iterations_per_s": chunk / (cgc_ms * 1e-3),
            "cgc_compulsory_gbs": 24.0 * chunk * N * nx / (cgc_ms * 1e-3) / 1e9,
            "cgc_hbm_frac": 24.0 * chunk * N * nx / (cgc_ms * 1e-3) / 1e9 / load_peaks()["hbm_gbs"],
            "cgc_path": "cluster" if sfac is not None else "large (FFT / per-frequency solve / inverse FFT kernels)",
            "fgr_ms_per_launch": fgr_ms,
            "fgr_dof_updates_per_s": chunk * N * J * nx / (fgr_ms * 1e-3),
            "fgr_tflops_alg": FLOPS_PER_DOF * chunk * N * J * nx / (fgr_ms * 1e-3) / 1e12,
        }
        del U, R, op, scratch
    if not args.no_cpu_baseline:  # the reference path (SuperLU / LAPACK / pocketfft) on the host cores
        from concurrent.futures import ProcessPoolExecutor

        cores = os.cpu_count() or 1
        model_np = model
        tasks = []
        for i in range(cores):
            dia, off = model_np.tridiagonal(xi[i])
            tasks.append((dia, off, model_np.initial_condition(), N, J, 1e-1))
        t0 = time.time()
        with ProcessPoolExecutor(cores) as ex:
            cpu_it = list(ex.map(_cpu_c5, tasks))
        wall = time.time() - t0
        out["cpu_baseline"] = {"value": cores / wall, "unit": "KLE-CGC solves/s", "cores": cores, "kind": "port",
                               "sample": f"first {cores} samples at alpha = 0.1, coarse-sweep init, one per process "
                                         f"(oracle/ref_port: SuperLU, solve_banded, np.fft), {wall:.1f} s wall",
                               "iters": cpu_it}
    peaks = load_peaks()
    a4 = out["alphas"]["0.0001"]
    out["roofline"] = {"kernel": "large-block CGC (cgcl_fwd / cgcl_solve / cgcl_inv kernels, one launch)",
                       "bound": "hbm", "achieved": a4["cgc_compulsory_gbs"], "peak": peaks["hbm_gbs"], "unit": "GB/s",
                       "frac": a4["cgc_compulsory_gbs"] / peaks["hbm_gbs"],
                       "algorithmic": "24 B per (n, i) per sample-iteration (read R, read U, write U) x the chunk",
                       "fine_sweep_fp64_frac": (a4["fgr_tflops_alg"] / peaks["fp64_tflops"]
                                                if peaks.get("fp64_tflops") else None),
                       "traffic": None}
    print(json.dumps(out), flush=True)


def _cpu_c5(task):
    from oracle import ref_port

    dia, off, u0, N, J, alpha = task
    op = ref_port.SampleOperator(dia, off, np.ones(len(dia)))
    init = ref_port.coarse_sweep(op, u0, N, 1.0 / N)
    return ref_port.pcgc(op, u0, init, N, J, 1.0, alpha, 1e-8, 60)["iters"]


def _cpu_solve2d(task):
    """One c3 sample on the oracle (SuperLU paths): task = (stencil, U0, u0, n, N, J, alpha, tol)."""
    from oracle import ref_port

    (dia, ex, ey), U0, u0, n, N, J, alpha, tol = task
    op = ref_port.SampleOperator.from_stencil2d(dia, ex, ey, n, np.full(len(dia), 1.0))
    out = ref_port.pcgc(op, u0, U0, N, J, 1.0, alpha, tol, 60)
    return out["iters"]


def run_c3(args):
    """BASELINE configs[2]: 2D diffusion, 127 x 127 grid (nx = 16,129), N = 32,
    J = 16, d = 10, Hermite p = 2 (66 terms) fitted on --train seeded samples,
    alpha = 1e-3, tol = 1e-8. Timed step = U0 (gPC GEMM) + banded factors of
    I + dt A and of the 17 shifted matrices + PCGC to tol + moments, on
    --samples evaluation samples (default: the config's M = 4,096, a ~80 s
    step; the samples go through in batches sized to the free HBM, ~193).
    The CPU baseline is the oracle (SuperLU paths) on a bounded sample over
    all host cores."""
    import torch

    from paper_2510_26180_b200 import LogNormalKL2D, ParameterSample, RngStream, SolverConfig, make_time_grid
    from paper_2510_26180_b200.engine import KleCgcSolver
    from paper_2510_26180_b200.surrogate import build_surrogate

    n, N, J, d = 127, 32, 16, 10
    M = args.samples or 4096
    os.environ["KLE_2D_SOLVER"] = args.solver
    model = LogNormalKL2D(n=n, d=d, sigma=0.5, ell=0.25)
    grid = make_time_grid(1.0, N, J)
    cfg = SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60, seed=SEED)
    train_rng, eval_rng, _ = RngStream(SEED).split(3)
    train = train_rng.normal(0.0, 1.0, size=(args.train, d))
    t0 = time.time()
    sur = build_surrogate(model, grid, cfg, [ParameterSample(x, id=i) for i, x in enumerate(train)], eps_kl=1e-10,
                          degree=2)
    t_build = time.time() - t0
    print(f"c3: surrogate built in {t_build:.1f} s (m_q={sur.m_q})", file=sys.stderr, flush=True)
    solver = KleCgcSolver(model, grid, cfg, sur)
    xi_host = eval_rng.normal(0.0, 1.0, size=(M, d))
    xi_d = torch.as_tensor(xi_host, device="cuda")

    def step(x):
        res = solver.solve(x)
        mean, var = solver.moments(res, M_total=M)
        return res, mean, var

    res = mean = var = None
    for _ in range(args.warmup):
        tw = time.time()
        res = mean = var = None  # a step's fields are consumed before the next (c3's batches size to free HBM)
        res, mean, var = step(xi_d)
        torch.cuda.synchronize()
        print(f"c3: warm-up step {time.time() - tw:.1f} s", file=sys.stderr, flush=True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clocks:
        ev0.record()
        for _ in range(args.steps):
            res = mean = var = None
            res, mean, var = step(xi_d)
        ev1.record()
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    it = res.batch.iters.cpu().numpy()
    status = res.batch.status.cpu().numpy()
    # end to end: pinned host xi -> device -> host moments
    pinned = torch.from_numpy(xi_host).pin_memory()
    hm = torch.empty(mean.numel(), dtype=torch.float64).pin_memory()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res.batch.states = None
    e0.record()
    r2, m2, v2 = step(pinned.to("cuda", non_blocking=True))
    hm.copy_(m2.reshape(-1), non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    dof = float(it.sum()) * N * J * model.nx
    roof = c3_roofline(model, grid, cfg, xi_d, solver)
    cpu = None
    if not args.no_cpu_baseline:
        from concurrent.futures import ProcessPoolExecutor
        import multiprocessing as mp

        cores = os.cpu_count() or 1
        nb = min(M, cores)
        # spawned workers (a fork after the CUDA context and the BLAS thread pools
        # of the surrogate build can deadlock); U0 = surrogate_predict on the host
        from oracle import ref_port

        tasks = [(model.stencil(xi_host[i]),
                  ref_port.surrogate_predict(sur.mean_field, sur.eigenvalues, sur.modes, sur.coeffs, sur.degree,
                                             xi_host[i]),
                  model.initial_condition(), n, N, J, cfg.alpha, cfg.tol) for i in range(nb)]
        print(f"c3: CPU baseline on {nb} samples", file=sys.stderr, flush=True)
        # one BLAS thread per worker (SuperLU calls BLAS; cores x cores threads thrash)
        for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
            os.environ[var] = "1"
        with ProcessPoolExecutor(cores, mp_context=mp.get_context("spawn")) as ex:
            list(ex.map(_cpu_solve2d, tasks[:1]))  # start the workers
            t0 = time.time()
            its = list(ex.map(_cpu_solve2d, tasks))
            wall = time.time() - t0
        cpu = {"value": nb / wall, "unit": "KLE-CGC solves/s", "cores": cores, "kind": "port",
               "sample": f"first {nb} of the {M} evaluation samples, one per process, pcgc_solve from the "
                         f"host surrogate_predict U0 (oracle/ref_port: SuperLU of I + dt A and of each "
                         f"lambda_n I + dT A), {wall:.1f} s wall",
               "fine_dof_updates_per_s": float(np.sum(its)) * N * J * model.nx / wall}
    line = {"metric": METRIC, "value": M / (ms * 1e-3), "unit": "KLE-CGC solves/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded N(0,1) KL coordinates; no dataset exists)",
            "config": {"workload": f"BASELINE configs[2] (c3): 2D 127x127 5-point, N={N}, J={J}, d={d}, "
                                   f"Hermite p=2 on {args.train} training samples, alpha={cfg.alpha}, tol={cfg.tol}; "
                                   + ("direct banded LDL^T solves (the reference's SuperLU semantics)"
                                      if args.solver == "direct" else
                                      "matrix-free Jacobi-PCG / COCG solves to relative residual 1e-13"),
                       "samples": M, "l2": "state 8*M*N*nx bytes + factors 16*17*nx*n bytes per sample > L2"},
            "fine_dof_updates_per_s": dof / (ms * 1e-3), "avg_outer_iters": float(it.mean()),
            "max_outer_iters": int(it.max()), "all_converged": bool(np.all(status == 1)),
            "surrogate_build_s": t_build, "surrogate": {"m_q": sur.m_q, "P": solver.surrogate.P},
            "e2e": {"value": M / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(xi_host.nbytes),
                    "d2h_bytes_per_step": int(hm.numel() * 8), "ms_per_step": e2e_ms},
            "roofline": roof, "clocks": clocks.summary(), "cpu_baseline": cpu}
    print(json.dumps(line))


def c3_roofline(model, grid, cfg, xi_d, solver):
    """The dominant c3 kernel: the fused fine sweep + rhs of one batch
    (direct: fine2d_tma_kernel, banded forward/backward substitutions with the
    far parts on DMMA; krylov: cg_fine_kernel). Algorithmic work per
    backward-Euler step and DOF: 4 n + 1 flop (n-wide banded forward and
    backward substitutions + the D^-1 scale), x M N J nx per launch, against
    the measured DMMA peak; HBM fraction of the factor stream beside it."""
    import torch

    from paper_2510_26180_b200.device import AlphaTables, DeviceOperator, empty
    from paper_2510_26180_b200.pcgc import build_alpha_circulant

    op_all = DeviceOperator.from_model(model, xi_d)
    B = min(op_all.M, 192)
    op = op_all.select(0, B)
    N, J, n, nx = grid.n_coarse, grid.n_fine_per_coarse, model.n, model.nx
    tables = AlphaTables(build_alpha_circulant(N, cfg.alpha))
    U = solver.surrogate.predict(xi_d[:B])
    R = empty(B, N, nx)
    op.fgr(U, tables, grid, cfg.alpha, R)  # warm-up (+ factor / restage, untimed)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    op.fgr(U, tables, grid, cfg.alpha, R)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    peaks = load_peaks()
    flops = (4.0 * n + 1.0) * B * N * J * nx
    tf = flops / (ms * 1e-3) / 1e12
    return {"kernel": "fine2d_tma_kernel (banded L D L^T substitutions, DMMA far parts, TMA-streamed factors)"
                      if op.solver == "direct" else "cg_fine_kernel (Jacobi-PCG, matrix-free 5-point)",
            "bound": "tensor(dmma)", "achieved": tf, "peak": peaks.get("dmma_tflops"), "unit": "TFLOP/s",
            "frac": tf / peaks["dmma_tflops"] if peaks.get("dmma_tflops") else None,
            "algorithmic": "(4 n + 1) flop per DOF and backward-Euler step x M N J nx per launch (the banded "
                           "substitutions' work; for the Krylov variant the same useful work, so the fractions compare)",
            "ms_per_launch": ms, "samples_per_launch": B, "traffic": None}


# ---------------------------------------------------------------------------
# nonlinear models: PCGC with the simplified-Newton CGC and the
# classical parareal baseline, batched, at the reference harness settings
# ---------------------------------------------------------------------------
NL_CASES = {
    # pintuq/experiments.py:33-38 (BENCHMARK_DEFAULTS); Allen-Cahn at T = 3 instead of 30: with dT = 1 the
    # reference's own coarse Newton step from u0 fails (recorded in tests/golden/nl.npz)
    "burgers": dict(T=2.0, N=25, J=40),
    "allen-cahn": dict(T=3.0, N=30, J=48),
}


def _cpu_nl(task):
    from oracle import nonlinear_port as nlp

    m, u0, init, N, J, T = task
    return nlp.pcgc_newton(m, u0, init, N, J, T, 0.1, 1e-8, 60)["iters"]


def run_nonlinear(args):
    """Batched PCGC (and classical parareal) for Burgers1D / AllenCahn1D on the
    device from coarse-sweep initial guesses; CPU oracle (the reference's
    pure-Python path, bit-identical) on a bounded sample beside it."""
    import torch
    from concurrent.futures import ProcessPoolExecutor

    from paper_2510_26180_b200 import AllenCahn1D, Burgers1D, RngStream, SolverConfig, make_time_grid
    from paper_2510_26180_b200.nonlinear import NewtonOperator
    from paper_2510_26180_b200.parareal import parareal_solve_device
    from paper_2510_26180_b200.pcgc import pcgc_solve_device

    c = NL_CASES[args.config]
    model = Burgers1D(dx=1 / 100) if args.config == "burgers" else AllenCahn1D(dx=1 / 128)
    grid = make_time_grid(c["T"], c["N"], c["J"])
    cfg = SolverConfig(alpha=0.1, tol=1e-8, max_outer_iters=60, seed=SEED)
    M = args.samples or 4096
    xis = model.sample_parameters(M, RngStream(SEED).split(3)[1])
    op = NewtonOperator.from_model(model, xis, cfg)
    u0 = op.u0[None, None].expand(M, 1, model.nx).contiguous()

    def init():
        return op.sweep(u0, grid.deltaT, 1, nseg=grid.n_coarse)[0][:, 0].contiguous()

    def timed(fn):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = fn()
        b.record()
        torch.cuda.synchronize()
        return r, a.elapsed_time(b)

    for _ in range(max(1, args.warmup)):
        pcgc_solve_device(op, init(), grid, cfg)
    res, ms_pcgc = timed(lambda: pcgc_solve_device(op, init(), grid, cfg))
    res_p, ms_par = timed(lambda: parareal_solve_device(op, init(), grid, cfg))
    it, itp = res.iters.cpu().numpy(), res_p.iters.cpu().numpy()
    # CPU oracle: bounded sample over all cores
    cores = os.cpu_count() or 1
    U0 = init().cpu().numpy()
    n_cpu = min(M, max(cores, 2 * cores if args.config == "burgers" else cores))
    tasks = [((model.sweep_kind,) + model.sweep_params(xis[i].values), model.initial_condition(), U0[i],
              grid.n_coarse, grid.n_fine_per_coarse, grid.t_final) for i in range(n_cpu)]
    t0 = time.time()
    with ProcessPoolExecutor(cores) as ex:
        cpu_it = list(ex.map(_cpu_nl, tasks))
    cpu_s = time.time() - t0
    line = {"metric": f"PCGC solves/s, nonlinear model ({model.name})", "value": M / (ms_pcgc * 1e-3),
            "unit": "PCGC solves/s", "n_gpus": 1, "higher_is_better": True, "dtype": "f64",
            "config": {"workload": f"{model.name}: nx={model.nx}, T={grid.t_final}, N={grid.n_coarse}, "
                                   f"J={grid.n_fine_per_coarse}, alpha=0.1, tol=1e-8, coarse-sweep init",
                       "samples": M},
            "pcgc": {"ms": ms_pcgc, "iters_mean": float(it.mean()), "all_converged": bool(np.all(
                res.status.cpu().numpy() == 1)), "inner_iters_last_mean": float(res.imag.cpu().numpy().mean())},
            "parareal": {"ms": ms_par, "solves_per_s": M / (ms_par * 1e-3), "iters_mean": float(itp.mean())},
            "cpu_baseline": {"value": n_cpu / cpu_s, "unit": "PCGC solves/s", "cores": cores, "kind": "port",
                             "sample": f"first {n_cpu} samples, oracle/nonlinear_port.pcgc_newton (the reference's "
                                       f"pure-Python path, bit-identical), {cores} processes, {cpu_s:.1f} s wall",
                             "iters_match": bool(np.array_equal(np.array(cpu_it), it[:n_cpu]))}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    maybe_relaunch(a)
    if a.config in NL_CASES:
        run_nonlinear(a)
    elif a.config == "c5":
        run_c5(a)
    elif a.config == "c3" and a.impl == "b200":
        run_c3(a)
    elif a.impl == "reference":
        run_reference(a)
    else:
        run_b200(a)
