"""Drop-in for ``pintuq.parareal`` (``/root/reference/pkg/src/pintuq/parareal.py``):
the trace types, the initial guesses and the classical parareal solver,
the paper's comparison baseline, on the device.

``parareal_solve`` keeps the reference signature and semantics
(:100-191); each outer iteration is one fine-sweep launch (``fgr_kernel``
writing the F ends) and one sequential coarse-correction launch
(``kle_parareal_step_f64``). ``parareal_solve_device`` runs the whole loop
for M samples at once (``kle_parareal_solve_f64``), each sample frozen at
its own iteration count. Linear tridiagonal (1D) models.
"""
from __future__ import annotations

import time

import numpy as np

from . import _lib
from .core import (CoarseTrajectory, IterationRecord, IterationTrace, MaxItersExceededError, ParameterSample,
                   SolverConfig, TimeGrid)
from .device import DeviceOperator, empty, ptr, stream_ptr, to_dev, torch
from .pcgc import BatchResult
from .propagators import coarse_sweep_init, fine_reference, random_guess_init

__all__ = ["IterationRecord", "IterationTrace", "coarse_sweep_init", "fine_reference", "parareal_solve",
           "parareal_solve_device", "random_guess_init"]


def _check_1d(op):
    if not isinstance(op, DeviceOperator):
        raise NotImplementedError("the device parareal covers the tridiagonal (1D) operators")


def parareal_solve_device(op: DeviceOperator, U, grid: TimeGrid, cfg: SolverConfig, reference=None,
                          stop_on: str = "increment") -> BatchResult:
    """Batched ``parareal_solve`` for the M samples of ``op``: U (M, N, nx)
    (the initial guesses) is overwritten with the final states. ``op`` may be
    a ``nonlinear.NewtonOperator`` (Burgers, Allen-Cahn)."""
    from .nonlinear import NewtonOperator, parareal_solve_newton

    if isinstance(op, NewtonOperator):
        return parareal_solve_newton(op, U, grid, cfg, reference, stop_on)
    if stop_on not in ("increment", "reference"):
        raise ValueError(f"stop_on must be 'increment' or 'reference', not {stop_on!r}")
    if stop_on == "reference" and reference is None:
        raise ValueError("stop_on='reference' requires a reference trajectory")
    _check_1d(op)
    M, N, nx = U.shape
    if N != grid.n_coarse or nx != op.nx or M != op.M:
        raise ValueError("initial guess length does not match the time grid")
    nbytes = int(_lib.query("kle_parareal_workspace_bytes", M, N, nx))
    ws = torch.empty(max(nbytes, 8), dtype=torch.uint8, device="cuda")
    status = torch.empty(M, dtype=torch.int32, device="cuda")
    iters = torch.empty(M, dtype=torch.int32, device="cuda")
    inc = empty(M, cfg.max_outer_iters)
    ref = err = me = None
    if reference is not None:
        ref = to_dev(reference).contiguous()
        if tuple(ref.shape) != (M, N, nx):
            raise ValueError("reference trajectory shape does not match the initial guess")
        err = empty(M, cfg.max_outer_iters + 1, N)
        me = empty(M)
    _lib.call("kle_parareal_solve_f64", ptr(U), ptr(op.u0), ptr(op.dia), ptr(op.off), ptr(op.blob(grid.deltat)),
              ptr(op.blob(grid.deltaT)), M, N, nx, grid.n_fine_per_coarse, grid.t_final, op.g0, cfg.tol,
              cfg.max_outer_iters, ptr(ref), int(stop_on == "reference"), ptr(status), ptr(iters), ptr(inc),
              ptr(err), ptr(me), ptr(ws), nbytes, stream_ptr())
    return BatchResult(U, iters, status, inc, torch.zeros(M, dtype=torch.float64, device="cuda"), err, me)


def parareal_solve(model, xi: ParameterSample, grid: TimeGrid, cfg: SolverConfig, init: CoarseTrajectory,
                   reference: CoarseTrajectory | None = None, stop_on: str = "increment", store_states: bool = False,
                   executor=None, raise_on_max: bool = True) -> IterationTrace:
    """Single-sample drop-in for ``pintuq.parareal.parareal_solve`` (:100-191)."""
    if stop_on not in ("increment", "reference"):
        raise ValueError(f"stop_on must be 'increment' or 'reference', not {stop_on!r}")
    if stop_on == "reference" and reference is None:
        raise ValueError("stop_on='reference' requires a reference trajectory")
    if init.n_coarse != grid.n_coarse:
        raise ValueError("initial guess length does not match the time grid")
    model.validate(xi)
    from .nonlinear import NewtonOperator, is_newton_model

    if is_newton_model(model):
        return _parareal_newton_trace(model, xi, grid, cfg, init, reference, stop_on, raise_on_max)
    if not getattr(model, "is_linear", False):
        raise NotImplementedError("the device parareal covers linear and tridiagonal Newton models only")
    N = grid.n_coarse
    u0 = np.asarray(model.initial_condition(xi), dtype=float)
    op = DeviceOperator.from_model(model, [xi])
    _check_1d(op)
    nx = op.nx
    U = to_dev(init.states)[None].clone()
    F, G = empty(1, N, nx), empty(1, N, nx)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    inc = empty(1, cfg.max_outer_iters).fill_(float("nan"))

    def err(states):
        if reference is None:
            return None, None
        e = np.max(np.abs(states - reference.states), axis=1)
        return e, float(np.max(e))

    trace = IterationTrace(solver="parareal", stop_on=stop_on)
    host = np.asarray(init.states, dtype=float).copy()
    ev, me = err(host)
    trace.records.append(IterationRecord(0, None, ev, me, 0.0))
    if store_states:
        trace.states_history.append(host.copy())
    if stop_on == "reference" and me is not None and me <= cfg.tol:
        trace.converged = True
        trace.trajectory = CoarseTrajectory(u0, host)
        return trace
    fine, coarse = op.blob(grid.deltat), op.blob(grid.deltaT)
    _lib.call("kle_parareal_init_f64", ptr(U), ptr(op.u0), ptr(coarse), 1, N, nx, grid.deltaT, op.g0, ptr(G),
              stream_ptr())
    for k in range(1, cfg.max_outer_iters + 1):
        tic = time.perf_counter()
        _lib.call("kle_fgr_f64", ptr(U), ptr(op.u0), None, ptr(F), None, ptr(fine), ptr(op.dia), ptr(op.off), None,
                  None, 1, N, nx, grid.n_fine_per_coarse, grid.deltat, grid.deltaT, op.g0, 0.0, stream_ptr())
        # tol < 0 keeps the device from freezing the sample; the stop test is ours
        _lib.call("kle_parareal_step_f64", ptr(U), ptr(op.u0), ptr(F), ptr(G), ptr(coarse), 1, N, nx, grid.deltaT,
                  op.g0, k, cfg.max_outer_iters, -1.0, None, None, ptr(inc), None, stream_ptr())
        host = U[0].cpu().numpy()
        increment = float(inc[0, k - 1].item())
        wall_ms = 1e3 * (time.perf_counter() - tic)
        ev, me = err(host)
        trace.records.append(IterationRecord(k, increment, ev, me, wall_ms))
        if store_states:
            trace.states_history.append(host.copy())
        metric = increment if stop_on == "increment" else me
        if metric <= cfg.tol:
            trace.converged = True
            break
    trace.trajectory = CoarseTrajectory(u0, host)
    trace.trajectory.assert_finite()
    if not trace.converged and raise_on_max:
        raise MaxItersExceededError(
            f"parareal did not reach tol {cfg.tol:.1e} within {cfg.max_outer_iters} iterations", trace=trace
        )
    return trace


def _parareal_newton_trace(model, xi, grid, cfg, init, reference, stop_on, raise_on_max):
    """parareal_solve for one sample of a nonlinear model: the batched device
    loop with M = 1, the trace rebuilt from its records."""
    from .nonlinear import NewtonOperator, parareal_solve_newton

    u0 = np.asarray(model.initial_condition(xi), dtype=float)
    op = NewtonOperator.from_model(model, [xi], cfg)
    U = to_dev(init.states)[None].clone()
    ref = None if reference is None else to_dev(reference.states)[None]
    res = parareal_solve_newton(op, U, grid, cfg, ref, stop_on)
    k = int(res.iters[0].item())
    trace = IterationTrace(solver="parareal", stop_on=stop_on)
    errs = res.err_vs_ref[0].cpu().numpy() if res.err_vs_ref is not None else None
    incs = res.increments[0].cpu().numpy()
    for j in range(k + 1):
        ev = None if errs is None else errs[j]
        me = None if ev is None else float(np.max(ev))
        trace.records.append(IterationRecord(j, None if j == 0 else float(incs[j - 1]), ev, me, 0.0))
    trace.trajectory = CoarseTrajectory(u0, res.states[0].cpu().numpy())
    st = int(res.status[0].item())
    trace.converged = st == 1
    if st == 3:
        trace.trajectory.assert_finite()
    if not trace.converged and raise_on_max:
        raise MaxItersExceededError(
            f"parareal did not reach tol {cfg.tol:.1e} within {cfg.max_outer_iters} iterations", trace=trace
        )
    return trace
