"""Nonlinear tridiagonal models on the device (Burgers, Allen-Cahn;
``pintuq/models.py:269-379``): the fused Newton backward-Euler sweeps of the
reference's compiled kernels (``pintuq/_kernels.pyx``, dispatched by
``pintuq/propagators.py:82-99``) as one CUDA kernel over many systems, and
the classical parareal loop on top of them (``pintuq/parareal.py:100-191``).

``NewtonOperator`` plays the role ``DeviceOperator`` plays for the linear
models: per-sample parameters resident on the device and a ``sweep`` over
(sample, start) systems. Non-convergence maps to the reference's
``NonConvergenceError`` (status = first failing step, ``propagators.py:94-98``).
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .core import NonConvergenceError, ParameterSample, SolverConfig, TimeGrid
from .device import empty, ptr, require_cuda, stream_ptr, to_dev, torch


def is_newton_model(model) -> bool:
    return getattr(model, "sweep_kind", None) is not None and not getattr(model, "is_linear", False)


class NewtonOperator:
    """M samples of a nonlinear tridiagonal model resident on the device."""

    def __init__(self, model, p0, newton_tol: float, max_newton: int):
        self.model = model
        self.kind = int(model.sweep_kind)
        self.p0 = p0  # (M,) nu or eps
        self.M = int(p0.shape[0])
        self.nx = int(model.nx)
        _, self.dx, self.bc_lo, self.bc_hi = model.sweep_params(np.array([model.supports[0][0]]))
        self.newton_tol = float(newton_tol)
        self.max_newton = int(max_newton)
        self.u0 = to_dev(np.asarray(model.initial_condition(None), dtype=float))

    @classmethod
    def from_model(cls, model, xis, cfg: SolverConfig):
        require_cuda()
        if isinstance(xis, ParameterSample):
            xis = [xis]
        vals = [x.values if isinstance(x, ParameterSample) else np.atleast_1d(np.asarray(x, float)) for x in xis]
        p0 = np.array([model.sweep_params(v)[0] for v in vals], dtype=float)
        return cls(model, to_dev(p0), cfg.newton_tol, cfg.max_newton_iters)

    def sweep(self, start, h: float, J: int, nseg: int = 1, active=None, raise_on_fail: bool = True):
        """start: (M, Q, nx) device tensor -> (M, Q, nseg, nx), status (M, Q)."""
        M, Q, nx = start.shape
        out = empty(M, Q, nseg, nx)
        status = torch.zeros(M, Q, dtype=torch.int32, device="cuda")
        nbytes = int(_lib.query("kle_newton_work_bytes", M, Q, nx))
        work = torch.empty(max(nbytes, 8), dtype=torch.uint8, device="cuda")
        _lib.call("kle_newton_sweep_f64", self.kind, ptr(start.contiguous()), ptr(out), ptr(self.p0), M, Q, nx, J,
                  nseg, float(h), self.dx, self.bc_lo, self.bc_hi, self.newton_tol, self.max_newton, ptr(active),
                  ptr(status), ptr(work), nbytes, stream_ptr())
        if raise_on_fail:
            st = status.cpu().numpy()
            if st.any():
                i, q = np.argwhere(st)[0]
                raise NonConvergenceError(
                    f"Newton failed in fused sweep at step {int(st[i, q])}/{J * nseg} (dt={h})",
                    last_iterate=out[i, q, -1].cpu().numpy(),
                )
        return out, status


# ---------------------------------------------------------------------------
# classical parareal for the nonlinear models (batched)
# ---------------------------------------------------------------------------
def parareal_solve_newton(op: NewtonOperator, U, grid: TimeGrid, cfg: SolverConfig, reference=None,
                          stop_on: str = "increment"):
    """Batched ``parareal_solve`` (``pintuq/parareal.py:100-191``) for the M
    samples of ``op``; U (M, N, nx) initial guesses, overwritten. Fine ends
    and the N sequential coarse steps are Newton sweeps on the device; the
    correction U_n = (G(U_{n-1}^new) + F_n) - G(U_{n-1}^old) and the stop
    tests run as device kernels with per-sample freezing."""
    from .pcgc import BatchResult

    if stop_on not in ("increment", "reference"):
        raise ValueError(f"stop_on must be 'increment' or 'reference', not {stop_on!r}")
    if stop_on == "reference" and reference is None:
        raise ValueError("stop_on='reference' requires a reference trajectory")
    M, N, nx = U.shape
    if N != grid.n_coarse or nx != op.nx or M != op.M:
        raise ValueError("initial guess length does not match the time grid")
    K = cfg.max_outer_iters
    status = torch.zeros(M, dtype=torch.int32, device="cuda")
    iters = torch.zeros(M, dtype=torch.int32, device="cuda")
    inc_km = torch.full((K, M), float("nan"), dtype=torch.float64, device="cuda")  # row k-1: increments of k
    inc_rec = torch.full((M, K + 1, N), float("nan"), dtype=torch.float64, device="cuda")
    ref = err = me = None
    stop_ref = int(stop_on == "reference")
    if reference is not None:
        ref = to_dev(reference).contiguous()
        err = torch.full((M, K + 1, N), float("nan"), dtype=torch.float64, device="cuda")
        me = empty(M)
        _lib.call("kle_err_ref_f64", ptr(U), ptr(ref), M, N, nx, 0, K, cfg.tol, stop_ref, ptr(status), ptr(iters),
                  None, ptr(err), ptr(me), stream_ptr())
    u0b = op.u0[None, None].expand(M, 1, nx).contiguous()

    def starts(V):
        return torch.cat([u0b, V[:, :-1]], dim=1).contiguous()

    def n_active():
        return int(np.count_nonzero(status.cpu().numpy() == 0))

    G_prev, _ = op.sweep(starts(U), grid.deltaT, 1, active=status)
    G_prev = G_prev[:, :, 0].contiguous()
    k_done = 0
    for k in range(1, K + 1):
        if n_active() == 0:
            break
        k_done = k
        U_old = U.clone()
        F, _ = op.sweep(starts(U), grid.deltat, grid.n_fine_per_coarse, active=status)
        F = F[:, :, 0].contiguous()
        prev = u0b
        for n in range(N):
            Gn, _ = op.sweep(prev, grid.deltaT, 1, active=status)
            _lib.call("kle_para_combine_f64", ptr(U), ptr(Gn), ptr(F), ptr(G_prev), ptr(status), M, N, nx, n,
                      stream_ptr())
            prev = U[:, n:n + 1].contiguous()
        # the increment max|U_new - U_old| (pintuq/parareal.py:181) is an error
        # record against the previous iterate; it stops samples for stop_on="increment"
        _lib.call("kle_err_ref_f64", ptr(U), ptr(U_old), M, N, nx, k, K, cfg.tol, 1 - stop_ref, ptr(status),
                  ptr(iters), None, ptr(inc_rec), ptr(inc_km[k - 1]), stream_ptr())
        if ref is not None:
            _lib.call("kle_err_ref_f64", ptr(U), ptr(ref), M, N, nx, k, K, cfg.tol, stop_ref, ptr(status),
                      ptr(iters), None, ptr(err), ptr(me), stream_ptr())
    # samples still active after max_outer_iters: MaxItersExceeded (non-finite if the increment is NaN)
    st, it = status.cpu().numpy(), iters.cpu().numpy()
    last = inc_km[max(k_done - 1, 0)].cpu().numpy()
    still = st == 0
    st[still & ~np.isfinite(last)] = 3
    st[still & np.isfinite(last)] = 2
    it[still] = k_done
    status.copy_(torch.as_tensor(st))
    iters.copy_(torch.as_tensor(it))
    return BatchResult(U, iters, status, inc_km.t().contiguous(), torch.zeros(M, dtype=torch.float64, device="cuda"),
                       err, me)


# ---------------------------------------------------------------------------
# PCGC for the nonlinear models (batched): Newton fine / coarse sweeps and the
# simplified-Newton diagonalised CGC (pintuq/pcgc.py:245-270)
# ---------------------------------------------------------------------------
def pcgc_solve_newton(op: NewtonOperator, U, grid: TimeGrid, cfg: SolverConfig, reference=None,
                      stop_on: str = "increment"):
    """Batched ``pcgc_solve`` (``pintuq/pcgc.py:273-358``) for the M samples
    of a nonlinear model; U (M, N, nx) initial guesses, overwritten. Per outer
    iteration: the N fine Newton sweeps, the N coarse Newton steps of
    ``assemble_rhs_blocks`` (b = F - G(prev), prev = [alpha U_N, U_1..]),
    then ``kle_newton_cgc_f64`` (one CTA per sample runs the whole simplified
    Newton loop). ``BatchResult.imag`` carries the per-sample inner iteration
    count of the last correction (the reference's ``diag["inner_iters"]``)."""
    from .device import AlphaTables
    from .pcgc import BatchResult, build_alpha_circulant

    if stop_on not in ("increment", "reference"):
        raise ValueError(f"stop_on must be 'increment' or 'reference', not {stop_on!r}")
    if stop_on == "reference" and reference is None:
        raise ValueError("stop_on='reference' requires a reference trajectory")
    M, N, nx = U.shape
    if N != grid.n_coarse or nx != op.nx or M != op.M:
        raise ValueError("initial guess length does not match the time grid")
    K = cfg.max_outer_iters
    tables = AlphaTables(build_alpha_circulant(N, cfg.alpha))
    status = torch.zeros(M, dtype=torch.int32, device="cuda")
    iters = torch.zeros(M, dtype=torch.int32, device="cuda")
    inner = torch.zeros(M, dtype=torch.int32, device="cuda")
    inc_km = torch.full((K, M), float("nan"), dtype=torch.float64, device="cuda")
    inc_rec = torch.full((M, K + 1, N), float("nan"), dtype=torch.float64, device="cuda")
    ref = err = me = None
    stop_ref = int(stop_on == "reference")
    if reference is not None:
        ref = to_dev(reference).contiguous()
        err = torch.full((M, K + 1, N), float("nan"), dtype=torch.float64, device="cuda")
        me = empty(M)
        _lib.call("kle_err_ref_f64", ptr(U), ptr(ref), M, N, nx, 0, K, cfg.tol, stop_ref, ptr(status), ptr(iters),
                  None, ptr(err), ptr(me), stream_ptr())
    u0b = op.u0[None, None].expand(M, 1, nx).contiguous()
    b = empty(M, N, nx)
    k_done = 0
    for k in range(1, K + 1):
        if int(np.count_nonzero(status.cpu().numpy() == 0)) == 0:
            break
        k_done = k
        U_old = U.clone()
        F, _ = op.sweep(torch.cat([u0b, U_old[:, :-1]], dim=1).contiguous(), grid.deltat, grid.n_fine_per_coarse,
                        active=status)
        last = empty(M, 1, nx)
        _lib.call("kle_axpby_f64", ptr(U_old[:, -1:].contiguous()), ptr(U_old[:, -1:].contiguous()), ptr(last),
                  cfg.alpha, 0.0, M * nx, stream_ptr())
        G, _ = op.sweep(torch.cat([last, U_old[:, :-1]], dim=1).contiguous(), grid.deltaT, 1, active=status)
        _lib.call("kle_axpby_f64", ptr(F[:, :, 0].contiguous()), ptr(G[:, :, 0].contiguous()), ptr(b), 1.0, -1.0,
                  M * N * nx, stream_ptr())
        _lib.call("kle_newton_cgc_f64", op.kind, ptr(U_old), ptr(b), ptr(U), ptr(op.p0), ptr(tables.lam),
                  ptr(tables.scaling), ptr(tables.inv_scaling), M, N, nx, grid.deltaT, op.dx, op.bc_lo, op.bc_hi,
                  op.newton_tol, ptr(status), ptr(inner), stream_ptr())
        st_h = status.cpu().numpy()
        failed = (st_h == 4) & (iters.cpu().numpy() == 0)
        if failed.any():  # the simplified Newton stalled in this iteration (pcgc.py:264-269)
            it_h = iters.cpu().numpy()
            it_h[failed] = k
            iters.copy_(torch.as_tensor(it_h))
        _lib.call("kle_err_ref_f64", ptr(U), ptr(U_old), M, N, nx, k, K, cfg.tol, 1 - stop_ref, ptr(status),
                  ptr(iters), None, ptr(inc_rec), ptr(inc_km[k - 1]), stream_ptr())
        if ref is not None:
            _lib.call("kle_err_ref_f64", ptr(U), ptr(ref), M, N, nx, k, K, cfg.tol, stop_ref, ptr(status),
                      ptr(iters), None, ptr(err), ptr(me), stream_ptr())
    st, it = status.cpu().numpy(), iters.cpu().numpy()
    lastinc = inc_km[max(k_done - 1, 0)].cpu().numpy()
    still = st == 0
    st[still & ~np.isfinite(lastinc)] = 3
    st[still & np.isfinite(lastinc)] = 2
    it[still] = k_done
    status.copy_(torch.as_tensor(st))
    iters.copy_(torch.as_tensor(it))
    return BatchResult(U, iters, status, inc_km.t().contiguous(), inner.to(torch.float64), err, me)
