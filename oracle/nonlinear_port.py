"""Restatement of the reference's nonlinear-model path (test oracle and CPU
baseline only): the pure-Python Newton sweeps (``pintuq/_kernels_fallback.py``,
selected by ``PINTUQ_PURE_PYTHON``, the backend the golden vectors were made
with), the simplified-Newton CGC (``pintuq/pcgc.py:245-270`` with the banded
``factor_shifted`` branch :112-135 and ``three_step_solve`` :148-172) and the
classical / PCGC outer loops, with the same numpy / scipy calls in the same
order, so the results equal the reference's bit for bit (pinned in
tests/test_oracle.py against tests/golden/nl.npz).

Models are described by (kind, p0, dx, bc_lo, bc_hi): kind 0 Burgers
(p0 = nu), kind 1 Allen-Cahn (p0 = eps).
"""
from __future__ import annotations

import numpy as np
from scipy.linalg import solve_banded


def bands(kind, p0, dx, bc_lo, bc_hi, v):
    """f(v) and the Jacobian bands (sub, diag, sup) — the rhs_bands closures
    of ``_kernels_fallback.py:57-88``."""
    left = np.concatenate(([0.0], v[:-1]))
    right = np.concatenate((v[1:], [0.0]))
    if kind == 0:
        nu = p0
        up = v >= 0.0
        dudx = np.where(up, (v - left) / dx, (right - v) / dx)
        f = -v * dudx + nu * (left - 2.0 * v + right) / dx**2
        diag = np.where(up, -(2.0 * v - left) / dx, -(right - 2.0 * v) / dx) - 2.0 * nu / dx**2
        sub = np.where(up[1:], v[1:] / dx, 0.0) + nu / dx**2
        sup = np.where(up[:-1], 0.0, -v[:-1] / dx) + nu / dx**2
        return f, sub, diag, sup
    eps = p0
    lift = np.zeros(v.shape[0])
    lift[0] = bc_lo / dx**2
    lift[-1] = bc_hi / dx**2
    f = eps * ((left - 2.0 * v + right) / dx**2 + lift) - (v**3 - v)
    diag = -2.0 * eps / dx**2 - (3.0 * v**2 - 1.0)
    off = np.full(v.shape[0] - 1, eps / dx**2)
    return f, off, diag, off


def newton_step(kind, p0, dx, bc_lo, bc_hi, u, dt, tol, max_newton):
    """One backward-Euler step by damped Newton (``_kernels_fallback.py:13-47``):
    returns (v, converged)."""
    v = u.copy()
    ab = np.zeros((3, u.shape[0]))
    f, sub, diag, sup = bands(kind, p0, dx, bc_lo, bc_hi, v)
    r = v - u - dt * f
    rn, r2 = np.max(np.abs(r)), np.linalg.norm(r)
    for it in range(max_newton + 1):
        if rn <= tol:
            return v, True
        if it == max_newton:
            break
        ab[0, 1:] = -dt * sup
        ab[1, :] = 1.0 - dt * diag
        ab[2, :-1] = -dt * sub
        delta = solve_banded((1, 1), ab, -r)
        t = 1.0
        while True:
            v_t = v + t * delta
            f, sub, diag, sup = bands(kind, p0, dx, bc_lo, bc_hi, v_t)
            r_t = v_t - u - dt * f
            r2_t = np.linalg.norm(r_t)
            if r2_t <= (1.0 - 1e-4 * t) * r2 or t <= 2.0**-20:
                break
            t *= 0.5
        v, r, r2 = v_t, r_t, r2_t
        rn = np.max(np.abs(r))
    return v, False


def sweep(m, u, dt, nsteps, tol=1e-12, max_newton=50):
    """``be_sweep_*`` (``_kernels_fallback.py:50-90``): (state, status)."""
    u = np.array(u, dtype=float, copy=True)
    for step in range(nsteps):
        u, ok = newton_step(*m, u, dt, tol, max_newton)
        if not ok:
            return u, step + 1
    return u, 0


def _prop(m, u, dt, nsteps, tol, max_newton):
    out, status = sweep(m, u, dt, nsteps, tol, max_newton)
    if status:
        raise RuntimeError(f"Newton failed at step {status}/{nsteps}")
    return out


from .ref_port import alpha_circulant  # noqa: E402  (build_alpha_circulant, pcgc.py:68-76; pinned bitwise)


def coarse_dt(T, N, n):
    """The coarse step of block n as the reference forms it: propagate_coarse
    steps t_to - t_from = T_{n+1} - T_n (``propagators.py:148-157``, grid
    points n * deltaT, ``core.py:76-78``), which differs from deltaT in the
    last bit when deltaT is not a power of two."""
    dT = T / N
    return (n + 1) * dT - n * dT


def mean_jacobian(m, U, b, N):
    """(sum_n J(U_n - b_n)) / N as bands (sub, diag, sup) and the F_l rows
    (``pcgc.py:252-259``; scipy sparse sums are elementwise in n order)."""
    Fl = np.empty_like(U)
    acc = None
    for i in range(N):
        f, sub, diag, sup = bands(*m, U[i] - b[i])
        Fl[i] = f
        acc = (sub.copy(), diag.copy(), sup.copy()) if acc is None else (acc[0] + sub, acc[1] + diag, acc[2] + sup)
    inv = 1.0 / N  # scipy sparse / scalar multiplies by the reciprocal
    return Fl, (acc[0] * inv, acc[1] * inv, acc[2] * inv)


def three_step_tridiag(lam, scaling, J, dT, r):
    """``three_step_solve`` with the banded shifted solvers (``pcgc.py:112-135,
    148-172``) for a tridiagonal J given as (sub, diag, sup)."""
    sub_j, dia_j, sup_j = J
    N, nx = r.shape
    sub = -dT * sub_j
    dia = dT * dia_j
    sup = -dT * sup_j
    p = np.fft.fft(scaling[:, None] * r, axis=0, norm="ortho")
    q = np.empty_like(p)
    for n in range(N):
        ab = np.zeros((3, nx), dtype=complex)
        ab[0, 1:] = sup
        ab[1, :] = lam[n] - dia
        ab[2, :-1] = sub
        q[n] = solve_banded((1, 1), ab, p[n])
    u = (1.0 / scaling)[:, None] * np.fft.ifft(q, axis=0, norm="ortho")
    return np.ascontiguousarray(u.real)


def cgc_newton(m, lam, scaling, N, dT, U_prev, b, newton_tol, cap=150):
    """Simplified Newton with the averaged Jacobian (``pcgc.py:245-270``):
    (U_new, inner iterations)."""
    u_l = U_prev.copy()
    for inner in range(1, cap + 1):
        Fl, J = mean_jacobian(m, u_l, b, N)
        Ju = np.empty_like(u_l)
        for n in range(N):  # (mean_jac @ u_l.T).T as a banded product
            x = u_l[n]
            y = J[1] * x
            y[1:] = J[0] * x[:-1] + y[1:]
            y[:-1] = y[:-1] + J[2] * x[1:]
            Ju[n] = y
        rhs = dT * (Fl - Ju) + b
        u_next = three_step_tridiag(lam, scaling, J, dT, rhs)
        inc = float(np.max(np.abs(u_next - u_l)))
        u_l = u_next
        if inc <= newton_tol:
            return u_l, inner
    raise RuntimeError("simplified Newton stalled")


def pcgc_newton(m, u0, init, N, J, T, alpha, tol, max_iters, newton_tol=1e-12, max_newton=50):
    """Outer PCGC loop for a nonlinear model (``pcgc.py:273-358``)."""
    dT = T / N
    dt = dT / J
    lam, scaling = alpha_circulant(N, alpha)
    U = np.array(init, dtype=float, copy=True)
    incs = []
    for _k in range(1, max_iters + 1):
        starts = np.vstack([u0, U[:-1]])
        F = np.array([_prop(m, starts[n], dt, J, newton_tol, max_newton) for n in range(N)])
        prev = np.vstack([alpha * U[-1:], U[:-1]])
        G = np.array([_prop(m, prev[n], coarse_dt(T, N, n), 1, newton_tol, max_newton) for n in range(N)])
        U_new, _ = cgc_newton(m, lam, scaling, N, dT, U, F - G, newton_tol)
        inc = float(np.max(np.abs(U_new - U)))
        U = U_new
        incs.append(inc)
        if inc <= tol:
            return dict(states=U, iters=len(incs), increments=np.array(incs), converged=True)
    return dict(states=U, iters=len(incs), increments=np.array(incs), converged=False)


def parareal_newton(m, u0, init, N, J, T, tol, max_iters, newton_tol=1e-12, max_newton=50):
    """Classical parareal for a nonlinear model (``parareal.py:100-191``)."""
    dT = T / N
    dt = dT / J
    U = np.array(init, dtype=float, copy=True)
    starts = np.vstack([u0, U[:-1]])
    G_prev = np.array([_prop(m, starts[n], coarse_dt(T, N, n), 1, newton_tol, max_newton) for n in range(N)])
    incs = []
    for _k in range(1, max_iters + 1):
        starts = np.vstack([u0, U[:-1]])
        F = np.array([_prop(m, starts[n], dt, J, newton_tol, max_newton) for n in range(N)])
        U_new, G_new = np.empty_like(U), np.empty_like(U)
        prev = u0
        for n in range(N):
            G_new[n] = _prop(m, prev, coarse_dt(T, N, n), 1, newton_tol, max_newton)
            U_new[n] = G_new[n] + F[n] - G_prev[n]
            prev = U_new[n]
        inc = float(np.max(np.abs(U_new - U)))
        U, G_prev = U_new, G_new
        incs.append(inc)
        if inc <= tol:
            return dict(states=U, iters=len(incs), increments=np.array(incs), converged=True)
    return dict(states=U, iters=len(incs), increments=np.array(incs), converged=False)
