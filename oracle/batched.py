"""Sample-batched numpy restatement of the KLE-CGC path (test oracle only).

Same algorithm as the reference (``pintuq/propagators.py:121-157``,
``pintuq/pcgc.py:148-358``, ``pintuq/surrogate.py:321-333``) vectorised over
samples: pivot-free Thomas along x instead of SuperLU / LAPACK ?gbsv (A is a
symmetric diagonally dominant M-matrix, Re lambda_n > 0, so no pivoting
occurs — SURVEY.md §8 a9), ``np.fft`` along the time axis exactly as the
reference. Pinned against ``ref_port`` (bit-faithful to the reference) in
tests/test_oracle.py.
"""
from __future__ import annotations

import numpy as np

from . import ref_port


def tridiag_from_xi(xi, kl_table, h):
    """LogNormalKL1D operator for every sample: (dia (M, nx), off (M, nx-1))."""
    a = np.exp(np.asarray(xi, dtype=float) @ kl_table)
    inv_h2 = 1.0 / (h * h)
    return (a[:, :-1] + a[:, 1:]) * inv_h2, -a[:, 1:-1] * inv_h2


def thomas(dia, off, rhs):
    """Solve tridiag(off, dia, off) x = rhs along the last axis; dia/off are
    broadcastable to rhs[..., :] / rhs[..., :-1] (real or complex)."""
    nx = rhs.shape[-1]
    dia = np.broadcast_to(dia, rhs.shape)
    off = np.broadcast_to(off, rhs.shape[:-1] + (nx - 1,))
    y = np.empty(np.broadcast_shapes(rhs.shape, dia.shape), dtype=np.result_type(dia, rhs))
    c = np.empty(y.shape[:-1] + (max(nx - 1, 1),), dtype=y.dtype)
    beta = dia[..., 0]
    y[..., 0] = rhs[..., 0] / beta
    for i in range(1, nx):
        c[..., i - 1] = off[..., i - 1] / beta
        beta = dia[..., i] - off[..., i - 1] * c[..., i - 1]
        y[..., i] = (rhs[..., i] - off[..., i - 1] * y[..., i - 1]) / beta
    for i in range(nx - 2, -1, -1):
        y[..., i] -= c[..., i] * y[..., i + 1]
    return y


def be_steps(dia, off, u, h, g0, J):
    """J backward-Euler steps of (I + hA) v = u + h g0 for u (M, Q, nx)."""
    D = 1.0 + h * dia[:, None, :]
    E = h * off[:, None, :]
    v = u
    for _ in range(J):
        v = thomas(D, E, v + h * g0)
    return v


def fine_ends(dia, off, u0, U, J, dt, g0):
    """F over every subinterval from [u0, U_1..U_{N-1}] (``pcgc.py:321-330``)."""
    starts = np.concatenate([np.broadcast_to(u0, (U.shape[0], 1, U.shape[2])), U[:, :-1]], axis=1)
    return be_steps(dia, off, starts, dt, g0, J)


def cgc(dia, off, U, F, alpha, dT, g0):
    """Linear CGC for all samples (``pcgc.py:175-243``): returns (U_new, imag)."""
    M, N, nx = U.shape
    lam, scaling = ref_port.alpha_circulant(N, alpha)
    prev = np.concatenate([alpha * U[:, -1:], U[:, :-1]], axis=1)
    G = be_steps(dia, off, prev, dT, g0, 1)
    b = F - G
    Ab = dia[:, None, :] * b
    Ab[..., :-1] += off[:, None, :] * b[..., 1:]
    Ab[..., 1:] += off[:, None, :] * b[..., :-1]
    rhs = dT * (Ab + g0) + b
    p = np.fft.fft(scaling[None, :, None] * rhs, axis=1, norm="ortho")
    Dc = lam[None, :, None] + dT * dia[:, None, :]
    q = thomas(Dc, (dT * off)[:, None, :].astype(complex), p)
    u = (1.0 / scaling)[None, :, None] * np.fft.ifft(q, axis=1, norm="ortho")
    return np.ascontiguousarray(u.real), np.max(np.abs(u.imag), axis=(1, 2))


def pcgc(dia, off, u0, init, N, J, T, alpha, tol, max_iters, g0=1.0):
    """Per-sample-frozen outer loop (``pcgc.py:319-348``)."""
    dT = T / N
    dt = dT / J
    U = np.array(init, dtype=float, copy=True)
    M = U.shape[0]
    iters = np.zeros(M, dtype=np.int32)
    incs = np.full((M, max_iters), np.nan)
    imag = np.zeros(M)
    active = np.ones(M, dtype=bool)
    for k in range(1, max_iters + 1):
        idx = np.nonzero(active)[0]
        if idx.size == 0:
            break
        F = fine_ends(dia[idx], off[idx], u0, U[idx], J, dt, g0)
        Un, im = cgc(dia[idx], off[idx], U[idx], F, alpha, dT, g0)
        inc = np.max(np.abs(Un - U[idx]), axis=(1, 2))
        U[idx] = Un
        incs[idx, k - 1] = inc
        imag[idx] = np.maximum(imag[idx], im)
        done = inc <= tol
        iters[idx[done]] = k
        active[idx[done]] = False
    iters[active] = max_iters
    return dict(states=U, iters=iters, increments=incs, imag=imag, converged=~active)


def coarse_sweep(dia, off, u0, N, dT, g0=1.0):
    M, nx = dia.shape
    out = np.empty((M, N, nx))
    v = np.broadcast_to(u0, (M, 1, nx))
    for n in range(N):
        v = be_steps(dia, off, v, dT, g0, 1)
        out[:, n] = v[:, 0]
    return out


def hermite_predict(mean, lam, modes, coeffs, degree, xi):
    """Batched surrogate_predict (``surrogate.py:321-333``)."""
    xi = np.atleast_2d(xi)
    B = ref_port.basis_matrix(xi, degree)
    zeta = B @ coeffs.T
    w = zeta * np.sqrt(lam)[None, :]
    return mean[None] + (w @ modes.reshape(modes.shape[0], -1)).reshape((xi.shape[0],) + mean.shape)


def moments(U):
    return U.mean(axis=0), U.var(axis=0)
