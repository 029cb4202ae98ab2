"""Per-sample restatement of the reference KLE-CGC path (test oracle only).

Every function performs the same floating-point operations, through the same
numpy/scipy calls and in the same order, as the reference function it cites,
so its output equals the reference's bit-for-bit (checked against the golden
vectors generated from the unmodified reference: tests/golden/make_golden.py).

Inputs are plain arrays: a sample is described by its tridiagonal operator
``(dia, off)`` (A = tridiag(off, dia, off)), or the 2D 5-point stencil
``(dia, ex, ey)`` (``SampleOperator.from_stencil2d``), and a constant source
vector ``g`` (the linear_system contract, ``pintuq/models.py:114-116``,
specialised to the time-independent sources of the BASELINE models).
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
from scipy.linalg import solve_banded


class SampleOperator:
    """A, g and the cached SuperLU factors of (I + h A) for one sample
    (``pintuq/propagators.py:17-34`` caches per (sample, step))."""

    def __init__(self, dia, off, g, A=None):
        self.nx = len(dia) if A is None else A.shape[0]
        self.A = sp.diags([off, dia, off], [-1, 0, 1], format="csc") if A is None else sp.csc_matrix(A)
        self.g = np.asarray(g, dtype=float)
        self._lu = {}

    @classmethod
    def from_stencil2d(cls, dia, ex, ey, n, g):
        """2D 5-point operator (LogNormalKL2D.stencil layout): the wider-band
        sample of the same plugin contract."""
        A = sp.diags([ey[:-n], ex[:-1], dia, ex[:-1], ey[:-n]], [-n, -1, 0, 1, n], format="csc")
        return cls(None, None, g, A=A)

    def lu(self, h):
        key = float(h)
        if key not in self._lu:
            # pintuq/propagators.py:32
            self._lu[key] = spla.splu((sp.eye(self.nx, format="csc") + h * self.A).tocsc())
        return self._lu[key]

    def be_step(self, u, h):
        # pintuq/propagators.py:37-39 (g is time independent here)
        return self.lu(h).solve(u + h * self.g)


def fine(op: SampleOperator, u, J: int, dt: float):
    """F: J backward-Euler steps (``pintuq/propagators.py:121-145``)."""
    v = u
    for _ in range(J):
        v = op.be_step(v, dt)
    return v


def coarse(op: SampleOperator, u, dT: float):
    """G: one backward-Euler step of dT (``pintuq/propagators.py:148-157``)."""
    return op.be_step(u, dT)


def alpha_circulant(n: int, alpha: float):
    """(eigenvalues, scaling) of C_alpha (``pintuq/pcgc.py:68-76``)."""
    root = alpha ** (1.0 / n)
    lam = 1.0 - root * np.exp(-2j * np.pi * np.arange(n) / n)
    scaling = alpha ** (np.arange(n) / n)
    return lam, scaling


def shifted_solvers(op: SampleOperator, lam, dT: float):
    """Banded closures for (lam_n I + dT A) (``pintuq/pcgc.py:112-135``)."""
    J = sp.csr_matrix(-op.A)
    nx = J.shape[0]
    if nx == 1:
        jval = complex(J[0, 0])
        return [lambda p, d=(l - dT * jval): p / d for l in lam]
    coo = J.tocoo()
    if int(np.max(np.abs(coo.row - coo.col))) > 1:
        # wider band (2D): one complex SuperLU per eigenvalue (pcgc.py:137-145)
        eye = sp.eye(nx, format="csc", dtype=complex)
        shift = (dT * J.tocsc()).astype(complex)
        return [spla.splu((l * eye - shift).tocsc()).solve for l in lam]
    sub = -dT * J.diagonal(-1)
    dia = dT * J.diagonal(0)
    sup = -dT * J.diagonal(1)
    out = []
    for l in lam:
        ab = np.zeros((3, nx), dtype=complex)
        ab[0, 1:] = sup
        ab[1, :] = l - dia
        ab[2, :-1] = sub
        out.append(lambda p, ab=ab: solve_banded((1, 1), ab, p))
    return out


def three_step(lam, scaling, solvers, r):
    """Scaled DFT, N shifted solves, inverse (``pintuq/pcgc.py:148-172``).
    Returns (u real, max|Im u|)."""
    p = np.fft.fft(scaling[:, None] * r, axis=0, norm="ortho")
    q = np.array([solvers[n](p[n]) for n in range(len(lam))])
    u = (1.0 / scaling)[:, None] * np.fft.ifft(q, axis=0, norm="ortho")
    return np.ascontiguousarray(u.real), float(np.max(np.abs(u.imag)))


def cgc(op: SampleOperator, lam, scaling, solvers, alpha, dT, U, F_ends):
    """Linear coarse-grid correction (``pintuq/pcgc.py:175-197, 226-243``)."""
    N = U.shape[0]
    prev = np.vstack([alpha * U[-1], U[:-1]])
    b = np.array([F_ends[n] - coarse(op, prev[n], dT) for n in range(N)])
    rhs = np.empty_like(b)
    for n in range(N):
        rhs[n] = dT * (op.A @ b[n] + op.g) + b[n]
    return three_step(lam, scaling, solvers, rhs)


def coarse_sweep(op: SampleOperator, u0, N: int, dT: float):
    """N serial G steps from u0 (``pintuq/parareal.py:74-84``)."""
    out = np.empty((N, op.nx))
    v = u0
    for n in range(N):
        v = coarse(op, v, dT)
        out[n] = v
    return out


def fine_reference(op: SampleOperator, u0, N: int, J: int, dT: float):
    """Serial F trajectory (``pintuq/propagators.py:160-176``)."""
    out = np.empty((N, op.nx))
    v = u0
    for n in range(N):
        v = fine(op, v, J, dT / J)
        out[n] = v
    return out


def pcgc(op: SampleOperator, u0, init_states, N, J, T, alpha, tol, max_iters,
         keep_history=False, reference=None, stop_on="increment"):
    """Outer PCGC loop (``pintuq/pcgc.py:273-358``): increment stopping, or
    with ``reference`` (N, nx) the error records of ``_error_record``
    (``pintuq/parareal.py:87-91``) and, for stop_on="reference", stopping at
    the first record (k = 0 included, ``pcgc.py:312-316``) with max error <= tol.

    Returns dict(states, iters, converged, increments, imag, history, err, max_err)."""
    dT = T / N
    dt = dT / J
    lam, scaling = alpha_circulant(N, alpha)
    solvers = shifted_solvers(op, lam, dT)
    U = np.array(init_states, dtype=float, copy=True)
    increments, hist = [], [U.copy()] if keep_history else []
    errs = []

    def record(V):
        if reference is not None:
            errs.append(np.max(np.abs(V - reference), axis=1))
            return float(np.max(errs[-1]))
        return None

    imag = 0.0
    converged = False
    me = record(U)
    if stop_on == "reference" and me is not None and me <= tol:
        converged = True
        max_iters = 0
    for _k in range(1, max_iters + 1):
        starts = np.vstack([u0, U[:-1]])
        F_ends = np.array([fine(op, starts[n], J, dt) for n in range(N)])
        U_new, im = cgc(op, lam, scaling, solvers, alpha, dT, U, F_ends)
        inc = float(np.max(np.abs(U_new - U)))
        U = U_new
        imag = max(imag, im)
        increments.append(inc)
        me = record(U)
        if keep_history:
            hist.append(U.copy())
        metric = inc if stop_on == "increment" else me
        if metric <= tol:
            converged = True
            break
    err = np.array(errs) if reference is not None else None
    return dict(states=U, iters=len(increments), converged=converged,
                increments=np.array(increments), imag=imag, history=hist, err=err,
                max_err=None if err is None else err.max(axis=1))


def parareal(op: SampleOperator, u0, init_states, N, J, T, tol, max_iters, reference=None,
             stop_on="increment"):
    """Classical parareal (``pintuq/parareal.py:100-191``): sequential coarse
    correction U_n = G(U_{n-1}^new) + F(U_{n-1}^old) - G(U_{n-1}^old).

    Returns dict(states, iters, converged, increments, err, max_err)."""
    dT = T / N
    dt = dT / J
    U = np.array(init_states, dtype=float, copy=True)
    increments, errs = [], []

    def record(V):
        if reference is not None:
            errs.append(np.max(np.abs(V - reference), axis=1))
            return float(np.max(errs[-1]))
        return None

    def starts(V):
        return np.vstack([u0, V[:-1]])

    converged = False
    me = record(U)
    if stop_on == "reference" and me is not None and me <= tol:
        converged = True
        max_iters = 0
    cur = starts(U)
    G_prev = np.array([coarse(op, cur[n], dT) for n in range(N)]) if max_iters else None
    for _k in range(1, max_iters + 1):
        fs = starts(U)
        F_ends = np.array([fine(op, fs[n], J, dt) for n in range(N)])
        U_new = np.empty_like(U)
        G_new = np.empty_like(U)
        prev = u0
        for n in range(N):
            G_new[n] = coarse(op, prev, dT)
            U_new[n] = G_new[n] + F_ends[n] - G_prev[n]
            prev = U_new[n]
        inc = float(np.max(np.abs(U_new - U)))
        U, G_prev = U_new, G_new
        increments.append(inc)
        me = record(U)
        metric = inc if stop_on == "increment" else me
        if metric <= tol:
            converged = True
            break
    err = np.array(errs) if reference is not None else None
    return dict(states=U, iters=len(increments), converged=converged, increments=np.array(increments), err=err,
                max_err=None if err is None else err.max(axis=1))


# ---------------------------------------------------------------------------
# Hermite gPC surrogate (pintuq/surrogate.py:144-333)
# ---------------------------------------------------------------------------
def multi_indices(degree: int, dim: int) -> list:
    """Graded, reverse-lexicographic within degree (``surrogate.py:194-205``)."""
    out = []

    def rec(prefix, remaining, slots):
        if slots == 1:
            out.append(prefix + (remaining,))
            return
        for v in range(remaining, -1, -1):
            rec(prefix + (v,), remaining - v, slots - 1)

    for total in range(degree + 1):
        rec((), total, dim)
    return out


def hermite_table(x, degree: int):
    """Orthonormal probabilists' Hermite values (``surrogate.py:222-233``)."""
    x = np.asarray(x, dtype=float)
    T = np.empty((degree + 1,) + x.shape)
    T[0] = 1.0
    if degree >= 1:
        T[1] = x
    for k in range(1, degree):
        T[k + 1] = x * T[k] - k * T[k - 1]
    norms = np.array([1.0 / math.sqrt(math.factorial(k)) for k in range(degree + 1)])
    return T * norms.reshape((-1,) + (1,) * x.ndim)


def basis_matrix(points, degree: int):
    """Psi (n, P) in multi-index column order (``surrogate.py:236-248``)."""
    points = np.atleast_2d(np.asarray(points, dtype=float))
    n, dim = points.shape
    tabs = [hermite_table(points[:, d], degree) for d in range(dim)]
    idx = multi_indices(degree, dim)
    B = np.ones((n, len(idx)))
    for col, k in enumerate(idx):
        for d, kd in enumerate(k):
            if kd:
                B[:, col] *= tabs[d][kd]
    return B


def kl_build(fields, cell_weight, eps_kl):
    """Snapshot-method KL (``surrogate.py:59-64, 144-171``).
    Returns (mean, retained eigenvalues, modes (m_q, N, nx), X fluctuations)."""
    fields = np.asarray(fields, dtype=float)
    mean = fields.mean(axis=0)
    fl = fields - mean
    n_t = fields.shape[0]
    X = fl.reshape(n_t, -1)
    C = (cell_weight / n_t) * (X @ X.T)
    lam, E = np.linalg.eigh(C)
    lam = np.clip(lam[::-1], 0.0, None)
    E = E[:, ::-1]
    total = float(np.sum(lam))
    mean_energy = cell_weight * float(np.sum(mean ** 2))
    if total <= 1e-26 * max(mean_energy, 1.0):
        return mean, lam[:0], np.empty((0,) + fields.shape[1:]), X
    ratios = np.cumsum(lam) / total
    m_energy = int(np.searchsorted(ratios, 1.0 - eps_kl) + 1)
    m_floor = int(np.sum(lam > 1e-14 * lam[0]))
    m_q = min(m_energy, m_floor)
    scale = 1.0 / np.sqrt(lam[:m_q] * n_t)
    modes = (scale[:, None] * (E[:, :m_q].T @ X)).reshape((m_q,) + fields.shape[1:])
    return mean, lam[:m_q].copy(), modes, X


def kl_coefficients(X, modes, lam, cell_weight):
    """zeta (n_t, m_q) (``surrogate.py:174-184``)."""
    G = modes.reshape(modes.shape[0], -1)
    return cell_weight * (X @ G.T) / np.sqrt(lam)[None, :]


def gpc_fit(points, zeta, degree):
    """Least squares on the Hermite basis (``surrogate.py:264-288``);
    returns coeffs (m_q, P)."""
    B = basis_matrix(points, degree)
    coeffs, _, rank, _ = np.linalg.lstsq(B, zeta, rcond=None)
    if rank < B.shape[1]:
        raise RuntimeError("rank deficient gPC regression")
    return coeffs.T


def surrogate_predict(mean, lam, modes, coeffs, degree, xi):
    """U0 = mean + sum_i sqrt(lam_i) (H psi)_i g_i (``surrogate.py:321-333``)."""
    pred = mean.copy()
    if modes.shape[0]:
        psi = basis_matrix(np.atleast_2d(xi), degree)[0]
        zeta_hat = coeffs @ psi
        weights = np.sqrt(lam) * zeta_hat
        pred = pred + (weights @ modes.reshape(modes.shape[0], -1)).reshape(mean.shape)
    return pred
