"""Model plugins for the KLE-CGC hot path.

The reference's plugin surface is ``LinearModel`` (``pintuq/models.py:109-125``):
a model returns ``(A, g)`` with ``rhs(u, t) = -A u + g(t)``. The BASELINE
configs need a *random-coefficient* diffusion model that the reference does
not ship, so it is added here as a ``LinearModel`` subclass:

``LogNormalKL1D``  u_t - (a(x, w) u_x)_x = f on (0, 1), zero Dirichlet,
    u0 = sin(pi x), f = 1, nx interior nodes x_i = (i+1) h, h = 1/(nx+1);
    log a = sum_k sqrt(lam_k) phi_k(x) xi_k, the d-term KL expansion of the
    exponential covariance sigma^2 exp(-|x-y|/ell), xi_k iid N(0, 1).

Discretisation (flux form, conservative): a is evaluated at the nx+1 cell
midpoints m_j = (j + 1/2) h; A is tridiagonal with
    A_ii     = (a_i + a_{i+1}) / h^2
    A_i,i+1  = A_i+1,i = -a_{i+1} / h^2.
A is a symmetric, strictly diagonally dominant M-matrix, so both
(I + dt A) and (lambda_n I + dT A) (Re lambda_n > 0) admit pivot-free LU
(this is what makes the device's no-pivot tridiagonal solvers exact
restatements of SuperLU / LAPACK ?gbsv up to rounding).

KL eigenpairs: Nystrom on the midpoint grid with uniform weight h,
``eigh(sigma^2 exp(-|m_i - m_j|/ell) * h)``, eigenfunctions normalised to
sum(phi^2) h = 1 and signed so that phi_k(m_0) > 0. Computed once per model
on the host (the ``kl_table``), uploaded once, shared by all samples.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import ConfigError, ParameterSample, RngStream


@dataclass(frozen=True)
class ParameterMap:
    """Coordinate map used by the surrogate fit (``pintuq/models.py:25-52``),
    extended with ``identity`` for the Hermite (Gaussian) surrogates: the
    reference's ``affine(-1, 1)`` is not bit-exact identity."""

    kind: str
    lo: float
    hi: float

    def apply(self, v):
        v = np.asarray(v, dtype=float)
        if self.kind == "identity":
            return v.copy()
        if self.kind == "affine":
            return 2.0 * (v - self.lo) / (self.hi - self.lo) - 1.0
        if self.kind == "cos2pi":
            return np.cos(2.0 * np.pi * v)
        raise ConfigError(f"unknown parameter map kind {self.kind!r}")

    def to_dict(self) -> dict:
        return {"kind": self.kind, "lo": self.lo, "hi": self.hi}

    @staticmethod
    def from_dict(d: dict) -> "ParameterMap":
        return ParameterMap(str(d["kind"]), float(d["lo"]), float(d["hi"]))


class Model:
    """Interface shared by the models (``pintuq/models.py:61-106``)."""

    name: str = ""
    nx: int = 0
    parameter_dim: int = 1
    supports: tuple = ()
    is_linear: bool = False

    @property
    def cell_volume(self) -> float:
        raise NotImplementedError

    def rhs(self, u, t, xi):
        raise NotImplementedError

    def jacobian(self, u, t, xi):
        raise NotImplementedError

    def initial_condition(self, xi):
        raise NotImplementedError

    def sample_parameters(self, count: int, rng: RngStream) -> list:
        raise NotImplementedError

    def fit_maps(self) -> list:
        return [ParameterMap("affine", lo, hi) for lo, hi in self.supports]

    def validate(self, xi: ParameterSample):
        if xi.dim != self.parameter_dim:
            raise ValueError(f"{self.name}: expected {self.parameter_dim} parameters, got {xi.dim}")
        for v, (lo, hi) in zip(xi.values, self.supports):
            if not lo <= v <= hi:
                raise ValueError(f"{self.name}: parameter {v} outside support [{lo}, {hi}]")

    def check_state(self, u):
        u = np.asarray(u, dtype=float)
        if u.shape != (self.nx,):
            raise ValueError(f"{self.name}: state has shape {u.shape}, expected ({self.nx},)")
        return u


class LinearModel(Model):
    """rhs(u, t) = -A u + g(t) (``pintuq/models.py:109-125``)."""

    is_linear = True

    def linear_system(self, xi: ParameterSample):
        raise NotImplementedError

    def rhs(self, u, t, xi):
        u = self.check_state(u)
        A, g = self.linear_system(xi)
        return -(A @ u) + g(t)

    def jacobian(self, u, t, xi):
        A, _ = self.linear_system(xi)
        return -A


def exponential_kl_1d(points: np.ndarray, weight: float, sigma: float, ell: float, d: int):
    """Nystrom KL of sigma^2 exp(-|x-y|/ell) on ``points`` with quadrature
    ``weight``: returns (lam (d,), phi (d, len(points))) with sum(phi^2) w = 1
    and phi_k[0] > 0."""
    x = np.asarray(points, dtype=float)
    K = (sigma * sigma) * np.exp(-np.abs(x[:, None] - x[None, :]) / ell) * weight
    lam, vec = np.linalg.eigh(K)
    order = np.argsort(lam)[::-1][:d]
    lam = lam[order]
    phi = vec[:, order].T / np.sqrt(weight)
    phi *= np.where(phi[:, :1] < 0.0, -1.0, 1.0)
    return lam, phi


class LogNormalKL1D(LinearModel):
    """1D log-normal random-coefficient diffusion (BASELINE configs 1, 2, 4, 5)."""

    name = "lognormal-kl-1d"

    def __init__(self, nx: int = 127, d: int = 4, sigma: float = 0.5, ell: float = 0.3,
                 source: float = 1.0):
        if nx < 1 or d < 1:
            raise ConfigError("need nx >= 1 and d >= 1")
        self.nx = int(nx)
        self.parameter_dim = int(d)
        self.supports = tuple((-np.inf, np.inf) for _ in range(self.parameter_dim))
        self.h = 1.0 / (self.nx + 1)
        self.sigma = float(sigma)
        self.ell = float(ell)
        self.source = float(source)
        self.x = np.arange(1, self.nx + 1) * self.h
        self.midpoints = (np.arange(self.nx + 1) + 0.5) * self.h
        lam, phi = exponential_kl_1d(self.midpoints, self.h, self.sigma, self.ell, self.parameter_dim)
        self.kl_eigenvalues = lam
        self.kl_functions = phi
        # row k: sqrt(lam_k) phi_k(m_j); log a(m_j) = kl_table.T @ xi
        self.kl_table = np.ascontiguousarray(np.sqrt(lam)[:, None] * phi)
        self._cache: dict = {}

    @property
    def cell_volume(self) -> float:
        return self.h

    # xi ~ N(0, 1): the surrogate basis is the probabilists' Hermite family
    gpc_family = "hermite"

    def fit_maps(self):
        return [ParameterMap("identity", lo, hi) for lo, hi in self.supports]

    def log_coefficient(self, xi) -> np.ndarray:
        v = np.asarray(getattr(xi, "values", xi), dtype=float)
        return self.kl_table.T @ v

    def coefficient(self, xi) -> np.ndarray:
        """a at the nx+1 midpoints."""
        return np.exp(self.log_coefficient(xi))

    def tridiagonal(self, xi):
        """(diag (nx,), off (nx-1,)) of A."""
        a = self.coefficient(xi)
        inv_h2 = 1.0 / (self.h * self.h)
        return (a[:-1] + a[1:]) * inv_h2, -a[1:-1] * inv_h2

    def linear_system(self, xi):
        key = xi.key()
        hit = self._cache.get(key)
        if hit is not None:
            return hit
        import scipy.sparse as sp

        dia, off = self.tridiagonal(xi)
        A = sp.diags([off, dia, off], [-1, 0, 1], format="csc")
        g = np.full(self.nx, self.source)
        pair = (A, lambda t, g=g: g)
        self._cache[key] = pair
        return pair

    def initial_condition(self, xi=None):
        return np.sin(np.pi * self.x)

    def sample_parameters(self, count, rng: RngStream) -> list:
        draws = rng.normal(0.0, 1.0, size=(count, self.parameter_dim))
        return [ParameterSample(row, id=i) for i, row in enumerate(draws)]


class LogNormalKL2D(LinearModel):
    """2D log-normal random-coefficient diffusion on the unit square (BASELINE
    config 3): n x n interior nodes of a 5-point finite-difference grid, zero
    Dirichlet data, f = 1, u0 = sin(pi x) sin(pi y).

    log a is the KL expansion of the separable covariance
    sigma^2 exp(-|x1-x2|/ell) exp(-|y1-y2|/ell): the eigenpairs are products of
    the 1D Nystrom pairs on the n+1 cell-centre coordinates (exponential_kl_1d
    with sigma = 1), the d largest products kept (ties: lower (j, k) first).
    log a is evaluated at the (n+1)^2 cell centres; face coefficients are the
    arithmetic averages of the two cell centres a face separates. DOF order:
    x fastest, idx = (j-1) n + (i-1) for node (i h, j h). The assembled operator
    is symmetric, irreducibly diagonally dominant, bandwidth n.
    """

    name = "lognormal-kl-2d"

    def __init__(self, n: int = 127, d: int = 10, sigma: float = 0.5, ell: float = 0.25,
                 source: float = 1.0):
        if n < 1 or d < 1:
            raise ConfigError("need n >= 1 and d >= 1")
        self.n = int(n)
        self.nx = self.n * self.n
        self.parameter_dim = int(d)
        self.supports = tuple((-np.inf, np.inf) for _ in range(self.parameter_dim))
        self.h = 1.0 / (self.n + 1)
        self.sigma = float(sigma)
        self.ell = float(ell)
        self.source = float(source)
        nc = self.n + 1
        centres = (np.arange(nc) + 0.5) * self.h
        m1 = min(nc, self.parameter_dim)
        mu, phi = exponential_kl_1d(centres, self.h, 1.0, self.ell, m1)
        jj, kk = np.meshgrid(np.arange(m1), np.arange(m1), indexing="ij")
        jj, kk = jj.ravel(), kk.ravel()
        lam_all = (self.sigma * self.sigma) * mu[jj] * mu[kk]
        order = np.lexsort((kk, jj, -lam_all))[: self.parameter_dim]
        if len(order) < self.parameter_dim:
            raise ConfigError("d exceeds the number of product modes")
        self.kl_eigenvalues = lam_all[order]
        self.kl_pairs = np.stack([jj[order], kk[order]], axis=1)
        # row q: sqrt(lam_q) phi_j(x_p) phi_k(y_r) at centre (p, r), flattened r*(n+1)+p
        modes = np.stack([np.outer(phi[k], phi[j]).ravel() for j, k in self.kl_pairs])
        self.kl_table = np.ascontiguousarray(np.sqrt(self.kl_eigenvalues)[:, None] * modes)
        xs = np.arange(1, self.n + 1) * self.h
        self.x = np.tile(xs, self.n)
        self.y = np.repeat(xs, self.n)
        self._cache: dict = {}

    @property
    def cell_volume(self) -> float:
        return self.h * self.h

    # xi ~ N(0, 1): the surrogate basis is the probabilists' Hermite family
    gpc_family = "hermite"

    def fit_maps(self):
        return [ParameterMap("identity", lo, hi) for lo, hi in self.supports]

    def log_coefficient(self, xi) -> np.ndarray:
        """log a at the cell centres, shape (n+1, n+1) indexed [r (y), p (x)]."""
        v = np.asarray(getattr(xi, "values", xi), dtype=float)
        return (self.kl_table.T @ v).reshape(self.n + 1, self.n + 1)

    def faces(self, xi):
        """(ax (n, n+1): x-faces [j-1][i], ay (n+1, n): y-faces [j][i-1])."""
        a = np.exp(self.log_coefficient(xi))
        ax = 0.5 * (a[:-1, :] + a[1:, :])   # face (i+1/2, j): centres (i, j-1), (i, j)
        ay = 0.5 * (a[:, :-1] + a[:, 1:])   # face (i, j+1/2): centres (i-1, j), (i, j)
        return ax, ay

    def stencil(self, xi):
        """(dia, ex, ey), each (nx,): A[i,i], A[i,i+1] (0 at the row end), A[i,i+n] (0 in the last row)."""
        ax, ay = self.faces(xi)
        n, inv_h2 = self.n, 1.0 / (self.h * self.h)
        dia = (ax[:, :-1] + ax[:, 1:] + ay[:-1, :] + ay[1:, :]) * inv_h2
        ex = -ax[:, 1:].copy() * inv_h2
        ex[:, -1] = 0.0
        ey = -ay[1:, :].copy() * inv_h2
        ey[-1, :] = 0.0
        return dia.ravel(), ex.ravel(), ey.ravel()

    def linear_system(self, xi):
        key = xi.key()
        hit = self._cache.get(key)
        if hit is not None:
            return hit
        import scipy.sparse as sp

        dia, ex, ey = self.stencil(xi)
        n = self.n
        A = sp.diags([ey[:-n], ex[:-1], dia, ex[:-1], ey[:-n]], [-n, -1, 0, 1, n], format="csc")
        g = np.full(self.nx, self.source)
        pair = (A, lambda t, g=g: g)
        self._cache[key] = pair
        return pair

    def initial_condition(self, xi=None):
        return np.sin(np.pi * self.x) * np.sin(np.pi * self.y)

    def sample_parameters(self, count, rng: RngStream) -> list:
        draws = rng.normal(0.0, 1.0, size=(count, self.parameter_dim))
        return [ParameterSample(row, id=i) for i, row in enumerate(draws)]


# ---------------------------------------------------------------------------
# Nonlinear tridiagonal models (pintuq/models.py:269-379): the reference's
# fused Newton sweeps (_kernels.pyx) run on the device (kle_newton_sweep_f64).
# ---------------------------------------------------------------------------
class Burgers1D(Model):
    """Viscous Burgers u_t + u u_x = nu u_xx on (0, 1), zero Dirichlet, upwind
    convection switched on sign(u_i), nu = xi / 50, xi ~ U[1, 3]
    (``pintuq/models.py:269-323``)."""

    name = "burgers"
    parameter_dim = 1
    supports = ((1.0, 3.0),)
    sweep_kind = 0

    def __init__(self, dx: float = 1.0 / 100.0):
        self.dx = float(dx)
        self.m = round(1.0 / self.dx) - 1
        self.nx = self.m
        self.x = np.arange(1, self.m + 1) * self.dx

    @property
    def cell_volume(self) -> float:
        return self.dx

    @staticmethod
    def viscosity(xi_value: float) -> float:
        return xi_value / 50.0

    def rhs(self, u, t, xi):
        u = self.check_state(u)
        nu, dx = self.viscosity(xi.values[0]), self.dx
        left = np.concatenate(([0.0], u[:-1]))
        right = np.concatenate((u[1:], [0.0]))
        dudx = np.where(u >= 0.0, (u - left) / dx, (right - u) / dx)
        return -u * dudx + nu * (left - 2.0 * u + right) / dx**2

    def jacobian(self, u, t, xi):
        import scipy.sparse as sp

        u = self.check_state(u)
        nu, dx = self.viscosity(xi.values[0]), self.dx
        left = np.concatenate(([0.0], u[:-1]))
        right = np.concatenate((u[1:], [0.0]))
        up = u >= 0.0
        diag = np.where(up, -(2.0 * u - left) / dx, -(right - 2.0 * u) / dx) - 2.0 * nu / dx**2
        sub = np.where(up[1:], u[1:] / dx, 0.0) + nu / dx**2
        sup = np.where(up[:-1], 0.0, -u[:-1] / dx) + nu / dx**2
        return sp.diags([sub, diag, sup], [-1, 0, 1], format="csr")

    def initial_condition(self, xi=None):
        return np.sin(2.0 * np.pi * self.x)

    def sample_parameters(self, count, rng: RngStream) -> list:
        from .core import sample_uniform

        return sample_uniform(*self.supports[0], count, rng)

    def sweep_args(self, xi: ParameterSample) -> tuple:
        """(kernel kind, parameters) of the fused implicit sweeps (``models.py:320-323``)."""
        return "burgers", (self.viscosity(xi.values[0]), self.dx)

    def sweep_params(self, xi) -> tuple:
        """Device sweep parameters (p0 per sample; dx, bc_lo, bc_hi shared)."""
        return self.viscosity(float(np.asarray(xi.values if isinstance(xi, ParameterSample) else xi)[0])), \
            self.dx, 0.0, 0.0


class AllenCahn1D(Model):
    """Allen-Cahn u_t = eps u_xx - (u^3 - u) on (-1, 1), u(-1) = -1, u(1) = 1,
    eps a truncated Gaussian on [0.06, 1] (``pintuq/models.py:326-379``)."""

    name = "allen-cahn"
    parameter_dim = 1
    supports = ((0.06, 1.0),)
    bc = (-1.0, 1.0)
    gaussian = (0.53, 0.15)
    sweep_kind = 1

    def __init__(self, dx: float = 1.0 / 128.0):
        self.dx = float(dx)
        self.m = round(2.0 / self.dx) - 1
        self.nx = self.m
        self.x = -1.0 + np.arange(1, self.m + 1) * self.dx
        self._lift = np.zeros(self.m)
        self._lift[0] = self.bc[0] / self.dx**2
        self._lift[-1] = self.bc[1] / self.dx**2

    @property
    def cell_volume(self) -> float:
        return self.dx

    def rhs(self, u, t, xi):
        u = self.check_state(u)
        eps = xi.values[0]
        left = np.concatenate(([0.0], u[:-1]))
        right = np.concatenate((u[1:], [0.0]))
        d2 = (left - 2.0 * u + right) / self.dx**2 + self._lift
        return eps * d2 - (u**3 - u)

    def jacobian(self, u, t, xi):
        import scipy.sparse as sp

        u = self.check_state(u)
        eps = xi.values[0]
        m = self.m
        band = sp.diags([np.ones(m - 1), -2.0 * np.ones(m), np.ones(m - 1)], [-1, 0, 1], format="csr") / self.dx**2
        return eps * band - sp.diags(3.0 * u**2 - 1.0)

    def initial_condition(self, xi=None):
        return 0.53 * self.x + 0.47 * np.sin(-1.5 * np.pi * self.x)

    def sample_parameters(self, count, rng: RngStream) -> list:
        from .core import sample_truncated_gaussian

        mu, sigma = self.gaussian
        return sample_truncated_gaussian(mu, sigma, *self.supports[0], count, rng)

    def with_boundaries(self, u: np.ndarray) -> np.ndarray:
        return np.concatenate(([self.bc[0]], np.asarray(u, float), [self.bc[1]]))

    def sweep_args(self, xi: ParameterSample) -> tuple:
        return "allen-cahn", (xi.values[0], self.dx, self.bc[0], self.bc[1])

    def sweep_params(self, xi) -> tuple:
        return float(np.asarray(xi.values if isinstance(xi, ParameterSample) else xi)[0]), self.dx, \
            self.bc[0], self.bc[1]


_MODELS = {"lognormal-kl-1d": LogNormalKL1D, "lognormal-kl-2d": LogNormalKL2D, "burgers": Burgers1D,
           "allen-cahn": AllenCahn1D}


def get_model(name: str, **kwargs) -> Model:
    """Registry lookup (``pintuq/models.py:400-413``)."""
    try:
        cls = _MODELS[name]
    except KeyError:
        raise ConfigError(f"unknown model {name!r}; known: {sorted(_MODELS)}") from None
    return cls(**kwargs)
