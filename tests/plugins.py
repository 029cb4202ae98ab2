"""Third-party model plugins for the tests: the reference's own linear
models (``pintuq/models.py:128-266``), restated as a user would write a
``LinearModel`` plugin for this package. They are not part of the product:
Diffusion1D exercises the generic tridiagonal plugin path (operator taken
from ``linear_system``), AdvectionDiffusion2D (non-symmetric 5-point
operator, time-dependent source) checks that unsupported plugins raise.
"""
from __future__ import annotations

import numpy as np

from paper_2510_26180_b200.core import ConfigError, RngStream
from paper_2510_26180_b200.models import LinearModel, ParameterMap

def laplacian_1d(m: int, dx: float):
    """Second-difference matrix on m interior nodes, homogeneous Dirichlet (``models.py:55-58``)."""
    import scipy.sparse as sp

    e = np.ones(m)
    return sp.diags([e[:-1], -2.0 * e, e[:-1]], [-1, 0, 1], format="csr") / dx**2


class Diffusion1D(LinearModel):
    """u_t = a u_xx on (0, 1), zero boundaries and source, a ~ U[0.5, 2] (``models.py:219-266``)."""

    name = "diffusion-1d"
    parameter_dim = 1
    supports = ((0.5, 2.0),)

    def __init__(self, h: float = 1.0 / 64.0):
        self.h = float(h)
        self.m = round(1.0 / self.h) - 1
        self.nx = self.m
        self.x = np.arange(1, self.m + 1) * self.h
        self._cache = {}

    @property
    def cell_volume(self) -> float:
        return self.h

    def linear_system(self, xi):
        key = xi.key()
        hit = self._cache.get(key)
        if hit is None:
            A = (-xi.values[0] * laplacian_1d(self.m, self.h)).tocsc()
            zero = np.zeros(self.nx)
            hit = (A, lambda t, z=zero: z)
            self._cache[key] = hit
        return hit

    def initial_condition(self, xi=None):
        return np.sin(np.pi * self.x)

    def sample_parameters(self, count, rng: RngStream) -> list:
        from paper_2510_26180_b200.core import sample_uniform

        return sample_uniform(*self.supports[0], count, rng)

    def diffusion_eigenvalues(self, xi):
        mm = np.arange(1, self.m + 1)
        return xi.values[0] * (4.0 / self.h**2) * np.sin(mm * np.pi * self.h / 2.0) ** 2

    def diffusion_eigenvectors(self):
        idx = np.arange(1, self.m + 1)
        return np.sqrt(2.0 * self.h) * np.sin(np.pi * self.h * np.outer(idx, idx))


class AdvectionDiffusion2D(LinearModel):
    """2D advection-diffusion on (0, 1)^2 (``models.py:128-216``): a(xi) =
    0.5 (2 + cos(pi xi)^2), velocity 0.1 (x2, x1), source exp(-t) w(x; xi).
    Host-only (non-symmetric operator, time-dependent source)."""

    name = "advection-diffusion"
    parameter_dim = 1
    supports = ((2.0, 6.0),)

    def __init__(self, h: float = 1.0 / 20.0, advection: bool = True):
        self.h = float(h)
        self.m = round(1.0 / self.h) - 1
        if abs((self.m + 1) * self.h - 1.0) > 1e-12:
            raise ConfigError(f"h={h} does not evenly divide the unit interval")
        self.nx = self.m * self.m
        self.advection = bool(advection)
        ii = np.arange(1, self.m + 1) * self.h
        self.x1 = np.repeat(ii, self.m)
        self.x2 = np.tile(ii, self.m)
        self._cache = {}

    @property
    def cell_volume(self) -> float:
        return self.h * self.h

    @staticmethod
    def diffusion_coefficient(xi_value: float) -> float:
        return 0.5 * (2.0 + np.cos(np.pi * xi_value) ** 2)

    def fit_maps(self):
        return [ParameterMap("cos2pi", *self.supports[0])]

    def linear_system(self, xi):
        import scipy.sparse as sp

        key = xi.key()
        hit = self._cache.get(key)
        if hit is not None:
            return hit
        a = self.diffusion_coefficient(xi.values[0])
        m, h = self.m, self.h
        L1 = laplacian_1d(m, h)
        I1 = sp.eye(m, format="csr")
        A = -a * (sp.kron(L1, I1) + sp.kron(I1, L1))
        if self.advection:
            D1 = sp.diags([-np.ones(m - 1), np.ones(m - 1)], [-1, 1], format="csr") / (2 * h)
            A = A + sp.diags(0.1 * self.x2) @ sp.kron(D1, I1) + sp.diags(0.1 * self.x1) @ sp.kron(I1, D1)
        A = A.tocsc()
        ss = np.sin(np.pi * self.x1) * np.sin(2 * np.pi * self.x2)
        w = ((a * np.pi**2 - 1.0) * ss
             + 0.05 * np.pi * self.x2 * np.cos(np.pi * self.x1) * np.sin(2 * np.pi * self.x2)
             + 0.1 * np.pi * self.x1 * np.sin(np.pi * self.x1) * np.cos(2 * np.pi * self.x2))
        hit = (A, lambda t, w=w: np.exp(-t) * w)
        self._cache[key] = hit
        return hit

    def source(self, t: float, xi):
        return self.linear_system(xi)[1](t)

    def initial_condition(self, xi=None):
        return np.sin(np.pi * self.x1) * np.sin(2 * np.pi * self.x2)

    def sample_parameters(self, count, rng: RngStream) -> list:
        from paper_2510_26180_b200.core import sample_uniform

        return sample_uniform(*self.supports[0], count, rng)
