"""Device-side operator batches and helpers (PyTorch is used only for device
memory and streams; every computation is a libkle_b200 kernel).

A ``DeviceOperator`` holds, for M samples of a tridiagonal linear model
(``pintuq/models.py:109-125`` contract, A symmetric tridiagonal, constant
uniform source g(t) = g0), the operator diagonals on the device and caches
the solver factor blobs per step size (the reference caches one SuperLU per
(sample, dt): ``pintuq/propagators.py:17-34``).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .core import DeviceError, ParameterSample

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None


def require_cuda():
    if torch is None or not torch.cuda.is_available():
        raise DeviceError("a CUDA device is required (libkle_b200 has no CPU path)")
    _lib.load()


def ptr(t):
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


def stream_ptr():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def to_dev(a, dtype=None):
    require_cuda()
    dtype = dtype or torch.float64
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


def empty(*shape, dtype=None):
    return torch.empty(*shape, dtype=dtype or torch.float64, device="cuda")


def fine_layout(nx: int):
    MR, P, nd = C.c_int(), C.c_int(), C.c_int()
    rc = _lib.query("kle_fine_layout", nx, C.byref(MR), C.byref(P), C.byref(nd))
    if rc != 0:
        raise DeviceError(_lib.load().kle_last_error().decode())
    return MR.value, P.value, nd.value


def constant_source(g) -> float:
    """g0 of a source g(t) = g0 * ones that is constant in time and uniform in
    space, else NotImplementedError. Probed at the interval ends and at
    irrational interior points (a source such as t (1 - t) w agrees at t = 0
    and t = 1 only)."""
    g_a = np.asarray(g(0.0), dtype=float)
    for t in (1.0, 0.5, 0.1234567890123, 0.7071067811865476, 3.0):
        if not np.array_equal(g_a, np.asarray(g(t), dtype=float)):
            raise NotImplementedError("the device path needs a constant, uniform source g(t) = g0")
    if g_a.size and not np.all(g_a == g_a.flat[0]):
        raise NotImplementedError("the device path needs a constant, uniform source g(t) = g0")
    return float(g_a.flat[0]) if g_a.size else 0.0


def tridiagonal_of(model, xi):
    """(dia, off, g0) of a tridiagonal plugin's operator, via its own
    ``linear_system`` (host-side model evaluation, as in the reference)."""
    import scipy.sparse as sp

    A, g = model.linear_system(xi)
    A = sp.csr_matrix(A)
    nx = A.shape[0]
    coo = A.tocoo()
    if coo.nnz and np.max(np.abs(coo.row - coo.col)) > 1:
        raise NotImplementedError("the device path supports tridiagonal operators only")
    dia = np.asarray(A.diagonal(0), dtype=float)
    off = np.zeros(nx)
    if nx > 1:
        lo, up = A.diagonal(-1), A.diagonal(1)
        if not np.array_equal(lo, up):
            raise NotImplementedError("the device path supports symmetric operators only")
        off[:-1] = up
    return dia, off, constant_source(g)


def shared_initial_condition(model, xis):
    """The plugin contract is ``initial_condition(xi)`` per sample
    (``pintuq/models.py:61-106``). The device kernels take one u0 shared by the
    batch, so every sample's initial state is evaluated and must be identical;
    a parameter-dependent u0 raises instead of silently using the first
    sample's. Array/tensor batches of a KL model evaluate ``initial_condition``
    at the first and last rows (the KL models' u0 does not depend on xi)."""
    if isinstance(xis, (list, tuple)):
        pts = list(xis)
    else:
        if hasattr(xis, "detach"):
            arr = xis.reshape(xis.shape[0], -1)[[0, -1]].cpu().numpy() if xis.shape[0] else np.zeros((0, 1))
        else:
            arr = np.atleast_2d(np.asarray(xis))
        pts = [ParameterSample(arr[0], id=0), ParameterSample(arr[-1], id=len(arr) - 1)] if len(arr) else []
    if not pts:
        return np.asarray(model.initial_condition(None), dtype=float)
    first = np.asarray(model.initial_condition(_as_sample(pts[0])), dtype=float)
    for x in pts[1:]:
        if not np.array_equal(first, np.asarray(model.initial_condition(_as_sample(x)), dtype=float)):
            raise NotImplementedError("the device path needs one initial state shared by all samples "
                                      "(initial_condition(xi) differs between samples)")
    return first


def _as_sample(x):
    if isinstance(x, ParameterSample):
        return x
    return ParameterSample(np.asarray(x, dtype=float), id=0)


class DeviceOperator:
    """Batch of M per-sample tridiagonal operators resident on the device."""

    def __init__(self, dia, off, g0: float, u0):
        self.dia = dia
        self.off = off
        self.M, self.nx = dia.shape
        self.g0 = float(g0)
        self.u0 = u0
        self.layout = fine_layout(self.nx)
        self._blobs = {}

    @classmethod
    def from_model(cls, model, xis):
        """xis: list of ParameterSample, an (M, d) array or a device tensor.
        5-point (2D) plugins get a ``twod.DeviceOperator2D``."""
        require_cuda()
        from .twod import DeviceOperator2D, is_five_point

        if is_five_point(model):
            return DeviceOperator2D.from_model(model, xis)
        if isinstance(xis, ParameterSample):
            xis = [xis]
        kl_table = getattr(model, "kl_table", None)
        if kl_table is not None:
            if isinstance(xis, (list, tuple)):
                arr = np.array([np.asarray(x.values if isinstance(x, ParameterSample) else x, dtype=float)
                                for x in xis])
            else:
                arr = xis
            xi_d = to_dev(arr).reshape(-1, model.parameter_dim)
            M = xi_d.shape[0]
            nx = model.nx
            dia, off = empty(M, nx), empty(M, nx)
            inv_h2 = 1.0 / (model.h * model.h)
            _lib.call("kle_kl_tridiag_f64", ptr(xi_d), M, model.parameter_dim, ptr(to_dev(kl_table)), nx,
                      inv_h2, ptr(dia), ptr(off), stream_ptr())
            g0 = model.source
        else:
            rows = [tridiagonal_of(model, x) for x in xis]
            g0s = {r[2] for r in rows}
            if len(g0s) != 1:
                raise NotImplementedError("all samples must share the source value g0")
            dia = to_dev(np.array([r[0] for r in rows]))
            off = to_dev(np.array([r[1] for r in rows]))
            g0 = rows[0][2]
        u0 = to_dev(shared_initial_condition(model, xis))
        return cls(dia, off, g0, u0)

    def blob(self, h: float):
        key = float(h)
        b = self._blobs.get(key)
        if b is None:
            b = empty(self.M, self.layout[2])
            _lib.call("kle_fine_factor_f64", ptr(self.dia), ptr(self.off), self.M, self.nx, key, self.g0, ptr(b),
                      stream_ptr())
            self._blobs[key] = b
        return b

    def sweep(self, start, h: float, J: int, nseg: int = 1):
        """start: (M, Q, nx) device tensor -> (M, Q, nseg, nx)."""
        M, Q, nx = start.shape
        out = empty(M, Q, nseg, nx)
        _lib.call("kle_sweep_f64", ptr(start.contiguous()), ptr(out), ptr(self.blob(h)), M, Q, nx, J, nseg, h,
                  self.g0, stream_ptr())
        return out


class AlphaTables:
    """Device copies of build_alpha_circulant's eigenvalues/scaling
    (computed on the host with the reference formula, pintuq/pcgc.py:68-76,
    so pow/exp rounding matches)."""

    def __init__(self, spec):
        lam = np.empty(2 * spec.n)
        lam[0::2] = spec.eigenvalues.real
        lam[1::2] = spec.eigenvalues.imag
        self.lam = to_dev(lam)
        self.scaling = to_dev(spec.scaling)
        self.inv_scaling = to_dev(1.0 / spec.scaling)
