"""2D (5-point) device path: BASELINE config 3 (``models.LogNormalKL2D``).

Same plugin contract and entry points as the 1D path: ``DeviceOperator.from_model``
returns a ``DeviceOperator2D`` for a 5-point operator, whose ``sweep`` serves
``propagate_fine`` / ``propagate_coarse`` / ``fine_reference`` /
``coarse_sweep_init``; ``pcgc.pcgc_solve_device`` dispatches here.

Two solver families for the implicit systems (``solver=``):

``"direct"`` (default), like the reference's SuperLU (``pintuq/propagators.py:
25-39``, ``pintuq/pcgc.py:137-145``): banded L D L^T factors of I + dt A
(real) and of the N/2+1 distinct shifted matrices lambda_f I + dT A (complex)
are built on the device once per solve (``kle_2d_factor_f64``) and reused by
every outer iteration. Samples are processed in batches sized to the free
device memory (the complex factors take 16 (N/2+1) n^3 bytes per sample).

``"krylov"`` (the north star's matrix-free variant): Jacobi-PCG
for every backward-Euler step (warm started) and Jacobi-COCG for the shifted
systems, applied matrix-free from the stencil (``kle_2d_krylov.cu``), to a
relative residual ``krylov_rtol``; no factors, so the batch is not limited by
factor memory. ``KLE_2D_SOLVER=krylov`` selects it by default.
"""
from __future__ import annotations

import os

import numpy as np

from . import _lib
from .core import DeviceError, ParameterSample
from .device import AlphaTables, empty, ptr, require_cuda, stream_ptr, to_dev

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None


# the TMA-staged fine sweeps (kle_2d_tma.cu); KLE_2D_TMA=0 selects the
# per-warp sweeps of kle_2d.cu (A/B measurements)
_USE_TMA = os.environ.get("KLE_2D_TMA", "1") != "0"


def stencil_of(model, xi):
    """(dia, ex, ey, g0) of a 5-point plugin's operator via its own
    ``linear_system`` (host-side model evaluation, as in the reference)."""
    import scipy.sparse as sp

    A, g = model.linear_system(xi)
    A = sp.csr_matrix(A)
    n = int(getattr(model, "n"))
    nx = A.shape[0]
    if nx != n * n:
        raise NotImplementedError("5-point operator size must be n*n")
    coo = A.tocoo()
    off = np.setdiff1d(np.unique(np.abs(coo.row - coo.col)), [0, 1, n])
    if off.size:
        raise NotImplementedError("the 2D device path supports 5-point operators only")
    if abs(A - A.T).max() if A.nnz else 0:
        raise NotImplementedError("the 2D device path supports symmetric operators only")
    dia = np.asarray(A.diagonal(0), dtype=float)
    ex = np.zeros(nx)
    ey = np.zeros(nx)
    if nx > 1:
        ex[:-1] = A.diagonal(1)
    if nx > n:
        ey[:-n] = A.diagonal(n)
    from .device import constant_source

    return dia, ex, ey, constant_source(g)


def is_five_point(model) -> bool:
    """True for plugins on an n x n grid with a 5-point operator (bandwidth n)."""
    n = getattr(model, "n", None)
    return hasattr(model, "stencil") or (n is not None and n > 1 and getattr(model, "nx", None) == n * n)


_SOLVERS = ("direct", "krylov")


class DeviceOperator2D:
    """Batch of M per-sample 5-point operators resident on the device."""

    # Krylov stopping rule: relative 2-norm residual (the probe in SURVEY §8(c):
    # 1e-12 reproduced the reference iteration counts with 1.9e-11 field error)
    krylov_rtol = 1e-13
    krylov_max_its = 20000

    def __init__(self, dia, ex, ey, n: int, g0: float, u0, solver: str | None = None):
        require_cuda()
        self.solver = solver or os.environ.get("KLE_2D_SOLVER", "direct")
        if self.solver not in _SOLVERS:
            raise ValueError(f"solver must be one of {_SOLVERS}, not {self.solver!r}")
        self.krylov_its = torch.zeros(1, dtype=torch.int64, device="cuda")  # accumulated PCG/COCG iterations
        self.dia, self.ex, self.ey = dia, ex, ey
        self.M, self.nx = dia.shape
        self.n = int(n)
        if self.n * self.n != self.nx or self.n > 127:
            raise DeviceError("2D operator: need nx = n*n with n <= 127")
        self.g0 = float(g0)
        self.u0 = u0
        self.layout = (0, 0, 0)
        self._fine = {}
        self._stage = {}

    @classmethod
    def from_model(cls, model, xis):
        require_cuda()
        if isinstance(xis, ParameterSample):
            xis = [xis]
        table = getattr(model, "kl_table", None)
        n = int(model.n)
        if table is not None and hasattr(model, "stencil"):
            if isinstance(xis, (list, tuple)):
                arr = np.array([np.asarray(x.values if isinstance(x, ParameterSample) else x, dtype=float)
                                for x in xis])
            else:
                arr = xis
            xi_d = to_dev(arr).reshape(-1, model.parameter_dim)
            M = xi_d.shape[0]
            dia, ex, ey = empty(M, n * n), empty(M, n * n), empty(M, n * n)
            _lib.call("kle_2d_kl5pt_f64", ptr(xi_d), M, model.parameter_dim, ptr(to_dev(table)), n,
                      1.0 / (model.h * model.h), ptr(dia), ptr(ex), ptr(ey), stream_ptr())
            g0 = model.source
        else:
            rows = [stencil_of(model, x) for x in xis]
            if len({r[3] for r in rows}) != 1:
                raise NotImplementedError("all samples must share the source value g0")
            dia, ex, ey = (to_dev(np.array([r[k] for r in rows])) for k in range(3))
            g0 = rows[0][3]
        from .device import shared_initial_condition

        return cls(dia, ex, ey, n, g0, to_dev(shared_initial_condition(model, xis)))

    def select(self, lo: int, hi: int) -> "DeviceOperator2D":
        o = DeviceOperator2D(self.dia[lo:hi], self.ex[lo:hi], self.ey[lo:hi], self.n, self.g0, self.u0, self.solver)
        o.krylov_its = self.krylov_its
        return o

    # -- factors -------------------------------------------------------------
    def fine_factor(self, h: float):
        """(Lt, Dinv) of I + h A for every sample (cached per h)."""
        key = float(h)
        f = self._fine.get(key)
        if f is None:
            M, nx, n = self.M, self.nx, self.n
            Lt, Dinv = empty(M, nx, n), empty(M, nx)
            _lib.call("kle_2d_factor_f64", ptr(self.dia), ptr(self.ex), ptr(self.ey), M, n, None, 1, 1.0, key,
                      ptr(Lt), ptr(Dinv), stream_ptr())
            f = (Lt, Dinv)
            self._fine[key] = f
        return f

    def fine_stage(self, h: float):
        """The factor of I + h A restaged for the TMA sweeps
        (``kle_2d_fine_stage_f64``: per row block, the skewed coefficient
        chunks of both substitution directions and D^{-1}), cached per h. The
        column-form factor is dropped unless ``fine_factor`` cached it."""
        key = float(h)
        st = self._stage.get(key)
        if st is None:
            cached = key in self._fine
            Lt, Dinv = self.fine_factor(key)
            st = empty(int(_lib.query("kle_2d_fine_stage_doubles", self.M, self.n)))
            _lib.call("kle_2d_fine_stage_f64", ptr(Lt), ptr(Dinv), self.M, self.n, ptr(st), stream_ptr())
            if not cached:
                del self._fine[key]
            self._stage[key] = st
        return st

    def shifted_factors(self, tables: AlphaTables, N: int, deltaT: float):
        """Complex (Lt, Dinv) of lambda_f I + dT A, f = 0..N/2 (B_{N-f} = conj B_f)."""
        NF = N // 2 + 1
        Lt = empty(self.M, NF, self.nx, self.n, 2)
        Dinv = empty(self.M, NF, self.nx, 2)
        _lib.call("kle_2d_factor_f64", ptr(self.dia), ptr(self.ex), ptr(self.ey), self.M, self.n,
                  ptr(tables.lam), NF, 0.0, deltaT, ptr(Lt), ptr(Dinv), stream_ptr())
        return Lt, Dinv

    # -- propagators ---------------------------------------------------------
    def sweep(self, start, h: float, J: int, nseg: int = 1):
        """start: (M, Q, nx) device tensor -> (M, Q, nseg, nx)."""
        M, Q, nx = start.shape
        out = empty(M, Q, nseg, nx)
        if self.solver == "krylov":
            cur = start.contiguous()
            seg = empty(M, Q, nx)
            for g in range(nseg):
                _lib.call("kle_2d_sweep_krylov_f64", ptr(cur), ptr(self.dia), ptr(self.ex), ptr(self.ey), M, Q,
                          self.n, J, h, self.g0, self.krylov_rtol, self.krylov_max_its, ptr(seg),
                          ptr(self.krylov_its), stream_ptr())
                out[:, :, g].copy_(seg)
                cur = out[:, :, g].contiguous()
            return out
        nw = int(_lib.query("kle_2d_fine_work_doubles", M, Q, self.n))
        work = empty(max(nw, 1))
        if _USE_TMA:
            st = self.fine_stage(h)
            _lib.call("kle_2d_sweep_staged_f64", ptr(start.contiguous()), ptr(st), M, Q, self.n, J, nseg, h, self.g0,
                      ptr(work), nw, ptr(out), stream_ptr())
            return out
        Lt, Dinv = self.fine_factor(h)
        _lib.call("kle_2d_sweep_f64", ptr(start.contiguous()), ptr(self.dia), ptr(self.ex), ptr(self.ey), ptr(Lt),
                  ptr(Dinv), M, Q, self.n, J, nseg, h, self.g0, ptr(work), nw, ptr(out), stream_ptr())
        return out

    def fgr(self, U, tables: AlphaTables, grid, alpha: float, R, status=None, F_given=None):
        M, N, nx = U.shape
        dT, dt = grid.deltaT, grid.deltat
        if self.solver == "krylov":
            _lib.call("kle_2d_fgr_krylov_f64", ptr(U), ptr(self.u0), ptr(F_given), ptr(self.dia), ptr(self.ex),
                      ptr(self.ey), ptr(tables.scaling), ptr(status), M, N, self.n, grid.n_fine_per_coarse, dt, dT,
                      self.g0, alpha, self.krylov_rtol, self.krylov_max_its, ptr(R), None, ptr(self.krylov_its),
                      stream_ptr())
            return
        nw = int(_lib.query("kle_2d_fine_work_doubles", M, N, self.n))
        work = empty(max(nw, 1))
        if _USE_TMA:
            st = self.fine_stage(dt)
            _lib.call("kle_2d_fgr_staged_f64", ptr(U), ptr(self.u0), ptr(F_given), ptr(self.dia), ptr(self.ex),
                      ptr(self.ey), ptr(st), ptr(tables.scaling), ptr(status), M, N, self.n,
                      grid.n_fine_per_coarse, dt, dT, self.g0, alpha, ptr(work), nw, ptr(R), stream_ptr())
            return
        Lt, Dinv = self.fine_factor(dt)
        _lib.call("kle_2d_fgr_f64", ptr(U), ptr(self.u0), ptr(F_given), ptr(self.dia), ptr(self.ex), ptr(self.ey),
                  ptr(Lt), ptr(Dinv), ptr(tables.scaling), ptr(status), M, N, self.n, grid.n_fine_per_coarse,
                  dt, dT, self.g0, alpha, ptr(work), nw, ptr(R), stream_ptr())


def cgc_krylov(op: DeviceOperator2D, tables: AlphaTables, N: int, deltaT: float, R, U=None, Uout=None,
               load_scale=None, k=1, max_iters=1, tol=0.0, status=None, iters=None, inc_hist=None, active=None,
               work=None):
    """kle_2d_cgc_krylov_f64: the scaled DFT, the COCG shifted solves and the
    inverse DFT (+ update / increment / stop test when U and status are given)."""
    M = R.shape[0]
    nw = int(_lib.query("kle_2d_cgc_krylov_work_doubles", M, N, op.n))
    if work is None or work.numel() < nw:
        work = torch.zeros(max(nw, 1), dtype=torch.float64, device="cuda")
    _lib.call("kle_2d_cgc_krylov_f64", ptr(R.contiguous()), ptr(load_scale), ptr(U), ptr(Uout), ptr(op.dia),
              ptr(op.ex), ptr(op.ey), ptr(tables.lam), ptr(tables.inv_scaling), M, N, op.n, k, max_iters, tol,
              ptr(status), ptr(iters), None, ptr(inc_hist), ptr(active), deltaT, op.krylov_rtol, op.krylov_max_its,
              ptr(work), work.numel(), ptr(op.krylov_its), stream_ptr())
    return work


def three_step_device2d(op: DeviceOperator2D, tables: AlphaTables, N: int, deltaT: float, r, prescaled=False,
                        factors=None):
    """u = V (Lambda (x) I + dT I (x) A)^{-1} V^{-1} r, r: (M, N, nx). Returns (u, imag)."""
    M, _, nx = r.shape
    if op.solver == "krylov":
        u = empty(M, N, nx)
        cgc_krylov(op, tables, N, deltaT, r, Uout=u, load_scale=None if prescaled else tables.scaling)
        return u, torch.zeros(M, dtype=torch.float64, device="cuda")
    Lt, Dinv = factors or op.shifted_factors(tables, N, deltaT)
    u = empty(M, N, nx)
    nw = int(_lib.query("kle_2d_cgc_work_doubles", M, N, op.n))
    work = empty(max(nw, 1))
    _lib.call("kle_2d_cgc_f64", ptr(r.contiguous()), None if prescaled else ptr(tables.scaling), None, ptr(u),
              ptr(Lt), ptr(Dinv), ptr(tables.inv_scaling), M, N, op.n, 0, 1, 0.0, None, None, None, None, None,
              ptr(work), nw, stream_ptr())
    return u, torch.zeros(M, dtype=torch.float64, device="cuda")


def _batch_size(op: DeviceOperator2D, N: int) -> int:
    NF = N // 2 + 1
    nblk = (op.nx + 7) // 8
    per = 8 * (2 * NF * op.nx * (op.n + 1) + 2 * op.nx * (op.n + 1) + 6 * N * op.nx + 2 * NF * op.nx
               + 2 * nblk * (op.n + 9) * 8)
    # the per-batch factors are single allocations of tens of GB: hand the
    # caching allocator's idle (possibly fragmented) blocks back first, so the
    # free figure is what one allocation can actually get
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    return max(1, min(op.M, int(0.85 * free) // per))


def pcgc_solve_device2d(op: DeviceOperator2D, U, grid, cfg, tables: AlphaTables = None, batch: int = None,
                        reference=None, stop_on: str = "increment"):
    """Batched PCGC loop for the 2D operator (``pintuq/pcgc.py:273-358``);
    U (M, N, nx) is overwritten with the final states. ``reference`` (M, N,
    nx) adds the error records; ``stop_on="reference"`` stops on them
    (``kle_err_ref_f64`` after every correction)."""
    from .pcgc import BatchResult, build_alpha_circulant

    M, N, nx = U.shape
    if N != grid.n_coarse or nx != op.nx or M != op.M:
        raise ValueError("initial guess length does not match the time grid")
    if N % 2:
        raise NotImplementedError("the 2D CGC needs an even number of subintervals")
    tables = tables or AlphaTables(build_alpha_circulant(N, cfg.alpha))
    status = torch.zeros(M, dtype=torch.int32, device="cuda")
    iters = torch.zeros(M, dtype=torch.int32, device="cuda")
    inc = torch.full((M, cfg.max_outer_iters), float("nan"), dtype=torch.float64, device="cuda")
    imag = torch.zeros(M, dtype=torch.float64, device="cuda")
    B = batch or _batch_size(op, N)
    active = torch.zeros(1, dtype=torch.int32, device="cuda")
    ref = err = me = None
    stop_ref = int(stop_on == "reference")
    if reference is not None:
        ref = reference.contiguous()
        if tuple(ref.shape) != (M, N, nx):
            raise ValueError("reference trajectory shape does not match the initial guess")
        err = torch.full((M, cfg.max_outer_iters + 1, N), float("nan"), dtype=torch.float64, device="cuda")
        me = empty(M)
    cgc_tol = -1.0 if (ref is not None and stop_ref) else cfg.tol

    def record(Ub, lo, Mb, k, st, it):
        _lib.call("kle_err_ref_f64", ptr(Ub), ptr(ref[lo:lo + Mb]), Mb, N, nx, k, cfg.max_outer_iters, cfg.tol,
                  stop_ref, ptr(st), ptr(it), ptr(active), ptr(err[lo:lo + Mb]), ptr(me[lo:lo + Mb]), stream_ptr())
    import os
    import time

    prof = os.environ.get("KLE_2D_PROFILE") == "1"

    def mark(msg, t0=[None]):
        if prof:
            torch.cuda.synchronize()
            t = time.time()
            if t0[0] is not None:
                print(f"[2d] {msg}: {t - t0[0]:.3f} s", flush=True)
            t0[0] = t

    mark("start")
    if op.solver == "krylov":  # no factors: one batch
        R = empty(M, N, nx)
        work = None
        if ref is not None:
            active.zero_()
            record(U, 0, M, 0, status, iters)
            if stop_ref and int(active.item()) == 0:
                return BatchResult(U, iters, status, inc, imag, err, me)
        for k in range(1, cfg.max_outer_iters + 1):
            op.fgr(U, tables, grid, cfg.alpha, R, status=status)
            active.zero_()
            work = cgc_krylov(op, tables, N, grid.deltaT, R, U=U, k=k, max_iters=cfg.max_outer_iters, tol=cgc_tol,
                              status=status, iters=iters, inc_hist=inc, active=active, work=work)
            if ref is not None:
                record(U, 0, M, k, status, iters)
            mark(f"k={k} krylov fgr + cgc")
            if int(active.item()) == 0:
                break
        return BatchResult(U, iters, status, inc, imag, err, me)
    for lo in range(0, M, B):
        hi = min(M, lo + B)
        ob = op.select(lo, hi)
        Ub = U[lo:hi]
        Mb = hi - lo
        ob.fine_factor(grid.deltat)
        mark(f"batch {lo}:{hi} real factor")
        Lt_c, Dinv_c = ob.shifted_factors(tables, N, grid.deltaT)
        mark("complex factors")
        R = empty(Mb, N, nx)
        nw = int(_lib.query("kle_2d_cgc_work_doubles", Mb, N, op.n))
        work = torch.zeros(max(nw, 1), dtype=torch.float64, device="cuda")
        st, it, ih = status[lo:hi], iters[lo:hi], inc[lo:hi]
        if ref is not None:
            active.zero_()
            record(Ub, lo, Mb, 0, st, it)
            if stop_ref and int(active.item()) == 0:
                del Lt_c, Dinv_c, R, work, ob
                continue
        for k in range(1, cfg.max_outer_iters + 1):
            ob.fgr(Ub, tables, grid, cfg.alpha, R, status=st)
            mark(f"k={k} fgr")
            active.zero_()
            _lib.call("kle_2d_cgc_f64", ptr(R), None, ptr(Ub), None, ptr(Lt_c), ptr(Dinv_c), ptr(tables.inv_scaling),
                      Mb, N, op.n, k, cfg.max_outer_iters, cgc_tol, ptr(st), ptr(it), None, ptr(ih), ptr(active),
                      ptr(work), nw, stream_ptr())
            if ref is not None:
                record(Ub, lo, Mb, k, st, it)
            mark(f"k={k} cgc")
            if int(active.item()) == 0:
                break
        del Lt_c, Dinv_c, R, work, ob
    return BatchResult(U, iters, status, inc, imag, err, me)
