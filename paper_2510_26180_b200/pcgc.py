"""Diagonalised parallel coarse-grid correction on the device — drop-in for
``pintuq.pcgc`` (``/root/reference/pkg/src/pintuq/pcgc.py``).

Same names, argument meaning and error behaviour as the reference:
``build_alpha_circulant`` (:68-76), ``three_step_solve`` (:148-172),
``assemble_rhs_blocks`` (:175-197), ``cgc_correct`` (:208-243, linear
branch), ``pcgc_solve`` (:273-358). The per-sample functions run batches of
one; ``pcgc_solve_batched`` is the production entry point (M samples, each
frozen at its own iteration count, one C-ABI call).
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import (
    NonConvergenceError,
    CoarseTrajectory,
    IterationRecord,
    IterationTrace,
    MaxItersExceededError,
    ParameterSample,
    SolverConfig,
    TimeGrid,
)
from .device import AlphaTables, DeviceOperator, empty, ptr, require_cuda, stream_ptr, to_dev, torch

SAMPLE_ACTIVE, SAMPLE_CONVERGED, SAMPLE_MAXITERS, SAMPLE_NONFINITE, SAMPLE_NEWTON = 0, 1, 2, 3, 4


@dataclass(frozen=True)
class AlphaCirculantSpec:
    """Eigenstructure of C_alpha (``pintuq/pcgc.py:35-65``)."""

    n: int
    alpha: float
    eigenvalues: np.ndarray
    scaling: np.ndarray

    def dense_matrix(self) -> np.ndarray:
        C = np.eye(self.n) - np.eye(self.n, k=-1)
        C[0, self.n - 1] -= self.alpha
        return C

    def dft_matrix(self) -> np.ndarray:
        jk = np.outer(np.arange(self.n), np.arange(self.n))
        return np.exp(2j * np.pi * jk / self.n) / np.sqrt(self.n)

    def eigenvector_matrix(self) -> np.ndarray:
        return (1.0 / self.scaling)[:, None] * self.dft_matrix()

    def inverse_eigenvector_matrix(self) -> np.ndarray:
        return self.dft_matrix().conj().T * self.scaling[None, :]


def build_alpha_circulant(n: int, alpha: float) -> AlphaCirculantSpec:
    """lambda_n = 1 - alpha^{1/N} e^{-2 pi i n/N}, scaling_j = alpha^{j/N}."""
    if n < 1:
        raise ValueError(f"need at least one subinterval, got {n}")
    if not 0.0 < alpha < 1.0:
        raise ValueError(f"alpha must lie in (0, 1), got {alpha}")
    root = alpha ** (1.0 / n)
    eigenvalues = 1.0 - root * np.exp(-2j * np.pi * np.arange(n) / n)
    scaling = alpha ** (np.arange(n) / n)
    return AlphaCirculantSpec(int(n), float(alpha), eigenvalues, scaling)


# ---------------------------------------------------------------------------
def _cgc_scratch(M, N, nx):
    nbytes = int(_lib.query("kle_cgc_scratch_bytes", M, N, nx))
    return torch.empty(max(nbytes, 8), dtype=torch.uint8, device="cuda"), nbytes


def shift_factors(op: DeviceOperator, tables: AlphaTables, N: int, deltaT: float):
    """Pivots of (lambda_f I + dT A) for every sample (iteration invariant), or
    None for shapes that form them on the fly (``kle_shift_factor_f64``)."""
    nbytes = int(_lib.query("kle_shift_factor_bytes", op.M, N, op.nx))
    if nbytes == 0:
        return None
    sfac = empty(nbytes // 8)
    _lib.call("kle_shift_factor_f64", ptr(op.dia), ptr(op.off), ptr(tables.lam), op.M, N, op.nx, deltaT, ptr(sfac),
              stream_ptr())
    return sfac


def imag_residue_device(op: DeviceOperator, tables: AlphaTables, N: int, deltaT: float, r, prescaled=False,
                        imag=None, status=None):
    """max|Im u| of the reference's three-step solve (``pintuq/pcgc.py:170-172``)
    for every sample: all N shifted systems solved independently and no
    Hermitian completion (``kle_imag_residue_f64``), max-accumulated into
    ``imag`` (M,). The production CGC kernels use the Hermitian symmetry and
    return real fields, so this is a separate diagnostic launch."""
    M, _, nx = r.shape
    if imag is None:
        imag = torch.zeros(M, dtype=torch.float64, device="cuda")
    nbytes = int(_lib.query("kle_imag_residue_scratch_bytes", M, N, nx))
    scratch = torch.empty(max(nbytes, 8), dtype=torch.uint8, device="cuda")
    _lib.call("kle_imag_residue_f64", ptr(r.contiguous()), None if prescaled else ptr(tables.scaling),
              ptr(tables.inv_scaling), ptr(tables.lam), ptr(op.dia), ptr(op.off), ptr(status), M, N, nx, deltaT,
              ptr(imag), ptr(scratch), nbytes, stream_ptr())
    return imag


def three_step_device(op: DeviceOperator, tables: AlphaTables, N: int, deltaT: float, r, prescaled=False,
                      sfac="auto", diagnostics: bool = True):
    """u = V (Lambda (x) I + dT I (x) A)^{-1} V^{-1} r for every sample;
    r: (M, N, nx) device tensor. Returns (u, imag (M,)); ``imag`` is the
    max_imag_residue diagnostic when ``diagnostics`` (else zeros)."""
    M, _, nx = r.shape
    u = empty(M, N, nx)
    imag = torch.zeros(M, dtype=torch.float64, device="cuda")
    if diagnostics:
        imag_residue_device(op, tables, N, deltaT, r, prescaled, imag)
    if isinstance(sfac, str):
        sfac = shift_factors(op, tables, N, deltaT)
    if sfac is not None:  # cluster path: per-sample reduction slots (zeroed by the call)
        scratch, nbytes = torch.empty(16 * M, dtype=torch.uint8, device="cuda"), 16 * M
    else:
        scratch, nbytes = _cgc_scratch(M, N, nx)
    _lib.call("kle_three_step_f64", ptr(r.contiguous()), None if prescaled else ptr(tables.scaling),
              ptr(tables.inv_scaling), ptr(tables.lam), ptr(op.dia), ptr(op.off), ptr(sfac), M, N, nx, deltaT,
              ptr(u), None, ptr(scratch), nbytes, stream_ptr())
    return u, imag


def _block_dft(v, sign: int) -> np.ndarray:
    require_cuda()
    v = np.asarray(v)
    shape = v.shape
    c = np.ascontiguousarray(v.reshape(shape[0], -1), dtype=np.complex128)
    src = torch.as_tensor(c.view(np.float64), device="cuda")
    out = torch.empty_like(src)
    _lib.call("kle_block_dft_f64", ptr(src), ptr(out), shape[0], c.shape[1], sign, stream_ptr())
    return out.cpu().numpy().view(np.complex128).reshape(shape)


def forward_dft(v) -> np.ndarray:
    """F (x) I on a block vector of shape (N, ...), entries omega^(jk)/sqrt(N),
    omega = exp(+2 pi i / N) (``pintuq/pcgc.py:79-82``); on the device."""
    return _block_dft(v, +1)


def inverse_dft(v) -> np.ndarray:
    """F* (x) I, the inverse of :func:`forward_dft` (``pintuq/pcgc.py:85-87``)."""
    return _block_dft(v, -1)


def factor_shifted(spec: AlphaCirculantSpec, mean_jac, deltaT: float) -> list:
    """Solver callables for the N shifted systems (lambda_n I - deltaT J)
    (``pintuq/pcgc.py:90-145``) for a tridiagonal J (nx = 1 included); each
    callable solves one right-hand side (or a stack, last axis nx) on the
    device and raises ``SingularShiftError`` on a zero pivot. Wider
    Jacobians: the batched 2D path (``three_step_solve``) factors them."""
    import scipy.sparse as sp

    from .core import SingularShiftError

    J = sp.csr_matrix(np.atleast_2d(mean_jac) if not sp.issparse(mean_jac) else mean_jac)
    nx = J.shape[0]
    coo = J.tocoo()
    if coo.nnz and int(np.max(np.abs(coo.row - coo.col))) > 1:
        raise NotImplementedError("device factor_shifted covers tridiagonal Jacobians")
    require_cuda()
    sub = to_dev(np.asarray(J.diagonal(-1), dtype=float) if nx > 1 else np.zeros(1))
    dia = to_dev(np.asarray(J.diagonal(0), dtype=float))
    sup = to_dev(np.asarray(J.diagonal(1), dtype=float) if nx > 1 else np.zeros(1))

    def make(lam):
        def solve(p):
            p = np.asarray(p)
            c = np.ascontiguousarray(p.reshape(-1, nx), dtype=np.complex128)
            src = torch.as_tensor(c.view(np.float64), device="cuda")
            q = torch.empty_like(src)
            work = torch.empty_like(src)
            st = torch.zeros(c.shape[0], dtype=torch.int32, device="cuda")
            _lib.call("kle_shifted_tridiag_solve_f64", ptr(sub), ptr(dia), ptr(sup), float(lam.real), float(lam.imag),
                      float(deltaT), ptr(src), ptr(q), ptr(work), nx, c.shape[0], ptr(st), stream_ptr())
            if bool(st.any().item()):
                raise SingularShiftError(f"shifted system at lambda={lam} is singular")
            return q.cpu().numpy().view(np.complex128).reshape(p.shape)

        return solve

    return [make(complex(lam)) for lam in spec.eigenvalues]


def three_step_solve(spec: AlphaCirculantSpec, mean_jac, deltaT: float, r, solvers=None, executor=None):
    """Solve (C_alpha (x) I - dT I (x) J) u = r (``pintuq/pcgc.py:148-172``)
    for a symmetric tridiagonal J on the device. Returns (u, imag_residue)."""
    import scipy.sparse as sp

    r = np.asarray(r, dtype=float)
    if r.shape[0] != spec.n:
        raise ValueError(f"block count {r.shape[0]} does not match N={spec.n}")
    require_cuda()
    A = -sp.csr_matrix(np.atleast_2d(mean_jac) if not sp.issparse(mean_jac) else mean_jac)
    nx = A.shape[0]
    r2 = r.reshape(spec.n, nx)
    coo = A.tocoo()
    bw = int(np.max(np.abs(coo.row - coo.col))) if coo.nnz else 0
    if bw > 1:  # 5-point (2D) Jacobian of an n x n grid: bandwidth n
        from .twod import DeviceOperator2D, three_step_device2d

        n = bw
        if n * n != nx or spec.n % 2:
            raise NotImplementedError("device three_step_solve: 5-point operators on an n x n grid, N even")
        ex, ey = np.zeros(nx), np.zeros(nx)
        ex[:-1] = A.diagonal(1)
        ey[:-n] = A.diagonal(n)
        op = DeviceOperator2D(to_dev(A.diagonal(0)[None]), to_dev(ex[None]), to_dev(ey[None]), n, 0.0,
                              to_dev(np.zeros(nx)))
        u, imag = three_step_device2d(op, AlphaTables(spec), spec.n, deltaT, to_dev(r2[None]))
        return u[0].cpu().numpy().reshape(r.shape), float(imag[0].item())
    dia = np.asarray(A.diagonal(0), dtype=float)
    off = np.zeros(nx)
    if nx > 1:
        coo = A.tocoo()
        if coo.nnz and np.max(np.abs(coo.row - coo.col)) > 1:
            raise NotImplementedError("device three_step_solve supports tridiagonal Jacobians only")
        if not np.array_equal(A.diagonal(-1), A.diagonal(1)):
            raise NotImplementedError("device three_step_solve supports symmetric Jacobians only")
        off[:-1] = A.diagonal(1)
    op = DeviceOperator(to_dev(dia[None]), to_dev(off[None]), 0.0, to_dev(np.zeros(nx)))
    u, imag = three_step_device(op, AlphaTables(spec), spec.n, deltaT, to_dev(r2[None]))
    return u[0].cpu().numpy().reshape(r.shape), float(imag[0].item())


def _grid_steps(grid: TimeGrid):
    return grid.deltaT, grid.deltat


def assemble_rhs_blocks(model, xi: ParameterSample, grid: TimeGrid, cfg: SolverConfig, U_prev, fine_ends,
                        executor=None):
    """b_n = F_end_n - G(prev_n), prev = [alpha U_N, U_1..U_{N-1}]
    (``pintuq/pcgc.py:175-197``)."""
    op = DeviceOperator.from_model(model, [xi])
    U = to_dev(np.asarray(U_prev, dtype=float))
    prev = torch.cat([cfg.alpha * U[-1:], U[:-1]], dim=0) if U.shape[0] > 1 else cfg.alpha * U
    G = op.sweep(prev[None].contiguous(), grid.deltaT, 1)[:, :, 0]
    F = to_dev(np.asarray(fine_ends, dtype=float))[None]
    b = empty(*F.shape)
    _lib.call("kle_axpby_f64", ptr(F), ptr(G.contiguous()), ptr(b), 1.0, -1.0, F.numel(), stream_ptr())
    return b[0].cpu().numpy()


def _fgr(op, tables, U, R, J, grid, alpha, F_given=None, F_out=None, status=None):
    M, N, nx = U.shape
    dT, dt = _grid_steps(grid)
    blob = op.blob(dt) if F_given is None else op.dia  # blob unused with F_given
    _lib.call("kle_fgr_f64", ptr(U), ptr(op.u0), ptr(F_given), ptr(F_out), ptr(R), ptr(blob), ptr(op.dia),
              ptr(op.off), ptr(tables.scaling), ptr(status), M, N, nx, J, dt, dT, op.g0, alpha, stream_ptr())


def cgc_correct(model, xi: ParameterSample, grid: TimeGrid, cfg: SolverConfig, U_prev: CoarseTrajectory,
                fine_ends, spec=None, shifted_solvers=None, executor=None):
    """One linear coarse-grid correction (``pintuq/pcgc.py:208-243``):
    returns (CoarseTrajectory, {"inner_iters": 1, "imag_residue": ...})."""
    if not getattr(model, "is_linear", False):
        raise NotImplementedError("the device CGC covers linear models only")
    N = grid.n_coarse
    spec = spec or build_alpha_circulant(N, cfg.alpha)
    op = DeviceOperator.from_model(model, [xi])
    tables = AlphaTables(spec)
    U = to_dev(U_prev.states)[None]
    F = to_dev(np.asarray(fine_ends, dtype=float))[None]
    R = empty(*U.shape)
    from .twod import DeviceOperator2D, three_step_device2d

    if isinstance(op, DeviceOperator2D):
        op.fgr(U, tables, grid, cfg.alpha, R, F_given=F)
        u, imag = three_step_device2d(op, tables, N, grid.deltaT, R, prescaled=True)
    else:
        _fgr(op, tables, U, R, grid.n_fine_per_coarse, grid, cfg.alpha, F_given=F)
        u, imag = three_step_device(op, tables, N, grid.deltaT, R, prescaled=True)
    return CoarseTrajectory(U_prev.initial, u[0].cpu().numpy()), {"inner_iters": 1,
                                                                   "imag_residue": float(imag[0].item())}


# ---------------------------------------------------------------------------
@dataclass
class BatchResult:
    """Outcome of ``pcgc_solve_batched`` (device tensors)."""

    states: "torch.Tensor"      # (M, N, nx) final U
    iters: "torch.Tensor"       # (M,) int32 iteration counts (len(records) - 1)
    status: "torch.Tensor"      # (M,) int32 SAMPLE_* words
    increments: "torch.Tensor"  # (M, max_iters) per-k increments, NaN past the stop
    imag: "torch.Tensor"        # (M,) max imaginary residue (diagnostics=True), else zeros
    err_vs_ref: "torch.Tensor | None" = None  # (M, max_iters+1, N) err_n of record k (k = 0: guess), NaN past the stop
    max_err: "torch.Tensor | None" = None     # (M,) max error of the last record

    def error_summary(self, tol: float, max_iters: int | None = None, group=None):
        """The harness aggregation over this batch (``pintuq/experiments.py:
        314-334``): ``(mean_vectors (k_max+1, N), mean_max_error (k_max+1,),
        mean_iters)``. Error vectors of each good sample (all records finite)
        are padded with their last record and averaged over samples on the
        device (``kle_err_aggregate_f64``); ``mean_iters`` averages
        ``iters_to_tol(tol)`` with unreached tolerances counted as
        ``max_iters`` (the harness's cfg.max_iters). With a process ``group``
        (sharded samples) the per-rank sums and counts are allreduced."""
        if self.err_vs_ref is None:
            raise ValueError("no reference errors were recorded")
        import torch.distributed as dist

        M, K1, N = self.err_vs_ref.shape
        max_iters = K1 - 1 if max_iters is None else int(max_iters)
        err = self.err_vs_ref.contiguous()
        good = torch.empty(M, dtype=torch.int32, device="cuda")
        counts = torch.zeros(2, dtype=torch.int32, device="cuda")
        sums = empty(K1, N)

        def aggregate(k_pad):
            _lib.call("kle_err_aggregate_f64", ptr(err), ptr(self.iters), M, N, K1 - 1, k_pad, ptr(good),
                      ptr(counts), ptr(sums), stream_ptr())

        it = self.iters_to_tol(tol)
        it = torch.where(it < 0, torch.full_like(it, max_iters), it).to(torch.float64)
        sharded = group is not None or (dist.is_available() and dist.is_initialized())
        aggregate(-1)
        if sharded:  # pad every rank's samples to the global k_max, then sum sums and counts
            kmax = counts[1:2].clone()
            dist.all_reduce(kmax, op=dist.ReduceOp.MAX, group=group)
            aggregate(int(kmax.item()))
            stats = torch.stack([counts[0].to(torch.float64), it.sum(),
                                 torch.tensor(float(M), device="cuda", dtype=torch.float64)])
            dist.all_reduce(sums, group=group)
            dist.all_reduce(stats, group=group)
            n_good, k_max = float(stats[0].item()), int(kmax.item())
            mean_iters = float((stats[1] / stats[2]).item()) if stats[2] > 0 else float("nan")
        else:
            n_good, k_max = float(counts[0].item()), int(counts[1].item())
            mean_iters = float(it.mean().item()) if M else float("nan")
        if n_good == 0:
            return np.full((1, N), np.nan), np.array([np.nan]), mean_iters
        mv = (sums[:k_max + 1] / n_good).cpu().numpy()
        return mv, mv.max(axis=1), mean_iters

    def iters_to_tol(self, tol: float):
        """Per sample, the first k whose max error vs the reference is <= tol
        (IterationTrace.iters_to_tol, pintuq/parareal.py:49-54); -1 if none."""
        if self.err_vs_ref is None:
            raise ValueError("no reference errors were recorded")
        me = self.err_vs_ref.amax(dim=2)  # NaN rows (past the stop) stay NaN
        ok = me <= tol
        first = torch.where(ok.any(dim=1), ok.int().argmax(dim=1), torch.full_like(ok[:, 0], -1, dtype=torch.int64))
        return first

    def failures(self) -> dict:
        """{sample index: exception} for every sample that did not converge,
        mapped to the reference's error types (MaxItersExceededError,
        pintuq/pcgc.py:352-357; non-finite trajectory ValueError,
        pintuq/core.py:179-181)."""
        st = self.status.cpu().numpy()
        out = {}
        for i in np.nonzero(st != SAMPLE_CONVERGED)[0]:
            if st[i] == SAMPLE_MAXITERS:
                out[int(i)] = MaxItersExceededError(f"sample {int(i)} did not reach tol")
            elif st[i] == SAMPLE_NEWTON:
                out[int(i)] = NonConvergenceError(f"sample {int(i)}: simplified Newton CGC stalled")
            elif st[i] == SAMPLE_NONFINITE:
                out[int(i)] = ValueError(f"sample {int(i)}: trajectory contains non-finite entries")
            else:
                out[int(i)] = RuntimeError(f"sample {int(i)}: status {int(st[i])}")
        return out

    def raise_for_status(self):
        """Raise the first per-sample failure (reference ``raise_on_max=True`` behaviour)."""
        f = self.failures()
        if f:
            i = min(f)
            raise f[i]


def pcgc_solve_device(op: DeviceOperator, U, grid: TimeGrid, cfg: SolverConfig, tables: AlphaTables = None,
                      workspace=None, reference=None, stop_on: str = "increment",
                      diagnostics: bool = False) -> BatchResult:
    """The production loop: U (M, N, nx) device tensor is overwritten with the
    final states (``kle_pcgc_solve_f64``). ``reference`` (M, N, nx), e.g.
    ``fine_reference_batched``, adds the per-iteration error records of
    ``pcgc_solve(reference=...)``; ``stop_on="reference"`` stops each sample
    at its first record with max error <= tol (``kle_pcgc_solve_ref_f64``).
    ``diagnostics`` adds the per-iteration max_imag_residue diagnostic (an
    extra full-spectrum three-step launch per iteration; ``imag`` is zeros
    otherwise)."""
    from .twod import DeviceOperator2D, pcgc_solve_device2d

    if stop_on not in ("increment", "reference"):
        raise ValueError(f"stop_on must be 'increment' or 'reference', not {stop_on!r}")
    if stop_on == "reference" and reference is None:
        raise ValueError("stop_on='reference' requires a reference trajectory")
    if isinstance(op, DeviceOperator2D):
        return pcgc_solve_device2d(op, U, grid, cfg, tables, reference=reference, stop_on=stop_on)
    from .nonlinear import NewtonOperator, pcgc_solve_newton

    if isinstance(op, NewtonOperator):
        return pcgc_solve_newton(op, U, grid, cfg, reference=reference, stop_on=stop_on)
    M, N, nx = U.shape
    if N != grid.n_coarse or nx != op.nx or M != op.M:
        raise ValueError("initial guess length does not match the time grid")
    tables = tables or AlphaTables(build_alpha_circulant(N, cfg.alpha))
    nbytes = int(_lib.query("kle_pcgc_workspace_bytes", M, N, nx))
    if workspace is None or workspace.numel() < nbytes:
        workspace = torch.empty(max(nbytes, 8), dtype=torch.uint8, device="cuda")
    status = torch.empty(M, dtype=torch.int32, device="cuda")
    iters = torch.empty(M, dtype=torch.int32, device="cuda")
    inc = empty(M, cfg.max_outer_iters)
    imag = torch.zeros(M, dtype=torch.float64, device="cuda")
    imag_arg = ptr(imag) if diagnostics else None
    common = (ptr(U), ptr(op.u0), ptr(op.dia), ptr(op.off), ptr(op.blob(grid.deltat)), ptr(tables.scaling),
              ptr(tables.inv_scaling), ptr(tables.lam), M, N, nx, grid.n_fine_per_coarse, grid.t_final, cfg.alpha,
              op.g0, cfg.tol, cfg.max_outer_iters)
    if reference is None:
        _lib.call("kle_pcgc_solve_f64", *common, ptr(status), ptr(iters), ptr(inc), imag_arg, ptr(workspace),
                  nbytes, stream_ptr())
        return BatchResult(U, iters, status, inc, imag)
    ref = to_dev(reference).contiguous()
    if tuple(ref.shape) != (M, N, nx):
        raise ValueError("reference trajectory shape does not match the initial guess")
    err = empty(M, cfg.max_outer_iters + 1, N)
    me = empty(M)
    _lib.call("kle_pcgc_solve_ref_f64", *common, ptr(ref), int(stop_on == "reference"), ptr(status), ptr(iters),
              ptr(inc), ptr(err), ptr(me), imag_arg, ptr(workspace), nbytes, stream_ptr())
    return BatchResult(U, iters, status, inc, imag, err, me)


def pcgc_solve_batched(model, xis, grid: TimeGrid, cfg: SolverConfig, init_states, reference=None,
                       stop_on: str = "increment", diagnostics: bool = False) -> BatchResult:
    """Batched ``pcgc_solve`` over M samples (``reference``: (M, N, nx) or
    ``"fine"`` for the batched serial fine reference of every sample)."""
    op = DeviceOperator.from_model(model, xis)
    U = to_dev(init_states).clone()
    if isinstance(reference, str) and reference == "fine":
        from .propagators import fine_reference_batched

        reference = fine_reference_batched(op, grid)
    return pcgc_solve_device(op, U, grid, cfg, reference=reference, stop_on=stop_on, diagnostics=diagnostics)


def pcgc_solve(model, xi: ParameterSample, grid: TimeGrid, cfg: SolverConfig, init: CoarseTrajectory,
               reference: CoarseTrajectory | None = None, stop_on: str = "increment", store_states: bool = False,
               executor=None, raise_on_max: bool = True, solver_name: str = "pcgc") -> IterationTrace:
    """Single-sample drop-in for ``pintuq.pcgc.pcgc_solve`` (:273-358).

    Each outer iteration is one fused F + rhs launch and one CGC launch; the
    trace bookkeeping (errors vs the reference, stored states) is host side."""
    if stop_on not in ("increment", "reference"):
        raise ValueError(f"stop_on must be 'increment' or 'reference', not {stop_on!r}")
    if stop_on == "reference" and reference is None:
        raise ValueError("stop_on='reference' requires a reference trajectory")
    if init.n_coarse != grid.n_coarse:
        raise ValueError("initial guess length does not match the time grid")
    model.validate(xi)
    from .nonlinear import is_newton_model

    if is_newton_model(model):
        return _pcgc_newton_trace(model, xi, grid, cfg, init, reference, stop_on, raise_on_max, solver_name)
    if not getattr(model, "is_linear", False):
        raise NotImplementedError("the device PCGC covers linear and tridiagonal Newton models only")
    N = grid.n_coarse
    u0 = np.asarray(model.initial_condition(xi), dtype=float)
    op = DeviceOperator.from_model(model, [xi])
    tables = AlphaTables(build_alpha_circulant(N, cfg.alpha))
    U = to_dev(init.states)[None].clone()
    nx = U.shape[2]
    R = empty(1, N, nx)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    iters = torch.zeros(1, dtype=torch.int32, device="cuda")
    inc = empty(1, cfg.max_outer_iters).fill_(float("nan"))
    imag = torch.zeros(1, dtype=torch.float64, device="cuda")
    from .twod import DeviceOperator2D

    is2d = isinstance(op, DeviceOperator2D)
    krylov2d = is2d and op.solver == "krylov"
    if is2d:
        if N % 2:
            raise NotImplementedError("the 2D CGC needs an even number of subintervals")
        fac2d = None if krylov2d else op.shifted_factors(tables, N, grid.deltaT)
        nbytes = int(_lib.query("kle_2d_cgc_krylov_work_doubles" if krylov2d else "kle_2d_cgc_work_doubles", 1, N,
                                op.n))
        scratch = torch.zeros(max(nbytes, 1), dtype=torch.float64, device="cuda")
    else:
        sfac = shift_factors(op, tables, N, grid.deltaT)
        if sfac is not None:  # cluster path: zero-initialised reduction slots
            scratch, nbytes = torch.zeros(16, dtype=torch.uint8, device="cuda"), 16
        else:
            scratch, nbytes = _cgc_scratch(1, N, nx)

    def err(states):
        if reference is None:
            return None, None
        e = np.max(np.abs(states - reference.states), axis=1)
        return e, float(np.max(e))

    trace = IterationTrace(solver=solver_name, stop_on=stop_on)
    trace.diagnostics["max_imag_residue"] = 0.0
    host = np.asarray(init.states, dtype=float).copy()
    ev, me = err(host)
    trace.records.append(IterationRecord(0, None, ev, me, 0.0))
    if store_states:
        trace.states_history.append(host.copy())
    if stop_on == "reference" and me is not None and me <= cfg.tol:
        trace.converged = True
        trace.trajectory = CoarseTrajectory(u0, host)
        return trace
    dT = grid.deltaT
    for k in range(1, cfg.max_outer_iters + 1):
        tic = time.perf_counter()
        # tol < 0 keeps the device from freezing the sample; the stop test is ours
        if krylov2d:
            from .twod import cgc_krylov

            op.fgr(U, tables, grid, cfg.alpha, R, status=status)
            cgc_krylov(op, tables, N, dT, R, U=U, k=k, max_iters=cfg.max_outer_iters, tol=-1.0, status=status,
                       iters=iters, inc_hist=inc, work=scratch)
        elif is2d:
            op.fgr(U, tables, grid, cfg.alpha, R, status=status)
            _lib.call("kle_2d_cgc_f64", ptr(R), None, ptr(U), None, ptr(fac2d[0]), ptr(fac2d[1]),
                      ptr(tables.inv_scaling), 1, N, op.n, k, cfg.max_outer_iters, -1.0, ptr(status), ptr(iters),
                      None, ptr(inc), None, ptr(scratch), nbytes, stream_ptr())
        else:
            _fgr(op, tables, U, R, grid.n_fine_per_coarse, grid, cfg.alpha)
            imag_residue_device(op, tables, N, dT, R, prescaled=True, imag=imag)
            _lib.call("kle_cgc_update_f64", ptr(R), ptr(U), ptr(tables.inv_scaling), ptr(tables.lam), ptr(op.dia),
                      ptr(op.off), ptr(sfac), 1, N, nx, dT, k, cfg.max_outer_iters, -1.0, None, None, ptr(inc),
                      None, None, ptr(scratch), nbytes, stream_ptr())
        host = U[0].cpu().numpy()
        increment = float(inc[0, k - 1].item())
        wall_ms = 1e3 * (time.perf_counter() - tic)
        ev, me = err(host)
        trace.records.append(IterationRecord(k, increment, ev, me, wall_ms))
        trace.diagnostics["max_imag_residue"] = float(imag[0].item())
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
            f"{solver_name} did not reach tol {cfg.tol:.1e} within {cfg.max_outer_iters} iterations", trace=trace
        )
    return trace


def _pcgc_newton_trace(model, xi, grid, cfg, init, reference, stop_on, raise_on_max, solver_name):
    """pcgc_solve for one sample of a nonlinear model: the batched device loop
    with M = 1 (simplified-Newton CGC, pcgc.py:245-270), trace rebuilt from its
    records."""
    from .core import NonConvergenceError
    from .nonlinear import NewtonOperator, pcgc_solve_newton

    u0 = np.asarray(model.initial_condition(xi), dtype=float)
    op = NewtonOperator.from_model(model, [xi], cfg)
    U = to_dev(init.states)[None].clone()
    ref = None if reference is None else to_dev(reference.states)[None]
    res = pcgc_solve_newton(op, U, grid, cfg, ref, stop_on)
    st = int(res.status[0].item())
    if st == 4:
        raise NonConvergenceError("simplified Newton stalled after 150 diagonalized solves",
                                  last_iterate=res.states[0].cpu().numpy())
    k = int(res.iters[0].item())
    trace = IterationTrace(solver=solver_name, stop_on=stop_on)
    trace.diagnostics["max_imag_residue"] = 0.0
    errs = res.err_vs_ref[0].cpu().numpy() if res.err_vs_ref is not None else None
    incs = res.increments[0].cpu().numpy()
    for j in range(k + 1):
        ev = None if errs is None else errs[j]
        trace.records.append(IterationRecord(j, None if j == 0 else float(incs[j - 1]), ev,
                                             None if ev is None else float(np.max(ev)), 0.0))
    trace.trajectory = CoarseTrajectory(u0, res.states[0].cpu().numpy())
    trace.converged = st == 1
    trace.trajectory.assert_finite()
    if not trace.converged and raise_on_max:
        raise MaxItersExceededError(
            f"{solver_name} did not reach tol {cfg.tol:.1e} within {cfg.max_outer_iters} iterations", trace=trace
        )
    return trace
