"""End-to-end batched KLE-CGC solve (the composition the reference runs per
sample in ``_run_one_sample``, ``pintuq/experiments.py:212-235``, kle-pcgc
branch: ``surrogate_predict`` -> ``pcgc_solve``), for M samples at once on
one device, plus the sharded multi-GPU moments.

    xi (M, d)  --kl_tridiag-->  A_s                      (coefficient field)
               --fine_factor--> LDL^T blobs of I + dt A_s
               --gpc basis + DMMA GEMM--> U0 = mean + Psi C
               --kle_pcgc_solve_f64--> U, iteration counts, increments
               --col sums (+ NCCL allreduce)--> mean, variance
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import SolverConfig, TimeGrid
from .device import AlphaTables, DeviceOperator, require_cuda, to_dev, torch
from .moments import two_pass_moments
from .pcgc import BatchResult, build_alpha_circulant, pcgc_solve_device
from .surrogate import DeviceSurrogate, KLGpcSurrogate


@dataclass
class KleCgcResult:
    batch: BatchResult
    U0: "torch.Tensor | None" = None


class KleCgcSolver:
    """KLE-CGC for a batch of samples of a KL-coefficient model."""

    def __init__(self, model, grid: TimeGrid, cfg: SolverConfig, surrogate: KLGpcSurrogate):
        require_cuda()
        if getattr(model, "kl_table", None) is None:
            raise NotImplementedError("KleCgcSolver needs a KL-coefficient model (kl_table)")
        self.model, self.grid, self.cfg = model, grid, cfg
        self.surrogate = DeviceSurrogate(surrogate)
        self.tables = AlphaTables(build_alpha_circulant(grid.n_coarse, cfg.alpha))
        self._ws = None

    def solve(self, xi, keep_initial: bool = False, stop_on: str = "increment",
              with_reference: bool = False, diagnostics: bool = False) -> KleCgcResult:
        """xi: (M, d) host array or device tensor.

        ``stop_on="reference"`` (or ``with_reference``) computes the serial fine
        reference of every sample on the device and records the per-iteration
        errors against it, as the reference harness does for every solve
        (``_run_one_sample``, ``pintuq/experiments.py:212-235``: ``fine_reference``
        then ``pcgc_solve(..., reference=, stop_on="reference")``); the
        harness's mean-error tables are ``result.batch.error_summary(tol)``.
        ``diagnostics`` records max_imag_residue per sample (an extra
        full-spectrum three-step launch per iteration)."""
        xi_d = to_dev(xi).reshape(-1, self.model.parameter_dim)
        op = DeviceOperator.from_model(self.model, xi_d)
        reference = None
        if stop_on == "reference" or with_reference:
            from .propagators import fine_reference_batched

            reference = fine_reference_batched(op, self.grid)
        U = self.surrogate.predict(xi_d)
        U0 = U.clone() if keep_initial else None
        from .twod import DeviceOperator2D

        if isinstance(op, DeviceOperator2D):
            # the 2D loop sizes its own per-batch buffers from the free memory:
            # a 1D workspace here would only shrink its batches
            self._ws = None
        else:
            from . import _lib

            if self._ws is None:
                self._ws = torch.empty(0, dtype=torch.uint8, device="cuda")
            need = int(_lib.query("kle_pcgc_workspace_bytes", op.M, self.grid.n_coarse, self.model.nx))
            if self._ws.numel() < need:
                self._ws = torch.empty(need, dtype=torch.uint8, device="cuda")
        if isinstance(op, DeviceOperator2D):
            res = pcgc_solve_device(op, U, self.grid, self.cfg, self.tables, self._ws, reference=reference,
                                    stop_on=stop_on)
        else:
            res = pcgc_solve_device(op, U, self.grid, self.cfg, self.tables, self._ws, reference=reference,
                                    stop_on=stop_on, diagnostics=diagnostics)
        return KleCgcResult(res, U0)

    @staticmethod
    def moments(result: KleCgcResult, M_total: int | None = None, group=None):
        U = result.batch.states
        return two_pass_moments(U, M_total if M_total is not None else U.shape[0], group)


def gauss_hermite_grid(d: int, n: int) -> np.ndarray:
    """n^d probabilists' Gauss-Hermite tensor grid (last coordinate fastest)."""
    import itertools

    nodes, _ = np.polynomial.hermite_e.hermegauss(n)
    return np.array(list(itertools.product(nodes, repeat=d)))
