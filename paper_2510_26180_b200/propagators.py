"""Fine/coarse backward-Euler propagators on the device — drop-in for
``pintuq.propagators`` (``/root/reference/pkg/src/pintuq/propagators.py``)
plus the initial-guess builders of ``pintuq.parareal`` (:63-84).

Same signatures and error behaviour; batched variants operate on device
tensors of many samples / many start states at once.
"""
from __future__ import annotations

import numpy as np

from .core import CoarseTrajectory, ParameterSample, RngStream, SolverConfig, TimeGrid
from .device import DeviceOperator, to_dev

_STEP_MATCH_TOL = 1e-9  # pintuq/propagators.py:14


def _linear_only(model):
    if not getattr(model, "is_linear", False):
        raise NotImplementedError("the device propagators cover linear models only")


def _sweep1(model, xi, cfg, u, h, J, nseg=1):
    """One sample: (nseg, nx) states after J, 2J, ... steps of size h from u.
    Linear models: partitioned LDL^T sweeps; the nonlinear tridiagonal models
    (Burgers, Allen-Cahn): the fused Newton sweeps (pintuq/propagators.py:82-99)."""
    from .nonlinear import NewtonOperator, is_newton_model

    if is_newton_model(model):
        op = NewtonOperator.from_model(model, [xi], cfg)
        out, _ = op.sweep(to_dev(u)[None, None], h, J, nseg)
        return out[0, 0].cpu().numpy()
    _linear_only(model)
    op = DeviceOperator.from_model(model, [xi])
    return op.sweep(to_dev(u)[None, None], h, J, nseg=nseg)[0, 0].cpu().numpy()


def backward_euler_step(model, u, t_from: float, dt: float, xi: ParameterSample, cfg: SolverConfig):
    """One implicit Euler step (``pintuq/propagators.py:102-118``)."""
    if dt <= 0:
        raise ValueError(f"step size must be positive, got {dt}")
    u = model.check_state(u)
    return _sweep1(model, xi, cfg, u, dt, 1)[0]


def propagate_fine(model, u, t_from: float, t_to: float, grid: TimeGrid, xi: ParameterSample,
                   cfg: SolverConfig):
    """J backward-Euler steps of dt across one coarse subinterval
    (``pintuq/propagators.py:121-145``)."""
    if abs((t_to - t_from) - grid.deltaT) > _STEP_MATCH_TOL * grid.deltaT:
        raise ValueError(
            f"fine propagation interval [{t_from}, {t_to}] does not span one coarse step {grid.deltaT}"
        )
    u = model.check_state(u)
    return _sweep1(model, xi, cfg, u, grid.deltat, grid.n_fine_per_coarse)[0]


def propagate_coarse(model, u, t_from: float, t_to: float, xi: ParameterSample, cfg: SolverConfig):
    """One backward-Euler step over the interval (``pintuq/propagators.py:148-157``)."""
    return backward_euler_step(model, u, t_from, t_to - t_from, xi, cfg)


def fine_reference(model, xi: ParameterSample, grid: TimeGrid, cfg: SolverConfig) -> CoarseTrajectory:
    """Serial F trajectory at the coarse points (``pintuq/propagators.py:160-176``)."""
    u0 = np.asarray(model.initial_condition(xi), dtype=float)
    traj = CoarseTrajectory(u0, _sweep1(model, xi, cfg, u0, grid.deltat, grid.n_fine_per_coarse, grid.n_coarse))
    traj.assert_finite()
    return traj


def coarse_sweep_init(model, xi: ParameterSample, grid: TimeGrid, cfg: SolverConfig) -> CoarseTrajectory:
    """N serial coarse steps from u0 (``pintuq/parareal.py:74-84``)."""
    u0 = np.asarray(model.initial_condition(xi), dtype=float)
    return CoarseTrajectory(u0, _sweep1(model, xi, cfg, u0, grid.deltaT, 1, grid.n_coarse))


def random_guess_init(model, xi: ParameterSample, grid: TimeGrid, rng: RngStream) -> CoarseTrajectory:
    """Entrywise U[-1,1] * |u0|_inf (``pintuq/parareal.py:63-71``); the draws
    come from the host PCG64 stream so they match the reference's."""
    u0 = np.asarray(model.initial_condition(xi), dtype=float)
    scale = np.max(np.abs(u0))
    return CoarseTrajectory(u0, scale * rng.uniform(-1.0, 1.0, size=(grid.n_coarse, model.nx)))


# ---------------------------------------------------------------------------
# batched device entry points
# ---------------------------------------------------------------------------
def propagate_fine_batched(op: DeviceOperator, starts, grid: TimeGrid):
    """starts: (M, Q, nx) device tensor -> F of each start, (M, Q, nx)."""
    return op.sweep(starts, grid.deltat, grid.n_fine_per_coarse)[:, :, 0]


def coarse_sweep_init_batched(op: DeviceOperator, grid: TimeGrid):
    """(M, N, nx) coarse-sweep initial guesses for all samples of ``op``."""
    start = op.u0[None, None].expand(op.M, 1, op.nx).contiguous()
    return op.sweep(start, grid.deltaT, 1, nseg=grid.n_coarse)[:, 0]


def fine_reference_batched(op: DeviceOperator, grid: TimeGrid):
    start = op.u0[None, None].expand(op.M, 1, op.nx).contiguous()
    return op.sweep(start, grid.deltat, grid.n_fine_per_coarse, nseg=grid.n_coarse)[:, 0]
