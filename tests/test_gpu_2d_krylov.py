"""The matrix-free Krylov 2D path (Jacobi-PCG fine steps,
Jacobi-COCG shifted solves, kle_2d_krylov.cu) against the same goldens of the
unmodified reference as the direct banded path (tests/test_gpu_2d.py), at the
small c3s shape and at the full config-3 shape. Tolerances are the direct
path's: iteration counts exact, fields within 1e-10 relative (the Krylov
solves stop at a relative residual of 1e-13)."""
import time

import numpy as np
import pytest

from tests import test_gpu_2d as direct

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def krylov(monkeypatch):
    monkeypatch.setenv("KLE_2D_SOLVER", "krylov")


def test_propagators_2d_krylov(cuda, golden):
    direct.test_propagators_2d(cuda, golden)


def test_three_step_and_cgc_correct_2d_krylov(cuda, golden):
    direct.test_three_step_and_cgc_correct_2d(cuda, golden)


def test_pcgc_batched_2d_small_krylov(cuda, golden):
    direct.test_pcgc_batched_2d_small(cuda, golden)


def test_pcgc_single_sample_dropin_2d_krylov(cuda, golden):
    direct.test_pcgc_single_sample_dropin_2d(cuda, golden)


def test_c3_full_shape_krylov(cuda, golden):
    """n = 127 (nx = 16,129), N = 32, J = 16: one sample, PCGC from the
    coarse sweep, against the reference (c3.npz); prints the PCG/COCG
    iteration totals and the solve time beside the direct path's."""
    import torch

    from paper_2510_26180_b200 import LogNormalKL2D, SolverConfig, make_time_grid
    from paper_2510_26180_b200.device import DeviceOperator
    from paper_2510_26180_b200.pcgc import pcgc_solve_device
    from paper_2510_26180_b200.propagators import coarse_sweep_init_batched

    g = golden("c3")
    model = LogNormalKL2D(n=127, d=10, sigma=0.5, ell=0.25)
    grid = make_time_grid(1.0, 32, 16)
    cfg = SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60)
    op = DeviceOperator.from_model(model, g["xi"])
    assert op.solver == "krylov"
    U = coarse_sweep_init_batched(op, grid).contiguous()
    op.krylov_its.zero_()
    t0 = time.time()
    res = pcgc_solve_device(op, U, grid, cfg)
    torch.cuda.synchronize()
    dt = time.time() - t0
    its = int(op.krylov_its.item())
    k = int(res.iters[0])
    print(f"\nc3 krylov: {k} outer iterations, {its} PCG+COCG iterations "
          f"({its / (k * (32 * 16 + 17)):.0f} per solve), {dt:.1f} s for one sample")
    np.testing.assert_array_equal(res.iters.cpu().numpy(), g["iters"])
    assert direct.rel(res.states.cpu().numpy(), g["final"]) <= direct.RTOL
