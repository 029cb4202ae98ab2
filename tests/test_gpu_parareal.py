"""Classical parareal on the device (the paper's comparison
baseline, pintuq/parareal.py:100-191) against the goldens of the unmodified
reference (tests/golden/para.npz) and the pinned oracle.

Tolerances as everywhere: iteration counts exact, fields 1e-10 relative,
increments and error records (differences of O(1) fields) 1e-11 absolute.
"""
import numpy as np
import pytest

from oracle import ref_port
from tests.conftest import c1_config

pytestmark = pytest.mark.gpu
ATOL = 1e-11


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - b)) / np.max(np.abs(b)))


def test_parareal_batched_increment_stop(cuda, golden):
    from paper_2510_26180_b200.device import DeviceOperator
    from paper_2510_26180_b200.parareal import parareal_solve_device
    from paper_2510_26180_b200.propagators import coarse_sweep_init_batched

    model, grid, cfg = c1_config()
    g1, g = golden("c1"), golden("para")
    op = DeviceOperator.from_model(model, g1["xi_all"][:4])
    U = coarse_sweep_init_batched(op, grid).contiguous()
    assert rel(U.cpu().numpy(), g["cs_init"]) <= 1e-13
    res = parareal_solve_device(op, U, grid, cfg)
    iters = res.iters.cpu().numpy()
    np.testing.assert_array_equal(iters, g["cs_iters"])
    assert np.all(res.status.cpu().numpy() == 1)
    assert rel(res.states.cpu().numpy(), g["cs_final"]) <= 1e-10
    inc = res.increments.cpu().numpy()
    for i, k in enumerate(iters):
        np.testing.assert_allclose(inc[i, :k], g["cs_incs"][i, 1:k + 1], rtol=0, atol=ATOL)
        assert np.all(np.isnan(inc[i, k:]))


def test_parareal_batched_reference_stop(cuda, golden):
    """The harness's "parareal" solver: random_guess_init, stop_on="reference"."""
    import torch
    from paper_2510_26180_b200.device import DeviceOperator
    from paper_2510_26180_b200.parareal import parareal_solve_device
    from paper_2510_26180_b200.propagators import fine_reference_batched

    model, grid, cfg = c1_config()
    g1, gr, g = golden("c1"), golden("ref"), golden("para")
    op = DeviceOperator.from_model(model, g1["xi_all"][:4])
    ref = fine_reference_batched(op, grid)
    U = torch.as_tensor(gr["rnd_init"], device="cuda").clone()
    res = parareal_solve_device(op, U, grid, cfg, reference=ref, stop_on="reference")
    iters = res.iters.cpu().numpy()
    np.testing.assert_array_equal(iters, g["rnd_iters"])
    np.testing.assert_array_equal(res.iters_to_tol(cfg.tol).cpu().numpy(), g["rnd_to_tol"])
    assert rel(res.states.cpu().numpy(), g["rnd_final"]) <= 1e-10
    err = res.err_vs_ref.cpu().numpy()
    for i, K in enumerate(iters + 1):
        np.testing.assert_allclose(err[i, :K], g["rnd_err"][i, :K], rtol=0, atol=ATOL)


def test_parareal_solve_dropin_trace(cuda, golden):
    """Single-sample drop-in: the same IterationTrace as the reference."""
    from paper_2510_26180_b200 import CoarseTrajectory, MaxItersExceededError, ParameterSample, SolverConfig
    from paper_2510_26180_b200.parareal import parareal_solve

    model, grid, cfg = c1_config()
    g1, g = golden("c1"), golden("para")
    for i in range(2):
        xi = ParameterSample(g1["xi_all"][i], id=i)
        tr = parareal_solve(model, xi, grid, cfg, CoarseTrajectory(model.initial_condition(), g["cs_init"][i]),
                            store_states=True)
        assert tr.converged and tr.iterations == g["cs_iters"][i]
        assert len(tr.states_history) == tr.iterations + 1
        assert rel(tr.trajectory.states, g["cs_final"][i]) <= 1e-10
        incs = np.array([r.increment_inf for r in tr.records[1:]])
        np.testing.assert_allclose(incs, g["cs_incs"][i, 1:tr.iterations + 1], rtol=0, atol=ATOL)
    with pytest.raises(MaxItersExceededError) as ei:
        parareal_solve(model, xi, grid, SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=3),
                       CoarseTrajectory(model.initial_condition(), g["cs_init"][1]))
    assert ei.value.trace.iterations == 3
    with pytest.raises(ValueError):
        parareal_solve(model, xi, grid, cfg, CoarseTrajectory(model.initial_condition(), g["cs_init"][1]),
                       stop_on="reference")


def test_parareal_c2_shape_vs_oracle(cuda, golden):
    """Config-2 shapes (nx = 511, N = 64, J = 64), 2 samples against the
    per-sample oracle (reference arithmetic)."""
    from paper_2510_26180_b200 import LogNormalKL1D, SolverConfig, make_time_grid
    from paper_2510_26180_b200.device import DeviceOperator
    from paper_2510_26180_b200.parareal import parareal_solve_device
    from paper_2510_26180_b200.propagators import coarse_sweep_init_batched

    g = golden("c2")
    model = LogNormalKL1D(nx=511, d=8)
    grid = make_time_grid(1.0, 64, 64)
    cfg = SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60)
    xi = g["xi"][:2]
    op = DeviceOperator.from_model(model, xi)
    U = coarse_sweep_init_batched(op, grid).contiguous()
    U0 = U.cpu().numpy()
    res = parareal_solve_device(op, U, grid, cfg)
    for i in range(2):
        dia, off = model.tridiagonal(xi[i])
        out = ref_port.parareal(ref_port.SampleOperator(dia, off, np.ones(511)), model.initial_condition(), U0[i],
                                64, 64, 1.0, 1e-8, 60)
        assert int(res.iters[i]) == out["iters"]
        assert rel(res.states[i].cpu().numpy(), out["states"]) <= 1e-10
