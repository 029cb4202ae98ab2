"""Nonlinear models on the device: the fused Newton sweeps of
pintuq/_kernels.pyx and classical parareal for Burgers1D / AllenCahn1D,
against the goldens of the unmodified reference (tests/golden/nl.npz, the
reference harness settings).

Tolerances: the Newton iterations stop on a 1e-12 residual, so the device and
the reference agree to the Newton tolerance, not to round-off: fields within
1e-9 relative, increments within 1e-10 absolute; parareal iteration counts
exact.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
RT = 1e-9

CASES = {"bu": dict(T=2.0, N=25, J=40, ns=3), "ac": dict(T=3.0, N=30, J=48, ns=2)}


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - b)) / np.max(np.abs(b)))


def _setup(tag):
    from paper_2510_26180_b200 import AllenCahn1D, Burgers1D, SolverConfig, make_time_grid

    c = CASES[tag]
    model = Burgers1D(dx=1 / 100) if tag == "bu" else AllenCahn1D(dx=1 / 128)
    grid = make_time_grid(c["T"], c["N"], c["J"])
    cfg = SolverConfig(alpha=0.1, tol=1e-8, max_outer_iters=60, seed=2718)
    return model, grid, cfg


@pytest.mark.parametrize("tag", ["bu", "ac"])
def test_newton_propagators_match_reference(cuda, golden, tag):
    from paper_2510_26180_b200 import ParameterSample
    from paper_2510_26180_b200.propagators import fine_reference, propagate_coarse, propagate_fine

    g = golden("nl")
    model, grid, cfg = _setup(tag)
    xi0 = ParameterSample(g[f"{tag}_xi"][0], id=0)
    u0 = model.initial_condition(xi0)
    u_keep = u0.copy()
    assert rel(propagate_fine(model, u0, 0.0, grid.deltaT, grid, xi0, cfg), g[f"{tag}_pf"]) <= RT
    assert rel(propagate_coarse(model, u0, 0.0, grid.deltaT, xi0, cfg), g[f"{tag}_pc"]) <= RT
    np.testing.assert_array_equal(u0, u_keep)  # the input is never mutated (_kernels.pyx:149)
    assert rel(fine_reference(model, xi0, grid, cfg).states, g[f"{tag}_ref"]) <= RT


@pytest.mark.parametrize("tag", ["bu", "ac"])
def test_newton_parareal_batched_matches_reference(cuda, golden, tag):
    import torch
    from paper_2510_26180_b200.nonlinear import NewtonOperator
    from paper_2510_26180_b200.parareal import parareal_solve_device
    from paper_2510_26180_b200.propagators import coarse_sweep_init
    from paper_2510_26180_b200 import ParameterSample

    g = golden("nl")
    model, grid, cfg = _setup(tag)
    xis = [ParameterSample(v, id=i) for i, v in enumerate(g[f"{tag}_xi"])]
    for i, xi in enumerate(xis):  # the device coarse sweep reproduces the reference's initial guesses
        assert rel(coarse_sweep_init(model, xi, grid, cfg).states, g[f"{tag}_init"][i]) <= RT
    op = NewtonOperator.from_model(model, xis, cfg)
    U = torch.as_tensor(g[f"{tag}_init"], device="cuda").clone()
    res = parareal_solve_device(op, U, grid, cfg)
    iters = res.iters.cpu().numpy()
    np.testing.assert_array_equal(iters, g[f"{tag}_iters"])
    assert np.all(res.status.cpu().numpy() == 1)
    assert rel(res.states.cpu().numpy(), g[f"{tag}_final"]) <= RT
    inc = res.increments.cpu().numpy()
    for i, k in enumerate(iters):
        np.testing.assert_allclose(inc[i, :k], g[f"{tag}_incs"][i, 1:k + 1], rtol=0, atol=1e-10)


def test_newton_parareal_dropin_and_failure_status(cuda, golden):
    from paper_2510_26180_b200 import CoarseTrajectory, NonConvergenceError, ParameterSample, SolverConfig
    from paper_2510_26180_b200.parareal import parareal_solve
    from paper_2510_26180_b200.propagators import propagate_coarse

    g = golden("nl")
    model, grid, cfg = _setup("bu")
    xi = ParameterSample(g["bu_xi"][1], id=1)
    tr = parareal_solve(model, xi, grid, cfg, CoarseTrajectory(model.initial_condition(xi), g["bu_init"][1]))
    assert tr.converged and tr.iterations == g["bu_iters"][1]
    assert rel(tr.trajectory.states, g["bu_final"][1]) <= RT
    # Allen-Cahn at the harness's coarse step dT = 1: Newton fails at step 1, as in the reference
    ac, _, _ = _setup("ac")
    xa = ParameterSample(g["ac_xi"][0], id=0)
    with pytest.raises(NonConvergenceError) as ei:
        propagate_coarse(ac, ac.initial_condition(xa), 0.0, 1.0, xa, SolverConfig(alpha=0.1, tol=1e-8))
    assert f"step {int(g['ac_fail_status'])}/1" in str(ei.value)
    assert ei.value.last_iterate.shape == (ac.nx,)


@pytest.mark.parametrize("tag", ["bu", "ac"])
def test_newton_pcgc_matches_reference(cuda, golden, tag):
    """pcgc_solve with the simplified-Newton averaged-Jacobian CGC
    (pintuq/pcgc.py:245-270) for the nonlinear models, batched."""
    import torch
    from paper_2510_26180_b200 import ParameterSample
    from paper_2510_26180_b200.nonlinear import NewtonOperator
    from paper_2510_26180_b200.pcgc import pcgc_solve_device

    g = golden("nl")
    model, grid, cfg = _setup(tag)
    xis = [ParameterSample(v, id=i) for i, v in enumerate(g[f"{tag}_xi"])]
    op = NewtonOperator.from_model(model, xis, cfg)
    U = torch.as_tensor(g[f"{tag}_init"], device="cuda").clone()
    res = pcgc_solve_device(op, U, grid, cfg)
    iters = res.iters.cpu().numpy()
    np.testing.assert_array_equal(iters, g[f"{tag}_pcgc_iters"])
    assert np.all(res.status.cpu().numpy() == 1)
    assert rel(res.states.cpu().numpy(), g[f"{tag}_pcgc_final"]) <= RT
    inc = res.increments.cpu().numpy()
    for i, k in enumerate(iters):
        np.testing.assert_allclose(inc[i, :k], g[f"{tag}_pcgc_incs"][i, 1:k + 1], rtol=0, atol=1e-10)


@pytest.mark.parametrize("tag", ["bu", "ac"])
def test_newton_cgc_single_correction(cuda, golden, tag):
    """One simplified-Newton correction (cgc_correct, pcgc.py:245-270) from
    the reference's fine ends: result and inner iteration count."""
    import torch
    from paper_2510_26180_b200 import ParameterSample, _lib
    from paper_2510_26180_b200.device import AlphaTables, empty, ptr, stream_ptr
    from paper_2510_26180_b200.nonlinear import NewtonOperator
    from paper_2510_26180_b200.pcgc import build_alpha_circulant

    g = golden("nl")
    model, grid, cfg = _setup(tag)
    N, nx = grid.n_coarse, model.nx
    xi0 = ParameterSample(g[f"{tag}_xi"][0], id=0)
    op = NewtonOperator.from_model(model, [xi0], cfg)
    U = torch.as_tensor(g[f"{tag}_init"][:1], device="cuda").contiguous()
    prev = np.vstack([cfg.alpha * g[f"{tag}_init"][0][-1:], g[f"{tag}_init"][0][:-1]])
    G, _ = op.sweep(torch.as_tensor(prev[None], device="cuda"), grid.deltaT, 1)
    b = torch.as_tensor(g[f"{tag}_cgc_F"][None], device="cuda") - G[:, :, 0]
    tables = AlphaTables(build_alpha_circulant(N, cfg.alpha))
    out = empty(1, N, nx)
    inner = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("kle_newton_cgc_f64", op.kind, ptr(U), ptr(b.contiguous()), ptr(out), ptr(op.p0), ptr(tables.lam),
              ptr(tables.scaling), ptr(tables.inv_scaling), 1, N, nx, grid.deltaT, op.dx, op.bc_lo, op.bc_hi,
              op.newton_tol, None, ptr(inner), stream_ptr())
    assert rel(out[0].cpu().numpy(), g[f"{tag}_cgc_out"]) <= RT
    assert abs(int(inner.item()) - int(g[f"{tag}_cgc_inner"])) <= 1  # the 1e-12 inner stop may flip by one step


def test_newton_status_words_and_maxiters(cuda, golden):
    """Per-system Newton status (first failing step, 0 = ok) in a mixed batch,
    MaxItersExceeded mapping of the batched loops, and the single-sample
    pcgc_solve drop-in for a nonlinear model."""
    import torch
    from paper_2510_26180_b200 import (CoarseTrajectory, MaxItersExceededError, ParameterSample, SolverConfig)
    from paper_2510_26180_b200.nonlinear import NewtonOperator
    from paper_2510_26180_b200.parareal import parareal_solve_device
    from paper_2510_26180_b200.pcgc import pcgc_solve, pcgc_solve_device

    g = golden("nl")
    ac, _, cfg_ac = _setup("ac")
    xs = [ParameterSample(v, id=i) for i, v in enumerate(g["ac_xi"])]
    op = NewtonOperator.from_model(ac, xs, cfg_ac)
    u0 = op.u0[None, None].expand(2, 1, ac.nx).contiguous()
    # dT = 1 fails at step 1 (the reference's status), dT = 0.1 succeeds, in the same launch
    out, st = op.sweep(torch.cat([u0, u0], dim=1).contiguous(), 1.0, 1, raise_on_fail=False)
    assert st.cpu().numpy()[:, 0].tolist() == [int(g["ac_fail_status"])] * 2
    out, st = op.sweep(u0, 0.1, 1, raise_on_fail=False)
    assert not st.cpu().numpy().any()

    model, grid, cfg = _setup("bu")
    xis = [ParameterSample(v, id=i) for i, v in enumerate(g["bu_xi"])]
    op = NewtonOperator.from_model(model, xis, cfg)
    short = SolverConfig(alpha=0.1, tol=1e-8, max_outer_iters=3)
    for solve in (pcgc_solve_device, parareal_solve_device):
        U = torch.as_tensor(g["bu_init"], device="cuda").clone()
        res = solve(op, U, grid, short)
        assert np.all(res.status.cpu().numpy() == 2) and np.all(res.iters.cpu().numpy() == 3)
        assert isinstance(res.failures()[0], MaxItersExceededError)
    tr = pcgc_solve(model, xis[2], grid, cfg, CoarseTrajectory(model.initial_condition(), g["bu_init"][2]))
    assert tr.converged and tr.iterations == g["bu_pcgc_iters"][2]
    assert rel(tr.trajectory.states, g["bu_pcgc_final"][2]) <= RT


def test_newton_pcgc_reference_stop(cuda, golden):
    """stop_on="reference" for a nonlinear model: the device loop stops at the
    first record within tol of the fine reference, and matches the oracle."""
    import torch
    from oracle import nonlinear_port as nlp
    from paper_2510_26180_b200 import ParameterSample
    from paper_2510_26180_b200.nonlinear import NewtonOperator
    from paper_2510_26180_b200.pcgc import pcgc_solve_device

    g = golden("nl")
    model, grid, cfg = _setup("bu")
    xis = [ParameterSample(v, id=i) for i, v in enumerate(g["bu_xi"][:2])]
    op = NewtonOperator.from_model(model, xis, cfg)
    ref, _ = op.sweep(op.u0[None, None].expand(2, 1, model.nx).contiguous(), grid.deltat,
                      grid.n_fine_per_coarse, nseg=grid.n_coarse)
    ref = ref[:, 0].contiguous()
    U = torch.as_tensor(g["bu_init"][:2], device="cuda").clone()
    res = pcgc_solve_device(op, U, grid, cfg, reference=ref, stop_on="reference")
    it = res.iters.cpu().numpy()
    assert np.all(res.status.cpu().numpy() == 1)
    np.testing.assert_array_equal(res.iters_to_tol(cfg.tol).cpu().numpy(), it)
    err = res.err_vs_ref.cpu().numpy()
    for i in range(2):
        assert np.max(err[i, it[i]]) <= cfg.tol < np.max(err[i, it[i] - 1])
