"""Device parity for the 2D (5-point) path, BASELINE config 3, against the
golden vectors of the unmodified reference (SuperLU paths) run on the
``LogNormalKL2D`` plugin (tests/golden/make_golden.py c3s, c3).

Tolerances as in test_gpu_parity: iteration counts exact, fields within 1e-10
relative (max-norm over the field's max)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RTOL = 1e-10


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def small():
    from paper_2510_26180_b200 import LogNormalKL2D, SolverConfig, make_time_grid

    return (LogNormalKL2D(n=15, d=10, sigma=0.5, ell=0.25), make_time_grid(1.0, 8, 4),
            SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60))


def test_stencil_on_device_matches_model(cuda, golden):
    from paper_2510_26180_b200.device import DeviceOperator

    model, _, _ = small()
    xi = golden("c3s")["xi"]
    op = DeviceOperator.from_model(model, xi)
    for s in range(len(xi)):
        dia, ex, ey = model.stencil(xi[s])
        assert rel(op.dia[s].cpu().numpy(), dia) <= 1e-14
        assert rel(op.ex[s].cpu().numpy(), ex) <= 1e-14
        assert rel(op.ey[s].cpu().numpy(), ey) <= 1e-14


def test_propagators_2d(cuda, golden):
    from paper_2510_26180_b200 import ParameterSample
    from paper_2510_26180_b200.propagators import coarse_sweep_init, propagate_coarse, propagate_fine

    model, grid, cfg = small()
    g = golden("c3s")
    xi0 = ParameterSample(g["xi"][0], id=0)
    assert rel(propagate_fine(model, g["u_rand"], 2 * grid.deltaT, 3 * grid.deltaT, grid, xi0, cfg),
               g["pf_rand"]) <= 1e-12
    assert rel(propagate_coarse(model, g["u_rand"], 0.0, grid.deltaT, xi0, cfg), g["pc_rand"]) <= 1e-12
    assert rel(coarse_sweep_init(model, xi0, grid, cfg).states, g["coarse_sweep"][0]) <= 1e-12


def test_three_step_and_cgc_correct_2d(cuda, golden):
    from paper_2510_26180_b200 import CoarseTrajectory, ParameterSample
    from paper_2510_26180_b200.pcgc import build_alpha_circulant, cgc_correct, three_step_solve

    model, grid, cfg = small()
    g = golden("c3s")
    xi0 = ParameterSample(g["xi"][0], id=0)
    A, _ = model.linear_system(xi0)
    u, imag = three_step_solve(build_alpha_circulant(8, 1e-3), -A, grid.deltaT, g["r_rand"])
    assert rel(u, g["ts_u"]) <= 1e-11 and imag <= 1e-12
    out, _ = cgc_correct(model, xi0, grid, cfg, CoarseTrajectory(model.initial_condition(), g["coarse_sweep"][0]),
                         g["F_ends"])
    assert rel(out.states, g["cgc_states"]) <= 1e-11


def test_pcgc_batched_2d_small(cuda, golden):
    from paper_2510_26180_b200.device import DeviceOperator
    from paper_2510_26180_b200.pcgc import pcgc_solve_device
    from paper_2510_26180_b200.propagators import coarse_sweep_init_batched

    model, grid, cfg = small()
    g = golden("c3s")
    op = DeviceOperator.from_model(model, g["xi"])
    U = coarse_sweep_init_batched(op, grid).contiguous()
    assert rel(U.cpu().numpy(), g["coarse_sweep"]) <= 1e-12
    res = pcgc_solve_device(op, U, grid, cfg)
    np.testing.assert_array_equal(res.iters.cpu().numpy(), g["iters"])
    assert rel(res.states.cpu().numpy(), g["final"]) <= RTOL
    hist = res.increments.cpu().numpy()
    for s in range(3):
        k = int(g["iters"][s])
        np.testing.assert_allclose(hist[s, :k], g["increments"][s, :k], rtol=1e-6, atol=1e-12)


def test_pcgc_single_sample_dropin_2d(cuda, golden):
    from paper_2510_26180_b200 import CoarseTrajectory, ParameterSample
    from paper_2510_26180_b200.pcgc import pcgc_solve

    model, grid, cfg = small()
    g = golden("c3s")
    xi = ParameterSample(g["xi"][1], id=1)
    tr = pcgc_solve(model, xi, grid, cfg, CoarseTrajectory(model.initial_condition(), g["coarse_sweep"][1]))
    assert tr.iterations == int(g["iters"][1])
    assert rel(tr.trajectory.states, g["final"][1]) <= RTOL


def test_c3_full_shape_one_sample(cuda, golden):
    """n = 127 (nx = 16,129), N = 32, J = 16, d = 10: the config-3 shape."""
    from paper_2510_26180_b200 import LogNormalKL2D, SolverConfig, make_time_grid
    from paper_2510_26180_b200.device import DeviceOperator
    from paper_2510_26180_b200.pcgc import pcgc_solve_device
    from paper_2510_26180_b200.propagators import coarse_sweep_init_batched

    g = golden("c3")
    model = LogNormalKL2D(n=127, d=10, sigma=0.5, ell=0.25)
    grid = make_time_grid(1.0, 32, 16)
    cfg = SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60)
    op = DeviceOperator.from_model(model, g["xi"])
    U = coarse_sweep_init_batched(op, grid).contiguous()
    res = pcgc_solve_device(op, U, grid, cfg)
    np.testing.assert_array_equal(res.iters.cpu().numpy(), g["iters"])
    assert rel(res.states.cpu().numpy(), g["final"]) <= RTOL


def _dense_ops(op):
    """Dense I-free operator A (M, nx, nx) of a DeviceOperator2D batch (fp64,
    for small n only)."""
    import torch

    n = op.n
    A = torch.diag_embed(op.dia)
    A = A + torch.diag_embed(op.ex[:, :-1], 1) + torch.diag_embed(op.ex[:, :-1], -1)
    A = A + torch.diag_embed(op.ey[:, :-n], n) + torch.diag_embed(op.ey[:, :-n], -n)
    return A


@pytest.mark.parametrize("M,N", [(20, 32), (150, 32), (300, 32), (300, 40), (7, 5)])
def test_tma_sweeps_match_dense_solves(cuda, M, N):
    """kle_2d_fgr_staged_f64 / kle_2d_sweep_staged_f64 (the TMA + DMMA sweeps,
    8, 16 and 32 right-hand sides per CTA as the batch size selects them, and
    ragged subinterval counts) against dense fp64 solves of the same BE steps
    and the same CGC right-hand side (pintuq/propagators.py:37-39,121-145,
    pcgc.py:175-197,233-237)."""
    import torch

    from paper_2510_26180_b200 import LogNormalKL2D, make_time_grid
    from paper_2510_26180_b200.device import AlphaTables, DeviceOperator, empty
    from paper_2510_26180_b200.pcgc import build_alpha_circulant

    n, J, alpha = 15, 3, 1e-3
    model = LogNormalKL2D(n=n, d=10, sigma=0.5, ell=0.25)
    grid = make_time_grid(1.0, N, J)
    xi = np.random.default_rng(M + N).normal(size=(M, 10))
    op = DeviceOperator.from_model(model, xi)
    nx = n * n
    U = torch.as_tensor(np.random.default_rng(1).uniform(0.0, 1.0, size=(M, N, nx)), device="cuda")
    tables = AlphaTables(build_alpha_circulant(N, alpha))
    R = empty(M, N, nx)
    op.fgr(U, tables, grid, alpha, R)
    A = _dense_ops(op)
    eye = torch.eye(nx, dtype=torch.float64, device="cuda")
    T = eye + grid.deltat * A
    starts = torch.cat([op.u0.view(1, 1, nx).expand(M, 1, nx), U[:, :-1]], dim=1)
    x = starts.transpose(1, 2)  # (M, nx, N)
    for _ in range(J):
        x = torch.linalg.solve(T, x + grid.deltat * op.g0)
    F = x.transpose(1, 2)
    prev = torch.cat([alpha * U[:, -1:], U[:, :-1]], dim=1)
    AF = torch.einsum("sij,snj->sni", A, F)
    ref = tables.scaling.view(1, N, 1) * (F + grid.deltaT * AF - prev)
    assert rel(R.cpu().numpy(), ref.cpu().numpy()) <= 1e-12
    # the sweep entry (propagate_fine / fine_reference): two segments of J steps
    out = op.sweep(U.contiguous(), grid.deltat, J, nseg=2)
    x = U.transpose(1, 2)
    for seg in range(2):
        for _ in range(J):
            x = torch.linalg.solve(T, x + grid.deltat * op.g0)
        assert rel(out[:, :, seg].cpu().numpy(), x.transpose(1, 2).cpu().numpy()) <= 1e-12


@pytest.mark.parametrize("n", [15, 40, 127])
def test_complex_band_factors_reconstruct(cuda, n):
    """kle_2d_factor_f64 with complex shifts (the panel L D L^T): L D L^T
    rebuilt densely equals lambda_f I + dT A for every frequency (complex
    symmetric, pintuq/pcgc.py:137-145 factors the same matrices with SuperLU)."""
    import torch

    from paper_2510_26180_b200 import LogNormalKL2D
    from paper_2510_26180_b200.device import AlphaTables, DeviceOperator
    from paper_2510_26180_b200.pcgc import build_alpha_circulant

    N, dT = 8, 1.0 / 8
    model = LogNormalKL2D(n=n, d=10, sigma=0.5, ell=0.25)
    xi = np.random.default_rng(n).normal(size=(2, 10))
    op = DeviceOperator.from_model(model, xi)
    tables = AlphaTables(build_alpha_circulant(N, 1e-3))
    Lt, Dinv = op.shifted_factors(tables, N, dT)
    nx, NF = n * n, N // 2 + 1
    Lc = torch.view_as_complex(Lt.reshape(2, NF, nx, n, 2))
    Dc = torch.view_as_complex(Dinv.reshape(2, NF, nx, 2))
    A = _dense_ops(op).to(torch.complex128)
    lam = torch.view_as_complex(tables.lam.reshape(N, 2))
    rows = torch.arange(nx, device="cuda")
    for s_ in range(2):
        for f in (0, 1, NF - 1):
            L = torch.eye(nx, dtype=torch.complex128, device="cuda")
            for t in range(n):
                r = rows[: nx - 1 - t]
                L[r + 1 + t, r] = Lc[s_, f, : nx - 1 - t, t]
            D = torch.diag(1.0 / Dc[s_, f])
            Bf = lam[f] * torch.eye(nx, dtype=torch.complex128, device="cuda") + dT * A[s_]
            err = (L @ D @ L.T - Bf).abs().max() / Bf.abs().max()
            assert float(err) <= 1e-13, (s_, f, float(err))
