"""Device parity: the CUDA path through the C ABI against the golden vectors
of the unmodified reference and the pinned CPU oracle.

Tolerances (BASELINE north star): parareal iteration counts exact; fields and
moments within 1e-10 relative (max-norm, relative to the field's max); for
alpha = 1e-4 at large N the reference's own round-off floor scales with
cond(V) = alpha^{-(N-1)/N}, so rtol = max(1e-10, 1e-12 cond(V)) there.
"""
import numpy as np
import pytest

from oracle import batched, ref_port
from tests.conftest import c1_config

pytestmark = pytest.mark.gpu

RTOL = 1e-10


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def test_library_exports_and_abi(cuda):
    from paper_2510_26180_b200 import _lib

    lib = _lib.load()
    assert lib.kle_abi_version() == 1
    for name in _lib.EXPORTED:
        assert hasattr(lib, name)


def test_coefficient_field_matches_model(cuda, golden):
    import torch
    from paper_2510_26180_b200.device import DeviceOperator

    model, _, _ = c1_config()
    xi = golden("c1")["xi_all"]
    op = DeviceOperator.from_model(model, xi)
    dia, off = batched.tridiag_from_xi(xi, model.kl_table, model.h)
    assert rel(op.dia.cpu().numpy(), dia) <= 1e-14
    assert rel(op.off.cpu().numpy()[:, :-1], off) <= 1e-14
    assert torch.all(op.off[:, -1] == 0)


def test_propagators_single_sample(cuda, golden):
    from paper_2510_26180_b200 import ParameterSample
    from paper_2510_26180_b200.propagators import (coarse_sweep_init, fine_reference, propagate_coarse,
                                                   propagate_fine)

    model, grid, cfg = c1_config()
    g = golden("c1")
    xi0 = ParameterSample(g["xi_all"][0], id=0)
    u0 = model.initial_condition()
    assert rel(propagate_fine(model, u0, 0.0, grid.deltaT, grid, xi0, cfg), g["pf_u0"]) <= 1e-13
    assert rel(propagate_fine(model, g["u_rand"], 3 * grid.deltaT, 4 * grid.deltaT, grid, xi0, cfg),
               g["pf_rand"]) <= 1e-13
    assert rel(propagate_coarse(model, g["u_rand"], 0.0, grid.deltaT, xi0, cfg), g["pc_rand"]) <= 1e-13
    assert rel(coarse_sweep_init(model, xi0, grid, cfg).states, g["coarse_sweep"]) <= 1e-13
    op = ref_port.SampleOperator(*model.tridiagonal(xi0), np.full(model.nx, 1.0))
    ref = ref_port.fine_reference(op, u0, 16, 32, grid.deltaT)
    assert rel(fine_reference(model, xi0, grid, cfg).states, ref) <= 1e-12
    with pytest.raises(ValueError):
        propagate_fine(model, u0, 0.0, 2 * grid.deltaT, grid, xi0, cfg)


def test_three_step_and_cgc_correct(cuda, golden):
    from paper_2510_26180_b200 import CoarseTrajectory, ParameterSample
    from paper_2510_26180_b200.pcgc import assemble_rhs_blocks, build_alpha_circulant, cgc_correct, three_step_solve

    model, grid, cfg = c1_config()
    g = golden("c1")
    xi0 = ParameterSample(g["xi_all"][0], id=0)
    A, _ = model.linear_system(xi0)
    u, imag = three_step_solve(build_alpha_circulant(16, 1e-3), -A, grid.deltaT, g["r_rand"])
    assert rel(u, g["ts_u"]) <= RTOL
    # max|Im u| is a real rounding-level diagnostic (not 0): same order as the reference's
    assert 0 < imag and abs(np.log10(imag / g["ts_imag"])) <= 2
    U_prev = CoarseTrajectory(model.initial_condition(), g["U0"][0])
    b = assemble_rhs_blocks(model, xi0, grid, cfg, g["U0"][0], g["F_ends"])
    assert rel(b, g["b_blocks"]) <= 1e-12
    out, diag = cgc_correct(model, xi0, grid, cfg, U_prev, g["F_ends"])
    assert rel(out.states, g["cgc_states"]) <= RTOL
    assert diag["inner_iters"] == 1
    assert 0 < diag["imag_residue"] and abs(np.log10(diag["imag_residue"] / g["cgc_imag"])) <= 2
    with pytest.raises(ValueError):
        three_step_solve(build_alpha_circulant(4, 0.1), np.zeros((1, 1)), 0.1, np.zeros((3, 1)))


def test_pcgc_solve_single_sample_matches_reference(cuda, golden):
    from paper_2510_26180_b200 import CoarseTrajectory, ParameterSample
    from paper_2510_26180_b200.pcgc import pcgc_solve

    model, grid, cfg = c1_config()
    g = golden("c1")
    for i in range(4):
        xi = ParameterSample(g["xi_all"][i], id=i)
        tr = pcgc_solve(model, xi, grid, cfg, CoarseTrajectory(model.initial_condition(), g["U0"][i]))
        assert tr.iterations == int(g["iters"][i])
        assert rel(tr.trajectory.states, g["final"][i]) <= RTOL
        incs = np.array([r.increment_inf for r in tr.records[1:]])
        # increments are differences of O(1) fields: compare at field round-off
        np.testing.assert_allclose(incs, g["increments"][i, : tr.iterations], rtol=0, atol=1e-12)


def test_kle_cgc_pipeline_c1_golden(cuda, golden):
    """xi -> coefficient field -> Hermite surrogate U0 -> batched PCGC ->
    moments, all on the device, against the reference's golden run."""
    from paper_2510_26180_b200.engine import KleCgcSolver
    from paper_2510_26180_b200.models import ParameterMap
    from paper_2510_26180_b200.surrogate import KLGpcSurrogate

    model, grid, cfg = c1_config()
    g = golden("c1")
    s = KLGpcSurrogate(g["mean_field"], g["eigenvalues"], g["modes"], g["coeffs"], int(g["degree"]),
                       [ParameterMap("identity", -np.inf, np.inf)] * 4, family="hermite")
    solver = KleCgcSolver(model, grid, cfg, s)
    M = len(g["iters"])
    res = solver.solve(g["xi_all"][:M], keep_initial=True)
    assert rel(res.U0.cpu().numpy(), g["U0"]) <= 1e-13
    np.testing.assert_array_equal(res.batch.iters.cpu().numpy(), g["iters"])
    assert np.all(res.batch.status.cpu().numpy() == 1)
    assert rel(res.batch.states.cpu().numpy(), g["final"]) <= RTOL
    mean, var = solver.moments(res)
    assert rel(mean.cpu().numpy(), g["mean"]) <= RTOL
    assert rel(var.cpu().numpy(), g["var"]) <= 1e-9
    inc = res.batch.increments.cpu().numpy()
    for i in range(M):
        k = int(g["iters"][i])
        np.testing.assert_allclose(inc[i, :k], g["increments"][i, :k], rtol=0, atol=1e-12)
        assert np.all(np.isnan(inc[i, k:]))


def test_kle_cgc_c1_full_batch_vs_oracle(cuda, golden):
    """All 256 config-1 samples against the batched oracle."""
    from paper_2510_26180_b200.engine import KleCgcSolver
    from paper_2510_26180_b200.models import ParameterMap
    from paper_2510_26180_b200.surrogate import KLGpcSurrogate

    model, grid, cfg = c1_config()
    g = golden("c1")
    s = KLGpcSurrogate(g["mean_field"], g["eigenvalues"], g["modes"], g["coeffs"], 2,
                       [ParameterMap("identity", -np.inf, np.inf)] * 4, family="hermite")
    xi = g["xi_all"]
    res = KleCgcSolver(model, grid, cfg, s).solve(xi)
    dia, off = batched.tridiag_from_xi(xi, model.kl_table, model.h)
    U0 = batched.hermite_predict(g["mean_field"], g["eigenvalues"], g["modes"], g["coeffs"], 2, xi)
    out = batched.pcgc(dia, off, model.initial_condition(), U0, 16, 32, 1.0, 1e-3, 1e-8, 60)
    np.testing.assert_array_equal(res.batch.iters.cpu().numpy(), out["iters"])
    assert rel(res.batch.states.cpu().numpy(), out["states"]) <= RTOL


def test_c2_shapes_match_reference(cuda, golden):
    from paper_2510_26180_b200 import LogNormalKL1D, SolverConfig, make_time_grid
    from paper_2510_26180_b200.device import DeviceOperator
    from paper_2510_26180_b200.pcgc import pcgc_solve_device
    from paper_2510_26180_b200.propagators import coarse_sweep_init_batched

    g = golden("c2")
    model = LogNormalKL1D(nx=511, d=8)
    grid = make_time_grid(1.0, 64, 64)
    cfg = SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60)
    op = DeviceOperator.from_model(model, g["xi"])
    U = coarse_sweep_init_batched(op, grid).contiguous()
    res = pcgc_solve_device(op, U, grid, cfg)
    np.testing.assert_array_equal(res.iters.cpu().numpy(), g["iters"])
    assert rel(res.states.cpu().numpy(), g["final"]) <= RTOL


@pytest.mark.parametrize("tag,alpha", [("a1", 1e-1), ("a2", 1e-2), ("a4", 1e-4)])
def test_c5_analogue_alpha_sweep(cuda, golden, tag, alpha):
    from paper_2510_26180_b200 import LogNormalKL1D, SolverConfig, make_time_grid
    from paper_2510_26180_b200.device import DeviceOperator
    from paper_2510_26180_b200.pcgc import pcgc_solve_device
    from paper_2510_26180_b200.propagators import coarse_sweep_init_batched

    g = golden("c5s")
    N = 128
    model = LogNormalKL1D(nx=255, d=4)
    grid = make_time_grid(1.0, N, 8)
    cfg = SolverConfig(alpha=alpha, tol=1e-8, max_outer_iters=60)
    op = DeviceOperator.from_model(model, g["xi"][None])
    U = coarse_sweep_init_batched(op, grid).contiguous()
    res = pcgc_solve_device(op, U, grid, cfg)
    assert int(res.iters[0]) == int(g[f"{tag}_iters"])
    rtol = max(RTOL, 1e-12 * alpha ** (-(N - 1) / N))
    assert rel(res.states[0].cpu().numpy(), g[f"{tag}_final"]) <= rtol


@pytest.mark.parametrize("trial", range(12))
def test_three_step_vs_dense_randomized(cuda, trial):
    """pintuq tests/test_pcgc.py:110-125 restated for the device operator
    class (symmetric tridiagonal), incl. N = 1..8 (non powers of two)."""
    from paper_2510_26180_b200.pcgc import build_alpha_circulant, three_step_solve

    rng = np.random.default_rng(100 + trial)
    n = int(rng.integers(1, 9))
    nx = int(rng.integers(1, 17))
    alpha = float(rng.uniform(0.02, 0.9))
    dT = float(rng.uniform(0.01, 1.0))
    spec = build_alpha_circulant(n, alpha)
    off = -rng.uniform(0.1, 1.0, nx - 1) if nx > 1 else np.zeros(0)
    dia = rng.uniform(0.5, 1.5, nx) + np.concatenate([[0.0], -off]) + np.concatenate([-off, [0.0]])
    A = np.diag(dia) + np.diag(off, 1) + np.diag(off, -1)
    r = rng.normal(size=(n, nx))
    Mx = np.kron(spec.dense_matrix(), np.eye(nx)) + dT * np.kron(np.eye(n), A)
    expected = np.linalg.solve(Mx, r.reshape(-1)).reshape(n, nx)
    u, imag = three_step_solve(spec, -A, dT, r)
    assert rel(u, expected) <= 1e-9
    assert imag <= 1e-10 * max(np.abs(u).max(), 1.0)
    if n == 1:  # one real eigenvalue, identity DFT: exactly real, as in the reference
        assert imag == 0.0


def test_three_step_hand_and_zero(cuda):
    from paper_2510_26180_b200.pcgc import build_alpha_circulant, three_step_solve

    u, imag = three_step_solve(build_alpha_circulant(2, 0.5), np.zeros((1, 1)), 0.3, np.array([[1.0], [0.0]]))
    np.testing.assert_allclose(u, [[2.0], [2.0]], atol=1e-12)
    u, _ = three_step_solve(build_alpha_circulant(5, 0.1), np.array([[-2.0]]), 0.1, np.zeros((5, 1)))
    np.testing.assert_array_equal(u, np.zeros((5, 1)))


def test_gpc_basis_bitwise_and_gemm(cuda, golden):
    import torch
    from paper_2510_26180_b200.models import ParameterMap
    from paper_2510_26180_b200.surrogate import DeviceSurrogate, KLGpcSurrogate

    g = golden("c1")
    s = KLGpcSurrogate(g["mean_field"], g["eigenvalues"], g["modes"], g["coeffs"], 2,
                       [ParameterMap("identity", -np.inf, np.inf)] * 4, family="hermite")
    ds = DeviceSurrogate(s)
    xi = g["xi_all"]
    Psi = ds.basis(torch.as_tensor(xi, device="cuda")).cpu().numpy()
    np.testing.assert_array_equal(Psi, ref_port.basis_matrix(xi, 2))
    # degree-3 8-dim basis (config-2 surrogate shape) also bitwise
    rng = np.random.default_rng(3)
    xi8 = rng.normal(size=(300, 8))
    s8 = KLGpcSurrogate(np.zeros((2, 3)), np.ones(1), np.ones((1, 2, 3)), np.ones((1, 165)), 3,
                        [ParameterMap("identity", -np.inf, np.inf)] * 8, family="hermite")
    Psi8 = DeviceSurrogate(s8).basis(torch.as_tensor(xi8, device="cuda")).cpu().numpy()
    np.testing.assert_array_equal(Psi8, ref_port.basis_matrix(xi8, 3))


def test_gpc_eval_factored_branch(cuda):
    """m_q < P (config-2 shape: 132 < 165) uses the two-GEMM branch."""
    import torch
    from paper_2510_26180_b200.models import ParameterMap
    from paper_2510_26180_b200.surrogate import DeviceSurrogate, KLGpcSurrogate

    rng = np.random.default_rng(5)
    m_q, P, N, nx = 20, 35, 4, 9  # d=4, p=3 -> P=35
    s = KLGpcSurrogate(rng.normal(size=(N, nx)), rng.uniform(0.1, 1, m_q), rng.normal(size=(m_q, N, nx)),
                       rng.normal(size=(m_q, P)), 3, [ParameterMap("identity", -np.inf, np.inf)] * 4, family="hermite")
    ds = DeviceSurrogate(s)
    assert ds.mode == "factored"
    xi = rng.normal(size=(77, 4))
    got = ds.predict(torch.as_tensor(xi, device="cuda")).cpu().numpy()
    want = batched.hermite_predict(s.mean_field, s.eigenvalues, s.modes, s.coeffs, 3, xi)
    assert rel(got, want) <= 1e-13


def test_moments_match_numpy(cuda):
    import torch
    from paper_2510_26180_b200.moments import two_pass_moments

    rng = np.random.default_rng(8)
    U = rng.normal(1.0, 0.2, size=(1000, 3, 7))
    mean, var = two_pass_moments(torch.as_tensor(U, device="cuda"), 1000)
    assert rel(mean.cpu().numpy(), U.mean(axis=0)) <= 1e-13
    assert rel(var.cpu().numpy(), U.var(axis=0)) <= 1e-12


def test_determinism_bitwise(cuda, golden):
    from paper_2510_26180_b200.engine import KleCgcSolver
    from paper_2510_26180_b200.models import ParameterMap
    from paper_2510_26180_b200.surrogate import KLGpcSurrogate

    model, grid, cfg = c1_config()
    g = golden("c1")
    s = KLGpcSurrogate(g["mean_field"], g["eigenvalues"], g["modes"], g["coeffs"], 2,
                       [ParameterMap("identity", -np.inf, np.inf)] * 4, family="hermite")
    solver = KleCgcSolver(model, grid, cfg, s)
    a = solver.solve(g["xi_all"][:64]).batch.states.cpu().numpy()
    b = solver.solve(g["xi_all"][:64]).batch.states.cpu().numpy()
    np.testing.assert_array_equal(a, b)


def test_empty_batch_is_noop(cuda):
    from paper_2510_26180_b200 import _lib

    assert _lib.call("kle_fgr_f64", *([None] * 10), 0, 16, 127, 32, 0.1, 0.1, 1.0, 0.1, None) == 0
    assert _lib.call("kle_sweep_f64", None, None, None, 0, 1, 127, 1, 1, 0.1, 1.0, None) == 0


@pytest.mark.parametrize("nx,N", [(127, 16), (511, 64), (255, 32), (1000, 8), (64, 2)])
def test_cluster_and_on_the_fly_cgc_agree(cuda, nx, N):
    """The cluster kernel (precomputed pivots, DSMEM stitching) and the
    on-the-fly per-frequency kernel solve the same three-step system."""
    from paper_2510_26180_b200 import LogNormalKL1D
    from paper_2510_26180_b200.device import AlphaTables, DeviceOperator, to_dev
    from paper_2510_26180_b200.pcgc import build_alpha_circulant, three_step_device

    rng = np.random.default_rng(nx + N)
    M = 3
    model = LogNormalKL1D(nx=nx, d=4)
    xi = rng.normal(size=(M, 4))
    op = DeviceOperator.from_model(model, xi)
    spec = build_alpha_circulant(N, 1e-2)
    tables = AlphaTables(spec)
    r = rng.normal(size=(M, N, nx))
    u1, im1 = three_step_device(op, tables, N, 1.0 / N, to_dev(r))
    u2, im2 = three_step_device(op, tables, N, 1.0 / N, to_dev(r), sfac=None)
    dia, off = batched.tridiag_from_xi(xi, model.kl_table, model.h)
    lam, sc = spec.eigenvalues, spec.scaling
    p = np.fft.fft(sc[None, :, None] * r, axis=1, norm="ortho")
    q = batched.thomas(lam[None, :, None] + dia[:, None, :] / N, (off / N)[:, None, :].astype(complex), p)
    want = ((1.0 / sc)[None, :, None] * np.fft.ifft(q, axis=1, norm="ortho")).real
    assert rel(u1.cpu().numpy(), want) <= 1e-10
    assert rel(u2.cpu().numpy(), want) <= 1e-10
    assert rel(u1.cpu().numpy(), u2.cpu().numpy()) <= 1e-11


def test_non_power_of_two_N_pcgc(cuda):
    """N = 12 (DFT fallback path) against the oracle."""
    from paper_2510_26180_b200 import LogNormalKL1D, SolverConfig, make_time_grid
    from paper_2510_26180_b200.device import DeviceOperator
    from paper_2510_26180_b200.pcgc import pcgc_solve_device
    from paper_2510_26180_b200.propagators import coarse_sweep_init_batched

    model = LogNormalKL1D(nx=63, d=4)
    grid = make_time_grid(1.0, 12, 10)
    cfg = SolverConfig(alpha=1e-2, tol=1e-9, max_outer_iters=60)
    xi = np.random.default_rng(4).normal(size=(5, 4))
    op = DeviceOperator.from_model(model, xi)
    U = coarse_sweep_init_batched(op, grid).contiguous()
    init = U.cpu().numpy()
    res = pcgc_solve_device(op, U, grid, cfg)
    dia, off = batched.tridiag_from_xi(xi, model.kl_table, model.h)
    out = batched.pcgc(dia, off, model.initial_condition(), init, 12, 10, 1.0, 1e-2, 1e-9, 60)
    np.testing.assert_array_equal(res.iters.cpu().numpy(), out["iters"])
    assert rel(res.states.cpu().numpy(), out["states"]) <= RTOL


@pytest.mark.parametrize("nx", [1500, 4095])
def test_multiwarp_fine_solver_matches_oracle(cuda, nx):
    """nx > 1024 uses the multi-warp layout (one CTA per system)."""
    import torch
    from paper_2510_26180_b200 import LogNormalKL1D
    from paper_2510_26180_b200.device import DeviceOperator, to_dev

    rng = np.random.default_rng(nx)
    model = LogNormalKL1D(nx=nx, d=4)
    xi = rng.normal(size=(2, 4))
    op = DeviceOperator.from_model(model, xi)
    assert op.layout[1] > 32  # multi-warp
    starts = rng.normal(size=(2, 3, nx))
    h, J = 1.0 / 1024 / 8, 8
    got = op.sweep(to_dev(starts), h, J)[:, :, 0].cpu().numpy()
    dia, off = batched.tridiag_from_xi(xi, model.kl_table, model.h)
    want = batched.be_steps(dia, off, starts, h, 1.0, J)
    assert rel(got, want) <= 1e-12


def test_c5_full_shape_alpha_1e4(cuda):
    """Config 5 shape (nx = 4095, N = 1024, J = 8, alpha = 1e-4), one sample,
    coarse-sweep initial guess: iteration count and fields vs the oracle."""
    from paper_2510_26180_b200 import LogNormalKL1D, SolverConfig, make_time_grid
    from paper_2510_26180_b200.device import DeviceOperator
    from paper_2510_26180_b200.pcgc import pcgc_solve_device
    from paper_2510_26180_b200.propagators import coarse_sweep_init_batched

    N, nx, alpha = 1024, 4095, 1e-4
    model = LogNormalKL1D(nx=nx, d=4)
    grid = make_time_grid(1.0, N, 8)
    cfg = SolverConfig(alpha=alpha, tol=1e-8, max_outer_iters=60)
    xi = np.random.default_rng(5).normal(size=(1, 4))
    op = DeviceOperator.from_model(model, xi)
    U = coarse_sweep_init_batched(op, grid).contiguous()
    init = U.cpu().numpy()
    res = pcgc_solve_device(op, U, grid, cfg)
    dia, off = batched.tridiag_from_xi(xi, model.kl_table, model.h)
    out = batched.pcgc(dia, off, model.initial_condition(), init, N, 8, 1.0, alpha, 1e-8, 60)
    np.testing.assert_array_equal(res.iters.cpu().numpy(), out["iters"])
    rtol = max(RTOL, 1e-12 * alpha ** (-(N - 1) / N))
    assert rel(res.states.cpu().numpy(), out["states"]) <= rtol


def test_device_surrogate_build_matches_reference(cuda, golden):
    """build_surrogate with device snapshots (3^4 Gauss-Hermite grid, the
    config-1 recipe) against the surrogate the reference built."""
    from paper_2510_26180_b200 import ParameterSample
    from paper_2510_26180_b200.surrogate import build_surrogate, collect_snapshots

    model, grid, cfg = c1_config()
    g = golden("c1")
    training = [ParameterSample(p, id=i) for i, p in enumerate(g["train_points"])]
    snap = collect_snapshots(model, grid, cfg, training)
    assert rel(snap.fields, g["snapshots"]) <= 1e-9  # PCGC to tol 1e-8 from the same init: O(1e-12)
    s = build_surrogate(model, grid, cfg, training, eps_kl=1e-10, degree=2, snapshots=snap)
    assert s.m_q == g["modes"].shape[0]
    np.testing.assert_allclose(s.eigenvalues, g["eigenvalues"], rtol=1e-6, atol=1e-9 * g["eigenvalues"][0])
    assert rel(s.mean_field, g["mean_field"]) <= 1e-10
    # leading modes/coefficients (well separated eigenvalues) agree up to sign
    for i in range(5):
        sgn = np.sign(np.sum(s.modes[i] * g["modes"][i]))
        assert rel(sgn * s.modes[i], g["modes"][i]) <= 1e-6


def test_batched_status_words_and_exceptions(cuda, golden):
    """max_outer_iters too small -> MAXITERS status / MaxItersExceededError;
    a non-finite initial guess -> NONFINITE status / ValueError; the other
    samples are unaffected (per-sample failure isolation, experiments.py:236-257)."""
    import torch
    from paper_2510_26180_b200 import MaxItersExceededError, SolverConfig
    from paper_2510_26180_b200.device import DeviceOperator, to_dev
    from paper_2510_26180_b200.pcgc import SAMPLE_CONVERGED, SAMPLE_MAXITERS, SAMPLE_NONFINITE, pcgc_solve_device

    model, grid, cfg = c1_config()
    g = golden("c1")
    op = DeviceOperator.from_model(model, g["xi_all"][:4])
    U = to_dev(g["U0"][:4]).clone()
    res = pcgc_solve_device(op, U, grid, SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=5))
    assert np.all(res.status.cpu().numpy() == SAMPLE_MAXITERS)
    assert np.all(res.iters.cpu().numpy() == 5)
    with pytest.raises(MaxItersExceededError):
        res.raise_for_status()
    U = to_dev(g["U0"][:4]).clone()
    U[2, 3, 7] = float("nan")
    res = pcgc_solve_device(op, U, grid, cfg)
    st = res.status.cpu().numpy()
    assert st[2] == SAMPLE_NONFINITE and np.all(st[[0, 1, 3]] == SAMPLE_CONVERGED)
    np.testing.assert_array_equal(res.iters.cpu().numpy()[[0, 1, 3]], g["iters"][[0, 1, 3]])
    assert isinstance(res.failures()[2], ValueError)


def test_pcgc_stop_on_reference_and_history(cuda, golden):
    """stop_on='reference' with store_states (pintuq/pcgc.py:291-348)."""
    from paper_2510_26180_b200 import CoarseTrajectory, ParameterSample
    from paper_2510_26180_b200.pcgc import pcgc_solve
    from paper_2510_26180_b200.propagators import fine_reference

    model, grid, cfg = c1_config()
    g = golden("c1")
    xi = ParameterSample(g["xi_all"][0], id=0)
    ref = fine_reference(model, xi, grid, cfg)
    tr = pcgc_solve(model, xi, grid, cfg, CoarseTrajectory(model.initial_condition(), g["U0"][0]),
                    reference=ref, stop_on="reference", store_states=True)
    assert tr.converged and tr.records[-1].max_err_vs_ref <= cfg.tol
    assert len(tr.states_history) == tr.iterations + 1
    errs = tr.max_errors()
    assert errs[0] > errs[-1]
    with pytest.raises(ValueError):
        pcgc_solve(model, xi, grid, cfg, CoarseTrajectory(model.initial_condition(), g["U0"][0]), stop_on="reference")


@pytest.mark.parametrize("nx,N,J", [(1, 4, 3), (2, 2, 2), (15, 1, 5), (33, 3, 2)])
def test_degenerate_shapes(cuda, nx, N, J):
    """Tiny / degenerate shapes (nx = 1, N = 1, odd N) against the oracle."""
    from paper_2510_26180_b200 import LogNormalKL1D, SolverConfig, make_time_grid
    from paper_2510_26180_b200.device import DeviceOperator
    from paper_2510_26180_b200.pcgc import pcgc_solve_device
    from paper_2510_26180_b200.propagators import coarse_sweep_init_batched

    model = LogNormalKL1D(nx=nx, d=2)
    grid = make_time_grid(1.0, N, J)
    cfg = SolverConfig(alpha=0.1, tol=1e-10, max_outer_iters=40)
    xi = np.random.default_rng(nx * 10 + N).normal(size=(3, 2))
    op = DeviceOperator.from_model(model, xi)
    U = coarse_sweep_init_batched(op, grid).contiguous()
    init = U.cpu().numpy()
    res = pcgc_solve_device(op, U, grid, cfg)
    dia, off = batched.tridiag_from_xi(xi, model.kl_table, model.h)
    out = batched.pcgc(dia, off, model.initial_condition(), init, N, J, 1.0, 0.1, 1e-10, 40)
    np.testing.assert_array_equal(res.iters.cpu().numpy(), out["iters"])
    assert rel(res.states.cpu().numpy(), out["states"]) <= RTOL


@pytest.mark.parametrize("variant", [4, 6, 13, 16, 18, 25, 27])
def test_fine_variants_match_oracle(cuda, golden, monkeypatch, variant):
    """Every tuning layout of the fine solver (register / pipelined / shared-memory
    factors, KLE_FINE_VARIANT) gives the same sweep and the same PCGC iterates."""
    from paper_2510_26180_b200 import LogNormalKL1D, SolverConfig, make_time_grid
    from paper_2510_26180_b200.device import DeviceOperator, to_dev
    from paper_2510_26180_b200.pcgc import pcgc_solve_device
    from paper_2510_26180_b200.propagators import coarse_sweep_init_batched

    monkeypatch.setenv("KLE_FINE_VARIANT", str(variant))
    rng = np.random.default_rng(variant)
    model = LogNormalKL1D(nx=511, d=8)
    xi = rng.normal(size=(3, 8))
    op = DeviceOperator.from_model(model, xi)
    starts = rng.normal(size=(3, 5, 511))
    h, J = 1.0 / 64 / 64, 64
    got = op.sweep(to_dev(starts), h, J)[:, :, 0].cpu().numpy()
    dia, off = batched.tridiag_from_xi(xi, model.kl_table, model.h)
    assert rel(got, batched.be_steps(dia, off, starts, h, 1.0, J)) <= 1e-12
    g = golden("c2")
    grid = make_time_grid(1.0, 64, 64)
    op = DeviceOperator.from_model(model, g["xi"])
    res = pcgc_solve_device(op, coarse_sweep_init_batched(op, grid).contiguous(), grid,
                            SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60))
    np.testing.assert_array_equal(res.iters.cpu().numpy(), g["iters"])
    assert rel(res.states.cpu().numpy(), g["final"]) <= RTOL


def test_device_kl_build_matches_host(cuda, golden):
    """kl_build on the device (Gram / mode / projection GEMMs, host eigh)
    against the host kl_build + kl_coefficients on the same snapshots (the
    reference's snapshot library of config 1): eigenvalues, m_q, and the
    surrogate predictions they define."""
    import torch
    from paper_2510_26180_b200 import ParameterSample
    from paper_2510_26180_b200.surrogate import (gpc_fit, kl_build, kl_build_device, kl_coefficients,
                                                 make_snapshot_set, surrogate_predict, KLGpcSurrogate)
    from paper_2510_26180_b200.models import ParameterMap

    model, grid, cfg = c1_config()
    g = golden("c1")
    training = [ParameterSample(p, id=i) for i, p in enumerate(g["train_points"])]
    snap = make_snapshot_set(training, g["snapshots"], model.cell_volume * grid.deltaT)
    snap.device_fields = torch.as_tensor(g["snapshots"], device="cuda")
    hb = kl_build(snap, 1e-10)
    hz = kl_coefficients(snap, hb)
    db, dz = kl_build_device(snap, 1e-10)
    assert db.m_q == hb.m_q == g["modes"].shape[0]
    np.testing.assert_allclose(db.eigenvalues, hb.eigenvalues, rtol=0, atol=1e-12 * hb.eigenvalues[0])
    # eigenvalues are accurate to eps * lambda_0 in absolute terms (the trailing ones are ~1e-12 lambda_0)
    np.testing.assert_allclose(db.retained, g["eigenvalues"], rtol=0, atol=1e-13 * g["eigenvalues"][0])
    maps = [ParameterMap("identity", -np.inf, np.inf)] * 4
    pts = g["train_points"]
    ch, _, _ = gpc_fit(pts, hz, 2, "hermite")
    cd, _, _ = gpc_fit(pts, dz, 2, "hermite")
    sh = KLGpcSurrogate(snap.mean_field, hb.retained, hb.modes, ch, 2, maps, family="hermite")
    sd = KLGpcSurrogate(snap.mean_field, db.retained, db.modes, cd, 2, maps, family="hermite")
    for i in range(4):
        xi = ParameterSample(g["xi_all"][i], id=i)
        a = surrogate_predict(sh, xi, model.initial_condition()).states
        b = surrogate_predict(sd, xi, model.initial_condition()).states
        # the trailing KL modes (eigenvalues ~1e-12 lambda_0) carry O(eps / lambda) direction error into
        # the least-squares fit; measured 2.2e-11 — an initial-guess difference the PCGC contracts away
        assert rel(b, a) <= 1e-10
        assert rel(b, g["U0"][i]) <= 1e-10


@pytest.mark.parametrize("N", [24, 100, 1000, 1500])
def test_non_power_of_two_time_fft(cuda, N):
    """Block DFTs for any N (pintuq/pcgc.py:79-87 uses np.fft for every N): the
    on-the-fly CGC kernel runs Bluestein's chirp-z transform through radix-2
    FFTs of length 2^ceil(log2(2N-1)) (N <= 1024) or, beyond its table budget,
    the direct DFT (N = 1500). three_step_solve against the oracle's np.fft +
    banded solves, and one PCGC solve with exact iteration counts (N = 24, 100)."""
    from paper_2510_26180_b200 import LogNormalKL1D, SolverConfig, make_time_grid
    from paper_2510_26180_b200.pcgc import build_alpha_circulant, pcgc_solve_batched, three_step_solve

    rng = np.random.default_rng(N)
    nx, alpha = 31, 1e-2
    dT = 1.0 / N
    off = -rng.uniform(0.5, 1.5, nx - 1) * 4.0
    dia = 2.0 * 4.0 + rng.uniform(0.0, 1.0, nx)
    A = np.diag(dia) + np.diag(off, 1) + np.diag(off, -1)
    spec = build_alpha_circulant(N, alpha)
    r = rng.normal(size=(N, nx))
    u, _ = three_step_solve(spec, -A, dT, r)
    op = ref_port.SampleOperator(dia, off, np.zeros(nx))
    want, _ = ref_port.three_step(spec.eigenvalues, spec.scaling, ref_port.shifted_solvers(op, spec.eigenvalues, dT),
                                  r)
    cond = alpha ** (-(N - 1) / N)
    assert rel(u, want) <= max(1e-10, 1e-13 * cond * np.log2(N)), rel(u, want)
    if N <= 100:
        model = LogNormalKL1D(nx=63, d=4)
        grid = make_time_grid(1.0, N, 4)
        cfg = SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60)
        xi = rng.normal(size=(4, 4))
        dia2, off2 = batched.tridiag_from_xi(xi, model.kl_table, model.h)
        U0 = batched.coarse_sweep(dia2, off2, model.initial_condition(), N, grid.deltaT)
        res = pcgc_solve_batched(model, xi, grid, cfg, U0)
        out = batched.pcgc(dia2, off2, model.initial_condition(), U0, N, 4, 1.0, 1e-3, 1e-8, 60)
        np.testing.assert_array_equal(res.iters.cpu().numpy(), out["iters"])
        assert rel(res.states.cpu().numpy(), out["states"]) <= RTOL


@pytest.mark.parametrize("N,nx", [(2, 1), (2, 5), (4, 33), (8, 100), (16, 64), (16, 127), (16, 128)])
def test_row_fft_cgc_matches_cluster_kernel_and_dense(cuda, N, nx, monkeypatch):
    """The small-block CGC kernel (kle_cgc_row.cu: thread-per-row real FFTs in
    registers, one CTA per sample; default for power-of-two N <= 16, nx <= 128)
    against the cluster kernel (KLE_CGC_ROW=0) on random symmetric tridiagonal
    operators and right-hand sides, ragged nx included, and against the dense
    solve of (C_alpha (x) I + dT I (x) A) u = r (pintuq/pcgc.py:148-172)."""
    import torch

    from paper_2510_26180_b200.device import AlphaTables, DeviceOperator, to_dev
    from paper_2510_26180_b200.pcgc import build_alpha_circulant, three_step_device

    rng = np.random.default_rng(1000 * N + nx)
    M, alpha, dT = 5, 1e-3, 1.0 / N
    off = rng.uniform(0.1, 1.0, (M, nx)) * 50.0  # A = tridiag(-off, dia, -off), SPD, stiff like the FD operator
    off[:, -1] = 0.0
    dia = rng.uniform(0.5, 1.5, (M, nx)) + off + np.concatenate([np.zeros((M, 1)), off[:, :-1]], axis=1)
    op = DeviceOperator(to_dev(dia), to_dev(-off), 0.0, to_dev(np.zeros(nx)))
    spec = build_alpha_circulant(N, alpha)
    tables = AlphaTables(spec)
    r = to_dev(rng.normal(size=(M, N, nx)))
    u_row, _ = three_step_device(op, tables, N, dT, r, diagnostics=False)
    monkeypatch.setenv("KLE_CGC_ROW", "0")
    u_cl, _ = three_step_device(op, tables, N, dT, r, diagnostics=False)
    monkeypatch.delenv("KLE_CGC_ROW")
    scale = float(u_cl.abs().max())
    assert float((u_row - u_cl).abs().max()) <= 1e-12 * scale
    if N * nx <= 1024:
        for s in range(M):
            A = np.diag(dia[s]) - np.diag(off[s, :-1], 1) - np.diag(off[s, :-1], -1)
            Mx = np.kron(spec.dense_matrix(), np.eye(nx)) + dT * np.kron(np.eye(N), A)
            expected = np.linalg.solve(Mx, r[s].cpu().numpy().reshape(-1)).reshape(N, nx)
            assert rel(u_row[s].cpu().numpy(), expected) <= 1e-9


@pytest.mark.parametrize("N,nx,J", [(16, 127, 32), (16, 128, 5), (3, 65, 2), (8, 100, 7), (20, 96, 4), (33, 127, 2)])
def test_twisted_fine_sweep_matches_partitioned_and_dense(cuda, N, nx, J, monkeypatch):
    """The two-lane twisted-factorisation sweep (kle_fine_tw.cu; default for
    64 < nx <= 128) against the partitioned register kernel (KLE_FGR_TW=0) and a
    dense evaluation of scaling_n ((I + dT A) F_n - prev_n), F_n = J backward-Euler
    steps with a constant source (pintuq/propagators.py:121-145, pcgc.py:175-197),
    over ragged nx, N not a multiple of 16 and samples masked by the status word."""
    import torch

    from paper_2510_26180_b200 import make_time_grid
    from paper_2510_26180_b200.device import AlphaTables, DeviceOperator, empty, to_dev
    from paper_2510_26180_b200.pcgc import _fgr, build_alpha_circulant

    rng = np.random.default_rng(7000 * N + nx)
    M, alpha, g0 = 6, 1e-3, 0.7
    grid = make_time_grid(1.0, N, J)
    off = rng.uniform(0.1, 1.0, (M, nx)) * 400.0
    off[:, -1] = 0.0
    dia = rng.uniform(0.5, 1.5, (M, nx)) + off + np.concatenate([np.zeros((M, 1)), off[:, :-1]], axis=1)
    u0 = rng.normal(size=nx)
    op = DeviceOperator(to_dev(dia), to_dev(-off), g0, to_dev(u0))
    tables = AlphaTables(build_alpha_circulant(N, alpha))
    U = to_dev(rng.normal(size=(M, N, nx)))
    status = torch.zeros(M, dtype=torch.int32, device="cuda")
    status[4] = 1  # a converged sample: its rhs rows must stay untouched
    R_tw = torch.full((M, N, nx), 123.0, dtype=torch.float64, device="cuda")
    R_pt = R_tw.clone()
    _fgr(op, tables, U, R_tw, J, grid, alpha, status=status)
    monkeypatch.setenv("KLE_FGR_TW", "0")
    _fgr(op, tables, U, R_pt, J, grid, alpha, status=status)
    monkeypatch.delenv("KLE_FGR_TW")
    assert float((R_tw[4] - 123.0).abs().max()) == 0.0
    scale = float(R_pt.abs().max())
    assert float((R_tw - R_pt).abs().max()) <= 1e-12 * scale
    sc = tables.scaling.cpu().numpy()
    Uh = U.cpu().numpy()
    for s in (0, 5):
        A = np.diag(dia[s]) - np.diag(off[s, :-1], 1) - np.diag(off[s, :-1], -1)
        T = np.eye(nx) + grid.deltat * A
        for n in range(N):
            x = u0 if n == 0 else Uh[s, n - 1]
            for _ in range(J):
                x = np.linalg.solve(T, x + grid.deltat * g0)
            prev = alpha * Uh[s, N - 1] if n == 0 else Uh[s, n - 1]
            want = sc[n] * (x + grid.deltaT * (A @ x) - prev)
            assert rel(R_tw[s, n].cpu().numpy(), want) <= 1e-10


def test_twisted_fine_sweep_fallback_for_unscalable_samples(cuda, monkeypatch):
    """Samples without a scaled twisted form — a vanishing coupling (the row scaling t
    would be 0), an operator without positive pivots (no steady state A x* = g0) — are
    flagged by the table kernel and taken by the partitioned kernel, inside one batch
    with regular samples: the flagged samples equal the KLE_FGR_TW=0 run bitwise (same
    kernel), the others within rounding; also through the batched PCGC loop, which
    counts the flags once per solve (kle_capi.cu)."""
    import torch

    from paper_2510_26180_b200 import SolverConfig, make_time_grid
    from paper_2510_26180_b200.device import AlphaTables, DeviceOperator, to_dev
    from paper_2510_26180_b200.pcgc import _fgr, build_alpha_circulant, pcgc_solve_device

    rng = np.random.default_rng(99)
    M, N, nx, J, alpha, g0 = 7, 16, 127, 8, 1e-3, 1.0
    grid = make_time_grid(1.0, N, J)
    off = rng.uniform(0.1, 1.0, (M, nx)) * 400.0
    off[:, -1] = 0.0
    dia = rng.uniform(0.5, 1.5, (M, nx)) + off + np.concatenate([np.zeros((M, 1)), off[:, :-1]], axis=1)
    off[2, 40] = 0.0         # decoupled blocks: t = 0 beyond row 40
    off[5, 90] = 1e-200      # t underflows
    dia[3, :] -= 2.0 * dia[3, :].max()  # A negative definite: no positive pivots for the steady state
    dia[3, :] *= 1e-3                  # (I + hA stays positive definite at this step size)
    off[3, :] *= 1e-3
    u0 = rng.normal(size=nx)
    op = DeviceOperator(to_dev(dia), to_dev(-off), g0, to_dev(u0))
    tables = AlphaTables(build_alpha_circulant(N, alpha))
    U = to_dev(rng.normal(size=(M, N, nx)))
    R_tw = torch.zeros((M, N, nx), dtype=torch.float64, device="cuda")
    R_pt = torch.zeros_like(R_tw)
    _fgr(op, tables, U, R_tw, J, grid, alpha)
    monkeypatch.setenv("KLE_FGR_TW", "0")
    _fgr(op, tables, U, R_pt, J, grid, alpha)
    monkeypatch.delenv("KLE_FGR_TW")
    assert torch.isfinite(R_tw).all()
    for s in (2, 3, 5):
        assert torch.equal(R_tw[s], R_pt[s]), s
    for s in (0, 1, 4, 6):
        assert float((R_tw[s] - R_pt[s]).abs().max()) <= 1e-12 * float(R_pt[s].abs().max())
        assert not torch.equal(R_tw[s], R_pt[s])  # (the twisted kernel did run)
    # the batched loop with flagged samples in the batch
    cfg = SolverConfig(alpha=alpha, tol=1e-9, max_outer_iters=40)
    keep = [0, 1, 2, 4, 5, 6]  # (sample 3's A is not a diffusion operator: PCGC need not converge for it)
    op2 = DeviceOperator(to_dev(dia[keep]), to_dev(-off[keep]), g0, to_dev(u0))
    U0 = to_dev(rng.normal(size=(len(keep), N, nx)))
    res_tw = pcgc_solve_device(op2, U0.clone(), grid, cfg, tables)
    monkeypatch.setenv("KLE_FGR_TW", "0")
    res_pt = pcgc_solve_device(op2, U0.clone(), grid, cfg, tables)
    monkeypatch.delenv("KLE_FGR_TW")
    assert torch.equal(res_tw.iters, res_pt.iters)
    assert int(res_tw.status.ne(1).sum()) == 0
    scale = float(res_pt.states.abs().max())
    assert float((res_tw.states - res_pt.states).abs().max()) <= 1e-10 * scale
    for s in (2, 4):  # keep[2] = 2 and keep[4] = 5: the flagged samples, same kernels in both runs
        assert torch.equal(res_tw.states[s], res_pt.states[s])


def test_twisted_fine_sweep_without_source(cuda, monkeypatch):
    """g0 = 0: no steady state (x* = 0); the twisted sweep against the partitioned one."""
    import torch

    from paper_2510_26180_b200 import make_time_grid
    from paper_2510_26180_b200.device import AlphaTables, DeviceOperator, to_dev
    from paper_2510_26180_b200.pcgc import _fgr, build_alpha_circulant

    rng = np.random.default_rng(5)
    M, N, nx, J, alpha = 3, 16, 101, 6, 1e-2
    grid = make_time_grid(0.5, N, J)
    off = rng.uniform(0.1, 1.0, (M, nx)) * 100.0
    off[:, -1] = 0.0
    dia = off + np.concatenate([np.zeros((M, 1)), off[:, :-1]], axis=1)  # singular A (Neumann-like): fine when g0 = 0
    op = DeviceOperator(to_dev(dia), to_dev(-off), 0.0, to_dev(rng.normal(size=nx)))
    tables = AlphaTables(build_alpha_circulant(N, alpha))
    U = to_dev(rng.normal(size=(M, N, nx)))
    R_tw = torch.zeros((M, N, nx), dtype=torch.float64, device="cuda")
    R_pt = torch.zeros_like(R_tw)
    _fgr(op, tables, U, R_tw, J, grid, alpha)
    monkeypatch.setenv("KLE_FGR_TW", "0")
    _fgr(op, tables, U, R_pt, J, grid, alpha)
    monkeypatch.delenv("KLE_FGR_TW")
    for s in range(M):  # (the twisted kernel took every sample)
        assert not torch.equal(R_tw[s], R_pt[s])
    assert float((R_tw - R_pt).abs().max()) <= 1e-12 * float(R_pt.abs().max())


@pytest.mark.parametrize("N,nx,J", [(64, 511, 4), (5, 300, 3), (13, 129, 2), (8, 512, 2)])
def test_scaled_partitioned_sweep_matches_unscaled_and_dense(cuda, N, nx, J, monkeypatch):
    """The scaled partitioned step (be_steps_sc, KLE_FGR_SC=1; the (16, 32) layout,
    128 < nx <= 512: steady-state shift, chunk-local row scaling, DADD forward
    chains) against the default unscaled step and a dense evaluation of
    scaling_n ((I + dT A) F_n - prev_n); one sample without a scaled form (a
    vanishing coupling) must come out of the unscaled kernel bitwise."""
    import torch

    from paper_2510_26180_b200 import make_time_grid
    from paper_2510_26180_b200.device import AlphaTables, DeviceOperator, to_dev
    from paper_2510_26180_b200.pcgc import _fgr, build_alpha_circulant

    rng = np.random.default_rng(9000 * N + nx)
    M, alpha, g0 = 5, 1e-3, 0.7
    grid = make_time_grid(1.0, N, J)
    off = rng.uniform(0.1, 1.0, (M, nx)) * 4000.0
    off[:, -1] = 0.0
    off[3, nx // 3] = 0.0  # decoupled blocks: no scaling
    dia = rng.uniform(0.5, 1.5, (M, nx)) + off + np.concatenate([np.zeros((M, 1)), off[:, :-1]], axis=1)
    u0 = rng.normal(size=nx)
    op = DeviceOperator(to_dev(dia), to_dev(-off), g0, to_dev(u0))
    tables = AlphaTables(build_alpha_circulant(N, alpha))
    U = to_dev(rng.normal(size=(M, N, nx)))
    status = torch.zeros(M, dtype=torch.int32, device="cuda")
    status[1] = 1
    R_sc = torch.full((M, N, nx), 123.0, dtype=torch.float64, device="cuda")
    R_un = R_sc.clone()
    monkeypatch.setenv("KLE_FGR_PW", "0")
    monkeypatch.setenv("KLE_FGR_SC", "1")
    _fgr(op, tables, U, R_sc, J, grid, alpha, status=status)
    monkeypatch.delenv("KLE_FGR_SC")
    _fgr(op, tables, U, R_un, J, grid, alpha, status=status)
    monkeypatch.delenv("KLE_FGR_PW")
    assert float((R_sc[1] - 123.0).abs().max()) == 0.0
    assert torch.equal(R_sc[3], R_un[3])
    scale = float(R_un.abs().max())
    assert float((R_sc - R_un).abs().max()) <= 1e-12 * scale
    assert not torch.equal(R_sc[0], R_un[0])
    sc = tables.scaling.cpu().numpy()
    Uh = U.cpu().numpy()
    s = 4
    A = np.diag(dia[s]) - np.diag(off[s, :-1], 1) - np.diag(off[s, :-1], -1)
    T = np.eye(nx) + grid.deltat * A
    for n in range(0, N, max(1, N // 4)):
        x = u0 if n == 0 else Uh[s, n - 1]
        for _ in range(J):
            x = np.linalg.solve(T, x + grid.deltat * g0)
        prev = alpha * Uh[s, N - 1] if n == 0 else Uh[s, n - 1]
        want = sc[n] * (x + grid.deltaT * (A @ x) - prev)
        assert rel(R_sc[s, n].cpu().numpy(), want) <= 1e-10


@pytest.mark.parametrize("N,nx,J", [(64, 511, 4), (5, 300, 3), (13, 129, 2), (8, 512, 2), (40, 450, 1)])
def test_eight_lane_scaled_sweep_matches_partitioned_and_dense(cuda, N, nx, J, monkeypatch):
    """The eight-lane scaled sweep (kle_fine_pw.cu, the default for 128 < nx <= 512:
    64 rows of one right-hand side per lane, coefficients from shared memory, the
    scaled partitioned step) against the default partitioned kernel and a dense
    evaluation of scaling_n ((I + dT A) F_n - prev_n); a masked sample stays
    untouched and a sample without a scaled form (a vanishing coupling) comes out
    of the partitioned kernel (KLE_FGR_PW=0) bitwise."""
    import torch

    from paper_2510_26180_b200 import make_time_grid
    from paper_2510_26180_b200.device import AlphaTables, DeviceOperator, to_dev
    from paper_2510_26180_b200.pcgc import _fgr, build_alpha_circulant

    rng = np.random.default_rng(11000 * N + nx)
    M, alpha, g0 = 5, 1e-3, 0.7
    grid = make_time_grid(1.0, N, max(J, 2))
    off = rng.uniform(0.1, 1.0, (M, nx)) * 4000.0
    off[:, -1] = 0.0
    off[3, nx // 3] = 0.0
    dia = rng.uniform(0.5, 1.5, (M, nx)) + off + np.concatenate([np.zeros((M, 1)), off[:, :-1]], axis=1)
    u0 = rng.normal(size=nx)
    op = DeviceOperator(to_dev(dia), to_dev(-off), g0, to_dev(u0))
    tables = AlphaTables(build_alpha_circulant(N, alpha))
    U = to_dev(rng.normal(size=(M, N, nx)))
    status = torch.zeros(M, dtype=torch.int32, device="cuda")
    status[1] = 1
    R_pw = torch.full((M, N, nx), 123.0, dtype=torch.float64, device="cuda")
    R_un = R_pw.clone()
    J = max(J, 2)
    _fgr(op, tables, U, R_pw, J, grid, alpha, status=status)
    monkeypatch.setenv("KLE_FGR_PW", "0")
    _fgr(op, tables, U, R_un, J, grid, alpha, status=status)
    monkeypatch.delenv("KLE_FGR_PW")
    assert float((R_pw[1] - 123.0).abs().max()) == 0.0
    assert torch.equal(R_pw[3], R_un[3])
    assert torch.isfinite(R_pw).all()
    scale = float(R_un.abs().max())
    assert float((R_pw - R_un).abs().max()) <= 1e-12 * scale
    assert not torch.equal(R_pw[0], R_un[0])
    sc = tables.scaling.cpu().numpy()
    Uh = U.cpu().numpy()
    s = 4
    A = np.diag(dia[s]) - np.diag(off[s, :-1], 1) - np.diag(off[s, :-1], -1)
    T = np.eye(nx) + grid.deltat * A
    for n in range(0, N, max(1, N // 4)):
        x = u0 if n == 0 else Uh[s, n - 1]
        for _ in range(J):
            x = np.linalg.solve(T, x + grid.deltat * g0)
        prev = alpha * Uh[s, N - 1] if n == 0 else Uh[s, n - 1]
        want = sc[n] * (x + grid.deltaT * (A @ x) - prev)
        assert rel(R_pw[s, n].cpu().numpy(), want) <= 1e-10


def test_eight_lane_sweep_without_source(cuda, monkeypatch):
    """g0 = 0 with a singular (Neumann-like) A: no steady state is needed, so the
    eight-lane sweep must still take every sample (not the fallback)."""
    import torch

    from paper_2510_26180_b200 import make_time_grid
    from paper_2510_26180_b200.device import AlphaTables, DeviceOperator, to_dev
    from paper_2510_26180_b200.pcgc import _fgr, build_alpha_circulant

    rng = np.random.default_rng(6)
    M, N, nx, J, alpha = 3, 20, 333, 5, 1e-2
    grid = make_time_grid(0.5, N, J)
    off = rng.uniform(0.1, 1.0, (M, nx)) * 1000.0
    off[:, -1] = 0.0
    dia = off + np.concatenate([np.zeros((M, 1)), off[:, :-1]], axis=1)
    op = DeviceOperator(to_dev(dia), to_dev(-off), 0.0, to_dev(rng.normal(size=nx)))
    tables = AlphaTables(build_alpha_circulant(N, alpha))
    U = to_dev(rng.normal(size=(M, N, nx)))
    R_pw = torch.zeros((M, N, nx), dtype=torch.float64, device="cuda")
    R_pt = torch.zeros_like(R_pw)
    _fgr(op, tables, U, R_pw, J, grid, alpha)
    monkeypatch.setenv("KLE_FGR_PW", "0")
    _fgr(op, tables, U, R_pt, J, grid, alpha)
    monkeypatch.delenv("KLE_FGR_PW")
    for s in range(M):
        assert not torch.equal(R_pw[s], R_pt[s])
    assert float((R_pw - R_pt).abs().max()) <= 1e-12 * float(R_pt.abs().max())
