"""Pin the CPU oracle against the golden vectors produced by the unmodified
reference (tests/golden/make_golden.py). CPU only."""
import numpy as np
import pytest

from oracle import batched, ref_port
from tests.conftest import c1_config


def _op(model, xi):
    dia, off = model.tridiagonal(xi)
    full_off = off
    return ref_port.SampleOperator(dia, full_off, np.full(model.nx, model.source))


def test_kl_table_matches_golden(golden):
    model, _, _ = c1_config()
    g = golden("c1")
    np.testing.assert_allclose(model.kl_table, g["kl_table"], rtol=0, atol=1e-13)


def test_ref_port_single_calls_bitwise(golden):
    model, grid, cfg = c1_config()
    g = golden("c1")
    xi0 = g["xi_all"][0]
    op = _op(model, xi0)
    u0 = model.initial_condition()
    np.testing.assert_array_equal(ref_port.fine(op, u0, grid.n_fine_per_coarse, grid.deltat), g["pf_u0"])
    np.testing.assert_array_equal(ref_port.fine(op, g["u_rand"], grid.n_fine_per_coarse, grid.deltat), g["pf_rand"])
    np.testing.assert_array_equal(ref_port.coarse(op, g["u_rand"], grid.deltaT), g["pc_rand"])
    lam, scaling = ref_port.alpha_circulant(16, 1e-3)
    np.testing.assert_array_equal(lam, g["lam"])
    np.testing.assert_array_equal(scaling, g["scaling"])
    solvers = ref_port.shifted_solvers(op, lam, grid.deltaT)
    u, imag = ref_port.three_step(lam, scaling, solvers, g["r_rand"])
    np.testing.assert_array_equal(u, g["ts_u"])
    assert imag == g["ts_imag"]
    Un, im = ref_port.cgc(op, lam, scaling, solvers, cfg.alpha, grid.deltaT, g["U0"][0], g["F_ends"])
    np.testing.assert_array_equal(Un, g["cgc_states"])
    cs = ref_port.coarse_sweep(op, u0, 16, grid.deltaT)
    np.testing.assert_array_equal(cs, g["coarse_sweep"])


def test_ref_port_pcgc_reproduces_reference_c1(golden):
    model, grid, cfg = c1_config()
    g = golden("c1")
    u0 = model.initial_condition()
    for i in range(len(g["iters"])):
        op = _op(model, g["xi_all"][i])
        out = ref_port.pcgc(op, u0, g["U0"][i], 16, 32, 1.0, cfg.alpha, cfg.tol, cfg.max_outer_iters)
        assert out["iters"] == g["iters"][i]
        np.testing.assert_array_equal(out["states"], g["final"][i])
        np.testing.assert_array_equal(out["increments"], g["increments"][i, : out["iters"]])


def test_ref_port_surrogate_bitwise(golden):
    g = golden("c1")
    for i in range(len(g["iters"])):
        pred = ref_port.surrogate_predict(g["mean_field"], g["eigenvalues"], g["modes"], g["coeffs"],
                                          int(g["degree"]), g["xi_all"][i])
        np.testing.assert_array_equal(pred, g["U0"][i])


def test_ref_port_kl_and_fit_from_snapshots(golden):
    model, grid, _ = c1_config()
    g = golden("c1")
    w = model.cell_volume * grid.deltaT
    mean, lam, modes, X = ref_port.kl_build(g["snapshots"], w, 1e-10)
    np.testing.assert_array_equal(mean, g["mean_field"])
    np.testing.assert_allclose(lam, g["eigenvalues"], rtol=1e-12)
    assert modes.shape == g["modes"].shape
    np.testing.assert_allclose(modes, g["modes"], rtol=0, atol=1e-9 * np.abs(g["modes"]).max())
    zeta = ref_port.kl_coefficients(X, modes, lam, w)
    coeffs = ref_port.gpc_fit(g["train_points"], zeta, 2)
    np.testing.assert_allclose(coeffs, g["coeffs"], rtol=0, atol=1e-9 * np.abs(g["coeffs"]).max())


def test_batched_oracle_matches_reference_c1(golden):
    model, grid, cfg = c1_config()
    g = golden("c1")
    xi = g["xi_all"][: len(g["iters"])]
    dia, off = batched.tridiag_from_xi(xi, model.kl_table, model.h)
    out = batched.pcgc(dia, off, model.initial_condition(), g["U0"], 16, 32, 1.0, cfg.alpha, cfg.tol,
                       cfg.max_outer_iters)
    np.testing.assert_array_equal(out["iters"], g["iters"])
    scale = np.abs(g["final"]).max()
    assert np.max(np.abs(out["states"] - g["final"])) / scale <= 1e-10
    mean, var = batched.moments(out["states"])
    np.testing.assert_allclose(mean, g["mean"], rtol=1e-11, atol=1e-14)
    np.testing.assert_allclose(var, g["var"], rtol=1e-9, atol=1e-16)
    U0 = batched.hermite_predict(g["mean_field"], g["eigenvalues"], g["modes"], g["coeffs"], 2, xi)
    np.testing.assert_allclose(U0, g["U0"], rtol=0, atol=1e-14)


def test_batched_oracle_c2_shapes(golden):
    from paper_2510_26180_b200 import LogNormalKL1D

    g = golden("c2")
    model = LogNormalKL1D(nx=511, d=8)
    np.testing.assert_allclose(model.kl_table, g["kl_table"], rtol=0, atol=1e-13)
    dia, off = batched.tridiag_from_xi(g["xi"], model.kl_table, model.h)
    init = batched.coarse_sweep(dia, off, model.initial_condition(), 64, 1.0 / 64)
    out = batched.pcgc(dia, off, model.initial_condition(), init, 64, 64, 1.0, 1e-3, 1e-8, 60)
    np.testing.assert_array_equal(out["iters"], g["iters"])
    assert np.max(np.abs(out["states"] - g["final"])) / np.abs(g["final"]).max() <= 1e-10


@pytest.mark.parametrize("tag,alpha", [("a1", 1e-1), ("a2", 1e-2), ("a4", 1e-4)])
def test_batched_oracle_c5_analogue(golden, tag, alpha):
    from paper_2510_26180_b200 import LogNormalKL1D

    g = golden("c5s")
    model = LogNormalKL1D(nx=255, d=4)
    dia, off = batched.tridiag_from_xi(g["xi"][None], model.kl_table, model.h)
    N = 128
    init = batched.coarse_sweep(dia, off, model.initial_condition(), N, 1.0 / N)
    out = batched.pcgc(dia, off, model.initial_condition(), init, N, 8, 1.0, alpha, 1e-8, 60)
    assert out["iters"][0] == int(g[f"{tag}_iters"])
    cond = alpha ** (-(N - 1) / N)
    rtol = max(1e-10, 1e-12 * cond)
    assert np.max(np.abs(out["states"][0] - g[f"{tag}_final"])) / np.abs(g[f"{tag}_final"]).max() <= rtol


# --- reference test pins restated on the oracle (pintuq tests/test_pcgc.py) ---
@pytest.mark.parametrize("n", [2, 4, 8, 16, 32])
@pytest.mark.parametrize("alpha", [0.05, 0.1, 0.5])
def test_alpha_circulant_diagonalises(n, alpha):
    from paper_2510_26180_b200.pcgc import build_alpha_circulant

    spec = build_alpha_circulant(n, alpha)
    V, Vinv = spec.eigenvector_matrix(), spec.inverse_eigenvector_matrix()
    np.testing.assert_allclose(V @ Vinv, np.eye(n), atol=1e-12)
    assert np.max(np.abs(V @ np.diag(spec.eigenvalues) @ Vinv - spec.dense_matrix())) <= 1e-12
    lam, sc = ref_port.alpha_circulant(n, alpha)
    np.testing.assert_array_equal(lam, spec.eigenvalues)
    np.testing.assert_array_equal(sc, spec.scaling)


def test_alpha_circulant_pins():
    from paper_2510_26180_b200.pcgc import build_alpha_circulant

    assert build_alpha_circulant(1, 0.5).eigenvalues[0] == pytest.approx(0.5, abs=1e-15)
    np.testing.assert_allclose(np.sort(build_alpha_circulant(2, 0.25).eigenvalues.real), [0.5, 1.5], atol=1e-14)
    assert np.prod(build_alpha_circulant(4, 0.1).eigenvalues) == pytest.approx(0.9, rel=1e-12)
    for n in (2, 8, 33, 64):
        cond = np.linalg.cond(build_alpha_circulant(n, 0.1).eigenvector_matrix())
        assert cond == pytest.approx(0.1 ** (-(n - 1) / n), rel=1e-10)
    for a in (0.0, 1.0, -0.2, 1.5):
        with pytest.raises(ValueError):
            build_alpha_circulant(4, a)


def _dense_all_at_once(spec_dense, J, dT, r):
    n, nx = r.shape
    Mx = np.kron(spec_dense, np.eye(nx)) - dT * np.kron(np.eye(n), J)
    return np.linalg.solve(Mx, r.reshape(-1)).reshape(n, nx)


@pytest.mark.parametrize("trial", range(12))
def test_oracle_three_step_vs_dense(trial):
    from paper_2510_26180_b200.pcgc import build_alpha_circulant

    rng = np.random.default_rng(100 + trial)
    n = int(rng.integers(1, 9))
    nx = int(rng.integers(1, 17))
    alpha = float(rng.uniform(0.02, 0.9))
    dT = float(rng.uniform(0.01, 1.0))
    spec = build_alpha_circulant(n, alpha)
    # symmetric diagonally dominant tridiagonal A (the device operator class)
    off = -rng.uniform(0.1, 1.0, nx - 1) if nx > 1 else np.zeros(0)
    dia = rng.uniform(0.5, 1.5, nx) + np.concatenate([[0.0], -off]) + np.concatenate([-off, [0.0]])
    A = np.diag(dia) + np.diag(off, 1) + np.diag(off, -1)
    r = rng.normal(size=(n, nx))
    expected = _dense_all_at_once(spec.dense_matrix(), -A, dT, r)
    op = ref_port.SampleOperator(dia, off, np.zeros(nx))
    u, imag = ref_port.three_step(spec.eigenvalues, spec.scaling, ref_port.shifted_solvers(op, spec.eigenvalues, dT), r)
    scale = max(np.abs(expected).max(), 1e-30)
    assert np.abs(u - expected).max() / scale <= 1e-9
    assert imag <= 1e-10 * max(np.abs(u).max(), 1.0)


def test_oracle_2d_matches_reference_goldens(golden):
    """The per-sample restatement on the 5-point operator (SuperLU paths of
    pcgc.py:137-145) reproduces the reference bit for bit."""
    from oracle import ref_port
    from paper_2510_26180_b200.models import LogNormalKL2D

    g = golden("c3s")
    m = LogNormalKL2D(n=15, d=10)
    np.testing.assert_array_equal(m.kl_table, g["kl_table"])
    for i in range(3):
        dia, ex, ey = m.stencil(g["xi"][i])
        op = ref_port.SampleOperator.from_stencil2d(dia, ex, ey, 15, np.ones(225))
        np.testing.assert_array_equal(ref_port.coarse_sweep(op, m.initial_condition(), 8, 1 / 8), g["coarse_sweep"][i])
        out = ref_port.pcgc(op, m.initial_condition(), g["coarse_sweep"][i], 8, 4, 1.0, 1e-3, 1e-8, 60)
        assert out["iters"] == g["iters"][i]
        np.testing.assert_array_equal(out["states"], g["final"][i])
    dia, ex, ey = m.stencil(g["xi"][0])
    op = ref_port.SampleOperator.from_stencil2d(dia, ex, ey, 15, np.ones(225))
    np.testing.assert_array_equal(ref_port.fine(op, g["u_rand"], 4, 1 / 32), g["pf_rand"])
    lam, sc = ref_port.alpha_circulant(8, 1e-3)
    u, _ = ref_port.three_step(lam, sc, ref_port.shifted_solvers(op, lam, 1 / 8), g["r_rand"])
    np.testing.assert_array_equal(u, g["ts_u"])


def _check_ref_run(out, g, tag, i):
    K = out["iters"] + 1
    assert out["iters"] == g[f"{tag}_iters"][i]
    np.testing.assert_array_equal(out["states"], g[f"{tag}_final"][i])
    np.testing.assert_array_equal(out["err"], g[f"{tag}_err"][i, :K])
    np.testing.assert_array_equal(out["max_err"], g[f"{tag}_max_err"][i, :K])
    np.testing.assert_array_equal(out["increments"], g[f"{tag}_incs"][i, 1:K])


def test_ref_port_stop_on_reference_bitwise(golden):
    """stop_on="reference" with the serial fine reference (the harness
    composition, pintuq/experiments.py:212-235): kle-pcgc from the surrogate
    U0, pcgc from random_guess_init, and reference= with increment stopping."""
    model, grid, cfg = c1_config()
    g1, g = golden("c1"), golden("ref")
    u0 = model.initial_condition()
    for tag, inits, stop in (("kle", g1["U0"], "reference"), ("rnd", g["rnd_init"], "reference"),
                             ("inc", g1["U0"], "increment")):
        for i in range(len(g[f"{tag}_iters"])):
            op = _op(model, g1["xi_all"][i])
            ref = ref_port.fine_reference(op, u0, 16, 32, grid.deltaT)
            np.testing.assert_array_equal(ref, g[f"{tag}_ref"][i])
            out = ref_port.pcgc(op, u0, inits[i], 16, 32, 1.0, cfg.alpha, cfg.tol, cfg.max_outer_iters,
                                reference=ref, stop_on=stop)
            _check_ref_run(out, g, tag, i)


def test_random_guess_init_matches_reference(golden):
    """random_guess_init draws (pintuq/parareal.py:63-71) from the harness's
    init stream are reproduced by the drop-in (same PCG64 derivation)."""
    from paper_2510_26180_b200 import ParameterSample, RngStream
    from paper_2510_26180_b200.propagators import random_guess_init

    model, grid, cfg = c1_config()
    g1, g = golden("c1"), golden("ref")
    _, _, init_rng = RngStream(2718).split(3)
    for i in range(4):
        tr = random_guess_init(model, ParameterSample(g1["xi_all"][i], id=i), grid, init_rng)
        np.testing.assert_array_equal(tr.states, g["rnd_init"][i])


def test_oracle_2d_stop_on_reference(golden):
    from paper_2510_26180_b200.models import LogNormalKL2D

    g3, g = golden("c3s"), golden("ref")
    m = LogNormalKL2D(n=15, d=10)
    for i in range(3):
        dia, ex, ey = m.stencil(g3["xi"][i])
        op = ref_port.SampleOperator.from_stencil2d(dia, ex, ey, 15, np.ones(225))
        ref = ref_port.fine_reference(op, m.initial_condition(), 8, 4, 1 / 8)
        np.testing.assert_array_equal(ref, g["c3s_ref"][i])
        out = ref_port.pcgc(op, m.initial_condition(), g3["coarse_sweep"][i], 8, 4, 1.0, 1e-3, 1e-8, 60,
                            reference=ref, stop_on="reference")
        _check_ref_run(out, g, "c3s", i)


def test_ref_port_parareal_bitwise(golden):
    """Classical parareal restatement (pintuq/parareal.py:100-191) against the
    reference: coarse-sweep init with increment stop, random init with the
    reference stop (1D), and the 2D plugin."""
    from paper_2510_26180_b200.models import LogNormalKL2D

    model, grid, cfg = c1_config()
    g1, gr, g = golden("c1"), golden("ref"), golden("para")
    u0 = model.initial_condition()
    for i in range(4):
        op = _op(model, g1["xi_all"][i])
        np.testing.assert_array_equal(ref_port.coarse_sweep(op, u0, 16, grid.deltaT), g["cs_init"][i])
        out = ref_port.parareal(op, u0, g["cs_init"][i], 16, 32, 1.0, cfg.tol, cfg.max_outer_iters)
        assert out["iters"] == g["cs_iters"][i]
        np.testing.assert_array_equal(out["states"], g["cs_final"][i])
        np.testing.assert_array_equal(out["increments"], g["cs_incs"][i, 1:out["iters"] + 1])
        ref = ref_port.fine_reference(op, u0, 16, 32, grid.deltaT)
        out = ref_port.parareal(op, u0, gr["rnd_init"][i], 16, 32, 1.0, cfg.tol, cfg.max_outer_iters,
                                reference=ref, stop_on="reference")
        _check_ref_run(out, g, "rnd", i)
    g3 = golden("c3s")
    m = LogNormalKL2D(n=15, d=10)
    for i in range(3):
        op = ref_port.SampleOperator.from_stencil2d(*m.stencil(g3["xi"][i]), 15, np.ones(225))
        out = ref_port.parareal(op, m.initial_condition(), g3["coarse_sweep"][i], 8, 4, 1.0, 1e-8, 60)
        assert out["iters"] == g["c3s_iters"][i]
        np.testing.assert_array_equal(out["states"], g["c3s_final"][i])


def test_nonlinear_models_match_reference(golden):
    """Burgers1D / AllenCahn1D host definitions (rhs, Jacobian, samplers,
    initial states) against the reference's (pintuq/models.py:269-379)."""
    from paper_2510_26180_b200 import AllenCahn1D, Burgers1D, ParameterSample, RngStream

    g = golden("nl")
    for tag, model, ns in (("bu", Burgers1D(dx=1 / 100), 3), ("ac", AllenCahn1D(dx=1 / 128), 2)):
        xis = model.sample_parameters(ns, RngStream(2718).split(3)[1])
        np.testing.assert_array_equal(np.array([x.values for x in xis]), g[f"{tag}_xi"])
        xi0 = ParameterSample(g[f"{tag}_xi"][0], id=0)
        u0 = model.initial_condition(xi0)
        np.testing.assert_array_equal(model.rhs(u0, 0.0, xi0), g[f"{tag}_rhs0"])
        np.testing.assert_array_equal(model.jacobian(u0, 0.0, xi0).toarray(), g[f"{tag}_jac0"])
        assert model.nx == g[f"{tag}_ref"].shape[1]


def test_nonlinear_port_bitwise(golden):
    """The nonlinear restatement (Newton sweeps, simplified-Newton CGC,
    parareal and PCGC loops) reproduces the reference bit for bit at the
    harness settings (tests/golden/nl.npz, pure-Python backend)."""
    from oracle import nonlinear_port as nlp
    from paper_2510_26180_b200 import AllenCahn1D, Burgers1D

    g = golden("nl")
    for tag, model, T, N, J in (("bu", Burgers1D(dx=1 / 100), 2.0, 25, 40), ("ac", AllenCahn1D(dx=1 / 128), 3.0, 30, 48)):
        xs = g[f"{tag}_xi"]
        m0 = (model.sweep_kind,) + model.sweep_params(xs[0])
        u0 = model.initial_condition()
        dT = T / N
        np.testing.assert_array_equal(nlp.sweep(m0, u0, dT / J, J)[0], g[f"{tag}_pf"])
        np.testing.assert_array_equal(nlp.sweep(m0, u0, dT, 1)[0], g[f"{tag}_pc"])
        lam, sc = ref_port.alpha_circulant(N, 0.1)
        U = g[f"{tag}_init"][0]
        prev = np.vstack([0.1 * U[-1:], U[:-1]])
        G = np.array([nlp.sweep(m0, prev[n], nlp.coarse_dt(T, N, n), 1)[0] for n in range(N)])
        out, inner = nlp.cgc_newton(m0, lam, sc, N, dT, U, g[f"{tag}_cgc_F"] - G, 1e-12)
        np.testing.assert_array_equal(out, g[f"{tag}_cgc_out"])
        assert inner == g[f"{tag}_cgc_inner"]
        i = len(xs) - 1  # one full loop of each kind per model (the longest runs are the GPU tests' job)
        mi = (model.sweep_kind,) + model.sweep_params(xs[i])
        pc = nlp.pcgc_newton(mi, u0, g[f"{tag}_init"][i], N, J, T, 0.1, 1e-8, 60)
        assert pc["iters"] == g[f"{tag}_pcgc_iters"][i]
        np.testing.assert_array_equal(pc["states"], g[f"{tag}_pcgc_final"][i])
        pa = nlp.parareal_newton(mi, u0, g[f"{tag}_init"][i], N, J, T, 1e-8, 60)
        assert pa["iters"] == g[f"{tag}_iters"][i]
        np.testing.assert_array_equal(pa["states"], g[f"{tag}_final"][i])


def test_reference_linear_models_match(golden):
    """Diffusion1D / AdvectionDiffusion2D host definitions equal the
    reference's (pintuq/models.py:128-266) bit for bit."""
    from paper_2510_26180_b200 import ParameterSample
    from tests.plugins import AdvectionDiffusion2D, Diffusion1D

    g = golden("models")
    xi = ParameterSample(np.array([1.3]), id=0)
    for tag, model in (("d1", Diffusion1D()), ("ad", AdvectionDiffusion2D())):
        A, src = model.linear_system(xi)
        np.testing.assert_array_equal(A.toarray(), g[f"{tag}_A"])
        np.testing.assert_array_equal(src(0.3), g[f"{tag}_g"])
        np.testing.assert_array_equal(model.initial_condition(xi), g[f"{tag}_u0"])
