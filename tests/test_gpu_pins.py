"""The reference's own hot-path pins (test_propagators.py / test_pcgc.py
of pintuq) replayed on the device path through the drop-in API, with a test-only
plugin like the reference's ``ScalarDecay`` (conftest.py:14-34)."""
import numpy as np
import pytest
import scipy.sparse as sp

from paper_2510_26180_b200 import (CoarseTrajectory, LinearModel, ParameterSample, SolverConfig,
                                   make_time_grid)

pytestmark = pytest.mark.gpu


class ScalarDecay(LinearModel):
    """u' = -lam u, nx = 1 (the reference's test plugin)."""

    name = "scalar-decay"

    def __init__(self, lam=1.0):
        self.lam, self.nx, self.parameter_dim = float(lam), 1, 1
        self.supports = ((-np.inf, np.inf),)

    @property
    def cell_volume(self):
        return 1.0

    def linear_system(self, xi):
        return sp.csc_matrix([[self.lam]]), (lambda t: np.zeros(1))

    def initial_condition(self, xi=None):
        return np.ones(1)


class Heat1D(LinearModel):
    """Constant-coefficient heat equation without source (a generic tridiagonal plugin)."""

    name = "heat-1d"

    def __init__(self, nx=31):
        self.nx, self.parameter_dim = nx, 1
        self.supports = ((-np.inf, np.inf),)
        self.h = 1.0 / (nx + 1)

    @property
    def cell_volume(self):
        return self.h

    def linear_system(self, xi):
        k = 1.0 + 0.1 * float(xi.values[0])
        main = np.full(self.nx, 2 * k / self.h ** 2)
        off = np.full(self.nx - 1, -k / self.h ** 2)
        return sp.diags([off, main, off], [-1, 0, 1], format="csc"), (lambda t: np.zeros(self.nx))

    def initial_condition(self, xi=None):
        return np.sin(np.pi * np.arange(1, self.nx + 1) * self.h)


def test_backward_euler_scalar_and_power_oracle(cuda):
    from paper_2510_26180_b200.propagators import backward_euler_step, propagate_fine

    m, xi, cfg = ScalarDecay(2.0), ParameterSample(np.zeros(1)), SolverConfig()
    v = backward_euler_step(m, np.ones(1), 0.0, 0.1, xi, cfg)
    np.testing.assert_allclose(v, [1.0 / (1.0 + 2.0 * 0.1)], rtol=1e-14)
    grid = make_time_grid(1.0, 1, 50)
    f = propagate_fine(ScalarDecay(1.0), np.ones(1), 0.0, 1.0, grid, xi, cfg)
    np.testing.assert_allclose(f, [(1.0 + 1.0 / 50) ** -50], rtol=1e-13)
    assert abs(f[0] - 0.371528) < 1e-6


def test_propagator_linearity_composition_and_errors(cuda):
    from paper_2510_26180_b200.propagators import propagate_coarse, propagate_fine

    m, xi, cfg = Heat1D(31), ParameterSample(np.array([0.7])), SolverConfig()
    grid = make_time_grid(1.0, 4, 8)
    rng = np.random.default_rng(3)
    u, v = rng.normal(size=31), rng.normal(size=31)
    fu = propagate_fine(m, u, 0.0, grid.deltaT, grid, xi, cfg)
    fv = propagate_fine(m, v, 0.0, grid.deltaT, grid, xi, cfg)
    fw = propagate_fine(m, 2.0 * u - 3.0 * v, 0.0, grid.deltaT, grid, xi, cfg)
    np.testing.assert_allclose(fw, 2.0 * fu - 3.0 * fv, rtol=1e-12, atol=1e-12 * np.abs(fw).max())
    # coarse step vs a dense solve
    A, _ = m.linear_system(xi)
    want = np.linalg.solve(np.eye(31) + grid.deltaT * A.toarray(), u)
    np.testing.assert_allclose(propagate_coarse(m, u, 0.0, grid.deltaT, xi, cfg), want, rtol=1e-12,
                               atol=1e-13 * np.abs(want).max())
    # composition is bitwise: two calls of one interval = the same twice
    a1 = propagate_fine(m, fu, grid.deltaT, 2 * grid.deltaT, grid, xi, cfg)
    a2 = propagate_fine(m, propagate_fine(m, u, 0.0, grid.deltaT, grid, xi, cfg), grid.deltaT,
                        2 * grid.deltaT, grid, xi, cfg)
    np.testing.assert_array_equal(a1, a2)
    u_copy = u.copy()
    propagate_fine(m, u, 0.0, grid.deltaT, grid, xi, cfg)
    np.testing.assert_array_equal(u, u_copy)  # the input is never mutated
    with pytest.raises(ValueError):
        propagate_fine(m, u, 0.0, 0.5 * grid.deltaT, grid, xi, cfg)


def test_three_step_block_mismatch_and_cgc_fixed_point(cuda):
    from paper_2510_26180_b200.pcgc import build_alpha_circulant, cgc_correct, three_step_solve
    from paper_2510_26180_b200.propagators import fine_reference, propagate_fine

    m, xi, cfg = Heat1D(15), ParameterSample(np.array([-0.4])), SolverConfig(alpha=1e-2)
    grid = make_time_grid(1.0, 8, 6)
    A, _ = m.linear_system(xi)
    with pytest.raises(ValueError):
        three_step_solve(build_alpha_circulant(8, 1e-2), -A, grid.deltaT, np.zeros((7, 15)))
    # the serial fine trajectory is a fixed point of the CGC (pcgc.py:208-243)
    ref = fine_reference(m, xi, grid, cfg)
    starts = np.vstack([ref.initial, ref.states[:-1]])
    F = np.array([propagate_fine(m, starts[n], n * grid.deltaT, (n + 1) * grid.deltaT, grid, xi, cfg)
                  for n in range(8)])
    out, diag = cgc_correct(m, xi, grid, cfg, CoarseTrajectory(ref.initial, ref.states), F)
    np.testing.assert_allclose(out.states, ref.states, rtol=0, atol=1e-10 * np.abs(ref.states).max())
    assert diag["imag_residue"] <= 1e-10


def test_pcgc_converges_to_fine_reference(cuda):
    from paper_2510_26180_b200.pcgc import pcgc_solve
    from paper_2510_26180_b200.propagators import coarse_sweep_init, fine_reference

    m, xi = Heat1D(31), ParameterSample(np.array([0.2]))
    grid, cfg = make_time_grid(1.0, 16, 8), SolverConfig(alpha=1e-3, tol=1e-10, max_outer_iters=60)
    ref = fine_reference(m, xi, grid, cfg)
    tr = pcgc_solve(m, xi, grid, cfg, coarse_sweep_init(m, xi, grid, cfg))
    assert tr.converged
    assert np.max(np.abs(tr.trajectory.states - ref.states)) <= 10 * cfg.tol
    assert tr.diagnostics["max_imag_residue"] <= 1e-10 * max(np.abs(tr.trajectory.states).max(), 1.0)


def test_block_dft_and_factor_shifted_api(cuda):
    """forward_dft / inverse_dft against np.fft and the naive DFT matrix
    (pintuq tests: test_pcgc.py:65-86 pins at 1e-13), and factor_shifted's
    solvers against dense solves; zero pivots raise SingularShiftError."""
    import scipy.sparse as sp
    from paper_2510_26180_b200 import SingularShiftError
    from paper_2510_26180_b200.pcgc import build_alpha_circulant, factor_shifted, forward_dft, inverse_dft

    rng = np.random.default_rng(4)
    for N in (1, 2, 5, 8, 33):
        v = rng.normal(size=(N, 7)) + 1j * rng.normal(size=(N, 7))
        np.testing.assert_allclose(forward_dft(v), np.fft.ifft(v, axis=0, norm="ortho"), rtol=0, atol=1e-13)
        np.testing.assert_allclose(inverse_dft(v), np.fft.fft(v, axis=0, norm="ortho"), rtol=0, atol=1e-13)
        np.testing.assert_allclose(inverse_dft(forward_dft(v)), v, rtol=0, atol=1e-13)
        w = np.exp(2j * np.pi * np.outer(np.arange(N), np.arange(N)) / N) / np.sqrt(N)
        np.testing.assert_allclose(forward_dft(v), w @ v, rtol=0, atol=1e-12)
    nx, dT = 12, 0.05
    J = sp.diags([rng.uniform(1, 2, nx - 1), -rng.uniform(4, 6, nx), rng.uniform(1, 2, nx - 1)], [-1, 0, 1])
    spec = build_alpha_circulant(6, 0.1)
    solvers = factor_shifted(spec, J, dT)
    for lam, solve in zip(spec.eigenvalues, solvers):
        p = rng.normal(size=nx) + 1j * rng.normal(size=nx)
        q = solve(p)
        dense = lam * np.eye(nx) - dT * J.toarray()
        np.testing.assert_allclose(dense @ q, p, rtol=0, atol=1e-12)
    scalar = factor_shifted(spec, np.array([[2.0]]), dT)
    np.testing.assert_allclose(scalar[1](np.array([1.0 + 0j])), 1.0 / (spec.eigenvalues[1] - dT * 2.0), rtol=1e-14)
    sing = factor_shifted(build_alpha_circulant(1, 0.5), np.array([[1.0]]), 0.5)  # lambda = 0.5 = dT J
    with pytest.raises(SingularShiftError):
        sing[0](np.array([1.0 + 0j]))


def test_reference_diffusion1d_model_on_device(cuda, golden):
    """The reference's Diffusion1D plugin (symmetric tridiagonal, zero source)
    runs through the generic plugin path: pcgc_solve matches the reference."""
    from paper_2510_26180_b200 import CoarseTrajectory, ParameterSample, SolverConfig, make_time_grid
    from tests.plugins import AdvectionDiffusion2D, Diffusion1D
    from paper_2510_26180_b200.pcgc import pcgc_solve

    g = golden("models")
    model, xi = Diffusion1D(), ParameterSample(np.array([1.3]), id=0)
    grid = make_time_grid(1.0, 16, 32)
    cfg = SolverConfig(alpha=0.1, tol=1e-10, max_outer_iters=60)
    tr = pcgc_solve(model, xi, grid, cfg, CoarseTrajectory(model.initial_condition(), g["d1_init"]))
    assert tr.iterations == int(g["d1_iters"])
    assert np.max(np.abs(tr.trajectory.states - g["d1_final"])) <= 1e-10 * np.max(np.abs(g["d1_final"]))
    ad = AdvectionDiffusion2D()
    with pytest.raises(NotImplementedError):
        pcgc_solve(ad, ParameterSample(np.array([3.0]), id=0), make_time_grid(1.0, 8, 4), cfg,
                   CoarseTrajectory(ad.initial_condition(), np.zeros((8, ad.nx))))


@pytest.mark.parametrize("pipes", [2, 3, 4])
def test_sample_pipelines_do_not_change_results(cuda, pipes, monkeypatch):
    """The batched loop's staggered sample pipelines (KLE_PCGC_PIPES) only
    regroup launches: states, iteration counts and increments are bitwise the
    single-pipeline ones (scheduling independence)."""
    import torch

    from paper_2510_26180_b200 import LogNormalKL1D
    from paper_2510_26180_b200.pcgc import pcgc_solve_batched

    model = LogNormalKL1D(nx=127, d=4)
    grid = make_time_grid(1.0, 16, 32)
    cfg = SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60)
    M = 301
    xi = np.random.default_rng(7).normal(size=(M, 4))
    U0 = np.random.default_rng(8).uniform(0.0, 1.0, size=(M, 16, 127))
    monkeypatch.setenv("KLE_PCGC_PIPES", "1")
    one = pcgc_solve_batched(model, xi, grid, cfg, U0)
    monkeypatch.setenv("KLE_PCGC_PIPES", str(pipes))
    many = pcgc_solve_batched(model, xi, grid, cfg, U0)
    assert torch.equal(one.iters, many.iters)
    assert torch.equal(one.status, many.status)
    assert torch.equal(one.states, many.states)
    assert torch.equal(torch.nan_to_num(one.increments, nan=-1.0), torch.nan_to_num(many.increments, nan=-1.0))


@pytest.mark.parametrize("env,val", [("KLE_FUSED", "1"), ("KLE_FUSED", "2"), ("KLE_CGC_SMALL", "1")])
def test_small_block_kernels_match_default_path(cuda, golden, env, val, monkeypatch):
    """The small-block kernels (kle_iter_small.cu: the fused whole-iteration
    kernel with one CTA or one warp per sample, and the CGC-only variant;
    opt-in A/B paths for nx <= 128, N <= 16) against the default fgr +
    cluster-CGC path on the
    config-1 goldens: iteration counts exact, fields within 1e-12."""
    import torch

    from paper_2510_26180_b200 import LogNormalKL1D
    from paper_2510_26180_b200.pcgc import pcgc_solve_batched

    g = golden("c1")
    model = LogNormalKL1D(nx=127, d=4)
    grid = make_time_grid(1.0, 16, 32)
    cfg = SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60)
    base = pcgc_solve_batched(model, g["xi_all"][:16], grid, cfg, g["U0"][:16])
    monkeypatch.setenv(env, val)
    alt = pcgc_solve_batched(model, g["xi_all"][:16], grid, cfg, g["U0"][:16])
    assert torch.equal(base.iters, alt.iters)
    np.testing.assert_array_equal(alt.iters.cpu().numpy(), g["iters"])
    d = float((base.states - alt.states).abs().max() / base.states.abs().max())
    assert d <= 1e-12, d


def test_streaming_large_cgc_is_bitwise_the_three_kernel_path(cuda, monkeypatch):
    """The opt-in streaming large-block CGC (KLE_CGCL_STREAM=1: per-sample CTAs
    walking row blocks, FFT + forward recurrence fused, back substitution +
    inverse FFT + update fused) performs the same operations per element as
    the three-kernel path: the updated U and increments are bitwise equal.
    Run in a subprocess per setting (the switch is read once per process)."""
    import subprocess
    import sys

    root = str(__import__("pathlib").Path(__file__).resolve().parents[1])
    outs = []
    for v in ("0", "1"):
        env = dict(__import__("os").environ, KLE_CGCL_STREAM=v)
        r = subprocess.run([sys.executable, "tools/ab_cgcl.py", "8"], capture_output=True, text=True, cwd=root,
                           env=env, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(r.stdout.split("checksum")[1].strip())
    assert outs[0] == outs[1], outs
