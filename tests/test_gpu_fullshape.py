"""Parity at the BASELINE configs' full shapes (round-2 corners):

- c5 (nx 4095, N 1024, J 8), every alpha in {1e-1, 1e-2, 1e-4}: 8 seeded
  samples from coarse-sweep init against the batched oracle, and the first
  two against the goldens of the unmodified reference (c5full.npz);
  iteration counts exact, fields within max(1e-10, 1e-12 cond V), the
  reference's own FFT-vs-DFT floor at alpha = 1e-4;
- c3 (127 x 127, N 32, J 16): eval samples 0..3 from coarse-sweep init
  against the reference (c3.npz, c3b.npz), and 4 samples from the config's
  own surrogate (p = 2 on 1,024 device-built training solves) against the
  oracle's SuperLU path run from the same U0;
- c4 (config 1 at M = 1,048,576 samples, the metric's scaling workload): the
  full batch on one GPU, all converged, a 32-sample seeded subset against the
  batched oracle with exact iteration counts, and the moments against numpy.
"""
import numpy as np
import pytest

from oracle import batched, ref_port

pytestmark = pytest.mark.gpu
RTOL = 1e-10


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("tag,alpha", [("a1", 1e-1), ("a2", 1e-2), ("a4", 1e-4)])
def test_c5_full_shape(cuda, golden, tag, alpha):
    import torch

    from paper_2510_26180_b200 import LogNormalKL1D, RngStream, SolverConfig, make_time_grid
    from paper_2510_26180_b200.device import DeviceOperator
    from paper_2510_26180_b200.pcgc import pcgc_solve_device
    from paper_2510_26180_b200.propagators import coarse_sweep_init_batched

    nx, N, J, M = 4095, 1024, 8, 8
    model = LogNormalKL1D(nx=nx, d=4, sigma=0.5, ell=0.3)
    grid = make_time_grid(1.0, N, J)
    cfg = SolverConfig(alpha=alpha, tol=1e-8, max_outer_iters=60)
    _, eval_rng, _ = RngStream(2718).split(3)
    xi = eval_rng.normal(0.0, 1.0, size=(M, 4))   # the c5 bench's first 8 samples
    op = DeviceOperator.from_model(model, xi)
    U = coarse_sweep_init_batched(op, grid).contiguous()
    init = U.cpu().numpy()
    res = pcgc_solve_device(op, U, grid, cfg)
    torch.cuda.synchronize()
    iters = res.iters.cpu().numpy()
    states = res.states.cpu().numpy()
    assert np.all(res.status.cpu().numpy() == 1)
    rtol = max(RTOL, 1e-12 * alpha ** (-(N - 1) / N))
    # the unmodified reference on samples 0 and 1
    g = golden("c5full")
    np.testing.assert_array_equal(g["xi"], xi[:2])
    np.testing.assert_array_equal(iters[:2], g[f"{tag}_iters"])
    for i in range(2):
        scale = np.abs(g[f"{tag}_rowmax"][i]).max()
        assert np.max(np.abs(states[i, ::8, ::8] - g[f"{tag}_sub"][i])) <= rtol * scale
        assert np.max(np.abs(np.abs(states[i]).max(axis=1) - g[f"{tag}_rowmax"][i])) <= rtol * scale
        assert np.max(np.abs(states[i].sum(axis=1) - g[f"{tag}_rowsum"][i])) <= rtol * scale * nx
        K = int(iters[i])
        np.testing.assert_allclose(res.increments[i, :K].cpu().numpy(), g[f"{tag}_incs"][i, :K], rtol=0,
                                   atol=max(1e-11, rtol))
    # all 8 against the batched oracle from the same initial guess
    dia, off = batched.tridiag_from_xi(xi, model.kl_table, model.h)
    out = batched.pcgc(dia, off, model.initial_condition(), init, N, J, 1.0, alpha, 1e-8, 60)
    np.testing.assert_array_equal(iters, out["iters"])
    assert rel(states, out["states"]) <= rtol


def _c3_setup():
    from paper_2510_26180_b200 import LogNormalKL2D, RngStream, SolverConfig, make_time_grid

    model = LogNormalKL2D(n=127, d=10, sigma=0.5, ell=0.25)
    grid = make_time_grid(1.0, 32, 16)
    cfg = SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60, seed=2718)
    train_rng, eval_rng, _ = RngStream(2718).split(3)
    return model, grid, cfg, train_rng, eval_rng


def test_c3_full_shape_four_samples(cuda, golden):
    from paper_2510_26180_b200.device import DeviceOperator
    from paper_2510_26180_b200.pcgc import pcgc_solve_device
    from paper_2510_26180_b200.propagators import coarse_sweep_init_batched

    model, grid, cfg, _, eval_rng = _c3_setup()
    g0, gb = golden("c3"), golden("c3b")
    xi = eval_rng.normal(0.0, 1.0, size=(4, 10))
    np.testing.assert_array_equal(xi[:1], g0["xi"])
    np.testing.assert_array_equal(xi[1:], gb["xi"])
    op = DeviceOperator.from_model(model, xi)
    res = pcgc_solve_device(op, coarse_sweep_init_batched(op, grid).contiguous(), grid, cfg)
    iters = res.iters.cpu().numpy()
    np.testing.assert_array_equal(iters, np.concatenate([g0["iters"], gb["iters"]]))
    states = res.states.cpu().numpy()
    want = np.concatenate([g0["final"], gb["final"]])
    for i in range(4):
        assert rel(states[i], want[i]) <= RTOL, i


def _c3_oracle(task):
    stencil, U0, u0 = task
    from threadpoolctl import threadpool_limits

    with threadpool_limits(1):
        op = ref_port.SampleOperator.from_stencil2d(*stencil, 127, np.full(127 * 127, 1.0))
        out = ref_port.pcgc(op, u0, U0, 32, 16, 1.0, 1e-3, 1e-8, 60)
    return out["iters"], out["states"]


def test_c3_from_config_surrogate(cuda):
    """Config 3 as specified: the degree-2 (66-term) Hermite surrogate fitted
    on 1,024 seeded training solves (built on the device), U0 for 4 eval
    samples, the device PCGC from it, against the oracle (the reference's
    SuperLU path, bit-identical to its goldens) from the same U0."""
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor

    from paper_2510_26180_b200 import ParameterSample
    from paper_2510_26180_b200.engine import KleCgcSolver
    from paper_2510_26180_b200.surrogate import build_surrogate

    model, grid, cfg, train_rng, eval_rng = _c3_setup()
    train = [ParameterSample(p, id=i) for i, p in enumerate(train_rng.normal(0.0, 1.0, size=(1024, 10)))]
    sur = build_surrogate(model, grid, cfg, train, eps_kl=1e-10, degree=2, family="hermite")
    assert sur.coeffs.shape[1] == 66
    xi = eval_rng.normal(0.0, 1.0, size=(4, 10))
    res = KleCgcSolver(model, grid, cfg, sur).solve(xi, keep_initial=True)
    iters = res.batch.iters.cpu().numpy()
    U0 = res.U0.cpu().numpy()
    tasks = [(model.stencil(xi[i]), U0[i], model.initial_condition()) for i in range(4)]
    with ProcessPoolExecutor(4, mp_context=mp.get_context("spawn")) as ex:
        outs = list(ex.map(_c3_oracle, tasks))
    np.testing.assert_array_equal(iters, [o[0] for o in outs])
    states = res.batch.states.cpu().numpy()
    for i in range(4):
        assert rel(states[i], outs[i][1]) <= RTOL, i


def test_c4_full_batch(cuda, golden):
    """M = 1,048,576 config-1 samples in one batch on one B200 (the c4 bench
    workload at one GPU)."""
    import torch

    from paper_2510_26180_b200 import LogNormalKL1D, RngStream, SolverConfig, make_time_grid
    from paper_2510_26180_b200.engine import KleCgcSolver, gauss_hermite_grid
    from paper_2510_26180_b200.models import ParameterMap
    from paper_2510_26180_b200.surrogate import KLGpcSurrogate

    M = 1048576
    g = golden("c1")
    model = LogNormalKL1D(nx=127, d=4, sigma=0.5, ell=0.3)
    grid = make_time_grid(1.0, 16, 32)
    cfg = SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60, seed=2718)
    np.testing.assert_array_equal(g["train_points"], gauss_hermite_grid(4, 3))
    sur = KLGpcSurrogate(g["mean_field"], g["eigenvalues"], g["modes"], g["coeffs"], 2,
                         [ParameterMap("identity", -np.inf, np.inf)] * 4, family="hermite")
    _, eval_rng, _ = RngStream(2718).split(3)
    xi = eval_rng.normal(0.0, 1.0, size=(M, 4))
    np.testing.assert_array_equal(xi[:256], g["xi_all"])
    solver = KleCgcSolver(model, grid, cfg, sur)
    res = solver.solve(xi)
    mean, var = solver.moments(res)
    torch.cuda.synchronize()
    assert torch.all(res.batch.status == 1)
    iters = res.batch.iters.cpu().numpy()
    np.testing.assert_array_equal(iters[:16], g["iters"])   # the reference's own counts (c1 golden)
    pick = np.sort(np.random.default_rng(11).choice(M, size=32, replace=False))
    dia, off = batched.tridiag_from_xi(xi[pick], model.kl_table, model.h)
    U0 = batched.hermite_predict(g["mean_field"], g["eigenvalues"], g["modes"], g["coeffs"], 2, xi[pick])
    out = batched.pcgc(dia, off, model.initial_condition(), U0, 16, 32, 1.0, 1e-3, 1e-8, 60)
    np.testing.assert_array_equal(iters[pick], out["iters"])
    assert rel(res.batch.states[pick].cpu().numpy(), out["states"]) <= RTOL
    # moments: two-pass device reduction vs numpy over the returned fields (float64, 16.6 GB on the host)
    U = res.batch.states.reshape(M, -1)
    want_mean = U.mean(dim=0)   # torch pairwise sums on the device, independent of the kle reduction
    want_var = ((U - want_mean) ** 2).mean(dim=0)
    assert rel(mean.reshape(-1).cpu().numpy(), want_mean.cpu().numpy()) <= 1e-12
    assert rel(var.reshape(-1).cpu().numpy(), want_var.cpu().numpy()) <= 1e-10
