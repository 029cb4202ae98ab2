"""Config-2 parity at the full BASELINE size (M = 65,536 samples, nx = 511,
N = 64, J = 64) through size-independent properties, plus a seeded subset
against the batched CPU oracle:

- every sample converges, with the iteration counts of the oracle on a
  seeded subset of 12 samples and fields within 1e-10 relative;
- per-sample arithmetic does not depend on the batch: a permuted batch gives
  the permuted results bit for bit, and so does the batch split into two
  sample pipelines (KLE_PCGC_PIPES) or solved as two halves;
- the converged iterate is a fixed point of one more correction up to tol;
- the moments equal numpy's two-pass mean / variance of the returned fields.

The surrogate is the config's own: a degree-3 Hermite fit on 2,048 seeded
training samples, built on the device (compared with the reference's build
in test_gpu_surrogate.py).
"""
import numpy as np
import pytest

from oracle import batched

pytestmark = pytest.mark.gpu

M = 65536


@pytest.fixture(scope="module")
def c2_run(cuda):
    import torch
    from paper_2510_26180_b200 import LogNormalKL1D, ParameterSample, RngStream, SolverConfig, make_time_grid
    from paper_2510_26180_b200.engine import KleCgcSolver
    from paper_2510_26180_b200.surrogate import build_surrogate

    model = LogNormalKL1D(nx=511, d=8, sigma=0.5, ell=0.3)
    grid = make_time_grid(1.0, 64, 64)
    cfg = SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60, seed=2718)
    train_rng, eval_rng, _ = RngStream(2718).split(3)
    train = [ParameterSample(p, id=i) for i, p in enumerate(train_rng.normal(0.0, 1.0, size=(2048, 8)))]
    sur = build_surrogate(model, grid, cfg, train, eps_kl=1e-10, degree=3)
    xi = eval_rng.normal(0.0, 1.0, size=(M, 8))
    solver = KleCgcSolver(model, grid, cfg, sur)
    res = solver.solve(xi, keep_initial=True)
    torch.cuda.synchronize()
    return dict(model=model, grid=grid, cfg=cfg, sur=sur, xi=xi, solver=solver, res=res)


def test_full_c2_all_converged_and_oracle_subset(c2_run):
    res, model, xi = c2_run["res"], c2_run["model"], c2_run["xi"]
    st = res.batch.status.cpu().numpy()
    assert np.all(st == 1)
    iters = res.batch.iters.cpu().numpy()
    assert 5 <= iters.min() and iters.max() <= 20
    pick = np.random.default_rng(7).choice(M, size=12, replace=False)
    dia, off = batched.tridiag_from_xi(xi[pick], model.kl_table, model.h)
    U0 = res.U0[pick].cpu().numpy()
    out = batched.pcgc(dia, off, model.initial_condition(), U0, 64, 64, 1.0, 1e-3, 1e-8, 60)
    np.testing.assert_array_equal(iters[pick], out["iters"])
    got = res.batch.states[pick].cpu().numpy()
    assert np.max(np.abs(got - out["states"])) / np.max(np.abs(out["states"])) <= 1e-10


def test_full_c2_permutation_and_split_invariance(c2_run, monkeypatch):
    import torch

    res, xi, solver = c2_run["res"], c2_run["xi"], c2_run["solver"]
    perm = np.random.default_rng(3).permutation(M)
    monkeypatch.setenv("KLE_PCGC_PIPES", "1")  # one pipeline for the permuted batch
    r2 = solver.solve(xi[perm])
    np.testing.assert_array_equal(r2.batch.iters.cpu().numpy(), res.batch.iters.cpu().numpy()[perm])
    assert torch.equal(r2.batch.states, res.batch.states[torch.as_tensor(perm, device="cuda")])
    del r2
    h = M // 2 + 17  # two ragged halves
    a, b = solver.solve(xi[:h]), solver.solve(xi[h:])
    assert torch.equal(a.batch.states, res.batch.states[:h])
    assert torch.equal(b.batch.states, res.batch.states[h:])


def test_full_c2_fixed_point(c2_run):
    """One more correction from the converged iterate moves it by at most
    tol-scale amounts (the CGC fixed point, pintuq/pcgc.py:345-348)."""
    from paper_2510_26180_b200 import SolverConfig
    from paper_2510_26180_b200.device import DeviceOperator
    from paper_2510_26180_b200.pcgc import pcgc_solve_device

    run = c2_run
    xi = run["xi"][:4096]
    op = DeviceOperator.from_model(run["model"], xi)
    U = run["res"].batch.states[:4096].clone()
    cfg1 = SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=1)
    r = pcgc_solve_device(op, U, run["grid"], cfg1)
    inc = r.increments[:, 0].cpu().numpy()
    # the stop increment was <= tol, and the iteration contracts (rho ~ 0.25)
    assert np.all(inc <= 1e-8)


def test_full_c2_moments(c2_run):
    res, solver = c2_run["res"], c2_run["solver"]
    mean, var = solver.moments(res)
    host = res.batch.states.cpu().numpy()
    m_ref = host.mean(axis=0)
    v_ref = host.var(axis=0)
    assert np.max(np.abs(mean.cpu().numpy() - m_ref)) / np.max(np.abs(m_ref)) <= 1e-12
    assert np.max(np.abs(var.cpu().numpy() - v_ref)) / np.max(np.abs(v_ref)) <= 1e-10
