"""stop_on="reference" on the device: the batched
serial fine reference, the per-record error vectors of _error_record
(pintuq/parareal.py:87-91) and the reference-stopping PCGC loop of the
harness composition (pintuq/experiments.py:212-235), against the goldens of
the unmodified reference (tests/golden/ref.npz).

Tolerances: iteration counts and iters_to_tol exact; fields 1e-10 relative;
the error records and increments are differences of O(1) fields, so they
are compared with an absolute 1e-11 (0.1% of tol; measured <= 1.0e-12).
"""
import numpy as np
import pytest

from tests.conftest import c1_config

pytestmark = pytest.mark.gpu
ATOL = 1e-11  # 0.1% of tol; the records are O(1)-field differences (measured up to 1.0e-12)


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - b)) / np.max(np.abs(b)))


def _check(res, g, tag, ref_dev=None):
    iters = res.iters.cpu().numpy()
    np.testing.assert_array_equal(iters, g[f"{tag}_iters"])
    np.testing.assert_array_equal(res.status.cpu().numpy(), np.ones_like(iters))
    assert rel(res.states.cpu().numpy(), g[f"{tag}_final"]) <= 1e-10
    err = res.err_vs_ref.cpu().numpy()
    for i, K in enumerate(iters + 1):
        np.testing.assert_allclose(err[i, :K], g[f"{tag}_err"][i, :K], rtol=0, atol=ATOL)
        assert np.all(np.isnan(err[i, K:]))
        inc = res.increments.cpu().numpy()[i, : K - 1]
        np.testing.assert_allclose(inc, g[f"{tag}_incs"][i, 1:K], rtol=0, atol=ATOL)
    np.testing.assert_allclose(res.max_err.cpu().numpy(), [g[f"{tag}_max_err"][i, K - 1] for i, K in
                                                           enumerate(iters + 1)], rtol=0, atol=ATOL)
    return iters


@pytest.mark.parametrize("tag", ["kle", "rnd", "inc"])
def test_pcgc_with_reference_1d(cuda, golden, tag):
    import torch
    from paper_2510_26180_b200.device import DeviceOperator
    from paper_2510_26180_b200.pcgc import pcgc_solve_device
    from paper_2510_26180_b200.propagators import fine_reference_batched

    model, grid, cfg = c1_config()
    g1, g = golden("c1"), golden("ref")
    M = len(g[f"{tag}_iters"])
    op = DeviceOperator.from_model(model, g1["xi_all"][:M])
    ref = fine_reference_batched(op, grid)
    assert rel(ref.cpu().numpy(), g[f"{tag}_ref"]) <= 1e-12
    init = g["rnd_init"] if tag == "rnd" else g1["U0"][:M]
    U = torch.as_tensor(np.ascontiguousarray(init), device="cuda").clone()
    res = pcgc_solve_device(op, U, grid, cfg, reference=ref, stop_on="increment" if tag == "inc" else "reference")
    iters = _check(res, g, tag)
    if tag != "inc":  # stop_on="reference": the stop record is the first one at or below tol
        np.testing.assert_array_equal(res.iters_to_tol(cfg.tol).cpu().numpy(), g[f"{tag}_to_tol"])
        np.testing.assert_array_equal(iters, g[f"{tag}_to_tol"])


def test_pcgc_with_reference_two_pipelines(cuda, golden, monkeypatch):
    """The same run with the batch split over two sample pipelines."""
    import torch
    from paper_2510_26180_b200.device import DeviceOperator
    from paper_2510_26180_b200.pcgc import pcgc_solve_device
    from paper_2510_26180_b200.propagators import fine_reference_batched

    monkeypatch.setenv("KLE_PCGC_PIPES", "2")
    model, grid, cfg = c1_config()
    g1, g = golden("c1"), golden("ref")
    op = DeviceOperator.from_model(model, g1["xi_all"][:8])
    U = torch.as_tensor(np.ascontiguousarray(g1["U0"][:8]), device="cuda").clone()
    res = pcgc_solve_device(op, U, grid, cfg, reference=fine_reference_batched(op, grid), stop_on="reference")
    _check(res, g, "kle")


def test_reference_stop_at_k0(cuda, golden):
    """An initial guess equal to the reference stops at k = 0
    (pintuq/pcgc.py:312-316): no correction, iters 0, zero error record."""
    from paper_2510_26180_b200.device import DeviceOperator
    from paper_2510_26180_b200.pcgc import pcgc_solve_device
    from paper_2510_26180_b200.propagators import fine_reference_batched

    model, grid, cfg = c1_config()
    g1 = golden("c1")
    op = DeviceOperator.from_model(model, g1["xi_all"][:4])
    ref = fine_reference_batched(op, grid)
    U = ref.clone()
    U[2:] += 1e-3  # samples 2, 3 must iterate
    res = pcgc_solve_device(op, U, grid, cfg, reference=ref, stop_on="reference")
    iters = res.iters.cpu().numpy()
    assert iters[0] == 0 and iters[1] == 0 and iters[2] > 0 and iters[3] > 0
    assert np.all(res.status.cpu().numpy() == 1)
    err = res.err_vs_ref.cpu().numpy()
    assert np.all(err[:2, 0] == 0.0) and np.all(np.isnan(err[:2, 1:]))
    assert np.array_equal(res.states[:2].cpu().numpy(), ref[:2].cpu().numpy())


def test_pcgc_with_reference_2d(cuda, golden):
    import torch
    from paper_2510_26180_b200.models import LogNormalKL2D
    from paper_2510_26180_b200 import SolverConfig, make_time_grid
    from paper_2510_26180_b200.pcgc import pcgc_solve_device
    from paper_2510_26180_b200.propagators import fine_reference_batched
    from paper_2510_26180_b200.twod import DeviceOperator2D

    g3, g = golden("c3s"), golden("ref")
    m = LogNormalKL2D(n=15, d=10)
    grid = make_time_grid(1.0, 8, 4)
    cfg = SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60)
    op = DeviceOperator2D.from_model(m, g3["xi"])
    ref = fine_reference_batched(op, grid)
    assert rel(ref.cpu().numpy(), g["c3s_ref"]) <= 1e-12
    U = torch.as_tensor(np.ascontiguousarray(g3["coarse_sweep"]), device="cuda").clone()
    res = pcgc_solve_device(op, U, grid, cfg, reference=ref, stop_on="reference")
    _check(res, g, "c3s")


def test_kle_cgc_engine_harness_mode(cuda, golden):
    """KleCgcSolver.solve(stop_on="reference"): xi -> U0 -> fine reference ->
    reference-stopped PCGC, the harness's kle-pcgc solve for 8 samples."""
    from paper_2510_26180_b200.engine import KleCgcSolver
    from paper_2510_26180_b200.models import ParameterMap
    from paper_2510_26180_b200.surrogate import KLGpcSurrogate

    model, grid, cfg = c1_config()
    g1, g = golden("c1"), golden("ref")
    s = KLGpcSurrogate(g1["mean_field"], g1["eigenvalues"], g1["modes"], g1["coeffs"], int(g1["degree"]),
                       [ParameterMap("identity", -np.inf, np.inf)] * 4, family="hermite")
    res = KleCgcSolver(model, grid, cfg, s).solve(g1["xi_all"][:8], stop_on="reference")
    _check(res.batch, g, "kle")


def harness_aggregate(err_rows, iters_to_tol, max_iters):
    """pintuq/experiments.py:314-334 verbatim in numpy over per-sample error
    vectors (each (K_s+1, N), finite): pad with the last record, mean over
    samples, row max; mean of iters_to_tol with None -> max_iters."""
    k_max = max(ev.shape[0] for ev in err_rows)
    stack = np.empty((len(err_rows), k_max, err_rows[0].shape[1]))
    for i, ev in enumerate(err_rows):
        stack[i] = np.vstack([ev, np.repeat(ev[-1:], k_max - ev.shape[0], axis=0)])
    mv = stack.mean(axis=0)
    its = [max_iters if t < 0 else t for t in iters_to_tol]
    return mv, mv.max(axis=1), float(np.mean(its))


@pytest.mark.parametrize("tag", ["kle", "rnd"])
def test_mean_error_aggregation(cuda, golden, tag):
    """BatchResult.error_summary (device padding + sample mean) equals the
    harness aggregation of the same records bit for bit, and the reference's
    own aggregation of its golden records within the record tolerance."""
    import torch
    from paper_2510_26180_b200.device import DeviceOperator
    from paper_2510_26180_b200.pcgc import pcgc_solve_device
    from paper_2510_26180_b200.propagators import fine_reference_batched

    model, grid, cfg = c1_config()
    g1, g = golden("c1"), golden("ref")
    M = len(g[f"{tag}_iters"])
    op = DeviceOperator.from_model(model, g1["xi_all"][:M])
    ref = fine_reference_batched(op, grid)
    init = g["rnd_init"] if tag == "rnd" else g1["U0"][:M]
    U = torch.as_tensor(np.ascontiguousarray(init), device="cuda").clone()
    res = pcgc_solve_device(op, U, grid, cfg, reference=ref, stop_on="reference")
    mv, mme, mit = res.error_summary(cfg.tol, cfg.max_outer_iters)
    iters = res.iters.cpu().numpy()
    err = res.err_vs_ref.cpu().numpy()
    own = harness_aggregate([err[i, :K + 1] for i, K in enumerate(iters)],
                            res.iters_to_tol(cfg.tol).cpu().numpy(), cfg.max_outer_iters)
    np.testing.assert_array_equal(mv, own[0])
    np.testing.assert_array_equal(mme, own[1])
    assert mit == own[2]
    gold = harness_aggregate([g[f"{tag}_err"][i, :K + 1] for i, K in enumerate(g[f"{tag}_iters"])],
                             g[f"{tag}_to_tol"], cfg.max_outer_iters)
    np.testing.assert_allclose(mv, gold[0], rtol=0, atol=ATOL)
    np.testing.assert_allclose(mme, gold[1], rtol=0, atol=ATOL)
    assert mit == gold[2]
    assert mv.shape[0] == int(g[f"{tag}_iters"].max()) + 1
