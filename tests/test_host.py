"""CPU tests of the host-side mirror of the reference API and of the C-ABI
library's exports (no device calls)."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2510_26180_b200 import (
    CoarseTrajectory,
    ConfigError,
    LogNormalKL1D,
    ParameterSample,
    RngStream,
    SolverConfig,
    make_time_grid,
)
from paper_2510_26180_b200.models import ParameterMap, get_model
from paper_2510_26180_b200.surrogate import (
    KLGpcSurrogate,
    gpc_basis_count,
    gpc_basis_matrix,
    gpc_multi_indices,
    hermite_norms,
    load_surrogate,
    save_surrogate,
)

ROOT = Path(__file__).resolve().parents[1]


def test_library_loads_and_exports_every_header_symbol():
    from paper_2510_26180_b200 import _lib

    lib = _lib.load()  # loads without a GPU (cudart is lazy)
    assert lib.kle_abi_version() == 1
    header = (ROOT / "include" / "kle_b200.h").read_text()
    declared = set(re.findall(r"\b(kle_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.EXPORTED)


def test_fine_layout_query():
    from paper_2510_26180_b200 import _lib

    lib = _lib.load()
    MR, P, nd = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    for nx in (1, 16, 127, 511, 1000):
        assert lib.kle_fine_layout(nx, ctypes.byref(MR), ctypes.byref(P), ctypes.byref(nd)) == 0
        assert MR.value * P.value >= nx
    assert lib.kle_fine_layout(4095, ctypes.byref(MR), ctypes.byref(P), ctypes.byref(nd)) == 0 and P.value == 256
    assert lib.kle_fine_layout(5000, ctypes.byref(MR), ctypes.byref(P), ctypes.byref(nd)) != 0
    assert b"nx" in lib.kle_last_error()


def test_invalid_arguments_rejected_without_device():
    from paper_2510_26180_b200 import _lib

    lib = _lib.load()
    assert lib.kle_sweep_f64(None, None, None, -1, 1, 10, 1, 1, 0.1, 1.0, None) != 0
    assert lib.kle_pcgc_solve_f64(None, None, None, None, None, None, None, None, 1, 4, 10, 2, 1.0, 1.5, 1.0,
                                  1e-8, 10, None, None, None, None, None, 0, None) != 0
    assert lib.kle_pcgc_workspace_bytes(0, 4, 10) == 0


def test_solver_modules_fail_loudly_without_cuda():
    import torch

    from paper_2510_26180_b200 import DeviceError
    from paper_2510_26180_b200.propagators import propagate_fine

    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    model = LogNormalKL1D(nx=15, d=2)
    grid = make_time_grid(1.0, 4, 4)
    with pytest.raises(DeviceError):
        propagate_fine(model, model.initial_condition(), 0.0, grid.deltaT, grid, ParameterSample(np.zeros(2)),
                       SolverConfig())


def test_config_validation():
    with pytest.raises(ConfigError):
        SolverConfig(alpha=1.0)
    with pytest.raises(ConfigError):
        SolverConfig(tol=0.0)
    with pytest.raises(ConfigError):
        make_time_grid(1.0, 0, 4)
    with pytest.raises(ConfigError):
        make_time_grid(1.0, 4, 1)
    g = make_time_grid(1.0, 16, 32)
    assert g.deltaT == 1 / 16 and g.deltat == 1 / 512
    np.testing.assert_allclose(g.coarse_points(), np.arange(17) / 16)


def test_trajectory_container():
    with pytest.raises(ValueError):
        CoarseTrajectory(np.zeros(3), np.zeros(3))
    with pytest.raises(ValueError):
        CoarseTrajectory(np.zeros(2), np.zeros((4, 3)))
    t = CoarseTrajectory(np.zeros(3), np.ones((4, 3)))
    t.states[0, 0] = np.nan
    with pytest.raises(ValueError):
        t.assert_finite()


def test_rng_stream_matches_numpy_seedsequence():
    a, b, c = RngStream(2718).split(3)
    ref = np.random.default_rng(np.random.SeedSequence(2718).spawn(3)[1])
    np.testing.assert_array_equal(b.normal(0.0, 1.0, size=(5, 4)), ref.normal(0.0, 1.0, size=(5, 4)))
    assert b.counter == 1


def test_model_plugin_contract():
    m = get_model("lognormal-kl-1d", nx=31, d=3)
    assert m.is_linear and m.nx == 31 and m.parameter_dim == 3
    xi = ParameterSample(np.array([0.3, -1.0, 2.0]))
    A, g = m.linear_system(xi)
    assert A.shape == (31, 31)
    Ad = A.toarray()
    np.testing.assert_array_equal(Ad, Ad.T)
    offsum = np.abs(Ad).sum(axis=1) - np.abs(np.diag(Ad))
    assert np.all(np.diag(Ad) >= offsum * (1 - 1e-14)) and np.any(np.diag(Ad) > offsum)  # irreducibly dominant
    np.testing.assert_array_equal(g(0.3), np.ones(31))
    np.testing.assert_allclose(m.rhs(m.initial_condition(), 0.0, xi), -Ad @ m.initial_condition() + 1.0)
    # KL eigenfunctions orthonormal under the midpoint quadrature
    np.testing.assert_allclose(m.kl_functions @ m.kl_functions.T * m.h, np.eye(3), atol=1e-12)
    assert np.all(np.diff(m.kl_eigenvalues) <= 0)
    with pytest.raises(ConfigError):
        get_model("nope")
    with pytest.raises(ValueError):
        m.validate(ParameterSample(np.zeros(2)))


def test_gpc_multi_indices_order_and_counts():
    for (p, d, P) in [(0, 1, 1), (0, 7, 1), (2, 3, 10), (3, 1, 4), (4, 2, 15), (2, 4, 15), (3, 8, 165), (2, 10, 66)]:
        assert gpc_basis_count(p, d) == P
        assert len(gpc_multi_indices(p, d)) == P
    idx = gpc_multi_indices(2, 2)
    assert idx == [(0, 0), (1, 0), (0, 1), (2, 0), (1, 1), (0, 2)]


def test_hermite_basis_orthonormal_under_gaussian_measure():
    nodes, weights = np.polynomial.hermite_e.hermegauss(16)
    B = gpc_basis_matrix(nodes.reshape(-1, 1), 4, family="hermite")
    gram = (B * (weights / np.sqrt(2 * np.pi))[:, None]).T @ B
    np.testing.assert_allclose(gram, np.eye(B.shape[1]), atol=1e-12)
    np.testing.assert_allclose(hermite_norms(3), [1, 1, 1 / np.sqrt(2), 1 / np.sqrt(6)])


def test_host_basis_matches_oracle_bitwise():
    from oracle import ref_port

    x = np.random.default_rng(0).normal(size=(50, 4))
    np.testing.assert_array_equal(gpc_basis_matrix(x, 2, "hermite"), ref_port.basis_matrix(x, 2))


def test_surrogate_npz_round_trip(tmp_path):
    rng = np.random.default_rng(1)
    s = KLGpcSurrogate(rng.normal(size=(3, 4)), rng.uniform(size=2), rng.normal(size=(2, 3, 4)),
                       rng.normal(size=(2, 6)), 2, [ParameterMap("identity", -np.inf, np.inf)] * 2,
                       provenance={"model": "x"}, family="hermite")
    path = tmp_path / "s.npz"
    save_surrogate(s, path)
    t = load_surrogate(path)
    for f in ("mean_field", "eigenvalues", "modes", "coeffs"):
        np.testing.assert_array_equal(getattr(s, f), getattr(t, f))
    assert [m.to_dict() for m in t.maps] == [m.to_dict() for m in s.maps]
    assert t.provenance == s.provenance and t.family == "hermite"


def test_host_kl_build_matches_golden(golden):
    from paper_2510_26180_b200.surrogate import gpc_fit, kl_build, kl_coefficients, make_snapshot_set

    g = golden("c1")
    model = LogNormalKL1D(nx=127, d=4)
    w = model.cell_volume * (1.0 / 16)
    snap = make_snapshot_set(list(range(81)), g["snapshots"], w)
    basis = kl_build(snap, 1e-10)
    assert basis.m_q == g["modes"].shape[0]
    np.testing.assert_allclose(basis.retained, g["eigenvalues"], rtol=1e-12)
    zeta = kl_coefficients(snap, basis)
    coeffs, _, deg = gpc_fit(g["train_points"], zeta, 2, "hermite")
    assert deg == 2
    np.testing.assert_allclose(coeffs, g["coeffs"], atol=1e-9 * np.abs(g["coeffs"]).max())


def test_model_2d_contract():
    from paper_2510_26180_b200.models import LogNormalKL2D

    m = get_model("lognormal-kl-2d", n=9, d=6)
    assert isinstance(m, LogNormalKL2D) and m.nx == 81 and m.parameter_dim == 6
    xi = ParameterSample(np.linspace(-1, 1, 6))
    A, g = m.linear_system(xi)
    Ad = A.toarray()
    np.testing.assert_array_equal(Ad, Ad.T)
    assert np.all(np.linalg.eigvalsh(Ad) > 0)
    coo = A.tocoo()
    assert set(np.unique(np.abs(coo.row - coo.col))) <= {0, 1, 9}
    dia, ex, ey = m.stencil(xi)
    assert np.all(ex.reshape(9, 9)[:, -1] == 0) and np.all(ey.reshape(9, 9)[-1] == 0)
    np.testing.assert_allclose(m.kl_table @ m.kl_table.T * m.h ** 2, np.diag(m.kl_eigenvalues), atol=1e-12)
    assert np.all(np.diff(m.kl_eigenvalues) <= 0)
    u0 = m.initial_condition()
    assert u0.shape == (81,) and abs(u0.max() - np.sin(np.pi * 0.5) ** 2) < 1e-12


def test_legendre_host_tables_match_reference_build(golden):
    """The reference's own build_surrogate output (Legendre family; affine and
    cos2pi maps), read through load_surrogate (its save_surrogate wire
    format): the host Legendre table + ParameterMap.apply reproduce its
    surrogate_predict."""
    from paper_2510_26180_b200 import ParameterSample
    from paper_2510_26180_b200.surrogate import gpc_eval_basis, load_surrogate

    root = Path(__file__).resolve().parent / "golden"
    for tag in ("d1", "ad"):
        s = load_surrogate(root / f"legendre_{tag}.npz")
        p = golden(f"legendre_{tag}_pred")
        for x, want in zip(p["xi"], p["pred"]):
            psi = gpc_eval_basis(s.map_parameters(ParameterSample(x, id=0)), s.degree, s.family)
            w = np.sqrt(s.eigenvalues) * (s.coeffs @ psi)
            pred = s.mean_field + (w @ s.modes.reshape(s.m_q, -1)).reshape(s.mean_field.shape)
            np.testing.assert_array_equal(pred, want)


def test_constant_source_and_shared_initial_condition():
    """The device path takes g(t) = g0 and one u0 per batch: a source that is
    only constant at t = 0 and t = 1, or a parameter-dependent initial state,
    must raise instead of being silently replaced."""
    from paper_2510_26180_b200 import ParameterSample
    from paper_2510_26180_b200.device import constant_source, shared_initial_condition

    w = np.ones(5)
    assert constant_source(lambda t: 2.5 * w) == 2.5
    with pytest.raises(NotImplementedError):
        constant_source(lambda t: t * (1.0 - t) * w)
    with pytest.raises(NotImplementedError):
        constant_source(lambda t: np.arange(5.0))

    class M:
        def initial_condition(self, xi):
            return np.full(3, xi.values[0] if xi is not None else 0.0)

    xs = [ParameterSample(np.array([1.0]), id=0), ParameterSample(np.array([1.0]), id=1)]
    np.testing.assert_array_equal(shared_initial_condition(M(), xs), np.ones(3))
    with pytest.raises(NotImplementedError):
        shared_initial_condition(M(), xs + [ParameterSample(np.array([2.0]), id=2)])
