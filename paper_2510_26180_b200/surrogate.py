"""KL + Hermite-gPC surrogate — drop-in for ``pintuq.surrogate``
(``/root/reference/pkg/src/pintuq/surrogate.py``).

Online evaluation (the hot path, ``surrogate_predict`` :321-333) runs on the
device: the Hermite basis kernel builds Psi(xi) (``gpc_basis_matrix`` +
``_hermite_table`` :222-248, same recurrence/normalisation/product order)
and one FP64 tensor-core GEMM forms ``U0 = mean + Psi C`` with the
precontracted ``C = H^T diag(sqrt(lam)) G`` (inner dimension P), or
``U0 = mean + (Psi H^T diag(sqrt lam)) G`` when m_q < P (inner dimension m_q).

The offline build (``build_surrogate`` :336-393): the snapshot library is
produced by the batched device PCGC solver (``collect_snapshots`` :67-117);
with the snapshots on the device, the snapshot-method KL runs its three
large products there (``kl_build_device``: the Gram matrix X X^T :153 and
the modes E^T X :167 as DMMA GEMMs, the coefficients X G^T :183), leaving
the n_t x n_t ``eigh`` and the least-squares fit (:264-288) — small dense
LAPACK problems — on the host, exactly as the reference solves them.
"""
from __future__ import annotations

import json
import math
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .core import CoarseTrajectory, ParameterSample, RankDeficientError, SnapshotError, SolverConfig, TimeGrid
from .models import ParameterMap

_ZERO_VARIANCE_REL = 1e-26
_EIGENVALUE_FLOOR_REL = 1e-14


# ---------------------------------------------------------------------------
# polynomial chaos basis (host tables; pintuq/surrogate.py:187-261)
# ---------------------------------------------------------------------------
def gpc_basis_count(degree: int, dim: int) -> int:
    if degree < 0 or dim < 1:
        raise ValueError("degree must be >= 0 and dimension >= 1")
    return math.comb(degree + dim, dim)


def gpc_multi_indices(degree: int, dim: int) -> list:
    """Total degree <= p, graded; within a degree the first coordinate runs
    from high to low (the reference's order, :194-205)."""
    def compositions(total, slots):
        if slots == 1:
            yield (total,)
            return
        for v in range(total, -1, -1):
            for rest in compositions(total - v, slots - 1):
                yield (v,) + rest

    return [k for total in range(degree + 1) for k in compositions(total, dim)]


def _hermite_table(x, degree: int) -> np.ndarray:
    x = np.asarray(x, dtype=float)
    T = np.empty((degree + 1,) + x.shape)
    T[0] = 1.0
    if degree >= 1:
        T[1] = x
    for k in range(1, degree):
        T[k + 1] = x * T[k] - k * T[k - 1]
    return T * hermite_norms(degree).reshape((-1,) + (1,) * x.ndim)


def _legendre_table(x, degree: int) -> np.ndarray:
    x = np.asarray(x, dtype=float)
    T = np.empty((degree + 1,) + x.shape)
    T[0] = 1.0
    if degree >= 1:
        T[1] = x
    for k in range(1, degree):
        T[k + 1] = ((2 * k + 1) * x * T[k] - k * T[k - 1]) / (k + 1)
    return T * np.sqrt(2.0 * np.arange(degree + 1) + 1.0).reshape((-1,) + (1,) * x.ndim)


def hermite_norms(degree: int) -> np.ndarray:
    return np.array([1.0 / math.sqrt(math.factorial(k)) for k in range(degree + 1)])


def gpc_basis_matrix(points, degree: int, family: str = "legendre") -> np.ndarray:
    """Host basis matrix (n, P) — used by the offline fit only."""
    points = np.atleast_2d(np.asarray(points, dtype=float))
    n, dim = points.shape
    table = {"legendre": _legendre_table, "hermite": _hermite_table}[family]
    tabs = [table(points[:, d], degree) for d in range(dim)]
    B = np.ones((n, gpc_basis_count(degree, dim)))
    for col, k in enumerate(gpc_multi_indices(degree, dim)):
        for d, kd in enumerate(k):
            if kd:
                B[:, col] *= tabs[d][kd]
    return B


def gpc_eval_basis(xi_mapped, degree: int, family: str = "legendre") -> np.ndarray:
    """All total-order basis functions at one mapped point, length P
    (``pintuq/surrogate.py:251-253``; host table, the batched evaluation of
    the hot path is ``DeviceSurrogate.basis``)."""
    return gpc_basis_matrix(np.atleast_2d(xi_mapped), degree, family)[0]


def default_degree(n_train: int, dim: int, cap: int = 6) -> int:
    p = 0
    while p < cap and gpc_basis_count(p + 1, dim) <= max(1, n_train // 2):
        p += 1
    return p


# ---------------------------------------------------------------------------
# snapshots + KL (pintuq/surrogate.py:39-184)
# ---------------------------------------------------------------------------
@dataclass
class SnapshotSet:
    samples: list
    fields: np.ndarray
    mean_field: np.ndarray
    fluctuations: np.ndarray
    cell_weight: float
    device_fields: object = None  # (n_t, N, nx) device tensor when collected on the device

    @property
    def n_train(self) -> int:
        return self.fields.shape[0]

    def inner(self, a, b) -> float:
        return self.cell_weight * float(np.sum(a * b))


def make_snapshot_set(samples, fields, cell_weight: float) -> SnapshotSet:
    fields = np.asarray(fields, dtype=float)
    if fields.ndim != 3:
        raise ValueError("snapshot fields must have shape (n_t, N, N_x)")
    mean = fields.mean(axis=0)
    return SnapshotSet(list(samples), fields, mean, fields - mean, float(cell_weight))


def collect_snapshots(model, grid: TimeGrid, cfg: SolverConfig, training: list, method: str = "pcgc",
                      executor=None) -> SnapshotSet:
    """Snapshot library by the batched device solver: coarse-sweep initial
    guess + PCGC to ``cfg.tol`` (``method='pcgc'``) or the serial fine
    reference (``method='fine'``)."""
    from .device import DeviceOperator
    from .pcgc import SAMPLE_CONVERGED, pcgc_solve_device
    from .propagators import coarse_sweep_init_batched, fine_reference_batched

    if not training:
        raise ValueError("training set must not be empty")
    if method not in ("pcgc", "fine"):
        raise ValueError(f"unknown snapshot method {method!r}")
    op = DeviceOperator.from_model(model, training)
    if method == "fine":
        fields = fine_reference_batched(op, grid)
    else:
        U = coarse_sweep_init_batched(op, grid).contiguous()
        res = pcgc_solve_device(op, U, grid, cfg)
        st = res.status.cpu().numpy()
        bad = np.nonzero(st != SAMPLE_CONVERGED)[0]
        if bad.size:
            raise SnapshotError(
                f"snapshot solves failed for samples {[training[i].id for i in bad]}",
                {training[i].id: RuntimeError(f"status {int(st[i])}") for i in bad},
            )
        fields = res.states
    snap = make_snapshot_set(training, fields.cpu().numpy(), model.cell_volume * grid.deltaT)
    snap.device_fields = fields
    return snap


@dataclass
class KLBasis:
    eigenvalues: np.ndarray
    modes: np.ndarray
    m_q: int
    cell_weight: float
    energy_ratio: float

    @property
    def retained(self) -> np.ndarray:
        return self.eigenvalues[: self.m_q]

    def discarded_energy(self) -> float:
        total = float(np.sum(self.eigenvalues))
        return float(np.sum(self.eigenvalues[self.m_q:])) if total > 0 else 0.0


def kl_build(snap: SnapshotSet, eps_kl: float) -> KLBasis:
    if not 0.0 < eps_kl < 1.0:
        raise ValueError(f"eps_kl must lie in (0, 1), got {eps_kl}")
    n_t = snap.n_train
    X = snap.fluctuations.reshape(n_t, -1)
    lam, E = np.linalg.eigh((snap.cell_weight / n_t) * (X @ X.T))
    lam = np.clip(lam[::-1], 0.0, None)
    E = E[:, ::-1]
    total = float(np.sum(lam))
    mean_energy = snap.cell_weight * float(np.sum(snap.mean_field ** 2))
    if total <= _ZERO_VARIANCE_REL * max(mean_energy, 1.0):
        return KLBasis(lam, np.empty((0,) + snap.fields.shape[1:]), 0, snap.cell_weight, 1.0)
    ratios = np.cumsum(lam) / total
    m_q = min(int(np.searchsorted(ratios, 1.0 - eps_kl) + 1), int(np.sum(lam > _EIGENVALUE_FLOOR_REL * lam[0])))
    modes = ((1.0 / np.sqrt(lam[:m_q] * n_t))[:, None] * (E[:, :m_q].T @ X)).reshape((m_q,) + snap.fields.shape[1:])
    return KLBasis(lam, modes, m_q, snap.cell_weight, float(ratios[m_q - 1]))


def _gemm(A, B, trans_b=False, bias=None):
    from .device import empty, ptr, stream_ptr

    M, K = A.shape
    L = B.shape[0] if trans_b else B.shape[1]
    C = empty(M, L)
    _lib.call("kle_gemm_f64", ptr(A.contiguous()), ptr(B.contiguous()), ptr(bias), ptr(C), M, K, L, int(trans_b),
              stream_ptr())
    return C


def kl_build_device(snap: SnapshotSet, eps_kl: float):
    """``kl_build`` + ``kl_coefficients`` (pintuq/surrogate.py:144-184) with
    the snapshot products on the device. Returns (KLBasis, zeta). The
    eigendecomposition of the n_t x n_t covariance is the reference's own
    host ``eigh``; mode selection is identical."""
    from .device import empty, ptr, stream_ptr, to_dev
    from .moments import device_col_sum, device_scale

    if not 0.0 < eps_kl < 1.0:
        raise ValueError(f"eps_kl must lie in (0, 1), got {eps_kl}")
    F = snap.device_fields
    n_t = snap.n_train
    F2 = F.reshape(n_t, -1)
    L = F2.shape[1]
    mean = device_scale(device_col_sum(F2), 1.0 / n_t)
    X = empty(n_t, L)
    _lib.call("kle_sub_row_f64", ptr(F2.contiguous()), ptr(mean), ptr(X), n_t, L, stream_ptr())
    gram = _gemm(X, X, trans_b=True).cpu().numpy()
    lam, E = np.linalg.eigh((snap.cell_weight / n_t) * gram)
    lam = np.clip(lam[::-1], 0.0, None)
    E = E[:, ::-1]
    total = float(np.sum(lam))
    mean_energy = snap.cell_weight * float(np.sum(snap.mean_field ** 2))
    if total <= _ZERO_VARIANCE_REL * max(mean_energy, 1.0):
        return KLBasis(lam, np.empty((0,) + snap.fields.shape[1:]), 0, snap.cell_weight, 1.0), np.empty((n_t, 0))
    ratios = np.cumsum(lam) / total
    m_q = min(int(np.searchsorted(ratios, 1.0 - eps_kl) + 1), int(np.sum(lam > _EIGENVALUE_FLOOR_REL * lam[0])))
    scale = 1.0 / np.sqrt(lam[:m_q] * n_t)
    G = _gemm(to_dev(np.ascontiguousarray(scale[:, None] * E[:, :m_q].T)), X)  # (m_q, L) modes
    zeta = snap.cell_weight * _gemm(X, G, trans_b=True).cpu().numpy() / np.sqrt(lam[:m_q])[None, :]
    modes = G.cpu().numpy().reshape((m_q,) + snap.fields.shape[1:])
    return KLBasis(lam, modes, m_q, snap.cell_weight, float(ratios[m_q - 1])), zeta


def kl_coefficients(snap: SnapshotSet, basis: KLBasis) -> np.ndarray:
    if basis.m_q == 0:
        return np.empty((snap.n_train, 0))
    X = snap.fluctuations.reshape(snap.n_train, -1)
    G = basis.modes.reshape(basis.m_q, -1)
    return snap.cell_weight * (X @ G.T) / np.sqrt(basis.retained)[None, :]


def gpc_fit(points, zeta, degree: int, family: str = "legendre"):
    points = np.atleast_2d(np.asarray(points, dtype=float))
    zeta = np.asarray(zeta, dtype=float)
    n, dim = points.shape
    while degree > 0 and gpc_basis_count(degree, dim) > n:
        degree -= 1
    if gpc_basis_count(degree, dim) > n:
        warnings.warn("fewer samples than basis functions even at degree 0")
    B = gpc_basis_matrix(points, degree, family)
    coeffs, _, rank, _ = np.linalg.lstsq(B, zeta, rcond=None)
    if rank < B.shape[1]:
        raise RankDeficientError(f"regression matrix rank {rank} < basis size {B.shape[1]}")
    resid = B @ coeffs - zeta
    residuals = np.sqrt(np.mean(resid ** 2, axis=0)) if zeta.size else np.zeros(0)
    return coeffs.T, residuals, degree


# ---------------------------------------------------------------------------
# surrogate object + device evaluation
# ---------------------------------------------------------------------------
@dataclass
class KLGpcSurrogate:
    mean_field: np.ndarray
    eigenvalues: np.ndarray
    modes: np.ndarray
    coeffs: np.ndarray
    degree: int
    maps: list
    family: str = "legendre"
    cell_weight: float = 1.0
    provenance: dict = field(default_factory=dict)
    ls_residuals: np.ndarray | None = None
    training_errors: np.ndarray | None = None

    @property
    def m_q(self) -> int:
        return self.modes.shape[0]

    def map_parameters(self, xi: ParameterSample) -> np.ndarray:
        if xi.dim != len(self.maps):
            raise ValueError(f"sample has {xi.dim} coordinates, surrogate expects {len(self.maps)}")
        return np.array([m.apply(v) for m, v in zip(self.maps, xi.values)])


_FAMILY_CODE = {"hermite": 0, "legendre": 1}
_MAP_CODE = {"identity": 0, "affine": 1, "cos2pi": 2}


def family_norms(family: str, degree: int) -> np.ndarray:
    if family == "hermite":
        return hermite_norms(degree)
    return np.sqrt(2.0 * np.arange(degree + 1) + 1.0)


class DeviceSurrogate:
    """Device-resident evaluation tables of a ``KLGpcSurrogate`` (Hermite or
    Legendre family; identity, affine or cos2pi parameter maps applied in the
    basis kernel)."""

    def __init__(self, s: KLGpcSurrogate):
        from .core import ConfigError
        from .device import to_dev, torch

        if s.family not in _FAMILY_CODE:
            raise ConfigError(f"unknown gPC family {s.family!r}")
        if any(m.kind not in _MAP_CODE for m in s.maps):
            raise ConfigError(f"unknown parameter map kind in {[m.kind for m in s.maps]}")
        self.s = s
        self.family = _FAMILY_CODE[s.family]
        self.maps = (None if all(m.kind == "identity" for m in s.maps) else
                     to_dev(np.array([[_MAP_CODE[m.kind], m.lo, m.hi] for m in s.maps], dtype=float)))
        self.dim = len(s.maps)
        self.field_shape = s.mean_field.shape
        self.L = int(np.prod(self.field_shape))
        self.P = gpc_basis_count(s.degree, self.dim)
        self.mean = to_dev(s.mean_field.reshape(-1))
        self.midx = torch.as_tensor(np.array(gpc_multi_indices(s.degree, self.dim), dtype=np.int32),
                                    device="cuda").contiguous()
        self.norms = to_dev(family_norms(s.family, s.degree))
        m_q = s.m_q
        G = s.modes.reshape(m_q, -1)
        sq = np.sqrt(s.eigenvalues)
        if m_q == 0:
            self.mode = "mean"
        elif self.P <= m_q:
            self.mode = "direct"  # K_g = P
            self.C = to_dev(s.coeffs.T @ (sq[:, None] * G))
        else:
            self.mode = "factored"  # K_g = m_q
            self.HT = to_dev(s.coeffs.T * sq[None, :])  # (P, m_q)
            self.G = to_dev(G)

    @property
    def inner_dim(self) -> int:
        return {"mean": 0, "direct": self.P, "factored": self.s.m_q}[self.mode]

    def basis(self, xi_d):
        from .device import empty, ptr, stream_ptr

        M = xi_d.shape[0]
        Psi = empty(M, self.P)
        _lib.call("kle_gpc_basis_f64", ptr(xi_d), M, self.dim, self.s.degree, self.family, ptr(self.maps),
                  ptr(self.midx), self.P,
                  ptr(self.norms), ptr(Psi), stream_ptr())
        return Psi

    def predict(self, xi_d, out=None):
        """xi_d: (M, d) device tensor -> U0 (M, N, nx) device tensor."""
        from .device import empty, ptr, stream_ptr

        M = xi_d.shape[0]
        U0 = out if out is not None else empty(M, *self.field_shape)
        if self.mode == "mean":
            U0.copy_(self.mean.view(1, *self.field_shape).expand_as(U0))
            return U0
        Psi = self.basis(xi_d)
        if self.mode == "direct":
            _lib.call("kle_gpc_eval_f64", ptr(Psi), M, self.P, ptr(self.C), ptr(self.mean), self.L, ptr(U0),
                      stream_ptr())
        else:
            W = empty(M, self.s.m_q)
            _lib.call("kle_gpc_eval_f64", ptr(Psi), M, self.P, ptr(self.HT), None, self.s.m_q, ptr(W),
                      stream_ptr())
            _lib.call("kle_gpc_eval_f64", ptr(W), M, self.s.m_q, ptr(self.G), ptr(self.mean), self.L, ptr(U0),
                      stream_ptr())
        return U0


def surrogate_predict(s: KLGpcSurrogate, xi: ParameterSample, initial) -> CoarseTrajectory:
    """``pintuq/surrogate.py:321-333`` for one sample (device evaluation)."""
    from .device import to_dev

    if xi.dim != len(s.maps):
        raise ValueError(f"sample has {xi.dim} coordinates, surrogate expects {len(s.maps)}")
    ds = DeviceSurrogate(s)
    pred = ds.predict(to_dev(xi.values[None]))[0].cpu().numpy()
    return CoarseTrajectory(initial, pred)


def surrogate_predict_batched(ds: DeviceSurrogate, xi_d, out=None):
    return ds.predict(xi_d, out)


def build_surrogate(model, grid: TimeGrid, cfg: SolverConfig, training: list, eps_kl: float = 1e-10,
                    degree: int | None = None, snapshot_method: str = "pcgc", executor=None,
                    snapshots: SnapshotSet | None = None, family: str | None = None,
                    kl_on_device: bool = True) -> KLGpcSurrogate:
    """Snapshots (device) -> KL (device products, host eigh) -> least-squares
    gPC fit (host). ``kl_on_device=False`` runs the KL on the host.

    ``family``: the reference's build always fits Legendre
    (``pintuq/surrogate.py:336-393``); that stays the default. The Gaussian
    KL models of the BASELINE configs declare ``gpc_family = "hermite"``
    (probabilists' Hermite, orthonormal under N(0, 1)), which is used when
    ``family`` is not given."""
    if family is None:
        family = getattr(model, "gpc_family", "legendre")
    if snapshots is None:
        snapshots = collect_snapshots(model, grid, cfg, training, snapshot_method, executor)
    if kl_on_device and snapshots.device_fields is not None:
        basis, zeta = kl_build_device(snapshots, eps_kl)
    else:
        basis = kl_build(snapshots, eps_kl)
        zeta = kl_coefficients(snapshots, basis)
    maps = model.fit_maps()
    points = np.column_stack([m.apply([xi.values[d] for xi in snapshots.samples]) for d, m in enumerate(maps)])
    if degree is None:
        degree = default_degree(snapshots.n_train, points.shape[1])
    if basis.m_q:
        coeffs, residuals, degree = gpc_fit(points, zeta, degree, family)
    else:
        coeffs = np.empty((0, gpc_basis_count(degree, points.shape[1])))
        residuals = np.zeros(0)
    return KLGpcSurrogate(
        mean_field=snapshots.mean_field, eigenvalues=basis.retained.copy(), modes=basis.modes, coeffs=coeffs,
        degree=degree, maps=maps, family=family, cell_weight=snapshots.cell_weight,
        provenance={"model": model.name, "t_final": grid.t_final, "n_coarse": grid.n_coarse,
                    "n_fine_per_coarse": grid.n_fine_per_coarse, "seed": cfg.seed, "eps_kl": eps_kl,
                    "n_train": snapshots.n_train, "energy_ratio": basis.energy_ratio,
                    "snapshot_method": snapshot_method},
        ls_residuals=residuals,
    )


def save_surrogate(s: KLGpcSurrogate, path) -> None:
    """Self-describing .npz, bit-exact round trip (``pintuq/surrogate.py:396-415``)."""
    meta = {"degree": s.degree, "family": s.family, "cell_weight": s.cell_weight,
            "maps": [m.to_dict() for m in s.maps], "provenance": s.provenance, "format_version": 1}
    np.savez(path, mean_field=s.mean_field, eigenvalues=s.eigenvalues, modes=s.modes, coeffs=s.coeffs,
             ls_residuals=s.ls_residuals if s.ls_residuals is not None else np.zeros(0),
             training_errors=s.training_errors if s.training_errors is not None else np.zeros(0),
             meta=np.frombuffer(json.dumps(meta, sort_keys=True).encode(), dtype=np.uint8))


def load_surrogate(path) -> KLGpcSurrogate:
    with np.load(path) as data:
        meta = json.loads(bytes(data["meta"]).decode())
        return KLGpcSurrogate(
            mean_field=data["mean_field"], eigenvalues=data["eigenvalues"], modes=data["modes"],
            coeffs=data["coeffs"], degree=int(meta["degree"]),
            maps=[ParameterMap.from_dict(d) for d in meta["maps"]], family=meta["family"],
            cell_weight=float(meta["cell_weight"]), provenance=meta["provenance"],
            ls_residuals=data["ls_residuals"], training_errors=data["training_errors"],
        )
