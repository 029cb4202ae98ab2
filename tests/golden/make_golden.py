"""Generate the golden vectors by running the UNMODIFIED reference (pintuq)
on the BASELINE log-normal KL model plugin.

Run here (the reference tree exists only in the build container):

    python tests/golden/make_golden.py            # writes tests/golden/*.npz

The reference is imported read-only from /root/reference/pkg/src (pure-Python
backend; the Cython extension only serves the nonlinear models). The model is
plugged in through the reference's own plugin surface: a subclass of
``pintuq.models.LinearModel`` (models.py:109-125) delegating to
``paper_2510_26180_b200.models.LogNormalKL1D``. The Hermite surrogate is
composed from the reference's lower-level functions exactly as SURVEY.md §0.2
prescribes (collect_snapshots -> kl_build -> kl_coefficients ->
gpc_fit(family="hermite") -> KLGpcSurrogate(family="hermite")).

Outputs (np.savez_compressed):
  c1.npz   config-1 pipeline: KL table, 3^4 Gauss-Hermite surrogate, the
           first 16 of the 256 seeded eval samples: U0, iteration counts,
           per-k increments, final fields, imag residue, moments; plus
           single-call vectors for propagate_fine / propagate_coarse /
           cgc_correct / three_step_solve / coarse_sweep_init.
  c2.npz   config-2 shapes (nx=511, N=64, J=64, d=8): 3 samples from
           coarse-sweep init: iteration counts, increments, final fields.
  c5s.npz  config-5 analogue (nx=255, N=128, J=8), alpha in {1e-1,1e-2,1e-4}:
           coarse-sweep init, iteration counts, increments, final fields.
  c3s.npz  2D model (LogNormalKL2D) at small shapes (n=15, N=8, J=4, d=10):
           3 samples from coarse-sweep init; propagate_fine / propagate_coarse /
           three_step_solve / cgc_correct single-call vectors (SuperLU paths).
  ref.npz  stop_on="reference" (the harness composition, pintuq/experiments.py:
           212-257): c1 samples 0..7 from their surrogate U0 (kle-pcgc) and
           samples 0..3 from random_guess_init (pcgc), plus c3s samples 0..2,
           each against fine_reference: per-record error vectors, max errors,
           increments, iteration counts, final fields; one c1 sample with
           reference= but stop_on="increment".
  para.npz classical parareal_solve (pintuq/parareal.py:100-191), the
           paper's baseline: c1 samples 0..3 from coarse_sweep_init
           (increment stop) and from random_guess_init against
           fine_reference (reference stop, the harness's "parareal" solver),
           c3s samples 0..2 (increment stop).
  nl.npz   nonlinear models at the reference harness settings (BENCHMARK_DEFAULTS,
           pintuq/experiments.py:33-38): Burgers1D (dx 1/100, T 2, N 25,
           J 40) and AllenCahn1D (dx 1/128, N 30, J 48, T 3: at the harness's
           T 30 the coarse Newton step from u0 fails, which the file records as
           ac_fail_status), samples from
           the models' own samplers: propagate_fine / propagate_coarse /
           fine_reference single calls and classical parareal_solve from
           coarse_sweep_init (increment stop, tol 1e-8).
  c3.npz   2D model at the config-3 shape (n=127, N=32, J=16, d=10): one
           sample from coarse-sweep init (iteration count, increments, field).
  c3b.npz  the same for eval samples 1..3.
  c5full.npz  config 5 at full shape (nx 4095, N 1024, J 8), 2 samples x
           alpha in {1e-1, 1e-2, 1e-4}: iteration counts, increments, imag
           residues, final-field fingerprints.
  c2sur.npz   config 2's surrogate built by the reference (2,048 points,
           degree 3): KL spectrum, coefficients, U0 of 8 eval samples, and the
           KLE-CGC of 4 of them.
  legendre_{d1,ad}.npz / _pred.npz   the reference's own build_surrogate
           (Legendre; affine / cos2pi maps) in its save_surrogate wire
           format, with surrogate_predict at 6 seeded points.
"""
from __future__ import annotations

import itertools
import os
import sys
import time
from pathlib import Path

import numpy as np

os.environ.setdefault("PINTUQ_PURE_PYTHON", "1")
REF_SRC = "/root/reference/pkg/src"
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, REF_SRC)
sys.path.insert(0, str(ROOT))

from pintuq import core as rcore  # noqa: E402
from pintuq import models as rmodels  # noqa: E402
from pintuq import parareal as rpar  # noqa: E402
from pintuq import pcgc as rpcgc  # noqa: E402
from pintuq import propagators as rprop  # noqa: E402
from pintuq import surrogate as rsur  # noqa: E402

from paper_2510_26180_b200.models import LogNormalKL1D, LogNormalKL2D, ParameterMap  # noqa: E402

OUT = Path(__file__).resolve().parent


class RefLogNormalKL1D(rmodels.LinearModel):
    """Reference-side plugin: the reference's LinearModel interface over our
    model definition (what a maintainer adds to pintuq.models._MODELS)."""

    name = "lognormal-kl-1d"
    inner_cls = LogNormalKL1D

    def __init__(self, **kw):
        self.inner = self.inner_cls(**kw)
        self.nx = self.inner.nx
        self.parameter_dim = self.inner.parameter_dim
        self.supports = self.inner.supports
        self._cache = {}

    @property
    def cell_volume(self):
        return self.inner.cell_volume

    def linear_system(self, xi):
        key = xi.key()
        if key not in self._cache:
            self._cache[key] = self.inner.linear_system(rcore.ParameterSample(xi.values, id=xi.id))
        return self._cache[key]

    def initial_condition(self, xi):
        return self.inner.initial_condition(xi)

    def sample_parameters(self, count, rng):
        draws = rng.normal(0.0, 1.0, size=(count, self.parameter_dim))
        return [rcore.ParameterSample(r, id=i) for i, r in enumerate(draws)]

    def fit_maps(self):
        return [ParameterMap("identity", lo, hi) for lo, hi in self.supports]


class RefLogNormalKL2D(RefLogNormalKL1D):
    name = "lognormal-kl-2d"
    inner_cls = LogNormalKL2D


def hermite_surrogate(model, grid, cfg, training, degree, eps_kl=1e-10):
    snap = rsur.collect_snapshots(model, grid, cfg, training, method="pcgc")
    basis = rsur.kl_build(snap, eps_kl)
    zeta = rsur.kl_coefficients(snap, basis)
    points = np.array([xi.values for xi in training])
    coeffs, resid, deg = rsur.gpc_fit(points, zeta, degree, family="hermite")
    s = rsur.KLGpcSurrogate(
        mean_field=snap.mean_field, eigenvalues=basis.retained.copy(), modes=basis.modes,
        coeffs=coeffs, degree=deg, maps=model.fit_maps(), family="hermite",
        cell_weight=snap.cell_weight,
    )
    return s, snap


def solve_one(model, grid, cfg, xi, init_states):
    init = rcore.CoarseTrajectory(model.initial_condition(xi), init_states)
    tr = rpcgc.pcgc_solve(model, xi, grid, cfg, init, stop_on="increment")
    incs = np.array([r.increment_inf for r in tr.records[1:]])
    return tr.trajectory.states, tr.iterations, incs, tr.diagnostics["max_imag_residue"]


def make_c1():
    t0 = time.time()
    model = RefLogNormalKL1D(nx=127, d=4, sigma=0.5, ell=0.3)
    grid = rcore.make_time_grid(1.0, 16, 32)
    cfg = rcore.SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60, seed=2718)
    train_rng, eval_rng, init_rng = rcore.RngStream(2718).split(3)
    nodes, _ = np.polynomial.hermite_e.hermegauss(3)
    grid_pts = np.array(list(itertools.product(nodes, repeat=4)))
    training = [rcore.ParameterSample(p, id=i) for i, p in enumerate(grid_pts)]
    s, snap = hermite_surrogate(model, grid, cfg, training, degree=2)
    xi_all = eval_rng.normal(0.0, 1.0, size=(256, 4))
    M = 16
    U0 = np.empty((M, 16, 127))
    final = np.empty_like(U0)
    iters = np.empty(M, np.int32)
    incs = np.full((M, 60), np.nan)
    imag = np.empty(M)
    for i in range(M):
        xi = rcore.ParameterSample(xi_all[i], id=i)
        U0[i] = rsur.surrogate_predict(s, xi, model.initial_condition(xi)).states
        st, it, inc, im = solve_one(model, grid, cfg, xi, U0[i])
        final[i], iters[i], imag[i] = st, it, im
        incs[i, : len(inc)] = inc
    # single-call vectors on sample 0
    xi0 = rcore.ParameterSample(xi_all[0], id=0)
    u0 = model.initial_condition(xi0)
    rng = np.random.default_rng(11)
    u_rand = rng.normal(size=127)
    pf_u0 = rprop.propagate_fine(model, u0, 0.0, grid.deltaT, grid, xi0, cfg)
    pf_rand = rprop.propagate_fine(model, u_rand, 3 * grid.deltaT, 4 * grid.deltaT, grid, xi0, cfg)
    pc_rand = rprop.propagate_coarse(model, u_rand, 0.0, grid.deltaT, xi0, cfg)
    U_prev = rcore.CoarseTrajectory(u0, U0[0])
    starts = np.vstack([u0, U0[0][:-1]])
    F_ends = np.array([rprop.propagate_fine(model, starts[n], grid.coarse_point(n),
                                            grid.coarse_point(n + 1), grid, xi0, cfg)
                       for n in range(16)])
    cgc_out, cgc_diag = rpcgc.cgc_correct(model, xi0, grid, cfg, U_prev, F_ends)
    b_blocks = rpcgc.assemble_rhs_blocks(model, xi0, grid, cfg, U0[0], F_ends)
    spec = rpcgc.build_alpha_circulant(16, 1e-3)
    A, _ = model.linear_system(xi0)
    r_rand = rng.normal(size=(16, 127))
    ts_u, ts_imag = rpcgc.three_step_solve(spec, -A, grid.deltaT, r_rand)
    cs = rpar.coarse_sweep_init(model, xi0, grid, cfg).states
    cs_states, cs_iters, cs_incs, _ = solve_one(model, grid, cfg, xi0, cs)
    np.savez_compressed(
        OUT / "c1.npz",
        kl_table=model.inner.kl_table, xi_all=xi_all, train_points=grid_pts,
        mean_field=s.mean_field, eigenvalues=s.eigenvalues, modes=s.modes, coeffs=s.coeffs,
        degree=s.degree, U0=U0, final=final, iters=iters, increments=incs, imag=imag,
        mean=final.mean(axis=0), var=final.var(axis=0),
        pf_u0=pf_u0, u_rand=u_rand, pf_rand=pf_rand, pc_rand=pc_rand, F_ends=F_ends,
        b_blocks=b_blocks, cgc_states=cgc_out.states, cgc_imag=cgc_diag["imag_residue"],
        r_rand=r_rand, ts_u=ts_u, ts_imag=ts_imag, lam=spec.eigenvalues, scaling=spec.scaling,
        coarse_sweep=cs, cs_final=cs_states, cs_iters=cs_iters, cs_incs=cs_incs,
        snapshots=snap.fields,
    )
    print(f"c1 done in {time.time() - t0:.1f}s; iters {iters.tolist()}; m_q {s.m_q}")


def make_c2():
    t0 = time.time()
    model = RefLogNormalKL1D(nx=511, d=8, sigma=0.5, ell=0.3)
    grid = rcore.make_time_grid(1.0, 64, 64)
    cfg = rcore.SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60, seed=2718)
    _, eval_rng, _ = rcore.RngStream(2718).split(3)
    xi_all = eval_rng.normal(0.0, 1.0, size=(3, 8))
    final = np.empty((3, 64, 511))
    iters = np.empty(3, np.int32)
    incs = np.full((3, 60), np.nan)
    for i in range(3):
        xi = rcore.ParameterSample(xi_all[i], id=i)
        cs = rpar.coarse_sweep_init(model, xi, grid, cfg).states
        st, it, inc, _ = solve_one(model, grid, cfg, xi, cs)
        final[i], iters[i] = st, it
        incs[i, : len(inc)] = inc
    np.savez_compressed(OUT / "c2.npz", kl_table=model.inner.kl_table, xi=xi_all,
                        final=final, iters=iters, increments=incs)
    print(f"c2 done in {time.time() - t0:.1f}s; iters {iters.tolist()}")


def make_c5s():
    t0 = time.time()
    model = RefLogNormalKL1D(nx=255, d=4, sigma=0.5, ell=0.3)
    grid = rcore.make_time_grid(1.0, 128, 8)
    _, eval_rng, _ = rcore.RngStream(2718).split(3)
    xi = rcore.ParameterSample(eval_rng.normal(0.0, 1.0, size=4), id=0)
    out = {"kl_table": model.inner.kl_table, "xi": xi.values}
    for alpha in (1e-1, 1e-2, 1e-4):
        cfg = rcore.SolverConfig(alpha=alpha, tol=1e-8, max_outer_iters=60, seed=2718)
        cs = rpar.coarse_sweep_init(model, xi, grid, cfg).states
        st, it, inc, im = solve_one(model, grid, cfg, xi, cs)
        tag = f"a{-int(round(np.log10(alpha)))}"
        out[f"{tag}_final"] = st
        out[f"{tag}_iters"] = it
        out[f"{tag}_incs"] = inc
        out[f"{tag}_imag"] = im
    np.savez_compressed(OUT / "c5s.npz", **out)
    print(f"c5s done in {time.time() - t0:.1f}s")


def make_c3s():
    t0 = time.time()
    n, N, J, d = 15, 8, 4, 10
    model = RefLogNormalKL2D(n=n, d=d, sigma=0.5, ell=0.25)
    grid = rcore.make_time_grid(1.0, N, J)
    cfg = rcore.SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60, seed=2718)
    _, eval_rng, _ = rcore.RngStream(2718).split(3)
    xi_all = eval_rng.normal(0.0, 1.0, size=(3, d))
    final = np.empty((3, N, n * n))
    iters = np.empty(3, np.int32)
    incs = np.full((3, 60), np.nan)
    cs_all = np.empty_like(final)
    for i in range(3):
        xi = rcore.ParameterSample(xi_all[i], id=i)
        cs = rpar.coarse_sweep_init(model, xi, grid, cfg).states
        st, it, inc, _ = solve_one(model, grid, cfg, xi, cs)
        final[i], iters[i], cs_all[i] = st, it, cs
        incs[i, : len(inc)] = inc
    xi0 = rcore.ParameterSample(xi_all[0], id=0)
    rng = np.random.default_rng(13)
    u_rand = rng.normal(size=n * n)
    pf_rand = rprop.propagate_fine(model, u_rand, 2 * grid.deltaT, 3 * grid.deltaT, grid, xi0, cfg)
    pc_rand = rprop.propagate_coarse(model, u_rand, 0.0, grid.deltaT, xi0, cfg)
    A, _ = model.linear_system(xi0)
    spec = rpcgc.build_alpha_circulant(N, 1e-3)
    r_rand = rng.normal(size=(N, n * n))
    ts_u, ts_imag = rpcgc.three_step_solve(spec, -A, grid.deltaT, r_rand)
    U_prev = rcore.CoarseTrajectory(model.initial_condition(xi0), cs_all[0])
    starts = np.vstack([U_prev.initial, cs_all[0][:-1]])
    F_ends = np.array([rprop.propagate_fine(model, starts[k], grid.coarse_point(k), grid.coarse_point(k + 1),
                                            grid, xi0, cfg) for k in range(N)])
    cgc_out, _ = rpcgc.cgc_correct(model, xi0, grid, cfg, U_prev, F_ends)
    np.savez_compressed(OUT / "c3s.npz", kl_table=model.inner.kl_table, xi=xi_all, coarse_sweep=cs_all,
                        final=final, iters=iters, increments=incs, u_rand=u_rand, pf_rand=pf_rand,
                        pc_rand=pc_rand, r_rand=r_rand, ts_u=ts_u, ts_imag=ts_imag, F_ends=F_ends,
                        cgc_states=cgc_out.states)
    print(f"c3s done in {time.time() - t0:.1f}s; iters {iters.tolist()}")


def make_c3():
    t0 = time.time()
    n, N, J, d = 127, 32, 16, 10
    model = RefLogNormalKL2D(n=n, d=d, sigma=0.5, ell=0.25)
    grid = rcore.make_time_grid(1.0, N, J)
    cfg = rcore.SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60, seed=2718)
    _, eval_rng, _ = rcore.RngStream(2718).split(3)
    xi_all = eval_rng.normal(0.0, 1.0, size=(1, d))
    xi = rcore.ParameterSample(xi_all[0], id=0)
    cs = rpar.coarse_sweep_init(model, xi, grid, cfg).states
    st, it, inc, _ = solve_one(model, grid, cfg, xi, cs)
    np.savez_compressed(OUT / "c3.npz", xi=xi_all, final=st[None], iters=np.array([it], np.int32),
                        increments=inc[None])
    print(f"c3 done in {time.time() - t0:.1f}s; iters {it}")


def _ref_trace(model, grid, cfg, xi, init_states, stop_on="reference"):
    reference = rprop.fine_reference(model, xi, grid, cfg)
    init = rcore.CoarseTrajectory(model.initial_condition(xi), init_states)
    tr = rpcgc.pcgc_solve(model, xi, grid, cfg, init, reference=reference, stop_on=stop_on, raise_on_max=False)
    incs = np.array([np.nan] + [r.increment_inf for r in tr.records[1:]])
    return dict(ref=reference.states, err=tr.error_vectors(), max_err=tr.max_errors(), incs=incs,
                iters=tr.iterations, to_tol=tr.iters_to_tol(cfg.tol), final=tr.trajectory.states,
                converged=tr.converged)


def _pack(out, tag, runs, N, nx, K=61):
    M = len(runs)
    out[f"{tag}_ref"] = np.array([r["ref"] for r in runs])
    out[f"{tag}_final"] = np.array([r["final"] for r in runs])
    out[f"{tag}_iters"] = np.array([r["iters"] for r in runs], np.int32)
    out[f"{tag}_to_tol"] = np.array([-1 if r["to_tol"] is None else r["to_tol"] for r in runs], np.int32)
    err = np.full((M, K, N), np.nan)
    me = np.full((M, K), np.nan)
    inc = np.full((M, K), np.nan)
    for i, r in enumerate(runs):
        err[i, : len(r["err"])] = r["err"]
        me[i, : len(r["max_err"])] = r["max_err"]
        inc[i, : len(r["incs"])] = r["incs"]
    out[f"{tag}_err"], out[f"{tag}_max_err"], out[f"{tag}_incs"] = err, me, inc


def make_ref():
    t0 = time.time()
    out = {}
    g1 = np.load(OUT / "c1.npz")
    model = RefLogNormalKL1D(nx=127, d=4, sigma=0.5, ell=0.3)
    grid = rcore.make_time_grid(1.0, 16, 32)
    cfg = rcore.SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60, seed=2718)
    xs = g1["xi_all"]
    kle = [_ref_trace(model, grid, cfg, rcore.ParameterSample(xs[i], id=i), g1["U0"][i]) for i in range(8)]
    _pack(out, "kle", kle, 16, 127)
    _, _, init_rng = rcore.RngStream(2718).split(3)
    rnd_init, rnd = [], []
    for i in range(4):
        xi = rcore.ParameterSample(xs[i], id=i)
        init = rpar.random_guess_init(model, xi, grid, init_rng).states
        rnd_init.append(init)
        rnd.append(_ref_trace(model, grid, cfg, xi, init))
    _pack(out, "rnd", rnd, 16, 127)
    out["rnd_init"] = np.array(rnd_init)
    inc = [_ref_trace(model, grid, cfg, rcore.ParameterSample(xs[0], id=0), g1["U0"][0], stop_on="increment")]
    _pack(out, "inc", inc, 16, 127)
    g3 = np.load(OUT / "c3s.npz")
    m2 = RefLogNormalKL2D(n=15, d=10, sigma=0.5, ell=0.25)
    grid2 = rcore.make_time_grid(1.0, 8, 4)
    c3 = [_ref_trace(m2, grid2, cfg, rcore.ParameterSample(g3["xi"][i], id=i), g3["coarse_sweep"][i])
          for i in range(3)]
    _pack(out, "c3s", c3, 8, 225)
    np.savez_compressed(OUT / "ref.npz", **out)
    print(f"ref done in {time.time() - t0:.1f}s; kle iters {out['kle_iters'].tolist()} "
          f"rnd iters {out['rnd_iters'].tolist()} c3s iters {out['c3s_iters'].tolist()}")


def _para_trace(model, grid, cfg, xi, init_states, reference=None, stop_on="increment"):
    init = rcore.CoarseTrajectory(model.initial_condition(xi), init_states)
    tr = rpar.parareal_solve(model, xi, grid, cfg, init, reference=reference, stop_on=stop_on,
                             raise_on_max=False)
    incs = np.array([np.nan] + [r.increment_inf for r in tr.records[1:]])
    out = dict(ref=None if reference is None else reference.states, iters=tr.iterations,
               to_tol=tr.iters_to_tol(cfg.tol), final=tr.trajectory.states, incs=incs, converged=tr.converged)
    if reference is not None:
        out.update(err=tr.error_vectors(), max_err=tr.max_errors())
    else:
        out.update(err=np.zeros((0, grid.n_coarse)), max_err=np.zeros(0), ref=np.zeros((grid.n_coarse, model.nx)))
    return out


def make_para():
    t0 = time.time()
    out = {}
    g1 = np.load(OUT / "c1.npz")
    model = RefLogNormalKL1D(nx=127, d=4, sigma=0.5, ell=0.3)
    grid = rcore.make_time_grid(1.0, 16, 32)
    cfg = rcore.SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60, seed=2718)
    xs = g1["xi_all"]
    cs_runs, cs_init = [], []
    for i in range(4):
        xi = rcore.ParameterSample(xs[i], id=i)
        cs = rpar.coarse_sweep_init(model, xi, grid, cfg).states
        cs_init.append(cs)
        cs_runs.append(_para_trace(model, grid, cfg, xi, cs))
    _pack(out, "cs", cs_runs, 16, 127)
    out["cs_init"] = np.array(cs_init)
    rnd = []
    g = np.load(OUT / "ref.npz")
    for i in range(4):
        xi = rcore.ParameterSample(xs[i], id=i)
        ref = rprop.fine_reference(model, xi, grid, cfg)
        rnd.append(_para_trace(model, grid, cfg, xi, g["rnd_init"][i], reference=ref, stop_on="reference"))
    _pack(out, "rnd", rnd, 16, 127)
    g3 = np.load(OUT / "c3s.npz")
    m2 = RefLogNormalKL2D(n=15, d=10, sigma=0.5, ell=0.25)
    grid2 = rcore.make_time_grid(1.0, 8, 4)
    c3 = [_para_trace(m2, grid2, cfg, rcore.ParameterSample(g3["xi"][i], id=i), g3["coarse_sweep"][i])
          for i in range(3)]
    _pack(out, "c3s", c3, 8, 225)
    np.savez_compressed(OUT / "para.npz", **out)
    print(f"para done in {time.time() - t0:.1f}s; cs iters {out['cs_iters'].tolist()} "
          f"rnd iters {out['rnd_iters'].tolist()} c3s iters {out['c3s_iters'].tolist()}")


def make_nl():
    t0 = time.time()
    out = {}
    for tag, model, T, N, J, ns in (("bu", rmodels.Burgers1D(dx=1 / 100), 2.0, 25, 40, 3),
                                    ("ac", rmodels.AllenCahn1D(dx=1 / 128), 3.0, 30, 48, 2)):
        grid = rcore.make_time_grid(T, N, J)
        cfg = rcore.SolverConfig(alpha=0.1, tol=1e-8, max_outer_iters=60, seed=2718)
        xis = model.sample_parameters(ns, rcore.RngStream(2718).split(3)[1])
        out[f"{tag}_xi"] = np.array([x.values for x in xis])
        xi0 = xis[0]
        u0 = model.initial_condition(xi0)
        out[f"{tag}_pf"] = rprop.propagate_fine(model, u0, 0.0, grid.deltaT, grid, xi0, cfg)
        out[f"{tag}_pc"] = rprop.propagate_coarse(model, u0, 0.0, grid.deltaT, xi0, cfg)
        out[f"{tag}_ref"] = rprop.fine_reference(model, xi0, grid, cfg).states
        out[f"{tag}_rhs0"] = model.rhs(u0, 0.0, xi0)
        out[f"{tag}_jac0"] = model.jacobian(u0, 0.0, xi0).toarray()
        finals, iters, incs, inits = [], [], np.full((ns, 61), np.nan), []
        for i, xi in enumerate(xis):
            cs = rpar.coarse_sweep_init(model, xi, grid, cfg)
            tr = rpar.parareal_solve(model, xi, grid, cfg, cs)
            inits.append(cs.states)
            finals.append(tr.trajectory.states)
            iters.append(tr.iterations)
            inc = [r.increment_inf for r in tr.records[1:]]
            incs[i, 1:len(inc) + 1] = inc
        out[f"{tag}_init"] = np.array(inits)
        # PCGC with the simplified-Newton CGC (pcgc.py:245-270) from the same initial guesses
        pf, pi_, pinc = [], [], np.full((ns, 61), np.nan)
        for i, xi in enumerate(xis):
            cs = rcore.CoarseTrajectory(model.initial_condition(xi), inits[i])
            tr = rpcgc.pcgc_solve(model, xi, grid, cfg, cs)
            pf.append(tr.trajectory.states)
            pi_.append(tr.iterations)
            inc = [r.increment_inf for r in tr.records[1:]]
            pinc[i, 1:len(inc) + 1] = inc
        out[f"{tag}_pcgc_final"] = np.array(pf)
        out[f"{tag}_pcgc_iters"] = np.array(pi_, np.int32)
        out[f"{tag}_pcgc_incs"] = pinc
        # one cgc_correct call: inner iteration count and result
        xi0 = xis[0]
        cs = rcore.CoarseTrajectory(model.initial_condition(xi0), inits[0])
        starts = np.vstack([cs.initial, cs.states[:-1]])
        fe = np.array([rprop.propagate_fine(model, starts[n], grid.coarse_point(n), grid.coarse_point(n + 1), grid,
                                            xi0, cfg) for n in range(N)])
        cc, diag = rpcgc.cgc_correct(model, xi0, grid, cfg, cs, fe)
        out[f"{tag}_cgc_F"] = fe
        out[f"{tag}_cgc_out"] = cc.states
        out[f"{tag}_cgc_inner"] = np.int32(diag["inner_iters"])
        out[f"{tag}_final"] = np.array(finals)
        out[f"{tag}_iters"] = np.array(iters, np.int32)
        out[f"{tag}_incs"] = incs
        print(f"  {tag}: parareal iters {iters}, pcgc iters {pi_}, cgc inner {diag['inner_iters']} "
              f"({time.time() - t0:.1f}s)", flush=True)
    # the harness's Allen-Cahn coarse step (dT = 1) from u0: Newton fails at step 1
    ac = rmodels.AllenCahn1D(dx=1 / 128)
    xi0 = rcore.ParameterSample(out["ac_xi"][0], id=0)
    try:
        rprop.propagate_coarse(ac, ac.initial_condition(xi0), 0.0, 1.0, xi0,
                               rcore.SolverConfig(alpha=0.1, tol=1e-8, max_outer_iters=60))
        out["ac_fail_status"] = np.int32(0)
    except rcore.NonConvergenceError as exc:
        out["ac_fail_status"] = np.int32(int(str(exc).split("step ")[1].split("/")[0]))
        out["ac_fail_last"] = exc.last_iterate
    np.savez_compressed(OUT / "nl.npz", **out)
    print(f"nl done in {time.time() - t0:.1f}s")


def make_models():
    """The reference's own linear models at one parameter value (operator,
    source, initial state) and a Diffusion1D PCGC run (coarse-sweep init)."""
    out = {}
    xi = rcore.ParameterSample(np.array([1.3]), id=0)
    for tag, model in (("d1", rmodels.Diffusion1D()), ("ad", rmodels.AdvectionDiffusion2D())):
        A, g = model.linear_system(xi)
        out[f"{tag}_A"] = A.toarray()
        out[f"{tag}_g"] = g(0.3)
        out[f"{tag}_u0"] = model.initial_condition(xi)
    d1 = rmodels.Diffusion1D()
    grid = rcore.make_time_grid(1.0, 16, 32)
    cfg = rcore.SolverConfig(alpha=0.1, tol=1e-10, max_outer_iters=60, seed=2718)
    cs = rpar.coarse_sweep_init(d1, xi, grid, cfg).states
    st, it, inc, _ = solve_one(d1, grid, cfg, xi, cs)
    out.update(d1_init=cs, d1_final=st, d1_iters=np.int32(it), d1_incs=inc)
    np.savez_compressed(OUT / "models.npz", **out)
    print(f"models done; diffusion-1d pcgc iters {it}")


# ---------------------------------------------------------------------------
# Full-shape goldens (round 2). The per-sample reference solves run in forked
# worker processes over the host cores; every solve is the unmodified
# reference's own coarse_sweep_init / pcgc_solve / surrogate_predict.
# ---------------------------------------------------------------------------
_G = {}


def _pool(n=None):
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor

    return ProcessPoolExecutor(n or os.cpu_count(), mp_context=mp.get_context("fork"))


def _coarse_then_pcgc(i):
    model, grid, cfg, xi_all = _G["model"], _G["grid"], _G["cfg"], _G["xi"]
    xi = rcore.ParameterSample(xi_all[i], id=i)
    cs = rpar.coarse_sweep_init(model, xi, grid, cfg).states
    return solve_one(model, grid, cfg, xi, cs)


def _subsample(st):
    """A committed fingerprint of a large final field: every 8th row of every
    8th time slice, plus the per-slice sums and max norms (size-independent
    checks of the whole field)."""
    return st[::8, ::8].copy(), st.sum(axis=1), np.abs(st).max(axis=1)


def make_c5full():
    """BASELINE configs[4] at its full shape (nx 4095, N 1024, J 8): the
    first two of the c5 bench's seeded samples, alpha in {1e-1, 1e-2, 1e-4},
    from coarse_sweep_init: iteration counts, increments, max_imag_residue
    and a fingerprint of the final fields (_subsample)."""
    t0 = time.time()
    model = RefLogNormalKL1D(nx=4095, d=4, sigma=0.5, ell=0.3)
    grid = rcore.make_time_grid(1.0, 1024, 8)
    _, eval_rng, _ = rcore.RngStream(2718).split(3)
    xi_all = eval_rng.normal(0.0, 1.0, size=(2, 4))
    out = {"xi": xi_all}
    for alpha in (1e-1, 1e-2, 1e-4):
        cfg = rcore.SolverConfig(alpha=alpha, tol=1e-8, max_outer_iters=60, seed=2718)
        _G.update(model=model, grid=grid, cfg=cfg, xi=xi_all)
        with _pool(2) as ex:
            runs = list(ex.map(_coarse_then_pcgc, range(2)))
        tag = f"a{-int(round(np.log10(alpha)))}"
        sub = [_subsample(r[0]) for r in runs]
        out[f"{tag}_sub"] = np.array([x[0] for x in sub])
        out[f"{tag}_rowsum"] = np.array([x[1] for x in sub])
        out[f"{tag}_rowmax"] = np.array([x[2] for x in sub])
        out[f"{tag}_iters"] = np.array([r[1] for r in runs], np.int32)
        incs = np.full((2, 60), np.nan)
        for j, r in enumerate(runs):
            incs[j, : len(r[2])] = r[2]
        out[f"{tag}_incs"] = incs
        out[f"{tag}_imag"] = np.array([r[3] for r in runs])
        print(f"  c5full alpha {alpha:g}: iters {out[f'{tag}_iters'].tolist()} ({time.time() - t0:.0f}s)")
    np.savez_compressed(OUT / "c5full.npz", **out)
    print(f"c5full done in {time.time() - t0:.1f}s")


def make_c3b():
    """Config 3 at its full shape (n 127, N 32, J 16): eval samples 1..3 (c3.npz
    holds sample 0), from coarse_sweep_init through the reference's SuperLU
    paths: iteration counts, increments, final-field fingerprints."""
    t0 = time.time()
    n, N, J, d = 127, 32, 16, 10
    model = RefLogNormalKL2D(n=n, d=d, sigma=0.5, ell=0.25)
    grid = rcore.make_time_grid(1.0, N, J)
    cfg = rcore.SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60, seed=2718)
    _, eval_rng, _ = rcore.RngStream(2718).split(3)
    xi_all = eval_rng.normal(0.0, 1.0, size=(4, d))
    _G.update(model=model, grid=grid, cfg=cfg, xi=xi_all)
    with _pool(3) as ex:
        runs = list(ex.map(_coarse_then_pcgc, [1, 2, 3]))
    incs = np.full((3, 60), np.nan)
    for j, r in enumerate(runs):
        incs[j, : len(r[2])] = r[2]
    np.savez_compressed(OUT / "c3b.npz", xi=xi_all[1:], final=np.array([r[0] for r in runs]),
                        iters=np.array([r[1] for r in runs], np.int32), increments=incs)
    print(f"c3b done in {time.time() - t0:.1f}s; iters {[r[1] for r in runs]}")


def _snap(i):
    model, grid, cfg, pts = _G["model"], _G["grid"], _G["cfg"], _G["train"]
    xi = rcore.ParameterSample(pts[i], id=i)
    init = rpar.coarse_sweep_init(model, xi, grid, cfg)   # collect_snapshots' `one` (surrogate.py:85-90)
    return rpcgc.pcgc_solve(model, xi, grid, cfg, init, stop_on="increment").trajectory.states


def _kle_one(i):
    model, grid, cfg, s, xi_all = _G["model"], _G["grid"], _G["cfg"], _G["sur"], _G["xi"]
    xi = rcore.ParameterSample(xi_all[i], id=i)
    U0 = rsur.surrogate_predict(s, xi, model.initial_condition(xi)).states
    return (U0,) + solve_one(model, grid, cfg, xi, U0)


def make_c2sur():
    """Config 2's own surrogate built by the reference: 2,048 seeded Gaussian
    training points (RngStream(2718).split(3)[0]), PCGC snapshots from
    coarse_sweep_init, snapshot KL at eps 1e-10, degree-3 Hermite least
    squares (P = 165); then the KLE-CGC of the first 4 eval samples from its
    surrogate_predict U0. Stores the KL spectrum, coefficients, U0 of 8 eval
    samples and the 4 solves (the modes, 34.5 MB, are not committed)."""
    t0 = time.time()
    model = RefLogNormalKL1D(nx=511, d=8, sigma=0.5, ell=0.3)
    grid = rcore.make_time_grid(1.0, 64, 64)
    cfg = rcore.SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60, seed=2718)
    train_rng, eval_rng, _ = rcore.RngStream(2718).split(3)
    train = train_rng.normal(0.0, 1.0, size=(2048, 8))
    _G.update(model=model, grid=grid, cfg=cfg, train=train)
    with _pool() as ex:
        fields = np.array(list(ex.map(_snap, range(len(train)), chunksize=8)))
    print(f"  c2sur snapshots {time.time() - t0:.0f}s")
    training = [rcore.ParameterSample(p, id=i) for i, p in enumerate(train)]
    snap = rsur.make_snapshot_set(training, fields, model.cell_volume * grid.deltaT)
    basis = rsur.kl_build(snap, 1e-10)
    zeta = rsur.kl_coefficients(snap, basis)
    coeffs, resid, deg = rsur.gpc_fit(train, zeta, 3, family="hermite")
    s = rsur.KLGpcSurrogate(mean_field=snap.mean_field, eigenvalues=basis.retained.copy(), modes=basis.modes,
                            coeffs=coeffs, degree=deg, maps=model.fit_maps(), family="hermite",
                            cell_weight=snap.cell_weight)
    xi_all = eval_rng.normal(0.0, 1.0, size=(8, 8))
    U0 = np.array([rsur.surrogate_predict(s, rcore.ParameterSample(x, id=i), model.initial_condition(None)).states
                   for i, x in enumerate(xi_all)])
    _G.update(sur=s, xi=xi_all)
    with _pool(4) as ex:
        runs = list(ex.map(_kle_one, range(4)))
    incs = np.full((4, 60), np.nan)
    for j, r in enumerate(runs):
        incs[j, : len(r[3])] = r[3]
    np.savez_compressed(OUT / "c2sur.npz", xi=xi_all, eigenvalues=s.eigenvalues, coeffs=s.coeffs, m_q=s.m_q,
                        degree=deg, U0=U0, final=np.array([r[1] for r in runs]),
                        iters=np.array([r[2] for r in runs], np.int32), increments=incs,
                        energy_ratio=basis.energy_ratio)
    print(f"c2sur done in {time.time() - t0:.1f}s; m_q {s.m_q}; iters {[r[2] for r in runs]}")


def make_legendre():
    """The reference's own build_surrogate (Legendre family, the models'
    fit_maps: affine for Diffusion1D, cos2pi for AdvectionDiffusion2D), saved
    with the reference's save_surrogate (the wire format), and its
    surrogate_predict at seeded evaluation points."""
    t0 = time.time()
    for tag, model, N, J in (("d1", rmodels.Diffusion1D(h=1.0 / 32.0), 8, 8),
                             ("ad", rmodels.AdvectionDiffusion2D(h=1.0 / 12.0), 8, 4)):
        grid = rcore.make_time_grid(1.0, N, J)
        cfg = rcore.SolverConfig(alpha=0.1, tol=1e-10, max_outer_iters=60, seed=2718)
        train_rng, eval_rng, _ = rcore.RngStream(2718).split(3)
        training = model.sample_parameters(12, train_rng)
        s = rsur.build_surrogate(model, grid, cfg, training, eps_kl=1e-10, degree=3)
        rsur.save_surrogate(s, OUT / f"legendre_{tag}.npz")
        evals = model.sample_parameters(6, eval_rng)
        pred = np.array([rsur.surrogate_predict(s, xi, model.initial_condition(xi)).states for xi in evals])
        np.savez_compressed(OUT / f"legendre_{tag}_pred.npz", xi=np.array([x.values for x in evals]), pred=pred,
                            family=s.family, maps=np.array([m.kind for m in s.maps]))
    print(f"legendre done in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c2", "c5s", "c3s", "c3", "ref", "para", "nl", "models", "legendre", "c5full",
                             "c3b", "c2sur"]
    for w in which:
        {"c1": make_c1, "c2": make_c2, "c5s": make_c5s, "c3s": make_c3s, "c3": make_c3, "ref": make_ref,
         "para": make_para, "nl": make_nl, "models": make_models, "legendre": make_legendre,
         "c5full": make_c5full, "c3b": make_c3b, "c2sur": make_c2sur}[w]()
