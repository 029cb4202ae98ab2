// Fused backward-Euler sweeps with a damped Newton iteration per step for the
// nonlinear tridiagonal models (Burgers, Allen-Cahn).
//
// Reference: the compiled sweeps of pintuq/_kernels.pyx (thomas 17-34,
// burgers_fill 37-58, allencahn_fill 61-73, eval_residual 76-97, newton_loop
// 100-143, run_sweep 146-163), dispatched by propagators.py:82-99. Same
// arithmetic and order of operations: the residual r = v - u - dt f(v), stop
// on max|r| <= newton_tol, Newton system (I - dt J) delta = -r by the
// pivot-free Thomas algorithm, step halved until the 2-norm residual drops
// by the Armijo factor (1 - 1e-4 t) or t <= 2^-20; status = 1-based index of
// the first step whose Newton iteration failed (0 = success).
//
// One thread per system (sample, start state); the ten work vectors of a
// system live in global memory interleaved across systems ([vec][row][sys]),
// so every load and store of a warp is one coalesced segment. nx <= a few
// hundred (99 for Burgers, 255 for Allen-Cahn) keeps them L1/L2 resident.
#include "kle_common.cuh"
#include "kle_internal.h"

namespace kle {

namespace {

struct NwView {
  double* base;
  size_t ns;  // systems (stride between rows)
  __device__ __forceinline__ double& at(int vec, int row, int nx, size_t sys) const {
    return base[((size_t)vec * nx + row) * ns + sys];
  }
};

enum { V_U, V_V, V_VT, V_F, V_SUB, V_DIAG, V_SUP, V_R, V_CP, V_DP, V_DELTA, NW_VECS };

// rhs f(v) and the Jacobian bands at v (burgers_fill / allencahn_fill)
__device__ __forceinline__ void fill(const NwView& w, int vv, int which, double p0, double dx, double bc_lo,
                                     double bc_hi, int m, size_t sy) {
  const double idx = 1.0 / dx, idx2 = 1.0 / (dx * dx);
  if (which == 0) {
    const double nu = p0;
    for (int i = 0; i < m; ++i) {
      const double vi = w.at(vv, i, m, sy);
      const double le = i > 0 ? w.at(vv, i - 1, m, sy) : 0.0;
      const double ri = i < m - 1 ? w.at(vv, i + 1, m, sy) : 0.0;
      if (vi >= 0.0) {
        w.at(V_F, i, m, sy) = -vi * (vi - le) * idx + nu * (le - 2.0 * vi + ri) * idx2;
        w.at(V_DIAG, i, m, sy) = -(2.0 * vi - le) * idx - 2.0 * nu * idx2;
        if (i > 0) w.at(V_SUB, i - 1, m, sy) = vi * idx + nu * idx2;
        if (i < m - 1) w.at(V_SUP, i, m, sy) = nu * idx2;
      } else {
        w.at(V_F, i, m, sy) = -vi * (ri - vi) * idx + nu * (le - 2.0 * vi + ri) * idx2;
        w.at(V_DIAG, i, m, sy) = -(ri - 2.0 * vi) * idx - 2.0 * nu * idx2;
        if (i > 0) w.at(V_SUB, i - 1, m, sy) = nu * idx2;
        if (i < m - 1) w.at(V_SUP, i, m, sy) = -vi * idx + nu * idx2;
      }
    }
  } else {
    const double eps = p0;
    for (int i = 0; i < m; ++i) {
      const double vi = w.at(vv, i, m, sy);
      const double le = i > 0 ? w.at(vv, i - 1, m, sy) : bc_lo;
      const double ri = i < m - 1 ? w.at(vv, i + 1, m, sy) : bc_hi;
      w.at(V_F, i, m, sy) = eps * (le - 2.0 * vi + ri) * idx2 - (vi * vi * vi - vi);
      w.at(V_DIAG, i, m, sy) = -2.0 * eps * idx2 - (3.0 * vi * vi - 1.0);
    }
    for (int i = 0; i < m - 1; ++i) {
      w.at(V_SUB, i, m, sy) = eps * idx2;
      w.at(V_SUP, i, m, sy) = eps * idx2;
    }
  }
}

// residual r = v - u - dt f(v); sup and 2-norms (eval_residual)
__device__ __forceinline__ void residual(const NwView& w, int vv, double dt, int which, double p0, double dx,
                                         double bc_lo, double bc_hi, int m, size_t sy, double& rn, double& r2) {
  fill(w, vv, which, p0, dx, bc_lo, bc_hi, m, sy);
  double res = 0.0, sq = 0.0;
  for (int i = 0; i < m; ++i) {
    const double r = w.at(vv, i, m, sy) - w.at(V_U, i, m, sy) - dt * w.at(V_F, i, m, sy);
    w.at(V_R, i, m, sy) = r;
    sq += r * r;
    if (r < 0.0) {
      if (-r > res) res = -r;
    } else if (r > res) {
      res = r;
    }
  }
  rn = res;
  r2 = sqrt(sq);
}

// pivot-free Thomas on (sub, diag, sup) with rhs r -> delta
__device__ __forceinline__ void thomas(const NwView& w, int m, size_t sy) {
  if (m == 1) {
    w.at(V_DELTA, 0, m, sy) = w.at(V_R, 0, m, sy) / w.at(V_DIAG, 0, m, sy);
    return;
  }
  double cp = w.at(V_SUP, 0, m, sy) / w.at(V_DIAG, 0, m, sy);
  double dp = w.at(V_R, 0, m, sy) / w.at(V_DIAG, 0, m, sy);
  w.at(V_CP, 0, m, sy) = cp;
  w.at(V_DP, 0, m, sy) = dp;
  for (int i = 1; i < m; ++i) {
    const double sb = w.at(V_SUB, i - 1, m, sy);
    const double denom = w.at(V_DIAG, i, m, sy) - sb * cp;
    if (i < m - 1) cp = w.at(V_SUP, i, m, sy) / denom;
    dp = (w.at(V_R, i, m, sy) - sb * dp) / denom;
    w.at(V_CP, i, m, sy) = cp;
    w.at(V_DP, i, m, sy) = dp;
  }
  double o = dp;
  w.at(V_DELTA, m - 1, m, sy) = o;
  for (int i = m - 2; i >= 0; --i) {
    o = w.at(V_DP, i, m, sy) - w.at(V_CP, i, m, sy) * o;
    w.at(V_DELTA, i, m, sy) = o;
  }
}

// one backward-Euler step of u (in V_U) in place; returns false if Newton failed
__device__ bool newton_step(const NwView& w, double dt, double tol, int max_newton, int which, double p0, double dx,
                            double bc_lo, double bc_hi, int m, size_t sy) {
  for (int i = 0; i < m; ++i) w.at(V_V, i, m, sy) = w.at(V_U, i, m, sy);
  double rn, r2;
  residual(w, V_V, dt, which, p0, dx, bc_lo, bc_hi, m, sy, rn, r2);
  for (int it = 0; it <= max_newton; ++it) {
    if (rn <= tol) {
      for (int i = 0; i < m; ++i) w.at(V_U, i, m, sy) = w.at(V_V, i, m, sy);
      return true;
    }
    if (it == max_newton) break;
    for (int i = 0; i < m; ++i) {
      w.at(V_DIAG, i, m, sy) = 1.0 - dt * w.at(V_DIAG, i, m, sy);
      w.at(V_R, i, m, sy) = -w.at(V_R, i, m, sy);
    }
    for (int i = 0; i < m - 1; ++i) {
      w.at(V_SUB, i, m, sy) = -dt * w.at(V_SUB, i, m, sy);
      w.at(V_SUP, i, m, sy) = -dt * w.at(V_SUP, i, m, sy);
    }
    thomas(w, m, sy);
    double t = 1.0, rn_t, r2_t;
    while (true) {
      for (int i = 0; i < m; ++i) w.at(V_VT, i, m, sy) = w.at(V_V, i, m, sy) + t * w.at(V_DELTA, i, m, sy);
      residual(w, V_VT, dt, which, p0, dx, bc_lo, bc_hi, m, sy, rn_t, r2_t);
      if (r2_t <= (1.0 - 1e-4 * t) * r2 || t <= 0x1p-20) break;
      t *= 0.5;
    }
    for (int i = 0; i < m; ++i) w.at(V_V, i, m, sy) = w.at(V_VT, i, m, sy);
    rn = rn_t;
    r2 = r2_t;
  }
  for (int i = 0; i < m; ++i) w.at(V_U, i, m, sy) = w.at(V_V, i, m, sy);
  return false;
}

}  // namespace

// out[s][q][g] = state after (g + 1) * J steps from start[s][q]; status[s][q]
// = 1-based first failing step (counting over all segments), 0 = success.
// Samples with active[s] != ACTIVE are skipped (optional).
__global__ void __launch_bounds__(128) newton_sweep_kernel(NewtonArgs a, double* __restrict__ work, size_t ns) {
  const size_t sy = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (sy >= (size_t)a.M * a.Q) return;
  const int s = (int)(sy / a.Q), q = (int)(sy - (size_t)s * a.Q);
  if (a.active && a.active[s] != KLE_SAMPLE_ACTIVE) return;
  const int m = a.nx;
  const NwView w{work, ns};
  const double* st = a.start + sy * m;
  for (int i = 0; i < m; ++i) w.at(V_U, i, m, sy) = st[i];
  const double p0 = a.p0[s];
  int bad = 0;
  for (int g = 0; g < a.nseg && !bad; ++g) {
    for (int k = 0; k < a.J; ++k) {
      if (!newton_step(w, a.h, a.newton_tol, a.max_newton, a.kind, p0, a.dx, a.bc_lo, a.bc_hi, m, sy)) {
        bad = g * a.J + k + 1;
        break;
      }
    }
    double* o = a.out + (sy * a.nseg + g) * m;
    for (int i = 0; i < m; ++i) o[i] = w.at(V_U, i, m, sy);
  }
  if (bad) {  // the reference returns the last iterate: fill the remaining segments with it
    const int g0 = (bad - 1) / a.J;
    for (int g = g0 + 1; g < a.nseg; ++g) {
      double* o = a.out + (sy * a.nseg + g) * m;
      for (int i = 0; i < m; ++i) o[i] = w.at(V_U, i, m, sy);
    }
  }
  if (a.status) a.status[sy] = bad;
}

// classical parareal correction of subinterval n for the active samples
// (pintuq/parareal.py:174-176): U[s][n] = (Gn[s] + F[s][n]) - Gp[s][n],
// then Gp[s][n] = Gn[s] (the "old" coarse value of the next iteration)
__global__ void para_combine_kernel(double* __restrict__ U, const double* __restrict__ Gn,
                                    const double* __restrict__ F, double* __restrict__ Gp,
                                    const int32_t* __restrict__ status, int M, int N, int nx, int n) {
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (t >= (size_t)M * nx) return;
  const int s = (int)(t / nx), i = (int)(t - (size_t)s * nx);
  if (status && status[s] != KLE_SAMPLE_ACTIVE) return;
  const size_t o = ((size_t)s * N + n) * nx + i;
  const double g = Gn[(size_t)s * nx + i];
  U[o] = (g + F[o]) - Gp[o];
  Gp[o] = g;
}

int para_combine(double* U, const double* Gn, const double* F, double* Gp, const int32_t* status, int M, int N,
                 int nx, int n, cudaStream_t st) {
  const size_t tot = (size_t)M * nx;
  if (tot == 0) return KLE_OK;
  para_combine_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(U, Gn, F, Gp, status, M, N, nx, n);
  return check_launch("para_combine_kernel");
}

size_t newton_work_doubles(int M, int Q, int nx) { return (size_t)NW_VECS * nx * ((size_t)M * Q); }

int newton_sweep(const NewtonArgs& a, double* work, cudaStream_t st) {
  const size_t ns = (size_t)a.M * a.Q;
  if (ns == 0) return KLE_OK;
  newton_sweep_kernel<<<(unsigned)((ns + 127) / 128), 128, 0, st>>>(a, work, ns);
  return check_launch("newton_sweep_kernel");
}

}  // namespace kle
