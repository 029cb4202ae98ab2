// Coarse-grid correction for the nonlinear tridiagonal models: the simplified
// Newton iteration with the averaged Jacobian of pintuq/pcgc.py:245-270, one
// CTA per sample running the whole inner loop on chip.
//
// Per inner iteration (u_l = current iterate, b = F - G(prev) from
// assemble_rhs_blocks, pcgc.py:175-197):
//   shifted_i = u_l[i] - b[i];  F_l[i] = f(shifted_i);  J_i = f'(shifted_i)
//   mean_jac = (J_0 + ... + J_{N-1}) * (1/N)              (tridiagonal)
//   rhs = dT (F_l - mean_jac u_l) + b
//   u_next = three_step_solve(spec, mean_jac, dT, rhs)      (pcgc.py:148-172:
//            scaled DFT along time, N shifted solves (lambda_n I - dT mean_jac)
//            -- banded, no pivoting: diagonally dominant for these models --
//            inverse DFT; the half spectrum f <= N/2 by Hermitian symmetry)
//   stop when max|u_next - u_l| <= newton_tol; NonConvergenceError after 150.
// The DFT is direct (N = 25 / 30 in the reference harness settings, not
// powers of two). Shared memory: u_l and rhs [N][nx] real, spectra
// [N/2+1][nx] complex; b is read from global (L2) memory.
#include <cmath>

#include "kle_common.cuh"
#include "kle_internal.h"

namespace kle {

namespace {

constexpr int NCGC_CAP = 150;  // _SIMPLIFIED_NEWTON_CAP, pcgc.py:205

// f(v)_i and the Jacobian row i (J[i][i-1], J[i][i], J[i][i+1]) of the model
// at the state v (neighbours vm, vp; 0 outside for Burgers), in the order of
// operations of models.py rhs / jacobian (numpy expressions).
__device__ __forceinline__ void row_fj(int kind, double p0, double dx, double bc_lo, double bc_hi, double vm,
                                       double v, double vp, int i, int m, double& f, double& jl, double& jd,
                                       double& ju) {
  const double dx2 = dx * dx;
  if (kind == 0) {  // Burgers: upwind on sign(v), nu = p0
    const double nu = p0;
    const double le = i > 0 ? vm : 0.0, ri = i < m - 1 ? vp : 0.0;
    const bool up = v >= 0.0;
    const double dudx = up ? (v - le) / dx : (ri - v) / dx;
    f = -v * dudx + nu * (le - 2.0 * v + ri) / dx2;
    jd = (up ? -(2.0 * v - le) / dx : -(ri - 2.0 * v) / dx) - 2.0 * nu / dx2;
    jl = (up ? v / dx : 0.0) + nu / dx2;
    ju = (up ? 0.0 : -v / dx) + nu / dx2;
  } else {  // Allen-Cahn: eps = p0, Dirichlet values lifted into the end rows
    const double eps = p0;
    const double le = i > 0 ? vm : 0.0, ri = i < m - 1 ? vp : 0.0;
    double d2 = (le - 2.0 * v + ri) / dx2;
    if (i == 0) d2 += bc_lo / dx2;
    if (i == m - 1) d2 += bc_hi / dx2;
    if (m == 1) d2 = (le - 2.0 * v + ri) / dx2 + (bc_lo / dx2 + bc_hi / dx2);
    f = eps * d2 - (v * v * v - v);
    jd = eps * (-2.0 / dx2) - (3.0 * v * v - 1.0);
    jl = eps * (1.0 / dx2);
    ju = eps * (1.0 / dx2);
  }
}

}  // namespace

__global__ void __launch_bounds__(256) newton_cgc_kernel(NewtonCgcArgs a) {
  const int s = blockIdx.x;
  if (a.status && a.status[s] != KLE_SAMPLE_ACTIVE) return;
  const int N = a.N, m = a.nx, NF = N / 2 + 1, tid = threadIdx.x, NT = blockDim.x;
  extern __shared__ __align__(16) double sm[];
  double* ul = sm;                                      // [N][m]
  double* rh = ul + (size_t)N * m;                      // [N + 2][m]: rhs, then the Thomas cp ([NF][m] complex)
  Cplx* P = reinterpret_cast<Cplx*>(rh + (size_t)(N + 2) * m);  // [NF][m]
  Cplx* tw = P + (size_t)NF * m;                        // [N]
  double* jb = reinterpret_cast<double*>(tw + N);       // [3][m]: mean Jacobian (sub, diag, sup)
  double* red = jb + 3 * m;                             // [32]
  const size_t sb = (size_t)s * N * m;
  const double* b = a.b + sb;
  const double p0 = a.p0[s];
  for (int e = tid; e < N * m; e += NT) ul[e] = a.U[sb + e];
  for (int j = tid; j < N; j += NT) {
    double sn, cs;
    sincospi(-2.0 * (double)j / (double)N, &sn, &cs);
    tw[j] = {cs, sn};
  }
  __syncthreads();
  const double rsN = 1.0 / sqrt((double)N), dT = a.dT;
  int inner = 0;
  bool ok = false;
  for (inner = 1; inner <= NCGC_CAP; ++inner) {
    // mean Jacobian (sums over the blocks in order, then / N)
    for (int i = tid; i < m; i += NT) {
      double sl = 0.0, sd = 0.0, su = 0.0;
      for (int n = 0; n < N; ++n) {
        const double* un = ul + (size_t)n * m;
        const double* bn = b + (size_t)n * m;
        const double v = un[i] - bn[i];
        const double vm = i > 0 ? un[i - 1] - bn[i - 1] : 0.0;
        const double vp = i < m - 1 ? un[i + 1] - bn[i + 1] : 0.0;
        double f, jl, jd, ju;
        row_fj(a.kind, p0, a.dx, a.bc_lo, a.bc_hi, vm, v, vp, i, m, f, jl, jd, ju);
        if (n == 0) {
          sl = jl;
          sd = jd;
          su = ju;
        } else {
          sl += jl;
          sd += jd;
          su += ju;
        }
        rh[(size_t)n * m + i] = f;  // F_l, completed to the rhs below
      }
      const double invN = 1.0 / N;  // mean_jac / N is a sparse scalar product with 1/N in scipy
      jb[i] = i > 0 ? sl * invN : 0.0;  // J[i][i-1]
      jb[m + i] = sd * invN;
      jb[2 * m + i] = i < m - 1 ? su * invN : 0.0;  // J[i][i+1]
    }
    __syncthreads();
    // rhs = dT (F_l - mean_jac u_l) + b, alpha-scaled for the DFT
    for (int e = tid; e < N * m; e += NT) {
      const int n = e / m, i = e - n * m;
      const double* un = ul + (size_t)n * m;
      double Ju = (i > 0 ? jb[i] * un[i - 1] : 0.0) + jb[m + i] * un[i];
      if (i < m - 1) Ju += jb[2 * m + i] * un[i + 1];
      rh[e] = a.scaling[n] * (dT * (rh[e] - Ju) + b[e]);
    }
    __syncthreads();
    // p_f = fft(scaling r)_f / sqrt(N), f <= N/2 (direct DFT along time)
    for (int e = tid; e < NF * m; e += NT) {
      const int f = e / m, i = e - f * m;
      double re = 0.0, im = 0.0;
      for (int n = 0; n < N; ++n) {
        const Cplx w = tw[(int)(((long long)f * n) % N)];
        const double r = rh[(size_t)n * m + i];
        re = fma(r, w.re, re);
        im = fma(r, w.im, im);
      }
      P[e] = {re * rsN, im * rsN};
    }
    __syncthreads();
    // (lambda_f I - dT mean_jac) q = p: pivot-free complex Thomas, one thread per f
    for (int f = tid; f < NF; f += NT) {
      const Cplx lam = {a.lam[2 * f], a.lam[2 * f + 1]};
      Cplx* p = P + (size_t)f * m;
      Cplx cpp = {0.0, 0.0}, dpp = {0.0, 0.0};
      // forward: cp_i = c_i / den_i, dp_i = (p_i - a_i dp_{i-1}) / den_i
      Cplx* cps = reinterpret_cast<Cplx*>(rh) + (size_t)f * m;  // rh is free now: reuse as cp storage
      for (int i = 0; i < m; ++i) {
        const Cplx d = {lam.re - dT * jb[m + i], lam.im};
        const double al = i > 0 ? -dT * jb[i] : 0.0;            // a_i = -dT J[i][i-1]
        const double cu = i < m - 1 ? -dT * jb[2 * m + i] : 0.0;  // c_i = -dT J[i][i+1]
        const Cplx den = i > 0 ? Cplx{d.re - al * cpp.re, d.im - al * cpp.im} : d;
        const Cplx iden = crcp(den);
        const Cplx num = i > 0 ? Cplx{p[i].re - al * dpp.re, p[i].im - al * dpp.im} : p[i];
        dpp = cmul(num, iden);
        cpp = {cu * iden.re, cu * iden.im};
        cps[i] = cpp;
        p[i] = dpp;
      }
      Cplx x = p[m - 1];
      for (int i = m - 2; i >= 0; --i) {
        const Cplx c = cps[i];
        x = {p[i].re - (c.re * x.re - c.im * x.im), p[i].im - (c.re * x.im + c.im * x.re)};
        p[i] = x;
      }
    }
    __syncthreads();
    // u = ifft(q)_n / sqrt(N) / scaling_n (Hermitian completion), increment vs u_l
    double inc = 0.0;
    bool bad = false;
    for (int e = tid; e < N * m; e += NT) {
      const int n = e / m, i = e - n * m;
      double re = P[i].re;  // f = 0
      for (int f = 1; f < NF; ++f) {
        const Cplx q = P[(size_t)f * m + i];
        const Cplx w = tw[(int)(((long long)f * n) % N)];  // conj for the inverse
        const double t = q.re * w.re + q.im * w.im;       // Re(q conj(w))
        re += (2 * f == N) ? t : 2.0 * t;
      }
      const double u = (re * rsN) * a.inv_scaling[n];
      const double d = fabs(u - ul[e]);
      inc = fmax(inc, d);
      bad |= (d != d);
      rh[e] = u;  // rh no longer needed: staged for the swap
    }
    if (__syncthreads_or(bad)) inc = __longlong_as_double(0x7ff8000000000000LL);
    inc = warp_max(inc);
    if ((tid & 31) == 0) red[tid >> 5] = inc;
    __syncthreads();
    double incmax = red[0];
    for (int w = 1; w < NT / 32; ++w) incmax = nanmax(incmax, red[w]);
    for (int e = tid; e < N * m; e += NT) ul[e] = rh[e];
    __syncthreads();
    if (incmax <= a.newton_tol) {
      ok = true;
      break;
    }
    if (incmax != incmax) break;
  }
  for (int e = tid; e < N * m; e += NT) a.Uout[sb + e] = ul[e];
  if (tid == 0) {
    if (a.inner) a.inner[s] = ok ? inner : NCGC_CAP;
    if (!ok && a.status) a.status[s] = KLE_SAMPLE_NEWTON;
  }
}

size_t newton_cgc_smem(int N, int nx) {
  const size_t NF = (size_t)N / 2 + 1;
  return sizeof(double) * ((2 * (size_t)N + 2) * nx + 3 * (size_t)nx + 32) + sizeof(Cplx) * (NF * nx + N);
}

int newton_cgc(const NewtonCgcArgs& a, cudaStream_t st) {
  if (a.M <= 0) return KLE_OK;
  const size_t smem = newton_cgc_smem(a.N, a.nx);
  if (smem > 220 * 1024) return set_error(KLE_ERR_UNSUPPORTED, "newton_cgc: N * nx too large for one CTA");
  static PerDeviceOnce attr_once;
  if (int rc = once_per_device(attr_once, "kle_newton_cgc: cudaFuncSetAttribute", [&] {
        return cudaFuncSetAttribute(newton_cgc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      }))
    return rc;
  newton_cgc_kernel<<<a.M, 256, smem, st>>>(a);
  return check_launch("newton_cgc_kernel");
}

}  // namespace kle
