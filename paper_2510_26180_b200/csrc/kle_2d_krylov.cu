// Matrix-free Krylov solvers for the 2D (5-point) path, BASELINE config 3
// (SURVEY.md §8 f1): the alternative to the direct banded L D L^T factors of
// kle_2d.cu / kle_2d_tma.cu, as the north star names it.
//
//   fine steps   (I + h A) x = x_prev + h g0 (pintuq/propagators.py:25-39,
//                121-145): Jacobi-preconditioned conjugate gradients, warm
//                started from x_prev, to ||r||_2 <= rtol ||b||_2;
//   CGC shifts   (lambda_f I + dT A) q = p_f, f = 0..N/2 (pintuq/pcgc.py:
//                137-145): Jacobi-preconditioned COCG (conjugate orthogonal
//                CG for complex-symmetric matrices: the unconjugated bilinear
//                form r^T z), from q = 0, to the same relative residual.
//
// A is applied matrix-free from the stencil (dia, ex, ey): (A v)_i = dia_i v_i
// + ex_{i-1} v_{i-1} + ex_i v_{i+1} + ey_{i-n} v_{i-n} + ey_i v_{i+n}, with
// ex[i] = A[i][i+1] (zero across a grid-row edge) and ey[i] = A[i][i+n].
//
// One 512-thread CTA per system (fine: per (sample, subinterval), all J steps
// in a row; CGC: per (sample, frequency)); every thread owns the DOFs
// i = tid + 512 j. Real CG keeps x, r, A p in registers and p in shared
// memory (zero-padded by n + 1 on both sides, so the stencil needs no bounds
// tests); COCG keeps A p in registers and x (in place in P), r, p in global
// memory (one complex vector of 16,129 DOFs is 258 KB, more than a CTA's
// shared memory). Two block reductions per iteration.
#include <cstdlib>

#include "kle_common.cuh"
#include "kle_internal.h"

namespace kle {
namespace kry {

constexpr int NT = 512;
constexpr int JJ = 32;  // DOFs per thread: nx <= 16384 (n <= 128)

// sum over the CTA of (a, b); `red` is [2][32][2] (double-buffered by `phase`)
__device__ __forceinline__ void block_sum2(double& a, double& b, double* red, int phase) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(KLE_FULL_MASK, a, o);
    b += __shfl_xor_sync(KLE_FULL_MASK, b, o);
  }
  double* buf = red + phase * 2 * (NT / 32);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    buf[2 * w] = a;
    buf[2 * w + 1] = b;
  }
  __syncthreads();
  a = 0.0;
  b = 0.0;
#pragma unroll 8
  for (int k = 0; k < NT / 32; ++k) {  // fixed order: every thread gets the same bits
    a += buf[2 * k];
    b += buf[2 * k + 1];
  }
}

struct Stencil {
  const double *dia, *ex, *ey;
  int n, nx;
  // (A v)_i - dia_i v_i, v from a zero-padded shared array (v[pad + i])
  __device__ __forceinline__ double offdiag(const double* v, int i) const {
    const double w = i > 0 ? __ldg(ex + i - 1) : 0.0;
    const double s = i >= n ? __ldg(ey + i - n) : 0.0;
    return fma(w, v[i - 1], fma(__ldg(ex + i), v[i + 1], fma(s, v[i - n], __ldg(ey + i) * v[i + n])));
  }
};

// One J-step fine sweep per (sample, subinterval) by PCG; optional F output and
// the CGC right-hand side rhs_n = scaling_n ((I + dT A) F_n - prev_n)
// (the same expression as the banded fgr kernels).
__global__ void __launch_bounds__(NT, 1) cg_fine_kernel(Kry2dArgs a) {
  extern __shared__ __align__(16) double smem[];
  const int n = a.n, nx = n * n, pad = n + 1;
  double* pv = smem + pad;  // p[-pad .. nx + pad)
  double* red = smem + nx + 2 * pad;
  const int s = blockIdx.x / a.Q, q = blockIdx.x % a.Q;
  if (a.status && a.status[s] != KLE_SAMPLE_ACTIVE) return;
  const int tid = threadIdx.x;
  const Stencil A{a.dia + (size_t)s * nx, a.ex + (size_t)s * nx, a.ey + (size_t)s * nx, n, nx};
  const double h = a.h, hg = a.h * a.g0;
  for (int e = tid; e < pad; e += NT) {
    smem[e] = 0.0;
    smem[pad + nx + e] = 0.0;
  }
  // start state
  const double* start = a.start_from_u
                            ? (q == 0 ? a.u0 : a.start + ((size_t)s * a.Q + q - 1) * nx)
                            : a.start + ((size_t)s * a.Q + q) * nx;
  double x[JJ], r[JJ], w[JJ];
  const double* x0 = a.F_given ? a.F_given + ((size_t)s * a.Q + q) * nx : start;
#pragma unroll
  for (int j = 0; j < JJ; ++j) {
    const int i = tid + NT * j;
    x[j] = i < nx ? x0[i] : 0.0;
  }
  int phase = 0;
  long long its = 0;
  const double tol2 = a.rtol * a.rtol;
  for (int step = 0; step < (a.F_given ? 0 : a.J); ++step) {
    // b = x + h g0; r = b - (I + hA) x, with x staged in p
#pragma unroll
    for (int j = 0; j < JJ; ++j) {
      const int i = tid + NT * j;
      if (i < nx) pv[i] = x[j];
    }
    __syncthreads();
    double bb = 0.0, rz = 0.0;
#pragma unroll
    for (int j = 0; j < JJ; ++j) {
      const int i = tid + NT * j;
      if (i < nx) {
        const double d = fma(h, __ldg(A.dia + i), 1.0);
        const double b = x[j] + hg;
        const double Ax = fma(d, x[j], h * A.offdiag(pv, i));
        r[j] = b - Ax;
        bb = fma(b, b, bb);
        rz = fma(r[j], r[j] / d, rz);
      }
    }
    block_sum2(bb, rz, red, phase);
    phase ^= 1;
    double rr_stop = tol2 * bb;
    // p = z
#pragma unroll
    for (int j = 0; j < JJ; ++j) {
      const int i = tid + NT * j;
      if (i < nx) pv[i] = r[j] / fma(h, __ldg(A.dia + i), 1.0);
    }
    __syncthreads();
    // r = 0 exactly (z = r / d with d > 0: rz = 0 iff r = 0): x already solves the step
    for (int it = 0; it < a.max_its && rz > 0.0; ++it) {
      double pq = 0.0, dummy = 0.0;
#pragma unroll
      for (int j = 0; j < JJ; ++j) {
        const int i = tid + NT * j;
        w[j] = 0.0;
        if (i < nx) {
          const double d = fma(h, __ldg(A.dia + i), 1.0);
          w[j] = fma(d, pv[i], h * A.offdiag(pv, i));
          pq = fma(pv[i], w[j], pq);
        }
      }
      block_sum2(pq, dummy, red, phase);
      phase ^= 1;
      const double alpha = rz / pq;
      double rzn = 0.0, rr = 0.0;
#pragma unroll
      for (int j = 0; j < JJ; ++j) {
        const int i = tid + NT * j;
        if (i < nx) {
          x[j] = fma(alpha, pv[i], x[j]);
          r[j] = fma(-alpha, w[j], r[j]);
          const double z = r[j] / fma(h, __ldg(A.dia + i), 1.0);
          rzn = fma(r[j], z, rzn);
          rr = fma(r[j], r[j], rr);
        }
      }
      block_sum2(rzn, rr, red, phase);
      phase ^= 1;
      ++its;
      if (rr <= rr_stop) break;
      const double beta = rzn / rz;
      rz = rzn;
#pragma unroll
      for (int j = 0; j < JJ; ++j) {
        const int i = tid + NT * j;
        if (i < nx) pv[i] = fma(beta, pv[i], r[j] / fma(h, __ldg(A.dia + i), 1.0));
      }
      __syncthreads();
    }
    __syncthreads();  // p is restaged at the next step
  }
  if (tid == 0 && a.its) atomicAdd(reinterpret_cast<unsigned long long*>(a.its), (unsigned long long)its);
  if (a.F_out) {
#pragma unroll
    for (int j = 0; j < JJ; ++j) {
      const int i = tid + NT * j;
      if (i < nx) a.F_out[((size_t)s * a.Q + q) * nx + i] = x[j];
    }
  }
  if (!a.R) return;
  // rhs = scaling_q ((I + dT A) F - prev), prev = alpha U_{N-1} (q = 0) or U_{q-1}
#pragma unroll
  for (int j = 0; j < JJ; ++j) {
    const int i = tid + NT * j;
    if (i < nx) pv[i] = x[j];
  }
  __syncthreads();
  const double sc = a.scaling[q];
  const double pmul = q == 0 ? a.alpha : 1.0;
  const double* prev = a.start + ((size_t)s * a.Q + (q == 0 ? a.Q - 1 : q - 1)) * nx;
#pragma unroll
  for (int j = 0; j < JJ; ++j) {
    const int i = tid + NT * j;
    if (i < nx) {
      const double Ax = fma(__ldg(A.dia + i), x[j], A.offdiag(pv, i));
      const double rhs = fma(a.dT, Ax, x[j]) - pmul * prev[i];
      a.R[((size_t)s * a.Q + q) * nx + i] = sc * rhs;
    }
  }
}

// (lambda_f I + dT A) q = p_f in place on P[s][f][:] by Jacobi-COCG from q = 0
__global__ void __launch_bounds__(NT, 1) cocg_shift_kernel(Cplx* __restrict__ P, const double* __restrict__ dia,
                                                           const double* __restrict__ ex,
                                                           const double* __restrict__ ey,
                                                           const double* __restrict__ lam,
                                                           const int32_t* __restrict__ status, int NF, int n,
                                                           double dT, double rtol, int max_its, Cplx* __restrict__ work,
                                                           long long* its_out) {
  __shared__ double red[128];
  const int s = blockIdx.x / NF, f = blockIdx.x % NF;
  if (status && status[s] != KLE_SAMPLE_ACTIVE) return;
  const int nx = n * n, tid = threadIdx.x;
  const Stencil A{dia + (size_t)s * nx, ex + (size_t)s * nx, ey + (size_t)s * nx, n, nx};
  const Cplx lm = {lam[2 * f], lam[2 * f + 1]};
  Cplx* x = P + (size_t)blockIdx.x * nx;            // in: p_f, out: q
  Cplx* r = work + (size_t)blockIdx.x * 2 * nx;     // residual
  Cplx* pp = r + nx;                                // search direction
  auto dinv = [&](int i) -> Cplx {                  // 1 / (lambda + dT dia_i)
    return crcp(Cplx{fma(dT, __ldg(A.dia + i), lm.re), lm.im});
  };
  auto apply = [&](const Cplx* v, int i) -> Cplx {  // ((lambda I + dT A) v)_i
    const Cplx vi = v[i];
    const double w = i > 0 ? __ldg(A.ex + i - 1) : 0.0, e = __ldg(A.ex + i);
    const double so = i >= n ? __ldg(A.ey + i - n) : 0.0, no = __ldg(A.ey + i);
    const Cplx vw = i > 0 ? v[i - 1] : Cplx{0.0, 0.0}, ve = i + 1 < nx ? v[i + 1] : Cplx{0.0, 0.0};
    const Cplx vs = i >= n ? v[i - n] : Cplx{0.0, 0.0}, vn = i + n < nx ? v[i + n] : Cplx{0.0, 0.0};
    const double d = fma(dT, __ldg(A.dia + i), 0.0);
    double re = fma(w, vw.re, fma(e, ve.re, fma(so, vs.re, no * vn.re)));
    double im = fma(w, vw.im, fma(e, ve.im, fma(so, vs.im, no * vn.im)));
    re = fma(dT, re, d * vi.re);
    im = fma(dT, im, d * vi.im);
    return {fma(lm.re, vi.re, fma(-lm.im, vi.im, re)), fma(lm.re, vi.im, fma(lm.im, vi.re, im))};
  };
  // r = b, x = 0, p = z = D^-1 r; rho = r^T z (unconjugated), bb = ||b||^2
  double bb = 0.0, rho_re = 0.0, rho_im = 0.0, dum = 0.0;
  for (int j = 0; j < JJ; ++j) {
    const int i = tid + NT * j;
    if (i < nx) {
      const Cplx b = x[i];
      r[i] = b;
      const Cplx z = cmul(b, dinv(i));
      pp[i] = z;
      x[i] = {0.0, 0.0};
      bb = fma(b.re, b.re, fma(b.im, b.im, bb));
      rho_re = fma(b.re, z.re, fma(-b.im, z.im, rho_re));
      rho_im = fma(b.re, z.im, fma(b.im, z.re, rho_im));
    }
  }
  block_sum2(rho_re, rho_im, red, 0);
  block_sum2(bb, dum, red, 1);
  const double stop = rtol * rtol * bb;
  Cplx w[JJ];
  int phase = 0;
  long long its = 0;
  for (int it = 0; it < max_its && bb > 0.0; ++it) {
    __syncthreads();  // p complete
    double pq_re = 0.0, pq_im = 0.0;
#pragma unroll
    for (int j = 0; j < JJ; ++j) {
      const int i = tid + NT * j;
      w[j] = {0.0, 0.0};
      if (i < nx) {
        w[j] = apply(pp, i);
        const Cplx pi = pp[i];
        pq_re = fma(pi.re, w[j].re, fma(-pi.im, w[j].im, pq_re));
        pq_im = fma(pi.re, w[j].im, fma(pi.im, w[j].re, pq_im));
      }
    }
    block_sum2(pq_re, pq_im, red, phase);
    phase ^= 1;
    const Cplx alpha = cmul(Cplx{rho_re, rho_im}, crcp(Cplx{pq_re, pq_im}));
    double rn_re = 0.0, rn_im = 0.0, rr = 0.0;
#pragma unroll
    for (int j = 0; j < JJ; ++j) {
      const int i = tid + NT * j;
      if (i < nx) {
        const Cplx pi = pp[i];
        const Cplx xi = x[i];
        x[i] = {fma(alpha.re, pi.re, fma(-alpha.im, pi.im, xi.re)), fma(alpha.re, pi.im, fma(alpha.im, pi.re, xi.im))};
        Cplx ri = r[i];
        ri = {fma(-alpha.re, w[j].re, fma(alpha.im, w[j].im, ri.re)),
              fma(-alpha.re, w[j].im, fma(-alpha.im, w[j].re, ri.im))};
        r[i] = ri;
        const Cplx z = cmul(ri, dinv(i));
        rn_re = fma(ri.re, z.re, fma(-ri.im, z.im, rn_re));
        rn_im = fma(ri.re, z.im, fma(ri.im, z.re, rn_im));
        rr = fma(ri.re, ri.re, fma(ri.im, ri.im, rr));
      }
    }
    double rr2 = rr;
    block_sum2(rn_re, rn_im, red, phase);
    phase ^= 1;
    block_sum2(rr2, dum, red, phase);
    phase ^= 1;
    ++its;
    if (rr2 <= stop) break;
    const Cplx beta = cmul(Cplx{rn_re, rn_im}, crcp(Cplx{rho_re, rho_im}));
    rho_re = rn_re;
    rho_im = rn_im;
#pragma unroll
    for (int j = 0; j < JJ; ++j) {
      const int i = tid + NT * j;
      if (i < nx) {
        const Cplx z = cmul(r[i], dinv(i));
        const Cplx pi = pp[i];
        pp[i] = {fma(beta.re, pi.re, fma(-beta.im, pi.im, z.re)), fma(beta.re, pi.im, fma(beta.im, pi.re, z.im))};
      }
    }
  }
  if (tid == 0 && its_out) atomicAdd(reinterpret_cast<unsigned long long*>(its_out), (unsigned long long)its);
}

}  // namespace kry

int kry2d_fine(const Kry2dArgs& a, cudaStream_t st) {
  if (a.M <= 0 || a.Q <= 0) return KLE_OK;
  const int nx = a.n * a.n;
  if (nx > kry::NT * kry::JJ) return set_error(KLE_ERR_UNSUPPORTED, "krylov2d: n > 128");
  const size_t smem = sizeof(double) * ((size_t)nx + 2 * (a.n + 1) + 128);
  static PerDeviceOnce attr_once;
  if (int rc = once_per_device(attr_once, "kle_2d_krylov: cudaFuncSetAttribute", [&] {
        return cudaFuncSetAttribute(kry::cg_fine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      }))
    return rc;
  kry::cg_fine_kernel<<<(unsigned)(a.M * a.Q), kry::NT, smem, st>>>(a);
  return check_launch("cg_fine_kernel");
}

int kry2d_shift_solve(Cplx* P, const double* dia, const double* ex, const double* ey, const double* lam,
                      const int32_t* status, int M, int NF, int n, double dT, double rtol, int max_its, Cplx* work,
                      long long* its, cudaStream_t st) {
  if (M <= 0) return KLE_OK;
  if (n * n > kry::NT * kry::JJ) return set_error(KLE_ERR_UNSUPPORTED, "krylov2d: n > 128");
  kry::cocg_shift_kernel<<<(unsigned)(M * NF), kry::NT, 0, st>>>(P, dia, ex, ey, lam, status, NF, n, dT, rtol,
                                                                  max_its, work, its);
  return check_launch("cocg_shift_kernel");
}

}  // namespace kle
