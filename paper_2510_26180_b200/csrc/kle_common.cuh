// Shared device helpers for libkle_b200 (sm_100a, fp64 throughout).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#define KLE_FULL_MASK 0xffffffffu

namespace kle {

// ---------------------------------------------------------------------------
// Layout of the fine-solver factor blob (one per sample and step size h).
//
// The tridiagonal T = I + h A (A = tridiag(off, dia, off)) is factored once
// as T = L D L^T (L unit lower bidiagonal with sub-diagonal l_i, D = 1/inv).
// Rows are padded to nxp = MR * P and split into P contiguous chunks of MR
// rows; chunk k is owned by lane k of a P-lane "system group" in a warp and
// lives in that lane's registers. The two first-order recurrences of the
// LDL^T solve are evaluated chunk-locally and stitched with a P-lane
// Kogge-Stone carry scan whose multipliers are data independent and
// precomputed here:
//
//   forward   yl_j = r_j - l_j yl_{j-1}                  (chunk local)
//             Y_k  = yl_e + pi_e Y_{k-1}                 (scan, mult Af)
//             z'_j = yl_j inv_j + (pihat_j Y_{k-1} + kap_j)
//   backward  xl_j = z'_j - l_{j+1} xl_{j+1}             (chunk local)
//             X_k  = xl_s + sig_s X_{k+1}                (scan, mult Bb)
//             x'_j = xl_j + sig_j X_{k+1}
//
// The state is carried as x' = x + h*g0 (g0 the constant source), which the
// kap_j = h g0 (1 + l_{j+1}) term absorbs, so one BE step costs exactly five
// FMAs per row: (I + hA) x_new = x + h g0  <=>  the recurrences above.
//
// Blob (doubles): [l | inv | pihat | kap | sig] each MR*P (index j*P + k),
// then Af[LOGP][P], Bb[LOGP][P].
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v >> 1); }

__host__ __device__ inline int fine_blob_doubles(int MR, int P) {
  int logp = 0;
  while ((1 << logp) < P) ++logp;
  // l, 1/beta, scan multipliers, lazy-stitch vectors; (16, 8): the twisted two-lane tables (kle_fine_tw.cu)
  // (16, 32): followed by the (64, 8) blob of the eight-lane sweep (kle_fine_pw.cu)
  return 6 * MR * P + 2 * logp * P + ((MR == 16 && P == 8) ? 256 : 0) + ((MR == 16 && P == 32) ? 8 * 512 + 72 : 0);
}

struct Cplx {
  double re, im;
};

__device__ __forceinline__ Cplx cmul(Cplx a, Cplx b) {
  return {fma(a.re, b.re, -a.im * b.im), fma(a.re, b.im, a.im * b.re)};
}
__device__ __forceinline__ Cplx crcp(Cplx a) {
  double d = 1.0 / fma(a.re, a.re, a.im * a.im);
  return {a.re * d, -a.im * d};
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(KLE_FULL_MASK, v, o));
  return v;
}

// NaN-propagating max for increments: a NaN increment must never look
// converged (the reference's `increment <= tol` is False for NaN).
__device__ __forceinline__ double nanmax(double a, double b) {
  return (a != a || b != b) ? __longlong_as_double(0x7ff8000000000000LL) : fmax(a, b);
}

}  // namespace kle

// Status codes shared with include/kle_b200.h
#ifndef KLE_OK
#define KLE_OK 0
#define KLE_ERR_INVALID 1
#define KLE_ERR_CUDA 2
#define KLE_ERR_UNSUPPORTED 3
#define KLE_ERR_WORKSPACE 4
#define KLE_SAMPLE_ACTIVE 0
#define KLE_SAMPLE_CONVERGED 1
#define KLE_SAMPLE_MAXITERS 2
#define KLE_SAMPLE_NONFINITE 3
#endif
#ifndef KLE_SAMPLE_NEWTON
#define KLE_SAMPLE_NEWTON 4
#endif
