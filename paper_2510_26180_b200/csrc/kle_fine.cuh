// Fine/coarse backward-Euler propagators for the 1D tridiagonal operator.
//
// Replaces the reference's per-sample, per-step SuperLU solves
// (pintuq/propagators.py:25-39, 121-157) by a register-resident partitioned
// LDL^T solve (see kle_common.cuh for the recurrences). One warp holds
// 32/P independent systems; each lane owns MR rows of R right-hand sides
// that share the sample's factor rows (read from shared memory).
#pragma once
#include "kle_common.cuh"

namespace kle {

template <int MR, int P>
struct FineLayout {
  static constexpr int LOGP = ilog2c(P);
  static constexpr int NXP = MR * P;
  static constexpr int L_OFF = 0;
  static constexpr int INV_OFF = NXP;
  static constexpr int PIH_OFF = 2 * NXP;
  static constexpr int KAP_OFF = 3 * NXP;
  static constexpr int SIG_OFF = 4 * NXP;
  static constexpr int AF_OFF = 5 * NXP;
  static constexpr int BB_OFF = 5 * NXP + LOGP * P;
  static constexpr int DOUBLES = 5 * NXP + 2 * LOGP * P;
};

// One backward-Euler solve (I + hA) x_new = x + h g0 on the x' = x + h g0
// representation, for R right-hand sides held in registers.
// `fac` points at the sample's blob (shared or global memory).
template <int MR, int P, int R>
__device__ __forceinline__ void be_solve(double (&x)[R][MR], const double* __restrict__ fac, int k) {
  using L = FineLayout<MR, P>;
  // forward, chunk local
#pragma unroll
  for (int j = 1; j < MR; ++j) {
    const double l = fac[L::L_OFF + j * P + k];
#pragma unroll
    for (int r = 0; r < R; ++r) x[r][j] = fma(-l, x[r][j - 1], x[r][j]);
  }
  // forward carry scan across the P chunks
  double Y[R];
#pragma unroll
  for (int r = 0; r < R; ++r) Y[r] = x[r][MR - 1];
#pragma unroll
  for (int t = 0; t < L::LOGP; ++t) {
    const int d = 1 << t;
    const double a = fac[L::AF_OFF + t * P + k];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double o = __shfl_up_sync(KLE_FULL_MASK, Y[r], d, P);
      if (k >= d) Y[r] = fma(a, o, Y[r]);
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const double o = __shfl_up_sync(KLE_FULL_MASK, Y[r], 1, P);
    Y[r] = (k == 0) ? 0.0 : o;
  }
  // stitch + diagonal scale (+ source term absorbed in kap)
#pragma unroll
  for (int j = 0; j < MR; ++j) {
    const double inv = fac[L::INV_OFF + j * P + k];
    const double ph = fac[L::PIH_OFF + j * P + k];
    const double kp = fac[L::KAP_OFF + j * P + k];
#pragma unroll
    for (int r = 0; r < R; ++r) x[r][j] = fma(x[r][j], inv, fma(ph, Y[r], kp));
  }
  // backward, chunk local
#pragma unroll
  for (int j = MR - 2; j >= 0; --j) {
    const double l = fac[L::L_OFF + (j + 1) * P + k];
#pragma unroll
    for (int r = 0; r < R; ++r) x[r][j] = fma(-l, x[r][j + 1], x[r][j]);
  }
  // backward carry scan
  double X[R];
#pragma unroll
  for (int r = 0; r < R; ++r) X[r] = x[r][0];
#pragma unroll
  for (int t = 0; t < L::LOGP; ++t) {
    const int d = 1 << t;
    const double b = fac[L::BB_OFF + t * P + k];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double o = __shfl_down_sync(KLE_FULL_MASK, X[r], d, P);
      if (k + d < P) X[r] = fma(b, o, X[r]);
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const double o = __shfl_down_sync(KLE_FULL_MASK, X[r], 1, P);
    X[r] = (k == P - 1) ? 0.0 : o;
  }
#pragma unroll
  for (int j = 0; j < MR; ++j) {
    const double sg = fac[L::SIG_OFF + j * P + k];
#pragma unroll
    for (int r = 0; r < R; ++r) x[r][j] = fma(sg, X[r], x[r][j]);
  }
}

}  // namespace kle
