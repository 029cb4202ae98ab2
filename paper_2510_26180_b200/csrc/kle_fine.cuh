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
  // chunk-major: lane k's MR values are contiguous (vector loads)
  static constexpr int L_OFF = 0;        // l_r   (LDL^T sub-diagonal), [k][j]
  static constexpr int INV_OFF = NXP;    // 1/beta_r,                 [k][j]
  static constexpr int AF_OFF = 2 * NXP; // forward scan multipliers  [t][k]
  static constexpr int BB_OFF = 2 * NXP + LOGP * P;  // backward scan multipliers
  static constexpr int DOUBLES = 2 * NXP + 2 * LOGP * P;
};

// Per-lane register copy of the factor rows it owns.
template <int MR, int P>
struct LaneFactors {
  double l[MR], inv[MR];
  double af[FineLayout<MR, P>::LOGP], bb[FineLayout<MR, P>::LOGP];
  double lnx;  // l of the next chunk's first row (0 for the last chunk)
  int nreal;   // rows of this chunk that are real (< nx)

  __device__ __forceinline__ void load(const double* __restrict__ blob, int k, int nx) {
    using L = FineLayout<MR, P>;
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      l[j] = blob[L::L_OFF + k * MR + j];
      inv[j] = blob[L::INV_OFF + k * MR + j];
    }
#pragma unroll
    for (int t = 0; t < L::LOGP; ++t) {
      af[t] = blob[L::AF_OFF + t * P + k];
      bb[t] = blob[L::BB_OFF + t * P + k];
    }
    const double o = __shfl_down_sync(KLE_FULL_MASK, l[0], 1, P);
    lnx = (k == P - 1) ? 0.0 : o;
    nreal = min(MR, max(0, nx - k * MR));
  }
};

// J backward-Euler solves (I + hA) x_new = x + h g0 on the x' = x + h g0
// representation, R right-hand sides in registers, factors in registers.
// Per step and row: five R-dependent FMAs
//   yl_j = x_j - l_j yl_{j-1}            (local forward)
//   y_j  = yl_j + pi_j Y                  (forward stitch, pi_j = prod -l)
//   z'_j = y_j inv_j + kap_j              (kap_j = h g0 (1 + l_{j+1}))
//   xl_j = z'_j - l_{j+1} xl_{j+1}        (local backward)
//   x'_j = xl_j + sig_j X                 (backward stitch, sig_j = prod -l_{+1})
// plus three R-independent products; Y, X come from P-lane carry scans.
// EXP (timing ablation only, wrong results): bit0 skips the carry scans,
// bit1 skips the stitch loops.
template <int MR, int P, int R, int EXP = 0>
__device__ __forceinline__ void be_steps(double (&x)[R][MR], const LaneFactors<MR, P>& f, int k, int J,
                                         double hg) {
  using L = FineLayout<MR, P>;
  constexpr bool SCAN = !(EXP & 1), STITCH = !(EXP & 2);
  for (int it = 0; it < J; ++it) {
#pragma unroll
    for (int j = 1; j < MR; ++j)
#pragma unroll
      for (int r = 0; r < R; ++r) x[r][j] = fma(-f.l[j], x[r][j - 1], x[r][j]);
    double Y[R];
#pragma unroll
    for (int r = 0; r < R; ++r) Y[r] = x[r][MR - 1];
    if constexpr (SCAN) {
#pragma unroll
    for (int t = 0; t < L::LOGP; ++t) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double o = __shfl_up_sync(KLE_FULL_MASK, Y[r], 1 << t, P);
        if (k >= (1 << t)) Y[r] = fma(f.af[t], o, Y[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double o = __shfl_up_sync(KLE_FULL_MASK, Y[r], 1, P);
      Y[r] = (k == 0) ? 0.0 : o;
    }
    }
    if constexpr (STITCH) {
      double pi = 1.0;
#pragma unroll
      for (int j = 0; j < MR; ++j) {
        pi *= -f.l[j];
#pragma unroll
        for (int r = 0; r < R; ++r) x[r][j] = fma(pi, Y[r], x[r][j]);
      }
    }
#pragma unroll
    for (int j = MR - 1; j >= 0; --j) {
      const double ln = (j + 1 < MR) ? f.l[j + 1] : f.lnx;
      const double kap = (j < f.nreal) ? hg * (1.0 + ln) : 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double z = fma(x[r][j], f.inv[j], kap);
        if (j + 1 < MR) z = fma(-ln, x[r][j + 1], z);
        x[r][j] = z;
      }
    }
    double X[R];
#pragma unroll
    for (int r = 0; r < R; ++r) X[r] = x[r][0];
    if constexpr (SCAN) {
#pragma unroll
    for (int t = 0; t < L::LOGP; ++t) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double o = __shfl_down_sync(KLE_FULL_MASK, X[r], 1 << t, P);
        if (k + (1 << t) < P) X[r] = fma(f.bb[t], o, X[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double o = __shfl_down_sync(KLE_FULL_MASK, X[r], 1, P);
      X[r] = (k == P - 1) ? 0.0 : o;
    }
    }
    if constexpr (STITCH) {
      double sg = 1.0;
#pragma unroll
      for (int j = MR - 1; j >= 0; --j) {
        sg *= -((j + 1 < MR) ? f.l[j + 1] : f.lnx);
#pragma unroll
        for (int r = 0; r < R; ++r) x[r][j] = fma(sg, X[r], x[r][j]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Software-pipelined variant: the R right-hand sides form two groups A and B
// (RG each) running half a step apart, so that every phase pairs one group's
// latency-bound carry scan with the other group's row recurrence:
//   S1 forward recurrence   S2 forward scan + stitch
//   S3 backward recurrence  S4 backward scan + stitch
//   schedule: B.S1 B.S2 | (A.S1,B.S3) (A.S2,B.S4) (A.S3,B.S1) (A.S4,B.S2) | ...
// Same arithmetic per right-hand side as be_steps.
template <int MR, int P, int RG>
struct PipeGroup {
  double x[RG][MR];
  double Y[RG], X[RG];
};

template <int MR, int P, int RG>
__device__ __forceinline__ void ph_s1(PipeGroup<MR, P, RG>& g, const LaneFactors<MR, P>& f) {
#pragma unroll
  for (int j = 1; j < MR; ++j)
#pragma unroll
    for (int r = 0; r < RG; ++r) g.x[r][j] = fma(-f.l[j], g.x[r][j - 1], g.x[r][j]);
}

template <int MR, int P, int RG>
__device__ __forceinline__ void ph_s2(PipeGroup<MR, P, RG>& g, const LaneFactors<MR, P>& f, int k) {
  using L = FineLayout<MR, P>;
#pragma unroll
  for (int r = 0; r < RG; ++r) g.Y[r] = g.x[r][MR - 1];
#pragma unroll
  for (int t = 0; t < L::LOGP; ++t)
#pragma unroll
    for (int r = 0; r < RG; ++r) {
      const double o = __shfl_up_sync(KLE_FULL_MASK, g.Y[r], 1 << t, P);
      if (k >= (1 << t)) g.Y[r] = fma(f.af[t], o, g.Y[r]);
    }
#pragma unroll
  for (int r = 0; r < RG; ++r) {
    const double o = __shfl_up_sync(KLE_FULL_MASK, g.Y[r], 1, P);
    g.Y[r] = (k == 0) ? 0.0 : o;
  }
  double pi = 1.0;
#pragma unroll
  for (int j = 0; j < MR; ++j) {
    pi *= -f.l[j];
#pragma unroll
    for (int r = 0; r < RG; ++r) g.x[r][j] = fma(pi, g.Y[r], g.x[r][j]);
  }
}

template <int MR, int P, int RG>
__device__ __forceinline__ void ph_s3(PipeGroup<MR, P, RG>& g, const LaneFactors<MR, P>& f, double hg) {
#pragma unroll
  for (int j = MR - 1; j >= 0; --j) {
    const double ln = (j + 1 < MR) ? f.l[j + 1] : f.lnx;
    const double kap = (j < f.nreal) ? hg * (1.0 + ln) : 0.0;
#pragma unroll
    for (int r = 0; r < RG; ++r) {
      double z = fma(g.x[r][j], f.inv[j], kap);
      if (j + 1 < MR) z = fma(-ln, g.x[r][j + 1], z);
      g.x[r][j] = z;
    }
  }
}

template <int MR, int P, int RG>
__device__ __forceinline__ void ph_s4(PipeGroup<MR, P, RG>& g, const LaneFactors<MR, P>& f, int k) {
  using L = FineLayout<MR, P>;
#pragma unroll
  for (int r = 0; r < RG; ++r) g.X[r] = g.x[r][0];
#pragma unroll
  for (int t = 0; t < L::LOGP; ++t)
#pragma unroll
    for (int r = 0; r < RG; ++r) {
      const double o = __shfl_down_sync(KLE_FULL_MASK, g.X[r], 1 << t, P);
      if (k + (1 << t) < P) g.X[r] = fma(f.bb[t], o, g.X[r]);
    }
#pragma unroll
  for (int r = 0; r < RG; ++r) {
    const double o = __shfl_down_sync(KLE_FULL_MASK, g.X[r], 1, P);
    g.X[r] = (k == P - 1) ? 0.0 : o;
  }
  double sg = 1.0;
#pragma unroll
  for (int j = MR - 1; j >= 0; --j) {
    sg *= -((j + 1 < MR) ? f.l[j + 1] : f.lnx);
#pragma unroll
    for (int r = 0; r < RG; ++r) g.x[r][j] = fma(sg, g.X[r], g.x[r][j]);
  }
}

template <int MR, int P, int R>
__device__ __forceinline__ void be_steps_pipe(double (&x)[R][MR], const LaneFactors<MR, P>& f, int k, int J,
                                              double hg) {
  static_assert(R % 2 == 0, "pipelined solve needs an even number of right-hand sides");
  constexpr int RG = R / 2;
  PipeGroup<MR, P, RG> A, B;
#pragma unroll
  for (int r = 0; r < RG; ++r)
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      A.x[r][j] = x[r][j];
      B.x[r][j] = x[RG + r][j];
    }
  if (J > 0) {
    ph_s1(B, f);
    ph_s2(B, f, k);
    for (int it = 0; it < J - 1; ++it) {
      ph_s1(A, f);
      ph_s3(B, f, hg);
      ph_s2(A, f, k);
      ph_s4(B, f, k);
      ph_s3(A, f, hg);
      ph_s1(B, f);
      ph_s4(A, f, k);
      ph_s2(B, f, k);
    }
    ph_s1(A, f);
    ph_s3(B, f, hg);
    ph_s2(A, f, k);
    ph_s4(B, f, k);
    ph_s3(A, f, hg);
    ph_s4(A, f, k);
  }
#pragma unroll
  for (int r = 0; r < RG; ++r)
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      x[r][j] = A.x[r][j];
      x[RG + r][j] = B.x[r][j];
    }
}

}  // namespace kle
