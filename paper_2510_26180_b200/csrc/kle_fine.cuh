// Fine/coarse backward-Euler propagators for the 1D tridiagonal operator.
//
// Replaces the reference's per-sample, per-step SuperLU solves
// (pintuq/propagators.py:25-39, 121-157) by a register-resident partitioned
// LDL^T solve (see kle_common.cuh for the recurrences). One warp holds
// 32/P independent systems; each lane owns MR rows of R right-hand sides
// that share the sample's factor rows (read from shared memory).
#pragma once
#include "kle_common.cuh"
#ifndef FGR_T
#define FGR_T(i) \
  do {           \
  } while (0)
#endif

namespace kle {

// The eight-lane sweep's tables (kle_fine_pw.cu), packed by fine_factor_kernel<64, 8> in the kernel's shared-
// memory order so that its prologue is a straight 16-byte copy: five tables of 16-byte entries (8 x 512
// doubles), the scan multipliers af[3][8], bb[3][8], rho[8], q[8], the flag
constexpr int kPwTables = 8 * 512, kPwAf = kPwTables, kPwBb = kPwAf + 24, kPwRho = kPwBb + 24, kPwQ = kPwRho + 8,
              kPwFlag = kPwQ + 8, kPwBlobDoubles = kPwFlag + 8;

template <int MR, int P>
struct FineLayout {
  static constexpr int LOGP = ilog2c(P);
  static constexpr int NXP = MR * P;
  // chunk-major: lane k's MR values are contiguous (vector loads)
  static constexpr int L_OFF = 0;        // l_r   (LDL^T sub-diagonal), [k][j]
  static constexpr int INV_OFF = NXP;    // 1/beta_r,                 [k][j]
  static constexpr int AF_OFF = 2 * NXP; // forward scan multipliers  [t][k]
  static constexpr int BB_OFF = 2 * NXP + LOGP * P;  // backward scan multipliers
  // lazy-stitch vectors (be_steps_lazy), chunk-major [k][j]
  static constexpr int PHI_OFF = 2 * NXP + 2 * LOGP * P;  // phi  = Bwd0(pi * inv)
  static constexpr int PHI2_OFF = PHI_OFF + NXP;          // phi2 = Fwd0(phi)
  static constexpr int SG_OFF = PHI2_OFF + NXP;           // sg_j = prod_{i=j+1}^{MR} (-l_i)
  static constexpr int SG2_OFF = SG_OFF + NXP;            // sg2  = Fwd0(sg)
  // Scaled partitioned sweep (be_steps_sc; P = 32 layouts), in the lazy-stitch part of the blob (unused unless
  // KLE_FINE_LAZY): steady state x*_r, chunk-local scaling t_r and 1 / t_r (chunk-major [k][j]), then the scan
  // multipliers of the scaled recurrences, rho_k, q_k and the per-sample "no scaled form" flag
  static constexpr int SC_XS = PHI_OFF, SC_T = PHI2_OFF, SC_IT = SG_OFF;
  static constexpr int SC_AF = SG2_OFF, SC_BB = SC_AF + LOGP * P, SC_RHO = SC_BB + LOGP * P, SC_Q = SC_RHO + P;
  static constexpr int SC_FLAG = SC_Q + P;
  static constexpr bool SC_FITS = 2 * LOGP * P + 2 * P + 1 <= NXP;
  // the (16, 8) blob carries the twisted two-lane tables (kle_fine_tw.cu) from PHI_OFF on; the (16, 32) blob
  // is followed by a (64, 8) blob with the scaled tables for the eight-lane sweep (kle_fine_pw.cu) at PW_OFF
  static constexpr int PW_OFF = 6 * NXP + 2 * LOGP * P;
  static constexpr int DOUBLES =
      6 * NXP + 2 * LOGP * P + ((MR == 16 && P == 8) ? 256 : 0) + ((MR == 16 && P == 32) ? kPwBlobDoubles : 0);
};
constexpr int kTwFlagOff = FineLayout<16, 8>::PHI_OFF + 640;  // per-sample "no twisted form" flag (double)

// Per-lane register copy of the factor rows it owns.
template <int MR, int P>
struct LaneFactors {
  double l[MR], inv[MR];
  double af[FineLayout<MR, P>::LOGP], bb[FineLayout<MR, P>::LOGP];
  double lnx;  // l of the next chunk's first row (0 for the last chunk)
  int nreal;   // rows of this chunk that are real (< nx)

  __device__ __forceinline__ void load(const double* __restrict__ blob, int k, int nx) {
    using L = FineLayout<MR, P>;
    if constexpr (MR % 2 == 0 && (L::DOUBLES % 2) == 0) {  // 16-byte loads (blob rows are 16-byte aligned)
      const double2* lp = reinterpret_cast<const double2*>(blob + L::L_OFF + k * MR);
      const double2* ip = reinterpret_cast<const double2*>(blob + L::INV_OFF + k * MR);
#pragma unroll
      for (int j = 0; j < MR / 2; ++j) {
        const double2 a = __ldg(lp + j), b = __ldg(ip + j);
        l[2 * j] = a.x;
        l[2 * j + 1] = a.y;
        inv[2 * j] = b.x;
        inv[2 * j + 1] = b.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < MR; ++j) {
        l[j] = blob[L::L_OFF + k * MR + j];
        inv[j] = blob[L::INV_OFF + k * MR + j];
      }
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
        Y[r] = fma(f.af[t], o, Y[r]);  // af = 0 for k < 2^t
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
        X[r] = fma(f.bb[t], o, X[r]);  // bb = 0 for k + 2^t >= P
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
// Scaled partitioned step (round 2, after the twisted kernel's rewrite of the recurrences). The steady state
// A x* = g0 removes the source (e = x - x* obeys (I + hA) e_new = e_old), and a chunk-local diagonal scaling
// e_j = t_j w_j, t_0 = 1, t_j = (-l_j) t_{j-1}, turns the in-chunk forward multipliers into 1 and, with
// them, every forward stitch coefficient pi_j / t_j into the same number: per step, row and right-hand side
//   yl_j = w_j + yl_{j-1}                 (DADD, local forward = prefix sums)
//   y_j  = yl_j + C                        (DADD, forward stitch; C = rho_k Y_{k-1}, rho_k = -l_{k,0} t_{k-1,last})
//   z_j  = y_j inv_j                       (DMUL)
//   wl_j = z_j + kk_j wl_{j+1}             (DFMA, local backward; kk_j = l_{j+1}^2)
//   w_j  = wl_j + sg_j X                   (DFMA, backward stitch; sg_last = q_k = -l_{k+1,0} / t_{k,last})
// against five three-operand DFMAs (a DFMA with three register operands issues in 3 cycles, DADD / DMUL in 2)
// and three R-independent products per row (here one). The carry scans keep their shape (Kogge-Stone with
// precomputed multipliers). Pad rows: inv = kk = 0, so they stay 0.
// ---------------------------------------------------------------------------
template <int MR, int P>
struct LaneFactorsSC {
  double inv[MR], kk[MR];  // kk[MR-1] unused
  double af[FineLayout<MR, P>::LOGP], bb[FineLayout<MR, P>::LOGP];
  double rho, q;
  int nreal;

  __device__ __forceinline__ void load(const double* __restrict__ blob, int k, int nx) {
    using L = FineLayout<MR, P>;
    nreal = min(MR, max(0, nx - k * MR));
    const double2* lp = reinterpret_cast<const double2*>(blob + L::L_OFF + k * MR);
    const double2* ip = reinterpret_cast<const double2*>(blob + L::INV_OFF + k * MR);
    double l[MR];
#pragma unroll
    for (int j = 0; j < MR / 2; ++j) {
      const double2 a = lp[j], b = ip[j];
      l[2 * j] = a.x;
      l[2 * j + 1] = a.y;
      inv[2 * j] = (2 * j < nreal) ? b.x : 0.0;
      inv[2 * j + 1] = (2 * j + 1 < nreal) ? b.y : 0.0;
    }
#pragma unroll
    for (int j = 0; j < MR; ++j) kk[j] = (j + 1 < MR) ? l[j + 1] * l[j + 1] : 0.0;
#pragma unroll
    for (int t = 0; t < L::LOGP; ++t) {
      af[t] = blob[L::SC_AF + t * P + k];
      bb[t] = blob[L::SC_BB + t * P + k];
    }
    rho = blob[L::SC_RHO + k];
    q = blob[L::SC_Q + k];
  }
};

template <int MR, int P, int R>
__device__ __forceinline__ void be_steps_sc(double (&x)[R][MR], const LaneFactorsSC<MR, P>& f, int J) {
  using L = FineLayout<MR, P>;
  for (int it = 0; it < J; ++it) {
#pragma unroll
    for (int j = 1; j < MR; ++j)
#pragma unroll
      for (int r = 0; r < R; ++r) x[r][j] += x[r][j - 1];
    double Y[R];
#pragma unroll
    for (int r = 0; r < R; ++r) Y[r] = x[r][MR - 1];
#pragma unroll
    for (int t = 0; t < L::LOGP; ++t) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double o = __shfl_up_sync(KLE_FULL_MASK, Y[r], 1 << t, P);
        Y[r] = fma(f.af[t], o, Y[r]);  // af = 0 for k < 2^t
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) Y[r] = f.rho * __shfl_up_sync(KLE_FULL_MASK, Y[r], 1, P);  // rho_0 = 0
#pragma unroll
    for (int j = MR - 1; j >= 0; --j) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double z = (x[r][j] + Y[r]) * f.inv[j];
        if (j + 1 < MR) z = fma(f.kk[j], x[r][j + 1], z);
        x[r][j] = z;
      }
    }
    double X[R];
#pragma unroll
    for (int r = 0; r < R; ++r) X[r] = x[r][0];
#pragma unroll
    for (int t = 0; t < L::LOGP; ++t) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double o = __shfl_down_sync(KLE_FULL_MASK, X[r], 1 << t, P);
        X[r] = fma(f.bb[t], o, X[r]);  // bb = 0 for k + 2^t >= P
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) X[r] = __shfl_down_sync(KLE_FULL_MASK, X[r], 1, P);  // (q = 0 in the last chunk)
    double sg = f.q;
#pragma unroll
    for (int j = MR - 1; j >= 0; --j) {
#pragma unroll
      for (int r = 0; r < R; ++r) x[r][j] = fma(sg, X[r], x[r][j]);
      if (j > 0) sg *= f.kk[j - 1];
    }
  }
}

// Same step with the R-independent chunk products (pi_j, sig_j, kap_j) read
// from shared memory (cs: [3][MR][P], written once per CTA) instead of being
// recomputed every step: they leave the FP64 pipe for the LSU. The loads are
// volatile so they are not hoisted into registers across the J loop.
__device__ __forceinline__ double lds_f64(unsigned addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

template <int MR, int P>
__device__ __forceinline__ void chunk_products(double* cs, const LaneFactors<MR, P>& f, int k, double hg) {
  double pi = 1.0;
#pragma unroll
  for (int j = 0; j < MR; ++j) {
    pi *= -f.l[j];
    cs[(0 * MR + j) * P + k] = pi;
  }
  double sg = 1.0;
#pragma unroll
  for (int j = MR - 1; j >= 0; --j) {
    const double ln = (j + 1 < MR) ? f.l[j + 1] : f.lnx;
    sg *= -ln;
    cs[(1 * MR + j) * P + k] = sg;
    cs[(2 * MR + j) * P + k] = (j < f.nreal) ? hg * (1.0 + ln) : 0.0;
  }
}

#ifndef KLE_FGR_EXP
#define KLE_FGR_EXP 0  // timing ablation only (wrong results): bit0 skips the carry scans, bit1 the stitch loops
#endif
template <int MR, int P, int R>
__device__ __forceinline__ void be_steps_cs(double (&x)[R][MR], const LaneFactors<MR, P>& f, int k, int J,
                                            const double* cs) {
  using L = FineLayout<MR, P>;
  constexpr bool SCAN = !(KLE_FGR_EXP & 1), STITCH = !(KLE_FGR_EXP & 2);
  const unsigned base = (unsigned)__cvta_generic_to_shared(cs) + (unsigned)(k * sizeof(double));
  for (int it = 0; it < J; ++it) {
    if (it == 1) FGR_T(8);
#pragma unroll
    for (int j = 1; j < MR; ++j)
#pragma unroll
      for (int r = 0; r < R; ++r) x[r][j] = fma(-f.l[j], x[r][j - 1], x[r][j]);
    if (it == 1) FGR_T(9);
    double Y[R];
#pragma unroll
    for (int r = 0; r < R; ++r) Y[r] = x[r][MR - 1];
    if constexpr (SCAN) {
#pragma unroll
    for (int t = 0; t < L::LOGP; ++t) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double o = __shfl_up_sync(KLE_FULL_MASK, Y[r], 1 << t, P);
        Y[r] = fma(f.af[t], o, Y[r]);  // af = 0 for k < 2^t
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double o = __shfl_up_sync(KLE_FULL_MASK, Y[r], 1, P);
      Y[r] = (k == 0) ? 0.0 : o;
    }
    }
    if (it == 1) FGR_T(10);
    if constexpr (STITCH) {
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      const double pi = lds_f64(base + (unsigned)((0 * MR + j) * P * sizeof(double)));
#pragma unroll
      for (int r = 0; r < R; ++r) x[r][j] = fma(pi, Y[r], x[r][j]);
    }
    }
    if (it == 1) FGR_T(11);
#pragma unroll
    for (int j = MR - 1; j >= 0; --j) {
      const double ln = (j + 1 < MR) ? f.l[j + 1] : f.lnx;
      const double kap = lds_f64(base + (unsigned)((2 * MR + j) * P * sizeof(double)));
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double z = fma(x[r][j], f.inv[j], kap);
        if (j + 1 < MR) z = fma(-ln, x[r][j + 1], z);
        x[r][j] = z;
      }
    }
    if (it == 1) FGR_T(12);
    double X[R];
#pragma unroll
    for (int r = 0; r < R; ++r) X[r] = x[r][0];
    if constexpr (SCAN) {
#pragma unroll
    for (int t = 0; t < L::LOGP; ++t) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double o = __shfl_down_sync(KLE_FULL_MASK, X[r], 1 << t, P);
        X[r] = fma(f.bb[t], o, X[r]);  // bb = 0 for k + 2^t >= P
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double o = __shfl_down_sync(KLE_FULL_MASK, X[r], 1, P);
      X[r] = (k == P - 1) ? 0.0 : o;
    }
    }
    if (it == 1) FGR_T(13);
    if constexpr (STITCH) {
#pragma unroll
    for (int j = MR - 1; j >= 0; --j) {
      const double sg = lds_f64(base + (unsigned)((1 * MR + j) * P * sizeof(double)));
#pragma unroll
      for (int r = 0; r < R; ++r) x[r][j] = fma(sg, X[r], x[r][j]);
    }
    }
    if (it == 1) FGR_T(14);
  }
}

// ---------------------------------------------------------------------------
// Lazy-stitch form of the same step (default). With chunk-local recurrences
//   Fwd0(v)_j = v_j - l_j Fwd0(v)_{j-1},  Bwd0(z)_j = z_j - l_{j+1} Bwd0(z)_{j+1}
// (zero carries) one BE step of the partitioned solve is
//   x' = Bwd0(Fwd0(x) inv + kap) + Y phi + X sg,   phi = Bwd0(pi inv)
// with Y, X the forward / backward chunk carries. The state is kept as
// yl = Fwd0(x), and the next step's forward pass is taken on the carry-free
// part, Fwd0(x') = Fwd0(xl0) + Y phi2 + X sg2 (phi2 = Fwd0(phi), sg2 = Fwd0(sg)).
// So neither carry scan waits for a stitch, and each scan runs concurrently
// with an independent local pass:
//   forward scan of last(yl)        ||  xl0 = Bwd0(yl inv + kap)
//   backward scan of xl0_0 + Y phi0 ||  Fwd0(xl0)
//   yl' = Fwd0(xl0) + Y phi2 + X sg2
// Five R-dependent FMAs per row and step, as in be_steps; same arithmetic up
// to the association of the carry terms.
template <int MR, int P, int R>
__device__ __forceinline__ void fwd_local(double (&x)[R][MR], const LaneFactors<MR, P>& f) {
#pragma unroll
  for (int j = 1; j < MR; ++j)
#pragma unroll
    for (int r = 0; r < R; ++r) x[r][j] = fma(-f.l[j], x[r][j - 1], x[r][j]);
}

template <int MR, int P, int R>
__device__ __forceinline__ void fwd_carry(const double (&x)[R][MR], const LaneFactors<MR, P>& f, int k,
                                          double (&Y)[R]) {
  using L = FineLayout<MR, P>;
#pragma unroll
  for (int r = 0; r < R; ++r) Y[r] = x[r][MR - 1];
#pragma unroll
  for (int t = 0; t < L::LOGP; ++t)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double o = __shfl_up_sync(KLE_FULL_MASK, Y[r], 1 << t, P);
      Y[r] = fma(f.af[t], o, Y[r]);  // af = 0 for k < 2^t
    }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const double o = __shfl_up_sync(KLE_FULL_MASK, Y[r], 1, P);
    Y[r] = (k == 0) ? 0.0 : o;
  }
}

template <int MR, int P, int R>
__device__ __forceinline__ void bwd_local(double (&x)[R][MR], const LaneFactors<MR, P>& f, double hg) {
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
}

template <int MR, int P, int R>
__device__ __forceinline__ void bwd_carry(const double (&x)[R][MR], const double (&Y)[R], double phi0,
                                          const LaneFactors<MR, P>& f, int k, double (&X)[R]) {
  using L = FineLayout<MR, P>;
#pragma unroll
  for (int r = 0; r < R; ++r) X[r] = fma(Y[r], phi0, x[r][0]);
#pragma unroll
  for (int t = 0; t < L::LOGP; ++t)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double o = __shfl_down_sync(KLE_FULL_MASK, X[r], 1 << t, P);
      X[r] = fma(f.bb[t], o, X[r]);  // bb = 0 for k + 2^t >= P
    }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const double o = __shfl_down_sync(KLE_FULL_MASK, X[r], 1, P);
    X[r] = (k == P - 1) ? 0.0 : o;
  }
}

// The scans interleaved into the concurrent local pass in source order (one
// shuffle round per segment of rows), so that each shuffle's latency is
// covered by independent row FMAs.
template <int MR, int P, int R>
__device__ __forceinline__ void fwdscan_bwdlocal(double (&x)[R][MR], const LaneFactors<MR, P>& f, int k, double hg,
                                                 double (&Y)[R]) {
  using L = FineLayout<MR, P>;
  constexpr int LOGP = L::LOGP, NS = LOGP + 1, SEG = (MR + NS - 1) / NS;
  double o[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    Y[r] = x[r][MR - 1];
    o[r] = __shfl_up_sync(KLE_FULL_MASK, Y[r], 1, P);
  }
  auto step = [&](int st) {
    if (st < LOGP) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        Y[r] = fma(f.af[st], o[r], Y[r]);
        o[r] = __shfl_up_sync(KLE_FULL_MASK, Y[r], (st + 1 < LOGP) ? (1 << (st + 1)) : 1, P);
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) Y[r] = (k == 0) ? 0.0 : o[r];
    }
  };
#pragma unroll
  for (int jj = 0; jj < MR; ++jj) {
    const int j = MR - 1 - jj;
    const double ln = (j + 1 < MR) ? f.l[j + 1] : f.lnx;
    const double kap = (j < f.nreal) ? hg * (1.0 + ln) : 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double z = fma(x[r][j], f.inv[j], kap);
      if (j + 1 < MR) z = fma(-ln, x[r][j + 1], z);
      x[r][j] = z;
    }
    if ((jj + 1) % SEG == 0 && (jj + 1) / SEG <= NS) step((jj + 1) / SEG - 1);
  }
#pragma unroll
  for (int st = MR / SEG; st < NS; ++st) step(st);
}

template <int MR, int P, int R>
__device__ __forceinline__ void bwdscan_fwdlocal(double (&x)[R][MR], const double (&Y)[R], double phi0,
                                                 const LaneFactors<MR, P>& f, int k, double (&X)[R]) {
  using L = FineLayout<MR, P>;
  constexpr int LOGP = L::LOGP, NS = LOGP + 1, SEG = (MR - 1 + NS - 1) / NS;
  double o[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    X[r] = fma(Y[r], phi0, x[r][0]);
    o[r] = __shfl_down_sync(KLE_FULL_MASK, X[r], 1, P);
  }
  auto step = [&](int st) {
    if (st < LOGP) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        X[r] = fma(f.bb[st], o[r], X[r]);
        o[r] = __shfl_down_sync(KLE_FULL_MASK, X[r], (st + 1 < LOGP) ? (1 << (st + 1)) : 1, P);
      }
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) X[r] = (k == P - 1) ? 0.0 : o[r];
    }
  };
#pragma unroll
  for (int j = 1; j < MR; ++j) {
#pragma unroll
    for (int r = 0; r < R; ++r) x[r][j] = fma(-f.l[j], x[r][j - 1], x[r][j]);
    if (SEG > 0 && j % SEG == 0 && j / SEG <= NS) step(j / SEG - 1);
  }
#pragma unroll
  for (int st = (SEG > 0 ? (MR - 1) / SEG : 0); st < NS; ++st) step(st);
}

// x (materialised) -> J steps -> x (materialised). blob: this sample's factor
// blob (the lazy vectors are read from it; the lane's l/inv/scan multipliers
// come in f).
template <int MR, int P, int R>
__device__ __forceinline__ void be_steps_lazy(double (&x)[R][MR], const LaneFactors<MR, P>& f,
                                              const double* __restrict__ blob, int k, int J, double hg) {
  using L = FineLayout<MR, P>;
  if (J <= 0) return;
  double phi2[MR], sg2[MR];
#pragma unroll
  for (int j = 0; j < MR; ++j) {
    phi2[j] = blob[L::PHI2_OFF + k * MR + j];
    sg2[j] = blob[L::SG2_OFF + k * MR + j];
  }
  const double phi0 = blob[L::PHI_OFF + k * MR];
  double Y[R], X[R];
  fwd_local<MR, P, R>(x, f);
  for (int it = 0; it < J - 1; ++it) {
    fwdscan_bwdlocal<MR, P, R>(x, f, k, hg, Y);
    bwdscan_fwdlocal<MR, P, R>(x, Y, phi0, f, k, X);
#pragma unroll
    for (int j = MR - 1; j >= 0; --j)
#pragma unroll
      for (int r = 0; r < R; ++r) x[r][j] = fma(X[r], sg2[j], fma(Y[r], phi2[j], x[r][j]));
  }
  fwdscan_bwdlocal<MR, P, R>(x, f, k, hg, Y);
  bwd_carry<MR, P, R>(x, Y, phi0, f, k, X);
#pragma unroll
  for (int j = 0; j < MR; ++j) {
    const double phi = blob[L::PHI_OFF + k * MR + j], sg = blob[L::SG_OFF + k * MR + j];
#pragma unroll
    for (int r = 0; r < R; ++r) x[r][j] = fma(X[r], sg, fma(Y[r], phi, x[r][j]));
  }
}

// ---------------------------------------------------------------------------
// Overlapped lazy-stitch step with the R-independent row vectors in shared
// memory (lz: [5][MR][P] = kap, phi2, sg2, phi, sg; built once per CTA by
// lazy_tables with the operations of fine_factor_kernel's lazy block). Same
// algebra as be_steps_lazy; the state between steps is yl = Fwd0(x). Every
// carry scan runs in the shadow of row work that does not depend on it:
//   A  forward scan of last(yl)            ||  xl0 = Bwd0(yl inv + kap)
//   B  backward scan of xl0_0 + Y phi_0    ||  w = Fwd0(xl0), then w += Y phi2 (one row behind the chain)
//   C  yl' = w + X sg2, last row first so that the next step's forward scan
//      starts under the remaining rows
// Five R-dependent FMAs per row and step, as in be_steps. One shuffle round
// is consumed per SEG rows (a round's latency ~ SEG R chain FMAs).
template <int MR, int P>
__device__ __forceinline__ void lazy_tables(double* lz, const LaneFactors<MR, P>& f, int k, double hg) {
  double phi[MR], sg[MR];
  double pi = 1.0;
#pragma unroll
  for (int j = 0; j < MR; ++j) {
    pi *= -f.l[j];
    phi[j] = pi * f.inv[j];
  }
#pragma unroll
  for (int j = MR - 2; j >= 0; --j) phi[j] = fma(-f.l[j + 1], phi[j + 1], phi[j]);
  double g = 1.0;
#pragma unroll
  for (int j = MR - 1; j >= 0; --j) {
    const double ln = (j + 1 < MR) ? f.l[j + 1] : f.lnx;
    g *= -ln;
    sg[j] = g;
    lz[(0 * MR + j) * P + k] = (j < f.nreal) ? hg * (1.0 + ln) : 0.0;
    lz[(3 * MR + j) * P + k] = phi[j];
    lz[(4 * MR + j) * P + k] = g;
  }
  double p2 = phi[0], s2 = sg[0];
  lz[(1 * MR + 0) * P + k] = p2;
  lz[(2 * MR + 0) * P + k] = s2;
#pragma unroll
  for (int j = 1; j < MR; ++j) {
    p2 = fma(-f.l[j], p2, phi[j]);
    s2 = fma(-f.l[j], s2, sg[j]);
    lz[(1 * MR + j) * P + k] = p2;
    lz[(2 * MR + j) * P + k] = s2;
  }
}

template <int MR, int P, int R>
__device__ __forceinline__ void be_steps_lz(double (&x)[R][MR], const LaneFactors<MR, P>& f, int k, int J,
                                            const double* lz) {
  using L = FineLayout<MR, P>;
  constexpr int LOGP = L::LOGP, NS = LOGP + 1;
  constexpr int SEG = (MR + NS - 1) / NS;  // rows per shuffle round
  if (J <= 0) return;
  const unsigned base = (unsigned)__cvta_generic_to_shared(lz) + (unsigned)(k * sizeof(double));
  auto tab = [&](int t, int j) { return lds_f64(base + (unsigned)((t * MR + j) * P * sizeof(double))); };
  double Y[R], X[R], o[R];
  // one consumption point of a scan: st < LOGP multiplies and re-shuffles, st = LOGP takes the neighbour's value
  auto ystep = [&](int st) {
    if (st < LOGP) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        Y[r] = fma(f.af[st], o[r], Y[r]);  // af = 0 for k < 2^st
        o[r] = __shfl_up_sync(KLE_FULL_MASK, Y[r], (st + 1 < LOGP) ? (1 << (st + 1)) : 1, P);
      }
    } else if (st == LOGP) {
#pragma unroll
      for (int r = 0; r < R; ++r) Y[r] = (k == 0) ? 0.0 : o[r];
    }
  };
  auto xstep = [&](int st) {
    if (st < LOGP) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        X[r] = fma(f.bb[st], o[r], X[r]);  // bb = 0 for k + 2^st >= P
        o[r] = __shfl_down_sync(KLE_FULL_MASK, X[r], (st + 1 < LOGP) ? (1 << (st + 1)) : 1, P);
      }
    } else if (st == LOGP) {
#pragma unroll
      for (int r = 0; r < R; ++r) X[r] = (k == P - 1) ? 0.0 : o[r];
    }
  };
  // phase A: xl0 = Bwd0(yl inv + kap) with the forward scan (round 0 already issued) consumed along the rows
  auto phaseA = [&]() {
#pragma unroll
    for (int jj = 0; jj < MR; ++jj) {
      const int j = MR - 1 - jj;
      const double ln = (j + 1 < MR) ? f.l[j + 1] : f.lnx;
      const double kap = tab(0, j);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double z = fma(x[r][j], f.inv[j], kap);
        if (j + 1 < MR) z = fma(-ln, x[r][j + 1], z);
        x[r][j] = z;
      }
      if ((jj + 1) % SEG == 0 && (jj + 1) / SEG <= NS) ystep((jj + 1) / SEG - 1);
    }
#pragma unroll
    for (int st = MR / SEG; st < NS; ++st) ystep(st);
  };

#pragma unroll
  for (int j = 1; j < MR; ++j)
#pragma unroll
    for (int r = 0; r < R; ++r) x[r][j] = fma(-f.l[j], x[r][j - 1], x[r][j]);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    Y[r] = x[r][MR - 1];
    o[r] = __shfl_up_sync(KLE_FULL_MASK, Y[r], 1, P);
  }
  const double phi0 = tab(3, 0);
  for (int it = 0; it < J - 1; ++it) {
    phaseA();
    // phase B
#pragma unroll
    for (int r = 0; r < R; ++r) {
      X[r] = fma(Y[r], phi0, x[r][0]);
      o[r] = __shfl_down_sync(KLE_FULL_MASK, X[r], 1, P);
    }
#pragma unroll
    for (int j = 1; j <= MR; ++j) {
      if (j < MR) {
#pragma unroll
        for (int r = 0; r < R; ++r) x[r][j] = fma(-f.l[j], x[r][j - 1], x[r][j]);
      }
      const double p2 = tab(1, j - 1);  // row j - 1 has left the chain
#pragma unroll
      for (int r = 0; r < R; ++r) x[r][j - 1] = fma(Y[r], p2, x[r][j - 1]);
      if (j % SEG == 0 && j / SEG <= NS) xstep(j / SEG - 1);
    }
#pragma unroll
    for (int st = MR / SEG; st < NS; ++st) xstep(st);
    // phase C, the last row first: it feeds round 0 of the next forward scan
    {
      const double s2 = tab(2, MR - 1);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        x[r][MR - 1] = fma(X[r], s2, x[r][MR - 1]);
        Y[r] = x[r][MR - 1];
        o[r] = __shfl_up_sync(KLE_FULL_MASK, Y[r], 1, P);
      }
    }
#pragma unroll
    for (int j = MR - 2; j >= 0; --j) {
      const double s2 = tab(2, j);
#pragma unroll
      for (int r = 0; r < R; ++r) x[r][j] = fma(X[r], s2, x[r][j]);
    }
  }
  // last step: materialise x' = xl0 + Y phi + X sg (the Y part runs under the backward scan)
  phaseA();
  {
    const double ph = tab(3, 0);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      x[r][0] = fma(Y[r], ph, x[r][0]);
      X[r] = x[r][0];
      o[r] = __shfl_down_sync(KLE_FULL_MASK, X[r], 1, P);
    }
  }
#pragma unroll
  for (int j = 1; j < MR; ++j) {
    const double ph = tab(3, j);
#pragma unroll
    for (int r = 0; r < R; ++r) x[r][j] = fma(Y[r], ph, x[r][j]);
    if (j % SEG == 0 && j / SEG <= NS) xstep(j / SEG - 1);
  }
#pragma unroll
  for (int st = (MR - 1) / SEG; st < NS; ++st) xstep(st);
#pragma unroll
  for (int j = 0; j < MR; ++j) {
    const double sgj = tab(4, j);
#pragma unroll
    for (int r = 0; r < R; ++r) x[r][j] = fma(X[r], sgj, x[r][j]);
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
      g.Y[r] = fma(f.af[t], o, g.Y[r]);
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
      g.X[r] = fma(f.bb[t], o, g.X[r]);
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
