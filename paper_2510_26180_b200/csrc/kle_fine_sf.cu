// Fine propagator, shared-memory-factor variant ("SF").
//
// Same LDL^T recurrences as kle_fine.cuh (pintuq/propagators.py:25-39,
// 121-157) but the per-row factors live in shared memory (one copy per CTA,
// shared by every right-hand side of the sample), so registers hold only the
// R x MR state and the kernel can run 4 CTAs per SM: the carry-scan latency of
// one warp is hidden behind the row recurrences of the others.
//
// Row record (6 doubles) per chunk row j of lane k, stored as three planes of
// 16-byte pairs, [plane][j][k] (consecutive lanes read consecutive pairs; the
// two P = 16 systems of a warp read the same pair, a broadcast):
//   plane 0 (sig_j, l_j) | plane 1 (inv_j, pihat_j) | plane 2 (kap_j, l_{j+1})
// Per step: forward loop x_j += sig_j X (previous back-stitch), yl_j = x_j -
// l_j yl_{j-1}; forward scan; backward loop z'_j = yl_j inv_j + pihat_j Y +
// kap_j, xl_j = z'_j - l_{j+1} xl_{j+1}; backward scan. Five FMAs per row.
#include "kle_fine.cuh"
#include "kle_internal.h"

namespace kle {

template <int MR, int P>
struct SfLayout {
  static constexpr int LOGP = ilog2c(P);
  static constexpr int NXP = MR * P;
  static constexpr int ROW = 6;
  static constexpr int AF_OFF = ROW * NXP;
  static constexpr int BB_OFF = ROW * NXP + LOGP * P;
  static constexpr int DOUBLES = ROW * NXP + 2 * LOGP * P;
  __host__ __device__ static constexpr int at(int q, int j, int k) { return ((q * MR + j) * P + k) * 2; }
};

template <int MR, int P>
__global__ void sf_factor_kernel(const double* __restrict__ dia, const double* __restrict__ off,
                                 double* __restrict__ blob, int M, int nx, double h, double g0) {
  using L = SfLayout<MR, P>;
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= M) return;
  const double* d = dia + (size_t)s * nx;
  const double* e = off + (size_t)s * nx;
  double* b = blob + (size_t)s * L::DOUBLES;
  auto el = [&](int row, int q) -> double& { return b[L::at(q / 2, row % MR, row / MR) + (q % 2)]; };
  double beta_prev = 1.0;
  for (int row = 0; row < L::NXP; ++row) {
    double l = 0.0, inv = 1.0;
    if (row < nx) {
      const double D = fma(h, d[row], 1.0);
      double beta = D;
      if (row > 0) {
        const double E = h * e[row - 1];
        l = E / beta_prev;
        beta = fma(-l, E, D);
      }
      inv = 1.0 / beta;
      beta_prev = beta;
    }
    el(row, 1) = l;
    el(row, 2) = inv;
  }
  const double hg = h * g0;
  double pie[P], sigs[P];
  for (int k = 0; k < P; ++k) {
    double pi = 1.0;
    for (int j = 0; j < MR; ++j) {
      const int row = k * MR + j;
      pi *= -el(row, 1);
      el(row, 3) = pi * el(row, 2);
      const double lnext = (row + 1 < L::NXP) ? el(row + 1, 1) : 0.0;
      el(row, 4) = (row < nx) ? hg * (1.0 + lnext) : 0.0;
      el(row, 5) = (j + 1 < MR) ? lnext : 0.0;
    }
    pie[k] = pi;
    double sg = 1.0;
    for (int j = MR - 1; j >= 0; --j) {
      const int row = k * MR + j;
      const double lnext = (row + 1 < L::NXP) ? el(row + 1, 1) : 0.0;
      sg *= -lnext;
      el(row, 0) = sg;
    }
    sigs[k] = sg;
  }
  for (int t = 0; t < L::LOGP; ++t) {
    const int dd = 1 << t;
    for (int k = 0; k < P; ++k) {
      double af = 0.0, bb = 0.0;
      if (k >= dd) {
        af = 1.0;
        for (int q = k - dd + 1; q <= k; ++q) af *= pie[q];
      }
      if (k + dd < P) {
        bb = 1.0;
        for (int q = k; q <= k + dd - 1; ++q) bb *= sigs[q];
      }
      b[L::AF_OFF + t * P + k] = af;
      b[L::BB_OFF + t * P + k] = bb;
    }
  }
}

// Shared-memory pair load through a 32-bit shared address (volatile: kept in
// program order, never hoisted out of the step loop into registers, which
// would spill; the row loops issue them a few rows ahead of use).
__device__ __forceinline__ double2 lds2(unsigned addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

template <int MR, int P, int R>
__device__ __forceinline__ void sf_steps(double (&x)[R][MR], const double* __restrict__ fac, int k, int J) {
  using L = SfLayout<MR, P>;
  double af[L::LOGP], bb[L::LOGP];
#pragma unroll
  for (int t = 0; t < L::LOGP; ++t) {
    af[t] = fac[L::AF_OFF + t * P + k];
    bb[t] = fac[L::BB_OFF + t * P + k];
  }
  double X[R];
#pragma unroll
  for (int r = 0; r < R; ++r) X[r] = 0.0;
  const unsigned fbase0 = (unsigned)__cvta_generic_to_shared(fac) + (unsigned)(k * 2 * sizeof(double));
  for (int it = 0; it < J; ++it) {
    unsigned fb = fbase0;
    asm volatile("" : "+r"(fb));
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      const double2 sl = lds2(fb + (unsigned)(L::at(0, j, 0) * sizeof(double)));
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double v = fma(sl.x, X[r], x[r][j]);
        if (j > 0) v = fma(-sl.y, x[r][j - 1], v);
        x[r][j] = v;
      }
    }
    double Y[R];
#pragma unroll
    for (int r = 0; r < R; ++r) Y[r] = x[r][MR - 1];
#pragma unroll
    for (int t = 0; t < L::LOGP; ++t)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double o = __shfl_up_sync(KLE_FULL_MASK, Y[r], 1 << t, P);
        Y[r] = fma(af[t], o, Y[r]);  // af = 0 for k < 2^t
      }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double o = __shfl_up_sync(KLE_FULL_MASK, Y[r], 1, P);
      Y[r] = (k == 0) ? 0.0 : o;
    }
#pragma unroll
    for (int j = MR - 1; j >= 0; --j) {
      const double2 ip = lds2(fb + (unsigned)(L::at(1, j, 0) * sizeof(double)));
      const double2 kl = lds2(fb + (unsigned)(L::at(2, j, 0) * sizeof(double)));
#pragma unroll
      for (int r = 0; r < R; ++r) {
        double z = fma(x[r][j], ip.x, fma(ip.y, Y[r], kl.x));
        if (j < MR - 1) z = fma(-kl.y, x[r][j + 1], z);
        x[r][j] = z;
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) X[r] = x[r][0];
#pragma unroll
    for (int t = 0; t < L::LOGP; ++t)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double o = __shfl_down_sync(KLE_FULL_MASK, X[r], 1 << t, P);
        X[r] = fma(bb[t], o, X[r]);  // bb = 0 for k + 2^t >= P
      }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double o = __shfl_down_sync(KLE_FULL_MASK, X[r], 1, P);
      X[r] = (k == P - 1) ? 0.0 : o;
    }
  }
#pragma unroll
  for (int j = 0; j < MR; ++j) {
    const double sg = fac[L::at(0, j, k)];
#pragma unroll
    for (int r = 0; r < R; ++r) x[r][j] = fma(sg, X[r], x[r][j]);
  }
}

template <int MR, int P, int R, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) fgr_sf_kernel(FgrArgs a) {
  using L = SfLayout<MR, P>;
  constexpr int SLOTS = 32 / P;
  constexpr int NC = (NT / 32) * SLOTS * R;
  extern __shared__ __align__(16) double sm[];
  double* fac = sm;  // [DOUBLES]
  const int s = blockIdx.x;
  if (a.active && a.active[s] != KLE_SAMPLE_ACTIVE) return;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int k = lane % P, slot = lane / P;
  const int nx = a.nx, N = a.N;
  const size_t sbase = (size_t)s * N * nx;
  const double* __restrict__ U = a.U;
  double* __restrict__ Rout = a.Rout;
  {
    const double* gb = a.ffac + (size_t)s * L::DOUBLES;
    for (int i = tid; i < L::DOUBLES / 2; i += NT)
      reinterpret_cast<double2*>(fac)[i] = __ldg(reinterpret_cast<const double2*>(gb) + i);
  }
  int n[R];
#pragma unroll
  for (int r = 0; r < R; ++r) n[r] = blockIdx.y * NC + (w * SLOTS + slot) * R + r;
  const double hg = a.dt * a.g0;
  double x[R][MR];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      const int row = k * MR + j;
      double v = 0.0;
      if (row < nx && n[r] < N) v = __ldg((n[r] == 0) ? a.u0 + row : U + sbase + (size_t)(n[r] - 1) * nx + row) + hg;
      x[r][j] = v;
    }
  __syncthreads();
  sf_steps<MR, P, R>(x, fac, k, a.J);
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int j = 0; j < MR; ++j) x[r][j] = (k * MR + j < nx) ? x[r][j] - hg : 0.0;
  // epilogue: R_n = scaling_n ((I + dT A) F_n - prev_n); operator rows and the
  // prev rows re-read through the read-only path (L2-resident), in batches of
  // EB rows to bound the live registers
  constexpr int EB = MR < 8 ? MR : 8;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const double left = __shfl_up_sync(KLE_FULL_MASK, x[r][MR - 1], 1, P);
    const double right = __shfl_down_sync(KLE_FULL_MASK, x[r][0], 1, P);
    if (n[r] >= N) continue;
    const double sc = a.scaling[n[r]];
    const double* pvr = U + ((n[r] == 0) ? sbase + (size_t)(N - 1) * nx : sbase + (size_t)(n[r] - 1) * nx);
    const double* dia = a.dia + (size_t)s * nx;
    const double* off = a.off + (size_t)s * nx;
    const double pmul = (n[r] == 0) ? a.alpha : 1.0;
#pragma unroll
    for (int j0 = 0; j0 < MR; j0 += EB) {
      double pv[EB], dd[EB], ee[EB + 1];
#pragma unroll
      for (int jj = 0; jj <= EB; ++jj) {
        const int row = k * MR + j0 + jj;
        if (jj < EB) {
          pv[jj] = (row < nx) ? __ldg(pvr + row) : 0.0;
          dd[jj] = (row < nx) ? __ldg(dia + row) : 0.0;
        }
        ee[jj] = (row >= 1 && row < nx) ? __ldg(off + row - 1) : 0.0;  // couples rows row-1, row
      }
#pragma unroll
      for (int jj = 0; jj < EB; ++jj) {
        const int j = j0 + jj, row = k * MR + j;
        if (row >= nx) continue;
        const double xm = (j > 0) ? x[r][j - 1] : left;
        const double xp = (j < MR - 1) ? x[r][j + 1] : right;
        const double Ax = fma(ee[jj], xm, fma(dd[jj], x[r][j], ee[jj + 1] * xp));
        const double rhs = fma(a.dT, Ax, x[r][j]) - pmul * pv[jj];
        Rout[sbase + (size_t)n[r] * nx + row] = sc * rhs;
      }
    }
  }
}

template <int MR, int P, int R, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) sweep_sf_kernel(SweepArgs a) {
  using L = SfLayout<MR, P>;
  constexpr int SLOTS = 32 / P;
  constexpr int NC = (NT / 32) * SLOTS * R;
  extern __shared__ __align__(16) double sm[];
  double* fac = sm;
  const int s = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int k = lane % P, slot = lane / P;
  const int nx = a.nx, Q = a.Q;
  {
    const double* gb = a.fac + (size_t)s * L::DOUBLES;
    for (int i = tid; i < L::DOUBLES / 2; i += NT)
      reinterpret_cast<double2*>(fac)[i] = reinterpret_cast<const double2*>(gb)[i];
  }
  int q[R];
#pragma unroll
  for (int r = 0; r < R; ++r) q[r] = blockIdx.y * NC + (w * SLOTS + slot) * R + r;
  const double hg = a.h * a.g0;
  double x[R][MR];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      const int row = k * MR + j;
      x[r][j] = (row < nx && q[r] < Q) ? a.start[((size_t)s * Q + q[r]) * nx + row] + hg : 0.0;
    }
  __syncthreads();
  for (int g = 0; g < a.nseg; ++g) {
    sf_steps<MR, P, R>(x, fac, k, a.J);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (q[r] >= Q) continue;
      double* o = a.out + (((size_t)s * Q + q[r]) * a.nseg + g) * nx;
#pragma unroll
      for (int j = 0; j < MR; ++j) {
        const int row = k * MR + j;
        if (row < nx) o[row] = x[r][j] - hg;
      }
    }
  }
}

template <int MR, int P, int R, int MINB>
struct SfInst {
  static constexpr int NT = 128;
  static constexpr int NC = (NT / 32) * (32 / P) * R;
  static int factor(const double* dia, const double* off, double* blob, int M, int nx, double h, double g0,
                    cudaStream_t st) {
    sf_factor_kernel<MR, P><<<(M + 63) / 64, 64, 0, st>>>(dia, off, blob, M, nx, h, g0);
    return check_launch("sf_factor_kernel");
  }
  static int fgr(const FgrArgs& a, cudaStream_t st) {
    using L = SfLayout<MR, P>;
    if (a.F_given) return set_error(KLE_ERR_UNSUPPORTED, "sf fgr: F_given uses the register variant");
    const size_t smem = (size_t)L::DOUBLES * sizeof(double);
    static PerDeviceOnce attr_once;
    if (int rc = once_per_device(attr_once, "kle_fine_sf: cudaFuncSetAttribute", [&] {
          return cudaFuncSetAttribute(fgr_sf_kernel<MR, P, R, NT, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           200 * 1024);
        }))
      return rc;
    fgr_sf_kernel<MR, P, R, NT, MINB><<<dim3(a.M, (a.N + NC - 1) / NC), NT, smem, st>>>(a);
    return check_launch("fgr_sf_kernel");
  }
  static int sweep(const SweepArgs& a, cudaStream_t st) {
    using L = SfLayout<MR, P>;
    const size_t smem = (size_t)L::DOUBLES * sizeof(double);
    static PerDeviceOnce attr_once;
    if (int rc = once_per_device(attr_once, "kle_fine_sf: cudaFuncSetAttribute", [&] {
          return cudaFuncSetAttribute(sweep_sf_kernel<MR, P, R, NT, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           200 * 1024);
        }))
      return rc;
    sweep_sf_kernel<MR, P, R, NT, MINB><<<dim3(a.M, (a.Q + NC - 1) / NC), NT, smem, st>>>(a);
    return check_launch("sweep_sf_kernel");
  }
};

#define KLE_SF_DISPATCH(MR_, P_, R_, MB_, CALL) \
  if (lay.MR == MR_ && lay.P == P_ && lay.R == R_ && lay.pipe == MB_) return SfInst<MR_, P_, R_, MB_>::CALL;
#define KLE_SF_ALL(CALL)                  \
  KLE_SF_DISPATCH(16, 32, 3, 4, CALL)     \
  KLE_SF_DISPATCH(16, 32, 3, 3, CALL)     \
  KLE_SF_DISPATCH(16, 32, 2, 4, CALL)     \
  KLE_SF_DISPATCH(16, 32, 4, 3, CALL)     \
  KLE_SF_DISPATCH(8, 16, 2, 4, CALL)      \
  KLE_SF_DISPATCH(8, 16, 4, 4, CALL)      \
  KLE_SF_DISPATCH(8, 32, 4, 4, CALL)      \
  KLE_SF_DISPATCH(32, 16, 2, 2, CALL)     \
  KLE_SF_DISPATCH(32, 16, 1, 3, CALL)     \
  KLE_SF_DISPATCH(16, 32, 3, 2, CALL)     \
  KLE_SF_DISPATCH(32, 16, 4, 3, CALL)     \
  KLE_SF_DISPATCH(32, 16, 3, 3, CALL)     \
  KLE_SF_DISPATCH(32, 16, 2, 4, CALL)     \
  KLE_SF_DISPATCH(32, 16, 4, 2, CALL)

int sf_blob_doubles(int MR, int P) {
  int logp = 0;
  while ((1 << logp) < P) ++logp;
  return 6 * MR * P + 2 * logp * P;
}
int sf_factor(FineLayoutRT lay, const double* dia, const double* off, double* blob, int M, int nx, double h,
              double g0, cudaStream_t st) {
  KLE_SF_ALL(factor(dia, off, blob, M, nx, h, g0, st))
  return set_error(KLE_ERR_UNSUPPORTED, "sf: variant");
}
int sf_fgr(FineLayoutRT lay, const FgrArgs& a, cudaStream_t st) {
  KLE_SF_ALL(fgr(a, st))
  return set_error(KLE_ERR_UNSUPPORTED, "sf: variant");
}
int sf_sweep(FineLayoutRT lay, const SweepArgs& a, cudaStream_t st) {
  KLE_SF_ALL(sweep(a, st))
  return set_error(KLE_ERR_UNSUPPORTED, "sf: variant");
}

}  // namespace kle
