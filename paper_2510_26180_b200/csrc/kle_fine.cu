// Fine propagator F, coarse propagator G and the fused "F + CGC right-hand
// side" kernel for the 1D KL-coefficient diffusion operator.
//
// Reference counterparts:
//   propagate_fine        pintuq/propagators.py:121-145  (J x splu.solve)
//   propagate_coarse      pintuq/propagators.py:148-157
//   assemble_rhs_blocks   pintuq/pcgc.py:175-197
//   cgc_correct (rhs)     pintuq/pcgc.py:233-237
//
// The fused kernel uses the identity (G = (I + dT A)^{-1}(prev + dT g)):
//   rhs_n = dT (A b_n + g) + b_n,  b_n = F_n - G(prev_n)
//         = (I + dT A) F_n - prev_n
// so the coarse solve of the reference collapses to one matvec.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "kle_common.cuh"
namespace kle {
#ifdef KLE_FGR_TIMING
// debug: per-CTA phase timestamps (SM clock), CTAs [KLE_FGR_T0, KLE_FGR_T0 + 4096)
#ifndef KLE_FGR_T0
#define KLE_FGR_T0 60000
#endif
__device__ long long g_fgr_t[4096][16];
#define FGR_T(i)                                                                              \
  do {                                                                                        \
    if (threadIdx.x == 0 && blockIdx.x >= KLE_FGR_T0 && blockIdx.x < KLE_FGR_T0 + 4096)       \
      g_fgr_t[blockIdx.x - KLE_FGR_T0][i] = (i == 7) ? (long long)__smid() : clock64();       \
    if (i == 7 && threadIdx.x == 0 && blockIdx.x >= KLE_FGR_T0 && blockIdx.x < KLE_FGR_T0 + 4096) {  \
      unsigned w_;                                                                            \
      asm volatile("mov.u32 %0, %%warpid;" : "=r"(w_));                                       \
      g_fgr_t[blockIdx.x - KLE_FGR_T0][15] = w_;                                              \
    }                                                                                         \
  } while (0)
__device__ __forceinline__ unsigned __smid() {
  unsigned v;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(v));
  return v;
}
extern "C" int kle_debug_fgr_timing(long long* host) { return (int)cudaMemcpyFromSymbol(host, g_fgr_t, sizeof(g_fgr_t)); }
#else
#define FGR_T(i) \
  do {           \
  } while (0)
#endif
}  // namespace kle
#include "kle_fine.cuh"
#include "kle_internal.h"

#ifndef KLE_FINE_LAZY
#define KLE_FINE_LAZY 0  // lazy-stitch step (kle_fine.cuh); measured slower, kept for A/B
#endif
#ifndef KLE_FINE_CS
#define KLE_FINE_CS 0  // chunk products from shared memory (be_steps_cs) for every variant: slower at c2
                       // (5.79 vs 5.43 ms), A/B only; the one-warp variants (NT = 32) always use them
#endif

#ifndef KLE_FGR_LZ
#define KLE_FGR_LZ 0  // 1: one-warp variants use the overlapped lazy-stitch step (be_steps_lz): solo warp 1,082 vs
                      // 1,301 cycles per step, but 4.69 vs 4.67 ms per 131k c4 launch at 2 warps per sub-partition (A/B)
#endif

namespace kle {



// ---------------------------------------------------------------------------
// Factor kernel: one warp builds the blobs of 32 / P samples, P lanes per sample (c4: four samples; with
// one sample per warp the kernel, a 128-step division chain in a single lane, took 8.7 ms per 1M samples):
// the operator rows are loaded coalesced into shared memory, lane 0 of each group runs the sequential
// LDL^T of T = I + h A, the group's lanes build the chunk / scan tables of the partitioned solve (layout:
// kle_common.cuh) with the same operations in the same order as the one-thread-per-sample original
// (bit-identical blob), and the warp stores the blobs coalesced.
// ---------------------------------------------------------------------------
template <int MR, int P>
struct FactorSmem {
  using L = FineLayout<MR, P>;
  static constexpr int SPW = 32 / P;                                  // samples per warp
  // scaled partitioned sweep (be_steps_sc): P = 32 layouts carry its tables in the lazy-stitch part
  static constexpr bool SC = !KLE_FINE_LAZY && (P == 32 || (MR == 64 && P == 8)) && L::SC_FITS;
  static constexpr int BS = KLE_FINE_LAZY ? L::DOUBLES : (SC ? L::SC_FLAG + 1 : L::PHI_OFF);  // staged (= stored) blob doubles
  static constexpr int PER = BS + 2 * L::NXP;                         // + the operator rows
  static constexpr size_t bytes = sizeof(double) * (size_t)SPW * PER;
};

template <int MR, int P>
__global__ void __launch_bounds__(32) fine_factor_kernel(const double* __restrict__ dia,
                                                         const double* __restrict__ off, double* __restrict__ blob,
                                                         int M, int nx, double h, double g0, int sc_on,
                                                         int stride, int offset) {
  using L = FineLayout<MR, P>;
  using FS = FactorSmem<MR, P>;
  constexpr int NXP = L::NXP;
  extern __shared__ __align__(16) double fsm[];
  const int lane = threadIdx.x, grp = lane / P, k = lane % P;
  const int s0 = blockIdx.x * FS::SPW;
  double* b = fsm + grp * FS::PER;  // [BS] the sample's blob
  double* dd = b + FS::BS;          // [NXP]
  double* ee = dd + NXP;            // [NXP]: ee[i] couples rows i, i+1
  for (int q = 0; q < FS::SPW; ++q) {
    const int sq = s0 + q;
    double* dq = fsm + q * FS::PER + FS::BS;
    for (int i = lane; i < NXP; i += 32) {
      dq[i] = (sq < M && i < nx) ? dia[(size_t)sq * nx + i] : 0.0;
      dq[NXP + i] = (sq < M && i < nx) ? off[(size_t)sq * nx + i] : 0.0;
    }
  }
  __syncwarp();
  if (k == 0) {  // LDL^T of I + hA: l_r (row r couples to r-1), inv_r = 1/beta_r; pad rows identity
    double beta_prev = 1.0;
    for (int row = 0; row < NXP; ++row) {
      double l = 0.0, inv = 1.0;
      if (row < nx) {
        const double D = fma(h, dd[row], 1.0);
        double beta = D;
        if (row > 0) {
          const double E = h * ee[row - 1];
          l = E / beta_prev;
          beta = fma(-l, E, D);
        }
        inv = 1.0 / beta;
        beta_prev = beta;
      }
      b[L::L_OFF + row] = l;
      b[L::INV_OFF + row] = inv;
    }
  }
  bool sc_bad = false;
  if (FS::SC && sc_on) {
    // steady state A x* = g0 (Thomas, one division per row; A needs positive pivots), lane 1, before dd / ee
    // are reused; the elimination multipliers wait in the 1/t slots
    if (k == 1) {
      double* xs = b + L::SC_XS;
      double* cw = b + L::SC_IT;
      if (g0 != 0.0) {
        double ib = 1.0 / dd[0];
        sc_bad |= !(dd[0] > 0.0);
        cw[0] = ee[0] * ib;
        xs[0] = g0 * ib;
        for (int i = 1; i < nx; ++i) {
          const double e = ee[i - 1];
          const double bt = fma(-e, cw[i - 1], dd[i]);
          sc_bad |= !(bt > 0.0);
          ib = 1.0 / bt;
          cw[i] = ee[i] * ib;
          xs[i] = fma(-e, xs[i - 1], g0) * ib;
        }
        for (int i = nx - 2; i >= 0; --i) xs[i] = fma(-cw[i], xs[i + 1], xs[i]);
        for (int i = 0; i < nx; ++i) sc_bad |= !(fabs(xs[i]) <= 1e150);
        for (int i = nx; i < NXP; ++i) xs[i] = 0.0;
      } else {
        for (int i = 0; i < NXP; ++i) xs[i] = 0.0;
      }
    }
  }
  __syncwarp();
  // chunk products: pie_k = prod_j (-l_j) over chunk k, sigs_k = prod_j (-l_{j+1}); staged in dd / ee
  double* pie = dd;
  double* sigs = ee;
  {
    double pi = 1.0, sg = 1.0;
    for (int j = 0; j < MR; ++j) pi *= -b[L::L_OFF + k * MR + j];
    for (int j = MR - 1; j >= 0; --j) {
      const int row = k * MR + j;
      sg *= -((row + 1 < NXP) ? b[L::L_OFF + row + 1] : 0.0);
    }
    __syncwarp();  // every lane has read what it needs of dd / ee
    pie[k] = pi;
    sigs[k] = sg;
  }
  __syncwarp();
  {
    for (int t = 0; t < L::LOGP; ++t) {
      const int d = 1 << t;
      double af = 0.0, bb = 0.0;
      if (k >= d) {
        af = 1.0;
        for (int q = k - d + 1; q <= k; ++q) af *= pie[q];
      }
      if (k + d < P) {
        bb = 1.0;
        for (int q = k; q <= k + d - 1; ++q) bb *= sigs[q];
      }
      b[L::AF_OFF + t * P + k] = af;
      b[L::BB_OFF + t * P + k] = bb;
    }
    // lazy-stitch vectors of chunk k: read only by be_steps_lazy (KLE_FINE_LAZY=1 builds), so neither
    // computed nor stored otherwise (they are two thirds of the blob)
    if (KLE_FINE_LAZY) {
      const double* l = b + L::L_OFF + k * MR;
      const double* inv = b + L::INV_OFF + k * MR;
      double* phi = b + L::PHI_OFF + k * MR;
      double* phi2 = b + L::PHI2_OFF + k * MR;
      double* sg = b + L::SG_OFF + k * MR;
      double* sg2 = b + L::SG2_OFF + k * MR;
      const double lnx = (k + 1 < P) ? b[L::L_OFF + (k + 1) * MR] : 0.0;
      double pi = 1.0;
      for (int j = 0; j < MR; ++j) {
        pi *= -l[j];
        phi[j] = pi * inv[j];
      }
      for (int j = MR - 2; j >= 0; --j) phi[j] = fma(-l[j + 1], phi[j + 1], phi[j]);
      double g = 1.0;
      for (int j = MR - 1; j >= 0; --j) {
        g *= -((j + 1 < MR) ? l[j + 1] : lnx);
        sg[j] = g;
      }
      phi2[0] = phi[0];
      sg2[0] = sg[0];
      for (int j = 1; j < MR; ++j) {
        phi2[j] = fma(-l[j], phi2[j - 1], phi[j]);
        sg2[j] = fma(-l[j], sg2[j - 1], sg[j]);
      }
    }
  }
  if (FS::SC && sc_on) {  // tables of the scaled partitioned sweep (kle_fine.cuh: be_steps_sc)
    __syncwarp();  // pie / sigs are consumed
    const double* l = b + L::L_OFF + k * MR;
    double t = 1.0, kprod = 1.0;
    for (int j = 0; j < MR; ++j) {
      const int row = k * MR + j;
      if (j > 0) t = (row < nx) ? -l[j] * t : 1.0;  // pad rows: 1 (never used, must not poison q)
      if (row < nx) sc_bad |= !(fabs(t) >= 1e-150 && fabs(t) <= 1e150);
      b[L::SC_T + row] = t;
      if (!(MR == 64 && P == 8)) b[L::SC_IT + row] = 1.0 / t;
      if (j + 1 < MR) kprod *= l[j + 1] * l[j + 1];
    }
    const double lnext = (k + 1 < P) ? b[L::L_OFF + (k + 1) * MR] : 0.0;
    const double qk = -lnext / t;  // t = t_{k,last}
    if constexpr (MR == 64 && P == 8) {
      // the eight-lane sweep (kle_fine_pw.cu) forms 1 / t itself and reads the backward stitch
      // coefficients sg_j = (prod_{i=j..MR-2} l_{i+1}^2) q_k from these slots
      double sg = qk;
      for (int j = MR - 1; j >= 0; --j) {
        b[L::SC_IT + k * MR + j] = sg;
        sg *= l[j] * l[j];
      }
    }
    __syncwarp();
    const double rho = (k > 0) ? -l[0] * b[L::SC_T + k * MR - 1] : 0.0;
    b[L::SC_RHO + k] = rho;
    b[L::SC_Q + k] = qk;
    dd[k] = rho;         // forward scan multiplier of chunk k
    ee[k] = kprod * qk;  // backward scan multiplier: sg_{k,0}
    __syncwarp();
    for (int tt = 0; tt < L::LOGP; ++tt) {
      const int d = 1 << tt;
      double af = 0.0, bb = 0.0;
      if (k >= d) {
        af = 1.0;
        for (int q = k - d + 1; q <= k; ++q) af *= dd[q];
      }
      if (k + d < P) {
        bb = 1.0;
        for (int q = k; q <= k + d - 1; ++q) bb *= ee[q];
      }
      b[L::SC_AF + tt * P + k] = af;
      b[L::SC_BB + tt * P + k] = bb;
    }
    const bool any_bad = ((__ballot_sync(KLE_FULL_MASK, sc_bad) >> (grp * P)) & (P == 32 ? 0xffffffffu : ((1u << P) - 1u))) != 0;
    if (k == 0) b[L::SC_FLAG] = any_bad ? 1.0 : 0.0;
  }
  __syncwarp();
  for (int q = 0; q < FS::SPW; ++q) {
    const int sq = s0 + q;
    if (sq >= M) break;
    double* out = blob + (size_t)sq * stride + offset;
    const double* bq = fsm + q * FS::PER;
    // l, 1/beta and the scan multipliers (+ lazy vectors / the scaled tables; without them every sample is
    // flagged, so a later KLE_FGR_SC=1 sweep on this blob falls through to the unscaled kernel)
    if constexpr (MR == 64 && P == 8) {
      // packed for kle_fine_pw.cu (kle_fine.cuh: kPw*): row r -> entry (j = r & 63, kq = r >> 6)
      //   T0 {1/beta, l_{r+1}^2}   T1 {sg pairs}   T2 {x*, 1/t}   T3 {t, dia}   T4 {off[r-1] pairs}
      for (int r = lane; r < NXP; r += 32) {
        const int j = r & 63, kq = r >> 6, e = (j * P + kq) * 2, e2 = ((j >> 1) * P + kq) * 2 + (j & 1);
        const bool real = r < nx;
        const double ln1 = (j < 63 && r + 1 < nx) ? bq[L::L_OFF + r + 1] : 0.0;
        const double tv = real ? bq[L::SC_T + r] : 0.0;
        out[0 * NXP + e] = real ? bq[L::INV_OFF + r] : 0.0;
        out[0 * NXP + e + 1] = ln1 * ln1;
        out[2 * NXP + e2] = bq[L::SC_IT + r];  // sg_r
        out[3 * NXP + e] = real ? bq[L::SC_XS + r] : 0.0;
        out[3 * NXP + e + 1] = real ? 1.0 / tv : 0.0;
        out[5 * NXP + e] = tv;
        out[5 * NXP + e + 1] = real ? dia[(size_t)sq * nx + r] : 0.0;
        out[7 * NXP + e2] = (real && r > 0) ? off[(size_t)sq * nx + r - 1] : 0.0;
      }
      for (int i = lane; i < 24; i += 32) {
        out[kPwAf + i] = bq[L::SC_AF + i];
        out[kPwBb + i] = bq[L::SC_BB + i];
      }
      if (lane < 8) {
        out[kPwRho + lane] = bq[L::SC_RHO + lane];
        out[kPwQ + lane] = bq[L::SC_Q + lane];
      }
      if (lane == 0) out[kPwFlag] = bq[L::SC_FLAG];
    } else {
      const int ns = (FS::SC && !sc_on) ? L::PHI_OFF : FS::BS;
      for (int i = lane; i < ns; i += 32) out[i] = bq[i];
      if (FS::SC && !sc_on && lane == 0) out[L::SC_FLAG] = 1.0;
    }
  }
  (void)g0;
}

template <int MR, int P>
constexpr size_t fine_factor_smem() {
  return FactorSmem<MR, P>::bytes;
}

// ---------------------------------------------------------------------------
// Fused F + rhs kernel. CTA = (sample, group of subintervals); samples on
// grid.x (grid.y is limited to 65535).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}

// shared-memory staging of the fused kernel: start rows (which are also the
// "prev" rows of the rhs for n >= 1), alpha-twisted prev row of n = 0, and
// the operator diagonals, all fetched with cp.async before the sweep.
template <int MR, int P, int NC>
struct FgrSmem {
  // rows are XOR-swizzled within their MR-row chunk (pidx), so that the P
  // lanes of a system (stride MR rows) hit distinct banks; a permutation of
  // each chunk, so no padding (ee needs one extra chunk for row nx)
  static constexpr int NXP = MR * P;
  static constexpr int LD = NXP;
  static constexpr int SWZ = (MR < 16 ? MR : 16) - 1;
  __device__ __forceinline__ static int pidx(int row) { return row ^ ((row / MR) & SWZ); }
  // TABS row vectors [MR][P] behind the staging: 3 chunk-product tables (be_steps_cs), 5 lazy tables
  // (be_steps_lz), none for the register-product variants (c2: 37 KB per CTA instead of 49)
  static constexpr size_t bytes(int tabs) { return ((size_t)(NC + 3) * LD + MR + 8 + (size_t)tabs * NXP) * sizeof(double); }
};

template <int MR, int P, int R, int NT, bool PIPE, bool SC = false>
#ifdef KLE_FGR_MINB_ALL  // tuning override
#define KLE_FGR_MINB(MR, R, NT) KLE_FGR_MINB_ALL
#else
#define KLE_FGR_MINB(MR, R, NT) ((NT) == 32 ? 8 : ((MR) * (R) > 32 ? 2 : 3))
#endif
__global__ void __launch_bounds__(NT, KLE_FGR_MINB(MR, R, NT)) fgr_kernel(FgrArgs a) {
  using L = FineLayout<MR, P>;
  constexpr int SLOTS = 32 / P;
  constexpr int NC = (NT / 32) * SLOTS * R;  // subintervals per CTA
  constexpr int NXP = MR * P;
  const int s = blockIdx.x;
  if (a.active && a.active[s] != KLE_SAMPLE_ACTIVE) return;
  if (a.tw_fallback && a.F_given == nullptr) {  // only the samples the twisted / scaled / eight-lane kernel skipped
    if (a.ffac[(size_t)s * L::DOUBLES + a.flag_off] == 0.0) return;
  }
  if constexpr (SC) {  // scaled step: flagged samples go to the unscaled kernel
    if (a.ffac[(size_t)s * L::DOUBLES + L::SC_FLAG] != 0.0) return;
  }
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int k = lane % P, slot = lane / P;
  const int nx = a.nx, N = a.N;
  const size_t sbase = (size_t)s * N * nx;
  const int n0 = blockIdx.y * NC;

  int nl[R];  // local subinterval index within the CTA
#pragma unroll
  for (int r = 0; r < R; ++r) nl[r] = (w * SLOTS + slot) * R + r;

  double x[R][MR];
  FGR_T(0);
  FGR_T(7);
  if (a.F_given == nullptr) {
    extern __shared__ __align__(16) double sm[];
    using SM = FgrSmem<MR, P, NC>;
    constexpr int LD = SM::LD;
    double* st = sm;              // [NC][LD]
    double* p0 = st + NC * LD;    // [LD]
    double* dd = p0 + LD;         // [LD]
    double* ee = dd + LD;         // [LD + MR]: ee[pidx(i)] couples rows i-1 and i
    // Two prologues. FAST (one-warp CTAs, c4 / c1 shapes, where the fixed cost was 31% of a launch): the
    // factor rows are requested first (the chunk products depend on them, the longest dependent chain), the
    // copy loops are straight predicated LDGSTS over per-thread row slots, and the start rows come out of
    // shared memory through unconditional volatile loads followed by selects. The compiler otherwise sinks
    // each load under its select and serialises 64 load-use pairs behind branches: 9.9k cycles per CTA at
    // c4 (tools/fgr_timing.py), 5.18 -> 4.56 ms per 131k-sample launch with this form. The multi-warp
    // variants keep the original form: at c2 the prologue is 7% of a CTA's life and the step loop's
    // register allocation is sensitive to it (10.17 ms per 8,192 samples against 10.6-11.0 with the fast form).
    constexpr bool FAST = NT == 32;
    constexpr int RPT = (NXP + NT - 1) / NT;
    std::conditional_t<SC, LaneFactorsSC<MR, P>, LaneFactors<MR, P>> fac;
    if constexpr (FAST) {
      fac.load(a.ffac + (size_t)s * L::DOUBLES, k, nx);
      int so[RPT];
      bool rv[RPT];
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int row = tid + i * NT;
        rv[i] = row < nx;
        so[i] = SM::pidx(rv[i] ? row : 0);
      }
      for (int ln = 0; ln < NC; ++ln) {
        const int n = n0 + ln;
        if (n >= N) break;
        const double* src = ((n == 0) ? a.u0 : a.U + sbase + (size_t)(n - 1) * nx) + tid;
        double* dst = st + ln * LD;
#pragma unroll
        for (int i = 0; i < RPT; ++i)
          if (rv[i]) cp_async8(dst + so[i], src + i * NT);
      }
      asm volatile("cp.async.commit_group;\n" ::);  // group 1: the start rows (needed first)
      const double* pl = a.U + sbase + (size_t)(N - 1) * nx + tid;
      const double* dg = a.dia + (size_t)s * nx + tid;
      const double* eg = a.off + (size_t)s * nx + tid;
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int row = tid + i * NT;
        if (rv[i]) {
          if (n0 == 0) cp_async8(p0 + so[i], pl + i * NT);
          cp_async8(dd + so[i], dg + i * NT);
          if (row + 1 < nx) cp_async8(ee + SM::pidx(row + 1), eg + i * NT);
        }
      }
    } else {
      for (int ln = 0; ln < NC; ++ln) {  // no division in the index math
        const int n = n0 + ln;
        if (n >= N) break;
        const double* src = (n == 0) ? a.u0 : a.U + sbase + (size_t)(n - 1) * nx;
        for (int row = tid; row < nx; row += NT) cp_async8(st + ln * LD + SM::pidx(row), src + row);
      }
      asm volatile("cp.async.commit_group;\n" ::);  // group 1: the start rows (needed first)
      if (n0 == 0)
        for (int row = tid; row < nx; row += NT) cp_async8(p0 + SM::pidx(row), a.U + sbase + (size_t)(N - 1) * nx + row);
      for (int row = tid; row < nx; row += NT) {
        cp_async8(dd + SM::pidx(row), a.dia + (size_t)s * nx + row);
        if (row + 1 < nx) cp_async8(ee + SM::pidx(row + 1), a.off + (size_t)s * nx + row);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);  // group 2: epilogue operands
    if (tid == 0) {
      ee[0] = 0.0;
      ee[SM::pidx(nx)] = 0.0;
    }
    if constexpr (!FAST) fac.load(a.ffac + (size_t)s * L::DOUBLES, k, nx);
    const double hg = a.dt * a.g0;
    double* cs = ee + LD + MR;  // [3][MR][P] chunk products (KLE_FINE_CS) / [5][MR][P] lazy tables (LZ)
    // chunk products from shared memory: the one-warp R = 4 variant (c4: 234 registers, 8 chains per
    // SMSP; 6.16 -> 5.17 ms per 131k-sample launch), or every variant under KLE_FINE_CS
    constexpr bool CS = (KLE_FINE_CS || NT == 32) && !PIPE && !KLE_FINE_LAZY && !SC;
    constexpr bool LZ = CS && KLE_FGR_LZ;
    if constexpr (LZ) {
      if (w == 0 && slot == 0) lazy_tables<MR, P>(cs, fac, k, hg);
    } else if constexpr (CS) {
      if (w == 0 && slot == 0) chunk_products<MR, P>(cs, fac, k, hg);
    }
    FGR_T(1);
    asm volatile("cp.async.wait_group 1;\n" ::);
    __syncthreads();
    FGR_T(2);
    if constexpr (FAST) {
      // the lane's rows k MR + j sit at k MR + (j ^ (k & SWZ)); pad rows and unused slots hold garbage
      // that the select drops
      const int kx = k & SM::SWZ;
      const unsigned sr0 = (unsigned)__cvta_generic_to_shared(st + nl[0] * LD + k * MR);
      unsigned xo[MR];
#pragma unroll
      for (int j = 0; j < MR; ++j) xo[j] = sr0 + (unsigned)((j ^ kx) * sizeof(double));
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int lim = (n0 + nl[r] < N) ? fac.nreal : 0;  // rows j < lim of this right-hand side are real
#pragma unroll
        for (int j = 0; j < MR; ++j) {
          const double v = lds_f64(xo[j] + (unsigned)(r * LD * sizeof(double)));
          x[r][j] = (j < lim) ? v + hg : 0.0;
        }
      }
    } else {
      if constexpr (SC) {  // w = (x - x*) / t
        const double* bl = a.ffac + (size_t)s * L::DOUBLES;
#pragma unroll
        for (int j = 0; j < MR; ++j) {
          const int row = k * MR + j;
          const double xs = bl[L::SC_XS + row], its = bl[L::SC_IT + row];
#pragma unroll
          for (int r = 0; r < R; ++r)
            x[r][j] = (row < nx && n0 + nl[r] < N) ? (st[nl[r] * LD + SM::pidx(row)] - xs) * its : 0.0;
        }
      } else {
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int j = 0; j < MR; ++j) {
          const int row = k * MR + j;
          x[r][j] = (row < nx && n0 + nl[r] < N) ? st[nl[r] * LD + SM::pidx(row)] + hg : 0.0;
        }
      }
    }
    FGR_T(3);
    if constexpr (SC) be_steps_sc<MR, P, R>(x, fac, a.J);
    else if constexpr (PIPE) be_steps_pipe<MR, P, R>(x, fac, k, a.J, hg);
    else if constexpr (KLE_FINE_LAZY) be_steps_lazy<MR, P, R>(x, fac, a.ffac + (size_t)s * L::DOUBLES, k, a.J, hg);
    else if constexpr (LZ) be_steps_lz<MR, P, R>(x, fac, k, a.J, cs);
    else if constexpr (CS) be_steps_cs<MR, P, R>(x, fac, k, a.J, cs);
    else be_steps<MR, P, R>(x, fac, k, a.J, hg);
    FGR_T(4);
    if constexpr (SC) {  // F = t w + x*
      const double* bl = a.ffac + (size_t)s * L::DOUBLES;
#pragma unroll
      for (int j = 0; j < MR; ++j) {
        const int row = k * MR + j;
        const double xs = bl[L::SC_XS + row], ts = bl[L::SC_T + row];
#pragma unroll
        for (int r = 0; r < R; ++r) x[r][j] = (row < nx) ? fma(ts, x[r][j], xs) : 0.0;
      }
    } else {
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int j = 0; j < MR; ++j) x[r][j] = (k * MR + j < nx) ? x[r][j] - hg : 0.0;
    }
    if (a.F_out) {
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int j = 0; j < MR; ++j) {
          const int row = k * MR + j;
          if (row < nx && n0 + nl[r] < N) a.F_out[sbase + (size_t)(n0 + nl[r]) * nx + row] = x[r][j];
        }
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
    if (a.Rout == nullptr) return;  // F ends only (classical parareal)
    __syncthreads();  // the epilogue operands (group 2) of every thread have landed
    // epilogue: rhs_n = scaling_n * ((I + dT A) F_n - prev_n), operands from shared memory;
    // each rhs row replaces its (consumed) prev row in st, then the CTA stores st coalesced.
    // Row-major over j with the R right-hand sides inner: the operator values of a row are
    // read once, every shared load precedes every store (no alias barriers between them),
    // and the rhs values overwrite x in place (the left neighbour is carried in xl).
    double left[R], right[R], sc[R], pmul[R];
    const double* pv[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      left[r] = __shfl_up_sync(KLE_FULL_MASK, x[r][MR - 1], 1, P);
      right[r] = __shfl_down_sync(KLE_FULL_MASK, x[r][0], 1, P);
      const int n = n0 + nl[r];
      sc[r] = (n < N) ? a.scaling[n] : 0.0;
      pmul[r] = (n == 0) ? a.alpha : 1.0;
      pv[r] = (n == 0) ? p0 : st + nl[r] * LD;
    }
    double xl[R];
#pragma unroll
    for (int r = 0; r < R; ++r) xl[r] = k > 0 ? left[r] : 0.0;
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      const int row = k * MR + j;
      const int pr = SM::pidx(row);
      const double dj = dd[pr], em = ee[pr], ep = ee[SM::pidx(row + 1)];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double xc = x[r][j];
        const double xp = (j < MR - 1) ? x[r][j + 1] : (k < P - 1 ? right[r] : 0.0);
        const double Ax = fma(em, xl[r], fma(dj, xc, ep * xp));
        const double rhs = fma(a.dT, Ax, xc) - pmul[r] * pv[r][pr];
        xl[r] = xc;
        x[r][j] = sc[r] * rhs;
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (n0 + nl[r] >= N) continue;
      double* rs = st + nl[r] * LD;
#pragma unroll
      for (int j = 0; j < MR; ++j) {
        const int row = k * MR + j;
        if (row < nx) rs[SM::pidx(row)] = x[r][j];
      }
    }
    __syncthreads();
    FGR_T(5);
    for (int ln = 0; ln < NC; ++ln) {
      const int n = n0 + ln;
      if (n >= N) break;
      double* out = a.Rout + sbase + (size_t)n * nx;
      const double* rs = st + ln * LD;
      if constexpr (FAST) {
        out += tid;
        double v[RPT];  // (row slots recomputed here: keeping them live over the step loop costs registers)
#pragma unroll
        for (int i = 0; i < RPT; ++i) v[i] = rs[SM::pidx(tid + i * NT < nx ? tid + i * NT : 0)];
#pragma unroll
        for (int i = 0; i < RPT; ++i)
          if (tid + i * NT < nx) out[i * NT] = v[i];
      } else {
        for (int row = tid; row < nx; row += NT) out[row] = rs[SM::pidx(row)];
      }
    }
    FGR_T(6);
    return;
  }
  // ---- F given (stand-alone cgc_correct): no sweep ----------------------------
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      const int row = k * MR + j;
      const int n = n0 + nl[r];
      x[r][j] = (row < nx && n < N) ? a.F_given[sbase + (size_t)n * nx + row] : 0.0;
    }
  const double* dd = a.dia + (size_t)s * nx;
  const double* ee = a.off + (size_t)s * nx;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const double left = __shfl_up_sync(KLE_FULL_MASK, x[r][MR - 1], 1, P);
    const double right = __shfl_down_sync(KLE_FULL_MASK, x[r][0], 1, P);
    const int n = n0 + nl[r];
    if (n >= N) continue;
    const double sc = a.scaling[n];
    const size_t prow = (n == 0) ? sbase + (size_t)(N - 1) * nx : sbase + (size_t)(n - 1) * nx;
    const double pmul = (n == 0) ? a.alpha : 1.0;
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      const int row = k * MR + j;
      if (row >= nx) continue;
      const double xm = (j > 0) ? x[r][j - 1] : (k > 0 ? left : 0.0);
      const double xp = (j < MR - 1) ? x[r][j + 1] : (k < P - 1 ? right : 0.0);
      const double em = (row > 0) ? ee[row - 1] : 0.0;
      const double ep = (row < nx - 1) ? ee[row] : 0.0;
      const double Ax = fma(em, xm, fma(dd[row], x[r][j], ep * xp));
      const double rhs = fma(a.dT, Ax, x[r][j]) - pmul * a.U[prow + row];
      a.Rout[sbase + (size_t)n * nx + row] = sc * rhs;
    }
  }
}

// ---------------------------------------------------------------------------
// Stand-alone sweep: out[s][q*nseg + g] = F^{(g+1)}(start[s][q]) where each
// segment is J steps of size h (blob built for that h). nseg = 1 gives
// propagate_fine / propagate_coarse (J=1, coarse blob); q = 1, nseg = N gives
// fine_reference / coarse_sweep_init.
// ---------------------------------------------------------------------------
template <int MR, int P, int R, int NT, bool PIPE>
__global__ void __launch_bounds__(NT) sweep_kernel(SweepArgs a) {
  using L = FineLayout<MR, P>;
  constexpr int SLOTS = 32 / P;
  constexpr int NC = (NT / 32) * SLOTS * R;
  const int s = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int k = lane % P, slot = lane / P;
  const int nx = a.nx, Q = a.Q;
  LaneFactors<MR, P> fac;
  fac.load(a.fac + (size_t)s * L::DOUBLES, k, nx);
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
  for (int g = 0; g < a.nseg; ++g) {
    if constexpr (PIPE) be_steps_pipe<MR, P, R>(x, fac, k, a.J, hg);
    else if constexpr (KLE_FINE_LAZY) be_steps_lazy<MR, P, R>(x, fac, a.fac + (size_t)s * L::DOUBLES, k, a.J, hg);
    else be_steps<MR, P, R>(x, fac, k, a.J, hg);
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

// ---------------------------------------------------------------------------
// host-side dispatch
// ---------------------------------------------------------------------------
// PI: 0 = eager step, 128 threads; 1 = software-pipelined step; 2 = eager, 64
// threads (finer CTA granularity: R = 3 wastes 2/66 instead of 8/72 slots at N = 64);
// 3 = eager, 32 threads (one warp: N = 16 with R = 4)
template <int MR, int P, int R_, int PI = 0>
struct FineInst {
  static constexpr bool PIPE = PI == 1;
  static constexpr int R = R_;
  static constexpr int NT = PI == 3 ? 32 : (PI == 2 ? 64 : 128);
  static constexpr int NC = (NT / 32) * (32 / P) * R;

  static int factor(const double* dia, const double* off, double* blob, int M, int nx, double h,
                    double g0, cudaStream_t st, int force_sc = 0, int stride = FineLayout<MR, P>::DOUBLES,
                    int offset = 0) {
    constexpr size_t smem = fine_factor_smem<MR, P>();
    static PerDeviceOnce attr_once;
    if (int rc = once_per_device(attr_once, "kle_fine(factor): cudaFuncSetAttribute", [&] {
          return cudaFuncSetAttribute(fine_factor_kernel<MR, P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem);
        }))
      return rc;
    constexpr int SPW = FactorSmem<MR, P>::SPW;
    const char* e = getenv("KLE_FGR_SC");
    const int sc_on = force_sc || (e && *e == '1');
    if (M > 0)
      fine_factor_kernel<MR, P><<<(unsigned)((M + SPW - 1) / SPW), 32, smem, st>>>(dia, off, blob, M, nx, h, g0, sc_on,
                                                                                   stride, offset);
    return check_launch("fine_factor_kernel");
  }
  static int fgr(const FgrArgs& a, cudaStream_t st) {
    dim3 grid(a.M, (a.N + NC - 1) / NC);
    constexpr bool CS = (KLE_FINE_CS || NT == 32) && !PIPE && !KLE_FINE_LAZY;  // as in fgr_kernel
    size_t smem = a.F_given ? 0 : FgrSmem<MR, P, NC>::bytes(CS ? (KLE_FGR_LZ ? 5 : 3) : 0);
    static const char* pad_env = getenv("KLE_FGR_PAD_SMEM");  // tuning: extra bytes per CTA (lowers CTAs/SM)
    if (pad_env && smem) smem = std::min<size_t>(smem + (size_t)atoi(pad_env), 200 * 1024);
    static PerDeviceOnce attr_once;
    if (int rc = once_per_device(attr_once, "kle_fine: cudaFuncSetAttribute", [&] {
          return cudaFuncSetAttribute(fgr_kernel<MR, P, R, NT, PIPE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        }))
      return rc;
    fgr_kernel<MR, P, R, NT, PIPE><<<grid, NT, smem, st>>>(a);
    return check_launch("fgr_kernel");
  }
  // scaled partitioned sweep (be_steps_sc), then the unscaled kernel for the samples flagged by the factor kernel
  static int fgr_sc(const FgrArgs& a, cudaStream_t st) {
    dim3 grid(a.M, (a.N + NC - 1) / NC);
    const size_t smem = FgrSmem<MR, P, NC>::bytes(0);
    static PerDeviceOnce attr_once;
    if (int rc = once_per_device(attr_once, "kle_fine(sc): cudaFuncSetAttribute", [&] {
          return cudaFuncSetAttribute(fgr_kernel<MR, P, R, NT, PIPE, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      200 * 1024);
        }))
      return rc;
    fgr_kernel<MR, P, R, NT, PIPE, true><<<grid, NT, smem, st>>>(a);
    if (int rc = check_launch("fgr_kernel(sc)")) return rc;
    if (a.tw_none_flagged) return KLE_OK;
    FgrArgs b = a;
    b.tw_fallback = 1;
    b.flag_off = FineLayout<MR, P>::SC_FLAG;
    return fgr(b, st);
  }
  static int sweep(const SweepArgs& a, cudaStream_t st) {
    dim3 grid(a.M, (a.Q + NC - 1) / NC);
    sweep_kernel<MR, P, R, NT, PIPE><<<grid, NT, 0, st>>>(a);
    return check_launch("sweep_kernel");
  }
};

// (MR, P, R) variants; the first entry whose MR*P covers nx is the default,
// KLE_FINE_VARIANT=<index> forces one (for tuning; blobs depend on MR, P).
struct FineVariant {
  int MR, P, R, pipe, kind = 0;  // kind 1 (shared-memory factors): `pipe` is the min CTAs/SM bound
};
static const FineVariant kVariants[] = {
    {1, 16, 4, 0},  {2, 16, 4, 0},  {4, 16, 4, 0},  {16, 8, 4, 3},  {16, 32, 3, 2}, {32, 32, 2, 0},  // defaults
    {8, 16, 2, 1},  {4, 32, 4, 0},  {8, 16, 4, 1},  {8, 16, 4, 0},  {16, 16, 2, 0}, {8, 32, 4, 0},
    {32, 16, 2, 0}, {16, 32, 2, 0}, {16, 32, 2, 1}, {16, 32, 4, 1}, {16, 32, 4, 0}, {4, 32, 4, 1},
    {16, 32, 3, 4, 1}, {16, 32, 3, 3, 1}, {16, 32, 2, 4, 1}, {16, 32, 4, 3, 1},  // 18..21 shared-memory factors
    {8, 16, 2, 4, 1},  {8, 16, 4, 4, 1},  {8, 32, 4, 4, 1},                     // 22..24
    {32, 16, 2, 2, 1}, {32, 16, 1, 3, 1}, {16, 32, 3, 2, 1},                     // 25..27
    {32, 16, 4, 3, 1}, {32, 16, 3, 3, 1}, {32, 16, 2, 4, 1}, {32, 16, 4, 2, 1},  // 28..31
    {16, 32, 3, 0}, {8, 16, 2, 2}, {16, 32, 2, 2},                                // 32..34
    {16, 8, 2, 0},  {16, 8, 3, 0},  {16, 8, 2, 2},  {16, 8, 3, 2},  {8, 8, 4, 0},   // 35..39 (nx <= 128)
    {16, 8, 4, 3},  {16, 8, 2, 3},  {16, 32, 4, 3}, {16, 32, 3, 3},                 // 40..43 (one-warp CTAs)
};
static const int kNumDefaults = 6;

#define KLE_FINE_DISPATCH(MR_, P_, R_, PI_, CALL) \
  if (lay.MR == MR_ && lay.P == P_ && lay.R == R_ && lay.pipe == PI_) return FineInst<MR_, P_, R_, PI_>::CALL;

#define KLE_FINE_ALL(CALL)                \
  KLE_FINE_DISPATCH(1, 16, 4, 0, CALL)    \
  KLE_FINE_DISPATCH(2, 16, 4, 0, CALL)    \
  KLE_FINE_DISPATCH(4, 16, 4, 0, CALL)    \
  KLE_FINE_DISPATCH(8, 16, 2, 0, CALL)    \
  KLE_FINE_DISPATCH(16, 32, 3, 0, CALL)   \
  KLE_FINE_DISPATCH(16, 32, 3, 2, CALL)   \
  KLE_FINE_DISPATCH(8, 16, 2, 2, CALL)    \
  KLE_FINE_DISPATCH(16, 32, 2, 2, CALL)   \
  KLE_FINE_DISPATCH(32, 32, 2, 0, CALL)   \
  KLE_FINE_DISPATCH(8, 16, 2, 1, CALL)    \
  KLE_FINE_DISPATCH(16, 32, 2, 1, CALL)   \
  KLE_FINE_DISPATCH(4, 32, 4, 0, CALL)    \
  KLE_FINE_DISPATCH(8, 16, 4, 1, CALL)    \
  KLE_FINE_DISPATCH(8, 16, 4, 0, CALL)    \
  KLE_FINE_DISPATCH(16, 16, 2, 0, CALL)   \
  KLE_FINE_DISPATCH(8, 32, 4, 0, CALL)    \
  KLE_FINE_DISPATCH(32, 16, 2, 0, CALL)   \
  KLE_FINE_DISPATCH(16, 32, 2, 0, CALL)   \
  KLE_FINE_DISPATCH(16, 32, 3, 0, CALL)   \
  KLE_FINE_DISPATCH(16, 32, 4, 1, CALL)   \
  KLE_FINE_DISPATCH(16, 32, 4, 0, CALL)   \
  KLE_FINE_DISPATCH(4, 32, 4, 1, CALL)    \
  KLE_FINE_DISPATCH(16, 8, 2, 0, CALL)    \
  KLE_FINE_DISPATCH(16, 8, 3, 0, CALL)    \
  KLE_FINE_DISPATCH(16, 8, 2, 2, CALL)    \
  KLE_FINE_DISPATCH(16, 8, 3, 2, CALL)    \
  KLE_FINE_DISPATCH(16, 8, 4, 3, CALL)    \
  KLE_FINE_DISPATCH(16, 8, 2, 3, CALL)    \
  KLE_FINE_DISPATCH(16, 32, 4, 3, CALL)   \
  KLE_FINE_DISPATCH(16, 32, 3, 3, CALL)   \
  KLE_FINE_DISPATCH(8, 8, 4, 0, CALL)

// scaled partitioned sweep (be_steps_sc) for the (16, 32) layout (128 < nx <= 512), KLE_FGR_SC=1
bool sc_supported(const FineLayoutRT& lay) {
  if (KLE_FINE_LAZY || lay.W || lay.kind || lay.P != 32) return false;
  if (!(lay.MR == 16 && lay.R == 3 && lay.pipe == 2)) return false;  // (32, 32, 2) spills with the scaled factors
  // opt-in: measured 9.63 against 9.85 ms per 8,192-sample config-2 launch (the step loop there is bound by the
  // latency of its carry scans, not by FP64 issue), so the unscaled step stays the default; read per call
  const char* e = getenv("KLE_FGR_SC");
  return e && *e == '1';
}

int sc_flag_offset(const FineLayoutRT& lay) { return FineLayout<16, 32>::SC_FLAG; }  // (the only scaled layout)

FineLayoutRT fine_layout(int nx) {
  const char* env = getenv("KLE_FINE_VARIANT");
  if (env && *env) {
    const int v = atoi(env);
    const int nv = (int)(sizeof(kVariants) / sizeof(kVariants[0]));
    if (v >= 0 && v < nv && kVariants[v].MR * kVariants[v].P >= nx) {
      const FineVariant& f = kVariants[v];
      FineLayoutRT l{f.MR, f.P, f.R, f.pipe, f.kind ? sf_blob_doubles(f.MR, f.P) : fine_blob_doubles(f.MR, f.P)};
      l.kind = f.kind;
      return l;
    }
  }
  for (int i = 0; i < kNumDefaults; ++i) {
    const FineVariant& f = kVariants[i];
    if (f.MR * f.P >= nx) return {f.MR, f.P, f.R, f.pipe, fine_blob_doubles(f.MR, f.P)};
  }
  const int W = mw_warps(nx);
  if (W) return {16, 32 * W, 1, 0, mw_blob_doubles(nx), W};
  return {0, 0, 0, 0, 0};
}

int fine_factor(FineLayoutRT lay, const double* dia, const double* off, double* blob, int M, int nx,
                double h, double g0, cudaStream_t st) {
  if (lay.W) return mw_factor(dia, off, blob, M, nx, h, st);
  if (lay.kind == 1) return sf_factor(lay, dia, off, blob, M, nx, h, g0, st);
  auto base = [&]() -> int {
    KLE_FINE_ALL(factor(dia, off, blob, M, nx, h, g0, st))
    return set_error(KLE_ERR_UNSUPPORTED, "fine_factor: unsupported nx");
  };
  if (int rc = base()) return rc;
  // the (64, 8) blob with the scaled tables of the eight-lane sweep (kle_fine_pw.cu) behind the (16, 32) blob
  if (lay.kind == 0 && !lay.W && lay.MR == 16 && lay.P == 32 && !KLE_FINE_LAZY)
    return FineInst<64, 8, 1, 0>::factor(dia, off, blob, M, nx, h, g0, st, 1, lay.doubles, FineLayout<16, 32>::PW_OFF);
  // the twisted two-lane tables (kle_fine_tw.cu) go into the blob's spare part
  if (tw_supported(lay, nx)) return tw_factor(dia, off, blob, M, nx, h, g0, st);
  return KLE_OK;
}

int fine_fgr(FineLayoutRT lay, const FgrArgs& a, cudaStream_t st) {
  if (lay.W) return mw_fgr(a, st);
  if (lay.kind == 1) {
    if (!a.F_given) return sf_fgr(lay, a, st);
    lay.kind = 0;  // F given: no sweep, any (MR, P) register variant serves the epilogue
    lay.pipe = 0;
    lay.R = (lay.MR == 16) ? 3 : (lay.P == 32 ? 4 : 2);
  }
  if (!a.F_given && !a.F_out && a.Rout && pw_supported(lay, a.nx)) {
    if (int rc = pw_fgr(a, st)) return rc;
    if (a.tw_none_flagged) return KLE_OK;
    FgrArgs b = a;  // samples without a scaled form: the partitioned kernel
    b.tw_fallback = 1;
    b.flag_off = pw_flag_offset();
    KLE_FINE_ALL(fgr(b, st))
  }
  if (!a.F_given && sc_supported(lay)) {
    return FineInst<16, 32, 3, 2>::fgr_sc(a, st);
  }
  if (!a.F_given && !a.F_out && a.Rout && tw_supported(lay, a.nx)) {
    if (int rc = tw_fgr(a, st)) return rc;
    if (a.tw_none_flagged) return KLE_OK;
    FgrArgs b = a;  // samples without a scaled twisted form (flagged by tw_factor): the partitioned kernel
    b.tw_fallback = 1;
    b.flag_off = kTwFlagOff;
    KLE_FINE_ALL(fgr(b, st))
  }
  KLE_FINE_ALL(fgr(a, st))
  return set_error(KLE_ERR_UNSUPPORTED, "fgr: unsupported nx");
}

int fine_sweep(FineLayoutRT lay, const SweepArgs& a, cudaStream_t st) {
  if (lay.W) return mw_sweep(a, st);
  if (lay.kind == 1) return sf_sweep(lay, a, st);
  KLE_FINE_ALL(sweep(a, st))
  return set_error(KLE_ERR_UNSUPPORTED, "sweep: unsupported nx");
}

}  // namespace kle
