// Twisted-factorisation fine sweep for small systems (64 < nx <= 128; configs 1 and 4).
//
// Reference counterparts: propagate_fine (pintuq/propagators.py:121-145, J x splu.solve) and the
// right-hand side of cgc_correct (pintuq/pcgc.py:175-197, 233-237), as kle_fine.cu.
//
// The partitioned solve of kle_fine.cu pays five FMAs per row and step plus two lane scans, because
// every chunk has two unknown neighbours. With exactly TWO lanes per system there is no unknown
// neighbour left: the "burn at both ends" (twisted) factorisation T = N D N^T eliminates from row 0
// downwards in one lane and from row nx-1 upwards in the other, the two eliminations meet in a 2 x 2
// system in the middle (one shuffle), and both lanes back-substitute outwards: the sequential Thomas
// count and no scan. Each lane keeps its H = 64 rows of ONE right-hand side in registers (local order
// j = 0 at the outer end .. H-1 in the middle; pad rows at the outer end), and the factor rows, which
// are per sample, come to the 16 lane pairs of a warp (= the N = 16 subintervals of a sample at c4) as
// broadcasts from shared memory.
//
// Shared-memory bandwidth is what such a kernel runs into (a broadcast 16-byte load still costs two
// wavefronts: measured 4.65 SM-cycles per warp-row with four coefficient doubles per row against 4.0
// for the partitioned kernel), so the recurrences are rewritten to need only TWO doubles per row:
//
//   * the constant source is removed by the steady state: with A x* = g0, e = x - x* obeys the
//     homogeneous step (I + hA) e_new = e_old;
//   * a diagonal scaling e_j = t_j w_j with t_j = nl_j t_{j-1} (t = 1 at the first real row) turns the
//     forward multipliers into 1:
//
//       forward   y_j = w_j + y_{j-1}                        (DADD, no coefficient)
//       middle    w_m = ca y_m + cb' y_m(partner)            (cb' carries the two lanes' t ratio)
//       backward  w_j = inv_j y_j + nl_{j+1}^2 w_{j+1}       (one 16-byte load {inv_j, nl_{j+1}^2})
//
//     Pad rows (inv = k = 0) stay exactly 0. t decays geometrically towards the middle (0.4^63 ~ 1e-25 at
//     c4); tw_factor_kernel flags a sample whose t leaves [1e-150, 1e150] or whose A has no positive
//     pivots (no steady state), fgr_tw_kernel skips flagged samples and the partitioned kernel, launched
//     right after with FgrArgs::tw_fallback, processes exactly those.
//
// The tables live behind the (16, 8) factor blob's scan multipliers (FineLayout::PHI_OFF .. DOUBLES), so
// every other consumer of the blob (sweeps, classical parareal, the fused small-block kernels) keeps its
// layout.
#include <algorithm>
#include <cstdlib>

#include "kle_common.cuh"
namespace kle {
#define FGR_T(i) \
  do {           \
  } while (0)
}
#include "kle_fine.cuh"
#include "kle_internal.h"

#ifndef KLE_FINE_LAZY
#define KLE_FINE_LAZY 0
#endif
#ifndef KLE_TW_SPLIT
#define KLE_TW_SPLIT 2  // independent forward chains per lane
#endif
#ifndef KLE_TW_NCACHE
#define KLE_TW_NCACHE 0  // rows whose backward coefficients stay in registers
#endif
#ifndef KLE_TW_PREFETCH
#define KLE_TW_PREFETCH 0  // L2 prefetch distance in CTAs (0: off)
#endif
#ifndef KLE_TW_HALVES
#define KLE_TW_HALVES 1  // lanes 0..15 top, 16..31 bottom: conflict-free staging rows (fixed cost 0.95 -> 0.83 ms per 131k launch)
#endif
#ifndef KLE_TW_MINB
#define KLE_TW_MINB 8  // CTAs (= warps) per SM the register allocation is bounded for
#endif

namespace kle {

namespace {
constexpr int TW_H = 64;  // rows per lane
// table layout (doubles), side 0 = top lane (rows ascending), side 1 = bottom lane (rows descending):
//   A [j][side][2]     = {inv_j, k_j = nl_{j+1}^2}   (j = H-1: {ca, cb'})      at (j * 2 + side) * 2
//   S [j][side][2]     = {x*_j, 1 / t_j}             (prologue)                at 4 H + (j * 2 + side) * 2
//   T [j/2][side][j&1] = t_j                         (epilogue)                at 8 H + ((j/2) * 2 + side) * 2 + (j & 1)
//   flag                                                                       at 10 H (kTwFlagOff - PHI_OFF)
// so that a warp's 16-byte load touches 32 contiguous bytes (even lanes one half, odd lanes the other).
constexpr int TW_DOUBLES = 10 * TW_H + 2;
__host__ __device__ constexpr int twA(int j, int side) { return (j * 2 + side) * 2; }
__host__ __device__ constexpr int twS(int j, int side) { return 4 * TW_H + (j * 2 + side) * 2; }
__host__ __device__ constexpr int twT(int j, int side) { return 8 * TW_H + ((j >> 1) * 2 + side) * 2 + (j & 1); }
constexpr int TW_FLAG = 10 * TW_H;

using TwL = FineLayout<16, 8>;
static_assert(TwL::DOUBLES - TwL::PHI_OFF >= TW_DOUBLES, "the twisted tables must fit the blob's spare part");
static_assert((TwL::PHI_OFF % 2) == 0 && (TwL::DOUBLES % 2) == 0, "16-byte aligned tables");
static_assert(kTwFlagOff == TwL::PHI_OFF + TW_FLAG, "flag offset shared with kle_fine.cu");

__device__ __forceinline__ double2 lds_v2(unsigned addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ void cp_async8(unsigned sa, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(unsigned sa, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
}  // namespace

// ---------------------------------------------------------------------------
// Tables. One warp builds the tables of TW_SPW = 8 samples, four lanes per sample, all running ONE
// recurrence shape (so the warp does not diverge over the roles):
//   role 0 / 1: twisted elimination of T = I + hA from the top / bottom end -> inv, nl^2, t;
//   role 2 / 3: twisted Thomas solve of the steady state A x* = g0 from the top / bottom end.
// Each lane walks its 64 rows with one division per row (the chain that bounds this kernel: a warp per
// sample with three active lanes took 18.6 ms per 1M samples, 4% of a config-4 step); the operator rows and
// the tables go through shared memory, so that every global access of the warp is coalesced, and 1 / t is
// formed by all lanes after the chains.
// ---------------------------------------------------------------------------
namespace {
constexpr int TW_SPW = 8;
// per sample: the tables (without the flag, which goes straight to global memory) and the operator rows
// (staged coalesced); the steady-state solve keeps (y, 1/b) in the S slots that x* and 1/t take over later.
// 896 doubles: four CTAs (32 samples) per SM
constexpr int TW_STAGED = 10 * TW_H;
constexpr int TW_FSM = TW_STAGED + 2 * 2 * TW_H;
}

__global__ void __launch_bounds__(32) tw_factor_kernel(const double* __restrict__ dia, const double* __restrict__ off,
                                                       double* __restrict__ blob, int M, int nx, double h, double g0) {
  constexpr int H = TW_H;
  extern __shared__ __align__(16) double fsm[];
  const int lane = threadIdx.x, ls = lane >> 2, role = lane & 3, side = role & 1;
  const bool steady = role >= 2;
  const int s = blockIdx.x * TW_SPW + ls;
  const bool live = s < M;
  double* tab = fsm + ls * TW_FSM;
  double* scr = tab + twS(0, side);               // y_j, 1 / b_j at scr[4 j], scr[4 j + 1] (the S slots)
  const double* dd = tab + TW_STAGED;             // [2 H]
  const double* ee = dd + 2 * H;                  // [2 H]: ee[i] couples rows i, i+1
  for (int q = 0; q < TW_SPW; ++q) {
    const int sq = blockIdx.x * TW_SPW + q;
    double* dq = fsm + q * TW_FSM + TW_STAGED;
    for (int i = lane; i < 2 * H; i += 32) {
      dq[i] = (sq < M && i < nx) ? dia[(size_t)sq * nx + i] : 1.0;
      dq[2 * H + i] = (sq < M && i + 1 < nx) ? off[(size_t)sq * nx + i] : 0.0;
    }
  }
  __syncwarp();
  const int mT = nx - nx / 2, mB = nx / 2;
  const int pad = H - (side ? mB : mT);
  const double hs = steady ? 1.0 : h, one = steady ? 0.0 : 1.0;
  double ib_prev = 0.0, y_prev = 0.0, t = 1.0, beta = 1.0;
  bool bad = false;
  for (int j = 0; j < H; ++j) {
    double nl = 0.0, ib = 0.0;
    if (j >= pad) {
      const int row = side ? nx - 1 - (j - pad) : j - pad;
      const double D = fma(hs, dd[row], one);
      const double E = (j > pad) ? hs * ee[side ? row : row - 1] : 0.0;  // coupling to the row before
      const double l = E * ib_prev;
      beta = fma(-l, E, D);
      ib = 1.0 / beta;
      y_prev = fma(-l, y_prev, g0);
      nl = -l;
      if (j > pad) t *= nl;  // t_j = nl_j t_{j-1}
      // (without a source there is no steady state to solve for: A may be singular then)
      bad |= (!(beta > 0.0) && (!steady || g0 != 0.0)) || (!steady && !(fabs(t) >= 1e-150 && fabs(t) <= 1e150));
    }
    if (!steady) {
      if (j > 0) {  // row j-1: its own inv (known one trip ago) and nl_j^2
        tab[twA(j - 1, side)] = ib_prev;
        tab[twA(j - 1, side) + 1] = nl * nl;
      }
      tab[twT(j, side)] = (j >= pad) ? t : 0.0;
    } else {
      scr[4 * j] = y_prev;
      scr[4 * j + 1] = ib;
    }
    ib_prev = ib;
  }
  // middle 2 x 2 systems [bT E; E bB] (x_p, x_q) = (yT, yB): of T in the scaled variables (roles 0 / 1),
  // of A for the steady state (roles 2 / 3)
  const int base = lane & ~3;
  const double b_o = __shfl_sync(KLE_FULL_MASK, beta, base + (role ^ 1));  // the partner's last pivot
  const double t_o = __shfl_sync(KLE_FULL_MASK, t, base + (role ^ 1));
  const double y_o = __shfl_sync(KLE_FULL_MASK, y_prev, base + (role ^ 1));
  const double E = hs * ee[mT - 1];
  const double idet = 1.0 / fma(beta, b_o, -E * E);
  bad |= !(fabs(idet) <= 1e150) && (!steady || g0 != 0.0);
  if (!steady) {
    tab[twA(H - 1, side)] = b_o * idet;                   // ca: own y
    tab[twA(H - 1, side) + 1] = -E * idet * (t_o / t);    // cb': partner's y
  } else {
    // x_mid = (b_o y - E y_o) / det, then outwards x_j = (y_j - e_{j,j+1} x_{j+1}) / b_j
    double xn = (g0 != 0.0) ? (b_o * y_prev - E * y_o) * idet : 0.0;
    tab[twS(H - 1, side)] = xn;
    for (int j = H - 2; j >= 0; --j) {
      double v = 0.0;
      if (j >= pad && g0 != 0.0) {
        const int row = side ? nx - 1 - (j - pad) : j - pad;
        const double e = ee[side ? row - 1 : row];  // couples local rows j, j+1
        v = fma(-e, xn, scr[4 * j]) * scr[4 * j + 1];
        bad |= !(fabs(v) <= 1e150);
      }
      tab[twS(j, side)] = v;
      xn = v;
    }
  }
  bad = (__ballot_sync(KLE_FULL_MASK, bad && live) >> base) & 0xfu;
  __syncwarp();
  if (role == 0 && live) {
    double* fl = blob + (size_t)s * TwL::DOUBLES + TwL::PHI_OFF + TW_FLAG;
    fl[0] = bad ? 1.0 : 0.0;
    fl[1] = 0.0;
  }
  // 1 / t_j by all lanes (off the chains)
  for (int i = lane; i < TW_SPW * 2 * H; i += 32) {
    const int sm_ = i / (2 * H), r = i % (2 * H), j = r >> 1, sd = r & 1;
    double* tb = fsm + sm_ * TW_FSM;
    const double tv = tb[twT(j, sd)];
    tb[twS(j, sd) + 1] = (tv != 0.0) ? 1.0 / tv : 0.0;
  }
  __syncwarp();
  for (int q = 0; q < TW_SPW; ++q) {
    const int sq = blockIdx.x * TW_SPW + q;
    if (sq >= M) break;
    double* out = blob + (size_t)sq * TwL::DOUBLES + TwL::PHI_OFF;
    const double* tb = fsm + q * TW_FSM;
    for (int i = lane; i < TW_STAGED; i += 32) out[i] = tb[i];
  }
}

__global__ void tw_count_flagged_kernel(const double* __restrict__ blob, int M, int stride, int off,
                                        int32_t* __restrict__ count) {
  int n = 0;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < M; s += gridDim.x * blockDim.x)
    n += blob[(size_t)s * stride + off] != 0.0;
  n = __reduce_add_sync(KLE_FULL_MASK, n);
  if ((threadIdx.x & 31) == 0 && n) atomicAdd(count, n);
}

// ---------------------------------------------------------------------------
// Fused F + rhs kernel: CTA = one warp = (sample, 16 subintervals); lane = 2 q + side.
//
// Shared memory, all in the lanes' LOCAL order (position side * H + j holds the row that lane `side`
// keeps in x[j]), so every per-row access of the unrolled loops is a load at an immediate offset:
//   tab [10 H + 2]      the twisted tables (above)
//   de  [H][2][2]       {dia, coupling of local rows j-1 and j} of the operator A (epilogue)
//   st  [17][LD]        start rows of the 16 subintervals (= prev rows of the rhs for n >= 1; the rhs rows
//                       replace them and the warp stores them coalesced), row 16: U_{N-1} (prev of n = 0)
// LD = 2 H + 1: the 16 lane pairs' rows fall into distinct banks.
// ---------------------------------------------------------------------------
namespace {
constexpr int TW_LD = 2 * TW_H + 1;
constexpr int TW_SMEM_DOUBLES = TW_DOUBLES + 4 * TW_H + 17 * TW_LD + 1;
static_assert(TW_DOUBLES % 2 == 0, "16-byte copies");
}

__global__ void __launch_bounds__(32, KLE_TW_MINB) fgr_tw_kernel(FgrArgs a) {
  constexpr int H = TW_H, LD = TW_LD;
  const int s = blockIdx.x;
  if (a.active && a.active[s] != KLE_SAMPLE_ACTIVE) return;
#if KLE_TW_HALVES  // lanes 0..15 = the top lanes of the 16 subintervals, 16..31 the bottom lanes
  const int lane = threadIdx.x, q = lane & 15, side = lane >> 4;
  constexpr int PARTNER = 16;
#else
  const int lane = threadIdx.x, q = lane >> 1, side = lane & 1;
  constexpr int PARTNER = 1;
#endif
  const int nx = a.nx, N = a.N;
  const size_t sbase = (size_t)s * N * nx;
  const int n0 = blockIdx.y * 16;
  const int n = n0 + q;
  const bool valid = n < N;
  const int mT = nx - nx / 2;
  const int padT = H - mT, padB = H - nx / 2;
  const int pad = side ? padB : padT;

  extern __shared__ __align__(16) double sm[];
  double* tab = sm;                  // [TW_DOUBLES]
  double* de = sm + TW_DOUBLES;      // [H][2][2]
  double* st = de + 4 * H;           // [17][LD]
  const unsigned tab_s = (unsigned)__cvta_generic_to_shared(tab);
  const unsigned de_s = (unsigned)__cvta_generic_to_shared(de);
  const unsigned st_s = (unsigned)__cvta_generic_to_shared(st);

  {  // tables (16-byte copies), then the start rows and the operator (coalesced 8-byte copies)
    const double* tg = a.ffac + (size_t)s * TwL::DOUBLES + TwL::PHI_OFF;
#pragma unroll
    for (int i = 0; i < (TW_DOUBLES / 2 + 31) / 32; ++i)
      if (lane + 32 * i < TW_DOUBLES / 2) cp_async16(tab_s + (unsigned)((lane + 32 * i) * 16), tg + (lane + 32 * i) * 2);
    bool rv[4];
    unsigned lo[4];  // byte offset of row lane + 32 i in the local order
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = lane + 32 * i;
      rv[i] = r < nx;
      lo[i] = (unsigned)((r < mT ? r + padT : H + (nx - 1 - r) + padB) * sizeof(double));
    }
    for (int ln = 0; ln < 16; ++ln) {
      const int nn = n0 + ln;
      if (nn >= N) break;
      const double* src = ((nn == 0) ? a.u0 : a.U + sbase + (size_t)(nn - 1) * nx) + lane;
      const unsigned dst = st_s + (unsigned)(ln * LD * sizeof(double));
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (rv[i]) cp_async8(dst + lo[i], src + i * 32);
    }
    asm volatile("cp.async.commit_group;\n" ::);  // group 1: what the sweep needs
    const double* pl = a.U + sbase + (size_t)(N - 1) * nx + lane;
    const double* dg = a.dia + (size_t)s * nx + lane;
    const double* eg = a.off + (size_t)s * nx + lane;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = lane + 32 * i;
      if (!rv[i]) continue;
      if (n0 == 0) cp_async8(st_s + (unsigned)(16 * LD * sizeof(double)) + lo[i], pl + i * 32);
      // de entry of local position p = side * H + j sits at ((j * 2 + side) * 2) doubles
      const int p = (int)(lo[i] / sizeof(double));
      const int sd = p >= H, j = p - sd * H;
      const unsigned e = de_s + (unsigned)(((j * 2 + sd) * 2) * sizeof(double));
      cp_async8(e, dg + i * 32);
      // coupling to the previously eliminated (outer) row: off[r-1] in the top half, off[r] in the bottom half
      if (sd ? (r + 1 < nx) : (r > 0)) cp_async8(e + 8, eg + i * 32 - (sd ? 0 : 1));
    }
    asm volatile("cp.async.commit_group;\n" ::);  // group 2: epilogue operands
#if KLE_TW_PREFETCH
    // L2 prefetch for the CTA that takes this SM slot later (sample s + KLE_TW_PREFETCH CTAs): with 8 latency-bound
    // warps per SM the memory phases of a CTA do not overlap the other CTAs' sweeps, so the fetch is started here
    if (blockIdx.y == 0) {
      const int sp = s + KLE_TW_PREFETCH;
      if (sp < a.M) {
        const char* pu = reinterpret_cast<const char*>(a.U + (size_t)sp * N * nx);
        const int nl_u = (int)(((size_t)N * nx * sizeof(double) + 127) / 128);
        for (int i = lane; i < nl_u; i += 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(pu + (size_t)i * 128));
        const char* pt = reinterpret_cast<const char*>(a.ffac + (size_t)sp * TwL::DOUBLES + TwL::PHI_OFF);
        for (int i = lane; i < (TW_DOUBLES * 8 + 127) / 128; i += 32)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(pt + (size_t)i * 128));
        const char* pd = reinterpret_cast<const char*>(a.dia + (size_t)sp * nx);
        const char* pe = reinterpret_cast<const char*>(a.off + (size_t)sp * nx);
        if (lane < 8) asm volatile("prefetch.global.L2 [%0];" ::"l"(pd + (size_t)lane * 128));
        else if (lane < 16) asm volatile("prefetch.global.L2 [%0];" ::"l"(pe + (size_t)(lane - 8) * 128));
      }
    }
#endif
    // entries no copy writes: the pad rows of this lane's start row (all of it for an unused lane pair),
    // the pad entries of de and the outer coupling of the two end rows
    const int nz = valid ? pad : H;
    for (int j = 0; j < nz; ++j) st[q * LD + side * H + j] = 0.0;
    if (q == 0) {
      for (int j = 0; j <= pad; ++j) {
        if (j < pad) de[(j * 2 + side) * 2] = 0.0;
        de[(j * 2 + side) * 2 + 1] = 0.0;
      }
    }
  }
  asm volatile("cp.async.wait_group 1;\n" ::);
  __syncwarp();
  if (tab[TW_FLAG] != 0.0) {  // no scaled form for this sample: the partitioned kernel takes it (tw_fallback)
    asm volatile("cp.async.wait_group 0;\n" ::);
    return;
  }

  // w_j = (x_j - x*_j) / t_j
  double x[H];
  const unsigned xs = st_s + (unsigned)((q * LD + side * H) * sizeof(double));
  const unsigned tS = tab_s + (unsigned)((4 * H) * sizeof(double) + side * 16);
#pragma unroll
  for (int j = 0; j < H; ++j) {
    const double2 sj = lds_v2(tS + (unsigned)(j * 32));
    x[j] = (lds_f64(xs + (unsigned)(j * sizeof(double))) - sj.x) * sj.y;
  }
  const unsigned tA = tab_s + (unsigned)(side * 16);
  const double2 cm = lds_v2(tA + (unsigned)((H - 1) * 32));  // {ca, cb'}

  // the kernel is bound by shared-memory wavefronts (ncu: 87% of peak, a broadcast 16-byte load costs two):
  // the coefficients of the first KLE_TW_NCACHE rows stay in registers over the J steps
  constexpr int NCACHE = KLE_TW_NCACHE;
  double2 cc[NCACHE > 0 ? NCACHE : 1];
#pragma unroll
  for (int j = 0; j < NCACHE; ++j) cc[j] = lds_v2(tA + (unsigned)(j * 32));
#pragma unroll 1
  for (int it = 0; it < a.J; ++it) {
    // forward prefix sums as KLE_TW_SPLIT independent chains (a warp's step is bound by the latency of its
    // dependent chains: 2 x 64 x ~8 cycles), the later chains corrected by the totals before them
    constexpr int NS = KLE_TW_SPLIT, SL = H / NS;
    double ys[NS];
#pragma unroll
    for (int c = 0; c < NS; ++c) ys[c] = x[c * SL];
#pragma unroll
    for (int j = 1; j < SL; ++j)
#pragma unroll
      for (int c = 0; c < NS; ++c) {
        ys[c] += x[c * SL + j];
        x[c * SL + j] = ys[c];
      }
#pragma unroll
    for (int c = 1; c < NS; ++c) ys[c] += ys[c - 1];  // ys[c]: the sum through chunk c
    const double y = ys[NS - 1];
    const double yp = __shfl_xor_sync(KLE_FULL_MASK, y, PARTNER);
    double xn = fma(cm.x, y, cm.y * yp);
    x[H - 1] = xn;
#pragma unroll
    for (int j = H - 2; j >= 0; --j) {
      const double2 c = (j < NCACHE) ? cc[j < NCACHE ? j : 0] : lds_v2(tA + (unsigned)(j * 32));  // {inv_j, nl_{j+1}^2}
      const double yj = (j >= SL) ? x[j] + ys[j / SL - 1] : x[j];
      xn = fma(c.y, xn, yj * c.x);
      x[j] = xn;
    }
  }
  {  // F_j = t_j w_j + x*_j
    const unsigned tT = tab_s + (unsigned)((8 * H + side * 2) * sizeof(double));
#pragma unroll
    for (int jp = 0; jp < H / 2; ++jp) {
      const double2 t2 = lds_v2(tT + (unsigned)(jp * 32));
      const double2 s0 = lds_v2(tS + (unsigned)((2 * jp) * 32));
      const double2 s1 = lds_v2(tS + (unsigned)((2 * jp + 1) * 32));
      x[2 * jp] = fma(t2.x, x[2 * jp], s0.x);
      x[2 * jp + 1] = fma(t2.y, x[2 * jp + 1], s1.x);
    }
  }

  // epilogue: rhs_n = scaling_n ((I + dT A) F_n - prev_n). In local order the neighbours of row j are
  // x[j-1] (outer; its coupling is 0 for the first real row) and x[j+1] (inner; the partner's middle
  // row for j = H-1). Pad rows compute finite values nobody reads.
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncwarp();
  const double xmid = __shfl_xor_sync(KLE_FULL_MASK, x[H - 1], PARTNER);
  const double sc = valid ? a.scaling[n] : 0.0;
  const double pmul = (n == 0) ? a.alpha : 1.0;
  const double emid = __ldg(a.off + (size_t)s * nx + mT - 1);  // couples the two middle rows
  const unsigned ps = (n == 0) ? st_s + (unsigned)((16 * LD + side * H) * sizeof(double)) : xs;
  const unsigned des = de_s + (unsigned)(side * 16);
  double xo = 0.0;
  double2 d0 = lds_v2(des);
#pragma unroll
  for (int j = 0; j < H; ++j) {
    double2 d1;
    if (j < H - 1) d1 = lds_v2(des + (unsigned)((j + 1) * 32));
    const double ei = (j < H - 1) ? d1.y : emid;
    const double xc = x[j];
    const double xi = (j < H - 1) ? x[j + 1] : xmid;
    const double prev = lds_f64(ps + (unsigned)(j * sizeof(double)));
    const double Ax = fma(d0.y, xo, fma(d0.x, xc, ei * xi));
    const double rhs = fma(a.dT, Ax, xc) - pmul * prev;
    xo = xc;
    x[j] = sc * rhs;
    if (j < H - 1) d0 = d1;
  }
  __syncwarp();  // every prev row (row 16 is shared by nobody else, but keep the reads before the writes)
#pragma unroll
  for (int j = 0; j < H; ++j) asm volatile("st.shared.f64 [%0], %1;" ::"r"(xs + (unsigned)(j * sizeof(double))), "d"(x[j]) : "memory");
  __syncwarp();
  for (int ln = 0; ln < 16; ++ln) {
    const int nn = n0 + ln;
    if (nn >= N) break;
    double* out = a.Rout + sbase + (size_t)nn * nx + lane;
    const double* rs = st + ln * LD;
    double v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = (lane + 32 * i < nx) ? lane + 32 * i : 0;
      v[i] = rs[r < mT ? r + padT : H + (nx - 1 - r) + padB];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (lane + 32 * i < nx) out[32 * i] = v[i];
  }
}

bool tw_supported(const FineLayoutRT& lay, int nx) {
  if (KLE_FINE_LAZY) return false;
  if (lay.W || lay.kind || lay.MR != 16 || lay.P != 8) return false;
  if (nx <= TW_H || nx > 2 * TW_H) return false;
  const char* e = getenv("KLE_FGR_TW");  // read per call (A/B in one process)
  return !(e && *e == '0');
}


int tw_factor(const double* dia, const double* off, double* blob, int M, int nx, double h, double g0,
              cudaStream_t st) {
  constexpr size_t smem = sizeof(double) * TW_SPW * TW_FSM;
  static PerDeviceOnce attr_once;
  if (int rc = once_per_device(attr_once, "kle_fine_tw(factor): cudaFuncSetAttribute", [&] {
        return cudaFuncSetAttribute(tw_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      }))
    return rc;
  if (M > 0) tw_factor_kernel<<<(unsigned)((M + TW_SPW - 1) / TW_SPW), 32, smem, st>>>(dia, off, blob, M, nx, h, g0);
  return check_launch("tw_factor_kernel");
}

// number of samples of the batch without a scaled twisted form (flagged by tw_factor) -> *count (device, += )
int tw_count_flagged(const double* blob, int M, int stride, int off, int32_t* count, cudaStream_t st) {
  if (stride == 0) {
    stride = TwL::DOUBLES;
    off = kTwFlagOff;
  }
  if (M > 0)
    tw_count_flagged_kernel<<<(unsigned)std::min((M + 255) / 256, 1184), 256, 0, st>>>(blob, M, stride, off, count);
  return check_launch("tw_count_flagged_kernel");
}

int tw_fgr(const FgrArgs& a, cudaStream_t st) {
  const size_t smem = sizeof(double) * (size_t)TW_SMEM_DOUBLES;
  static PerDeviceOnce attr_once;
  if (int rc = once_per_device(attr_once, "kle_fine_tw: cudaFuncSetAttribute", [&] {
        cudaError_t e = cudaFuncSetAttribute(fgr_tw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        if (e != cudaSuccess) return e;
        return cudaFuncSetAttribute(fgr_tw_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      }))
    return rc;
  dim3 grid(a.M, (a.N + 15) / 16);
  fgr_tw_kernel<<<grid, 32, smem, st>>>(a);
  return check_launch("fgr_tw_kernel");
}

}  // namespace kle
