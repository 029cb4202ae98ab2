// 2D fine sweeps with TMA-staged factor blocks (config 3, the fine half of
// pintuq/propagators.py:25-39,121-145 + the rhs of pcgc.py:175-197,233-237).
//
// Same arithmetic as fine2d_kernel (kle_2d.cu): every BE step is a forward
// and a backward banded substitution over the window of the last n solved
// rows, rows in blocks of RB = 8 (a register-blocked far part and an 8 x 8
// triangular near part). What changes is where the operands come from:
//
//   * the factor is restaged once per solve (fine2d_stage_kernel) into one
//     contiguous chunk per (direction, row block) that already has the skewed
//     coefficient layout the sweep reads, plus D^{-1} of the block's rows:
//     Lf/Lb[s][blk][(n + 8) * 8 + 8] — one cp.async.bulk per block instead of
//     1,016 gathered 8-byte loads;
//   * one CTA per (sample, 32 right-hand sides), NW warps of 32 / NW right-hand
//     sides each (the lane groups of a warp split the window sweep); the
//     coefficient chunk is shared by the CTA's warps and a block's 32
//     right-hand-side rows ([nx][32] layout, 2 KB contiguous) come in the same
//     stage;
//   * a D-stage ring fed by one elected thread (cp.async.bulk + mbarrier
//     complete_tx), so D - 1 blocks of loads are in flight while a block is
//     solved. The per-warp version it replaces kept one block of look-ahead in
//     registers (254 registers) and waited on HBM latency at every block.
#include <cstdlib>

#include "kle_common.cuh"
#include "kle_internal.h"

namespace kle {

namespace {

constexpr int TB_RB = 8;  // rows per block (as SB_RB)
#ifndef KLE_2D_TMA_STAGES
#define KLE_2D_TMA_STAGES 5
#endif
constexpr int TB_D = KLE_2D_TMA_STAGES;
#ifndef KLE_2D_TMA_U
#define KLE_2D_TMA_U 4
#endif
constexpr int TB_U = KLE_2D_TMA_U;  // window positions per register chunk of the far sweep

__host__ __device__ inline int tb_wp(int n) {
  int w = 1;
  while (w < n + 1) w <<= 1;
  return w;
}
// far rows padded to KP = 16 ceil(n/16) (zero rows n..KP-1: the DMMA loop runs whole groups of four
// 4-row k-steps with no bounds test), then 8 near rows and D^{-1}
__host__ __device__ inline int tb_kp(int n) { return (n + 15) / 16 * 16; }
__host__ __device__ inline int tb_ch(int n) { return (tb_kp(n) + TB_RB + 1) * TB_RB; }  // doubles per chunk
__host__ __device__ inline int tb_nblk(int n) { return (n * n + TB_RB - 1) / TB_RB; }

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "TB_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra TB_WAIT_%=;\n"
      "}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_async_global() { asm volatile("fence.proxy.async.global;\n" ::: "memory"); }

}  // namespace

// ---------------------------------------------------------------------------
// Restage: chunk e of block blk (p0 = 8 blk) in the unpadded row numbering u
// (far rows u < n, then rows KP.. hold u = n.., zero rows between), forward (dir 0):
//   e = u*8 + a, u < n:       L(p0+a, p0-n+u) = Lt[p0-n+u][n-1-u+a]   (a <= u)
//   e = (n+a2)*8 + a:         L(p0+a, p0+a2)  = Lt[p0+a2][a-a2-1]      (a2 < a)
//   e = (n+8)*8 + a:          Dinv[p0+a]
// backward (dir 1, sequence position p -> row nx-1-p):
//   e = v*8 + a:              Lt[nx-1-(p0+a)][a+n-1-v]                 (0 <= a+n-1-v < n)
// zero outside the band and beyond the last row (Dinv 1). These are the cst
// layouts of subst_pass (kle_2d.cu), so the sweep arithmetic is unchanged.
// ---------------------------------------------------------------------------
__global__ void fine2d_stage_kernel(const double* __restrict__ Lt, const double* __restrict__ Dinv, int M, int n,
                                    double* __restrict__ stage) {
  const int nx = n * n, CH = tb_ch(n), nb = tb_nblk(n);
  const long long per = 2LL * nb * CH;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)M * per) return;
  const int s = (int)(t / per);
  long long r = t - (long long)s * per;
  const int dir = (int)(r / ((long long)nb * CH));
  r -= (long long)dir * nb * CH;
  const int blk = (int)(r / CH), e = (int)(r - (long long)blk * CH);
  const double* L = Lt + (size_t)s * nx * n;
  const int p0 = blk * TB_RB, a = e % TB_RB, up = e / TB_RB, KP = tb_kp(n);
  // chunk row up -> row u of the unpadded layout (far rows < n, near rows n..n+7, D^{-1} at n+8)
  const int u = up < n ? up : (up >= KP ? up - KP + n : -1);
  const int p = p0 + a;
  double v = 0.0;
  if (u < 0) {
    v = 0.0;
  } else if (u == n + TB_RB) {
    v = (dir == 0 && p < nx) ? Dinv[(size_t)s * nx + p] : 1.0;
  } else if (p < nx) {
    if (dir == 0) {
      if (u < n) {
        const int k = p0 - n + u;
        if (a <= u && k >= 0) v = L[(size_t)k * n + (n - 1 - u + a)];
      } else {
        const int a2 = u - n;
        if (a2 < a) v = L[(size_t)(p0 + a2) * n + (a - a2 - 1)];
      }
    } else {
      const int uu = a + n - 1 - u;
      if (uu >= 0 && uu < n) v = L[(size_t)(nx - 1 - p) * n + uu];
    }
  }
  stage[t] = v;
}

struct Fine2dTmaArgs {
  const double* start;    // mode 0: U [M][N][nx]; mode 1: start rows [M][Q][nx]
  const double* u0;       // mode 0: [nx]
  const double* F_given;  // mode 0, optional
  const double *dia, *ex, *ey;
  const double* stage;    // [M][2][nblk][CH]
  const double* scaling;  // mode 0: [N]
  const int32_t* active;  // mode 0: [M] or null
  double* X;              // [M * G][nx][32]
  double* Z;              // [M * G][nx][32]
  double* out;            // mode 0: R [M][N][nx]; mode 1: [M][Q][nseg][nx]
  int M, N, n, J, nseg, mode;
  double dt, dT, g0, alpha;
};

// One pass (forward: Z = D^{-1} L^{-1} (X + h g); backward: X = L^{-T} Z) of
// the CTA's 32 right-hand sides. `it` counts the blocks the CTA has consumed
// (stage = it % D, parity = (it / D) & 1).
template <bool BACK, int NW>
__device__ __forceinline__ void tma_pass(const double* __restrict__ chunks, const double* __restrict__ bsrc,
                                         double badd, double* __restrict__ outp, double* stg, uint64_t* full,
                                         double* win, int n, int& it) {
  constexpr int RB = TB_RB, RW = 32 / NW;
  const int nx = n * n, CH = tb_ch(n), SZ = CH + RB * 32, nb = tb_nblk(n), WP = tb_wp(n), wm = WP - 1;
  const int KP = tb_kp(n);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int r = lane % RW, h = lane / RW, j = w * RW + r;
  auto issue = [&](int b, int st) {
    const int p0 = b * RB, cnt = min(RB, nx - p0);
    double* dst = stg + (size_t)st * SZ;
    const double* bs = bsrc + (size_t)(BACK ? nx - p0 - cnt : p0) * 32;
    mb_expect(&full[st], (unsigned)(CH * 8 + cnt * 256));
    bulk_g2s(dst, chunks + (size_t)b * CH, (unsigned)(CH * 8), &full[st]);
    bulk_g2s(dst + CH, bs, (unsigned)(cnt * 256), &full[st]);
  };
  for (int q = lane; q < WP * RW; q += 32) win[q] = 0.0;
  if (tid == 0)
    for (int b = 0; b < TB_D - 1 && b < nb; ++b) issue(b, (it + b) % TB_D);
  for (int b = 0; b < nb; ++b) {
    __syncthreads();  // every warp is done with block b - 1: its stage can be refilled
    if (tid == 0 && b + TB_D - 1 < nb) issue(b + TB_D - 1, (it + b + TB_D - 1) % TB_D);
    const int st = (it + b) % TB_D;
    mb_wait(&full[st], (unsigned)(((it + b) / TB_D) & 1));
    const double* cst = stg + (size_t)st * SZ;
    const double* bvs = cst + CH;
    const int p0 = b * RB, cnt = min(RB, nx - p0);
    double bv[RB], dv[RB];
#pragma unroll
    for (int a = 0; a < RB; ++a) {
      bv[a] = (a < cnt) ? bvs[(BACK ? cnt - 1 - a : a) * 32 + j] : 0.0;
      dv[a] = BACK ? 1.0 : cst[(KP + RB) * RB + a];
    }
    // near-part coefficients, loaded now (off the chain of the triangular fix-up)
    double nc[RB * (RB - 1) / 2];
#pragma unroll
    for (int a = 1, t = 0; a < RB; ++a)
#pragma unroll
      for (int a2 = 0; a2 < a; ++a2, ++t) nc[t] = cst[(KP + a2) * RB + a];
    // far part: this lane's window positions qq = h + NW m, m < nq, in chunks
    // of TB_U with the next chunk's shared-memory loads in flight (one warp per
    // SM sub-partition: nothing else hides their latency)
    double acc[RB];
#pragma unroll
    for (int a = 0; a < RB; ++a) acc[a] = 0.0;
    const int q0 = p0 - n;
    const int nq = (n - h + NW - 1) / NW;
    double yA[TB_U], yB[TB_U];
    double2 cA[TB_U][RB / 2], cB[TB_U][RB / 2];
    auto ld = [&](int m0, double* yy, double2 (*cc)[RB / 2]) {
#pragma unroll
      for (int u = 0; u < TB_U; ++u) {
        const int m = m0 + u;
        const int qq = min(h + NW * m, n - 1);
        const double y = win[((q0 + qq) & wm) * RW + r];
        yy[u] = m < nq ? y : 0.0;
#pragma unroll
        for (int k = 0; k < RB / 2; ++k) cc[u][k] = *reinterpret_cast<const double2*>(cst + qq * RB + 2 * k);
      }
    };
    auto fm = [&](const double* yy, const double2 (*cc)[RB / 2]) {
#pragma unroll
      for (int u = 0; u < TB_U; ++u)
#pragma unroll
        for (int k = 0; k < RB / 2; ++k) {
          acc[2 * k] = fma(cc[u][k].x, yy[u], acc[2 * k]);
          acc[2 * k + 1] = fma(cc[u][k].y, yy[u], acc[2 * k + 1]);
        }
    };
    ld(0, yA, cA);
    for (int m0 = 0; m0 < nq; m0 += 2 * TB_U) {
      ld(m0 + TB_U, yB, cB);
      fm(yA, cA);
      if (m0 + TB_U >= nq) break;
      ld(m0 + 2 * TB_U, yA, cA);
      fm(yB, cB);
    }
#pragma unroll
    for (int o = RW; o < 32; o <<= 1)
#pragma unroll
      for (int a = 0; a < RB; ++a) acc[a] += __shfl_xor_sync(KLE_FULL_MASK, acc[a], o);
    double yv[RB];
#pragma unroll
    for (int a = 0; a < RB; ++a) {
      double v = (bv[a] + badd) - acc[a];
#pragma unroll
      for (int a2 = 0; a2 < a; ++a2) v = fma(-nc[a * (a - 1) / 2 + a2], yv[a2], v);
      yv[a] = v;
      if (a < cnt && h == 0) {
        const int p = p0 + a;
        win[(p & wm) * RW + r] = v;
        outp[(size_t)(BACK ? nx - 1 - p : p) * 32 + j] = BACK ? v : v * dv[a];
      }
    }
  }
  it += nb;
  fence_async_global();  // this pass's stores are read by the next pass's bulk copies
  __syncthreads();
}

__device__ __forceinline__ void dmma_acc(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// The same pass with the far part on the FP64 tensor cores: per block, the
// 8 x 32 update D[a][rhs] = sum_qq cst[qq][a] win[q0 + qq][rhs] is a
// (8 x n) x (n x 32) product; warp w owns the 8 x 8 tile of right-hand sides
// 8w..8w+7 and runs ceil(n / 4) DMMA m8n8k4 steps (A fragment cst[4ks + k][a],
// 2 shared-memory wavefronts; B fragment from the warp's [WP][8] window, 2
// wavefronts) into two accumulators. The tile goes through a 64-double
// scratch so lanes 0..7 (one right-hand side each) run the triangular near
// part. 4 warps (one n-tile each), no cross-warp reduction.
template <bool BACK, int RPC>
__device__ __forceinline__ void tma_pass_mma(const double* __restrict__ chunks, const double* __restrict__ bsrc,
                                             double badd, double* __restrict__ outp, double* stg, uint64_t* full,
                                             double* win, double* xs, int n, int& it) {
  constexpr int RB = TB_RB;
  const int nx = n * n, CH = tb_ch(n), SZ = CH + RB * RPC, nb = tb_nblk(n), WP = tb_wp(n), wm = WP - 1;
  const int KP = tb_kp(n);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int fa = lane >> 2, fk = lane & 3, rl = lane & 7, j = w * 8 + rl;
  const int KS = KP / 4;  // a multiple of 4
  auto issue = [&](int b, int st) {
    const int p0 = b * RB, cnt = min(RB, nx - p0);
    double* dst = stg + (size_t)st * SZ;
    const double* bs = bsrc + (size_t)(BACK ? nx - p0 - cnt : p0) * RPC;
    mb_expect(&full[st], (unsigned)(CH * 8 + cnt * RPC * 8));
    bulk_g2s(dst, chunks + (size_t)b * CH, (unsigned)(CH * 8), &full[st]);
    bulk_g2s(dst + CH, bs, (unsigned)(cnt * RPC * 8), &full[st]);
  };
  for (int q = lane; q < WP * 8; q += 32) win[q] = 0.0;
  if (tid == 0)
    for (int b = 0; b < TB_D - 1 && b < nb; ++b) issue(b, (it + b) % TB_D);
  for (int b = 0; b < nb; ++b) {
    __syncthreads();  // every warp is done with block b - 1: its stage can be refilled
    if (tid == 0 && b + TB_D - 1 < nb) issue(b + TB_D - 1, (it + b + TB_D - 1) % TB_D);
    const int st = (it + b) % TB_D;
    mb_wait(&full[st], (unsigned)(((it + b) / TB_D) & 1));
    const double* cst = stg + (size_t)st * SZ;
    const double* bvs = cst + CH;
    const int p0 = b * RB, cnt = min(RB, nx - p0);
    double bv[RB], dv[RB], nc[RB * (RB - 1) / 2];
#pragma unroll
    for (int a = 0; a < RB; ++a) {
      bv[a] = (a < cnt) ? bvs[(BACK ? cnt - 1 - a : a) * RPC + j] : 0.0;
      dv[a] = BACK ? 1.0 : cst[(KP + RB) * RB + a];
    }
#pragma unroll
    for (int a = 1, t = 0; a < RB; ++a)
#pragma unroll
      for (int a2 = 0; a2 < a; ++a2, ++t) nc[t] = cst[(KP + a2) * RB + a];
    const int q0 = p0 - n;
    // four independent accumulators (8-deep DMMA chains at n = 127). A fragments at immediate
    // offsets (rows >= n of the chunk are zero); B fragment slot (q0 + 4 ks + fk) & wm advanced
    // by 4 per k-step on a pre-scaled index
    double c0[2] = {0.0, 0.0}, c1[2] = {0.0, 0.0}, c2[2] = {0.0, 0.0}, c3[2] = {0.0, 0.0};
    const double* ap = cst + fk * RB + fa;
    const int bmask = WP * 8 - 1;
    const int bb = ((q0 + fk) * 8 + fa) & bmask;
#pragma unroll 2
    for (int ks = 0; ks < KS; ks += 4) {
      const double A0 = ap[(4 * ks) * RB], A1 = ap[(4 * ks + 4) * RB];
      const double A2 = ap[(4 * ks + 8) * RB], A3 = ap[(4 * ks + 12) * RB];
      const double B0 = win[(bb + 32 * ks) & bmask], B1 = win[(bb + 32 * ks + 32) & bmask];
      const double B2 = win[(bb + 32 * ks + 64) & bmask], B3 = win[(bb + 32 * ks + 96) & bmask];
      dmma_acc(c0, A0, B0);
      dmma_acc(c1, A1, B1);
      dmma_acc(c2, A2, B2);
      dmma_acc(c3, A3, B3);
    }
    xs[fa * 8 + 2 * fk] = (c0[0] + c1[0]) + (c2[0] + c3[0]);
    xs[fa * 8 + 2 * fk + 1] = (c0[1] + c1[1]) + (c2[1] + c3[1]);
    __syncwarp();
    if (lane < 8) {
      double yv[RB];
#pragma unroll
      for (int a = 0; a < RB; ++a) {
        double v = (bv[a] + badd) - xs[a * 8 + lane];
#pragma unroll
        for (int a2 = 0; a2 < a; ++a2) v = fma(-nc[a * (a - 1) / 2 + a2], yv[a2], v);
        yv[a] = v;
        if (a < cnt) {
          const int p = p0 + a;
          win[(p & wm) * 8 + lane] = v;
          outp[(size_t)(BACK ? nx - 1 - p : p) * RPC + j] = BACK ? v : v * dv[a];
        }
      }
    }
  }
  it += nb;
  fence_async_global();  // this pass's stores are read by the next pass's bulk copies
  __syncthreads();
}

template <int NW, bool MMA>
__device__ __forceinline__ void tma_steps(const Fine2dTmaArgs& a, int s, double* X, double* Z, double* stg,
                                          uint64_t* full, double* win, double* xs, int& it) {
  const int n = a.n;
  const size_t per = 2ull * tb_nblk(n) * tb_ch(n);
  const double* Lf = a.stage + (size_t)s * per;
  const double* Lb = Lf + per / 2;
  const double hg = a.dt * a.g0;
  for (int step = 0; step < a.J; ++step) {
    if constexpr (MMA) {
      tma_pass_mma<false, 8 * NW>(Lf, X, hg, Z, stg, full, win, xs, n, it);
      tma_pass_mma<true, 8 * NW>(Lb, Z, 0.0, X, stg, full, win, xs, n, it);
    } else {
      tma_pass<false, NW>(Lf, X, hg, Z, stg, full, win, n, it);
      tma_pass<true, NW>(Lb, Z, 0.0, X, stg, full, win, n, it);
    }
  }
}

template <int NW, bool MMA>
__global__ void __launch_bounds__(32 * NW) fine2d_tma_kernel(Fine2dTmaArgs a) {
  constexpr int NT = 32 * NW, RW = 32 / NW;
  constexpr int RPC = MMA ? 8 * NW : 32;  // right-hand sides per CTA (one 8-wide DMMA tile per warp)
  constexpr int WW = MMA ? 8 : RW;        // window columns per warp
  static_assert(NT % RPC == 0, "the start-state load maps threads to right-hand sides");
  const int n = a.n, nx = n * n;
  const int G = (a.N + RPC - 1) / RPC;
  const int s = blockIdx.x / G, g = blockIdx.x % G;
  if (a.mode == 0 && a.active && a.active[s] != KLE_SAMPLE_ACTIVE) return;
  const int tid = threadIdx.x, w = tid >> 5;
  extern __shared__ __align__(128) double tsm[];
  const int SZ = tb_ch(n) + TB_RB * RPC;
  double* stg = tsm;                                         // [D][SZ]
  double* win = stg + (size_t)TB_D * SZ + (size_t)w * tb_wp(n) * WW;  // per warp [WP][RW]
  double* xs = stg + (size_t)TB_D * SZ + (size_t)NW * tb_wp(n) * WW + (size_t)w * 64;  // per warp [8][8]
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + (size_t)TB_D * SZ + (size_t)NW * tb_wp(n) * WW + NW * 64);
  if (tid == 0)
    for (int k = 0; k < TB_D; ++k) mb_init(&full[k], 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  double* X = a.X + (size_t)blockIdx.x * nx * RPC;
  double* Z = a.Z + (size_t)blockIdx.x * nx * RPC;
  // load the start states, X[i][jj] (RPC right-hand sides; dead ones zero):
  // consecutive threads write consecutive X entries (rows of RPC doubles)
  {
    // thread tid always handles the same right-hand side jj = tid % RPC (NT is a multiple of RPC)
    const int jj = tid % RPC;
    const int q = g * RPC + jj;
    const bool live = q < a.N;
    const double* src;
    if (a.mode == 0) {
      src = (q == 0 || !live) ? a.u0 : a.start + ((size_t)s * a.N + (q - 1)) * nx;
      if (a.F_given && live) src = a.F_given + ((size_t)s * a.N + q) * nx;
    } else {
      src = a.start + ((size_t)s * a.N + (live ? q : 0)) * nx;
    }
    for (int i = tid / RPC; i < nx; i += NT / RPC) X[(size_t)i * RPC + jj] = live ? src[i] : 0.0;
  }
  fence_async_global();
  __syncthreads();
  int it = 0;
  if (a.mode == 1) {
    for (int sg = 0; sg < a.nseg; ++sg) {
      tma_steps<NW, MMA>(a, s, X, Z, stg, full, win, xs, it);
      {
        const int jj = tid % RPC, q = g * RPC + jj;
        if (q < a.N) {
          double* o = a.out + (((size_t)s * a.N + q) * a.nseg + sg) * nx;
          for (int i = tid / RPC; i < nx; i += NT / RPC) o[i] = X[(size_t)i * RPC + jj];
        }
      }
      __syncthreads();
    }
    return;
  }
  if (!a.F_given) tma_steps<NW, MMA>(a, s, X, Z, stg, full, win, xs, it);
  // rhs_n = scaling_n ((I + dT A) F_n - prev_n); prev_0 = alpha U_{N-1}
  const double* dd = a.dia + (size_t)s * nx;
  const double* ex = a.ex + (size_t)s * nx;
  const double* ey = a.ey + (size_t)s * nx;
  {
    // thread tid keeps right-hand side jj = tid % RPC: X rows are read contiguously
    const int jj = tid % RPC;
    const int q = g * RPC + jj;
    if (q < a.N) {
      const double* pv = (q == 0) ? a.start + ((size_t)s * a.N + (a.N - 1)) * nx
                                  : a.start + ((size_t)s * a.N + (q - 1)) * nx;
      const double pmul = (q == 0) ? a.alpha : 1.0;
      const double sc = a.scaling[q];
      double* o = a.out + ((size_t)s * a.N + q) * nx;
      const double* Xq = X + jj;
      for (int i = tid / RPC; i < nx; i += NT / RPC) {
        const double x = Xq[(size_t)i * RPC];
        double Ax = dd[i] * x;
        if (i + 1 < nx) Ax = fma(ex[i], Xq[(size_t)(i + 1) * RPC], Ax);
        if (i >= 1) Ax = fma(ex[i - 1], Xq[(size_t)(i - 1) * RPC], Ax);
        if (i + n < nx) Ax = fma(ey[i], Xq[(size_t)(i + n) * RPC], Ax);
        if (i >= n) Ax = fma(ey[i - n], Xq[(size_t)(i - n) * RPC], Ax);
        const double rhs = fma(a.dT, Ax, x) - pmul * pv[i];
        o[i] = sc * rhs;
      }
    }
  }
}

size_t fine2d_stage_doubles(int M, int n) {
  return (M <= 0 || n <= 0) ? 0 : 2 * (size_t)M * tb_nblk(n) * tb_ch(n);
}

int fine2d_stage(const double* Lt, const double* Dinv, int M, int n, double* stage, cudaStream_t st) {
  const long long tot = (long long)fine2d_stage_doubles(M, n);
  if (tot == 0) return KLE_OK;
  fine2d_stage_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(Lt, Dinv, M, n, stage);
  return check_launch("fine2d_stage_kernel");
}

template <int NW, bool MMA>
static int tma_launch(const Fine2dTmaArgs& a, cudaStream_t st) {
  constexpr int RPC = MMA ? 8 * NW : 32;
  const size_t smem = sizeof(double) * ((size_t)TB_D * (tb_ch(a.n) + TB_RB * RPC) + (size_t)RPC * tb_wp(a.n) +
                                        (size_t)NW * 64) +
                      sizeof(uint64_t) * TB_D;
  cudaFuncSetAttribute(fine2d_tma_kernel<NW, MMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int G = (a.N + RPC - 1) / RPC;
  fine2d_tma_kernel<NW, MMA><<<(unsigned)(a.M * G), 32 * NW, smem, st>>>(a);
  return check_launch("fine2d_tma_kernel");
}

int fine2d_tma(const double* start, const double* u0, const double* F_given, const double* dia, const double* ex,
               const double* ey, const double* stage, const double* scaling, const int32_t* active, int M, int N,
               int n, int J, int nseg, int mode, double dt, double dT, double g0, double alpha, double* X, double* Z,
               double* out, cudaStream_t st) {
  Fine2dTmaArgs a{start, u0, F_given, dia, ex, ey, stage, scaling, active, X, Z, out,
                  M, N, n, J, nseg, mode, dt, dT, g0, alpha};
  static const int nw_env = [] {
    const char* e = getenv("KLE_2D_TMA_NW");
    return e ? atoi(e) : 0;
  }();
  static const bool mma = [] {
    const char* e = getenv("KLE_2D_TMA_MMA");
    return !(e && e[0] == '0');
  }();
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  if (!mma) return tma_launch<4, false>(a, st);
  // right-hand sides per CTA: 32 (4 warps) when the batch gives >= 2 CTAs per
  // SM, else 16 or 8 so the latency-bound per-block chain has company
  int nw = nw_env;
  if (nw != 1 && nw != 2 && nw != 4) {
    nw = N <= 8 ? 1 : (N <= 16 ? 2 : 4);
    while (nw > 1 && (long long)M * ((N + 8 * nw - 1) / (8 * nw)) < 2LL * sms) nw /= 2;
  }
  if (nw == 1) return tma_launch<1, true>(a, st);
  if (nw == 2) return tma_launch<2, true>(a, st);
  return tma_launch<4, true>(a, st);
}

}  // namespace kle

// ===========================================================================
// C ABI (declared in include/kle_b200.h)
// ===========================================================================
using namespace kle;
extern "C" size_t kle_2d_fine_work_doubles(int M, int N, int n);

extern "C" size_t kle_2d_fine_stage_doubles(int M, int n) { return fine2d_stage_doubles(M, n); }

extern "C" int kle_2d_fine_stage_f64(const double* Lt, const double* Dinv, int M, int n, double* stage,
                                     void* stream) {
  if (M < 0 || n < 1 || n > 127) return set_error(KLE_ERR_INVALID, "fine_stage2d: bad dims");
  return fine2d_stage(Lt, Dinv, M, n, stage, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int kle_2d_fgr_staged_f64(const double* U, const double* u0, const double* F_given, const double* dia,
                                     const double* ex, const double* ey, const double* stage,
                                     const double* scaling, const int32_t* active, int M, int N, int n, int J,
                                     double dt, double dT, double g0, double alpha, double* work,
                                     size_t work_doubles, double* Rout, void* stream) {
  if (M < 0 || N < 1 || n < 1 || n > 127 || J < 1) return set_error(KLE_ERR_INVALID, "fgr2d: bad dims");
  if (M == 0) return KLE_OK;
  const size_t need = kle_2d_fine_work_doubles(M, N, n);
  if (work_doubles < need) return set_error(KLE_ERR_WORKSPACE, "fgr2d: workspace too small");
  return fine2d_tma(U, u0, F_given, dia, ex, ey, stage, scaling, active, M, N, n, J, 1, 0, dt, dT, g0, alpha, work,
                    work + need / 2, Rout, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int kle_2d_sweep_staged_f64(const double* start, const double* stage, int M, int Q, int n, int J,
                                       int nseg, double h, double g0, double* work, size_t work_doubles,
                                       double* out, void* stream) {
  if (M < 0 || Q < 1 || n < 1 || n > 127 || J < 1 || nseg < 1) return set_error(KLE_ERR_INVALID, "sweep2d: bad dims");
  if (M == 0) return KLE_OK;
  const size_t need = kle_2d_fine_work_doubles(M, Q, n);
  if (work_doubles < need) return set_error(KLE_ERR_WORKSPACE, "sweep2d: workspace too small");
  return fine2d_tma(start, nullptr, nullptr, nullptr, nullptr, nullptr, stage, nullptr, nullptr, M, Q, n, J, nseg, 1,
                    h, 0.0, g0, 0.0, work, work + need / 2, out, reinterpret_cast<cudaStream_t>(stream));
}
