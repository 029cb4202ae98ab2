// Multi-warp fine propagator for large nx (config 5: nx = 4095).
//
// Same LDL^T recurrences as kle_fine.cuh (pintuq/propagators.py:25-39,
// 121-157), but one system spans W warps = one CTA: 32*W lanes own MR rows
// each (registers). Chunks are stitched in two levels per recurrence:
//   lane level  5-stage Kogge-Stone shuffle scan inside the warp
//   warp level  warp composites through shared memory; each warp composes
//               the composites of the warps before (forward) / after
//               (backward) it, then lanes apply their exclusive products.
// Two CTA barriers per backward-Euler step.
//
// Blob per sample (doubles): l[nxp] | inv[nxp] (lane-major, lane L owns rows
// L*MR..) | af[5][32W] | bb[5][32W] | aex[32W] | sex[32W] | aw[W] | sw[W]
//   af/bb  in-warp Kogge-Stone multipliers
//   aex    product of the chunk-end forward multipliers of the lanes before
//          this one in its warp;  sex  same for the backward, lanes after
//   aw/sw  whole-warp products
#include <cstdlib>

#include "kle_fine.cuh"
#include "kle_internal.h"

namespace kle {

template <int MR>
struct MwLayout {
  int W, nxp, lanes;
  __host__ __device__ MwLayout(int W_) : W(W_), nxp(32 * W_ * MR), lanes(32 * W_) {}
  __host__ __device__ int l_off() const { return 0; }
  __host__ __device__ int inv_off() const { return nxp; }
  __host__ __device__ int af_off() const { return 2 * nxp; }
  __host__ __device__ int bb_off() const { return 2 * nxp + 5 * lanes; }
  __host__ __device__ int aex_off() const { return 2 * nxp + 10 * lanes; }
  __host__ __device__ int sex_off() const { return 2 * nxp + 11 * lanes; }
  __host__ __device__ int aw_off() const { return 2 * nxp + 12 * lanes; }
  __host__ __device__ int sw_off() const { return 2 * nxp + 12 * lanes + W; }
  __host__ __device__ int doubles() const { return 2 * nxp + 12 * lanes + 2 * W; }
};

template <int MR>
__global__ void mw_factor_kernel(const double* __restrict__ dia, const double* __restrict__ off,
                                 double* __restrict__ blob, int M, int nx, int W, double h) {
  const MwLayout<MR> L(W);
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= M) return;
  const double* d = dia + (size_t)s * nx;
  const double* e = off + (size_t)s * nx;
  double* b = blob + (size_t)s * L.doubles();
  double beta_prev = 1.0;
  for (int row = 0; row < L.nxp; ++row) {
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
    b[L.l_off() + row] = l;
    b[L.inv_off() + row] = inv;
  }
  for (int w = 0; w < W; ++w) {
    double pie[32], sigs[32];
    for (int k = 0; k < 32; ++k) {
      const int lane = w * 32 + k;
      double pi = 1.0, sg = 1.0;
      for (int j = 0; j < MR; ++j) pi *= -b[L.l_off() + lane * MR + j];
      for (int j = MR - 1; j >= 0; --j) {
        const int row = lane * MR + j;
        sg *= -((row + 1 < L.nxp) ? b[L.l_off() + row + 1] : 0.0);
      }
      pie[k] = pi;
      sigs[k] = sg;
    }
    double ax = 1.0;
    for (int k = 0; k < 32; ++k) {
      b[L.aex_off() + w * 32 + k] = ax;
      ax *= pie[k];
    }
    b[L.aw_off() + w] = ax;
    double sx = 1.0;
    for (int k = 31; k >= 0; --k) {
      b[L.sex_off() + w * 32 + k] = sx;
      sx *= sigs[k];
    }
    b[L.sw_off() + w] = sx;
    for (int t = 0; t < 5; ++t) {
      const int dd = 1 << t;
      for (int k = 0; k < 32; ++k) {
        double af = 0.0, bb = 0.0;
        if (k >= dd) {
          af = 1.0;
          for (int q = k - dd + 1; q <= k; ++q) af *= pie[q];
        }
        if (k + dd < 32) {
          bb = 1.0;
          for (int q = k; q <= k + dd - 1; ++q) bb *= sigs[q];
        }
        b[L.af_off() + t * L.lanes + w * 32 + k] = af;
        b[L.bb_off() + t * L.lanes + w * 32 + k] = bb;
      }
    }
  }
}

// One system per CTA (W warps); returns after J steps with x' in registers.
template <int MR>
struct MwLane {
  double l[MR], inv[MR], af[5], bb[5], aex, sex, lnx;
  int nreal;
};

template <int MR>
__device__ __forceinline__ void mw_load(MwLane<MR>& f, const double* __restrict__ b, const MwLayout<MR>& L, int lane,
                                        int nx) {
#pragma unroll
  for (int j = 0; j < MR; ++j) {
    f.l[j] = b[L.l_off() + lane * MR + j];
    f.inv[j] = b[L.inv_off() + lane * MR + j];
  }
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    f.af[t] = b[L.af_off() + t * L.lanes + lane];
    f.bb[t] = b[L.bb_off() + t * L.lanes + lane];
  }
  f.aex = b[L.aex_off() + lane];
  f.sex = b[L.sex_off() + lane];
  f.lnx = ((lane + 1) * MR < L.nxp) ? b[L.l_off() + (lane + 1) * MR] : 0.0;
  f.nreal = min(MR, max(0, nx - lane * MR));
}

template <int MR>
__device__ void mw_steps(double (&x)[MR], const MwLane<MR>& f, const double* __restrict__ aw,
                         const double* __restrict__ sw, double* fw, double* bw, int W, int J, double hg) {
  const int k = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int it = 0; it < J; ++it) {
#pragma unroll
    for (int j = 1; j < MR; ++j) x[j] = fma(-f.l[j], x[j - 1], x[j]);
    double Y = x[MR - 1];
#pragma unroll
    for (int t = 0; t < 5; ++t) {
      const double o = __shfl_up_sync(KLE_FULL_MASK, Y, 1 << t);
      if (k >= (1 << t)) Y = fma(f.af[t], o, Y);
    }
    if (k == 31) fw[w] = Y;
    __syncthreads();
    double Yw = 0.0;
    for (int q = 0; q < w; ++q) Yw = fma(aw[q], Yw, fw[q]);
    double Yex = __shfl_up_sync(KLE_FULL_MASK, Y, 1);
    if (k == 0) Yex = 0.0;
    const double Cin = fma(f.aex, Yw, Yex);
    double pi = 1.0;
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      pi *= -f.l[j];
      x[j] = fma(pi, Cin, x[j]);
    }
#pragma unroll
    for (int j = MR - 1; j >= 0; --j) {
      const double ln = (j + 1 < MR) ? f.l[j + 1] : f.lnx;
      const double kap = (j < f.nreal) ? hg * (1.0 + ln) : 0.0;
      double z = fma(x[j], f.inv[j], kap);
      if (j + 1 < MR) z = fma(-ln, x[j + 1], z);
      x[j] = z;
    }
    double X = x[0];
#pragma unroll
    for (int t = 0; t < 5; ++t) {
      const double o = __shfl_down_sync(KLE_FULL_MASK, X, 1 << t);
      if (k + (1 << t) < 32) X = fma(f.bb[t], o, X);
    }
    if (k == 0) bw[w] = X;
    __syncthreads();
    double Xw = 0.0;
    for (int q = W - 1; q > w; --q) Xw = fma(sw[q], Xw, bw[q]);
    double Xex = __shfl_down_sync(KLE_FULL_MASK, X, 1);
    if (k == 31) Xex = 0.0;
    const double Xin = fma(f.sex, Xw, Xex);
    double sg = 1.0;
#pragma unroll
    for (int j = MR - 1; j >= 0; --j) {
      sg *= -((j + 1 < MR) ? f.l[j + 1] : f.lnx);
      x[j] = fma(sg, Xin, x[j]);
    }
  }
}

constexpr int MW_MR = 16;

// mode 0: fused F + CGC rhs (FgrArgs); mode 1: sweep (SweepArgs). One CTA = one
// (sample, subinterval) system of 32*W lanes.
template <int MR>
__global__ void __launch_bounds__(256, 2) fgr_mw_kernel(FgrArgs a, int W) {
  const MwLayout<MR> L(W);
  const int s = blockIdx.x, n = blockIdx.y;
  if (a.active && a.active[s] != KLE_SAMPLE_ACTIVE) return;
  __shared__ double fw[16], bw[16], aw[16], sw[16];
  const int lane = threadIdx.x, k = lane & 31;
  const int nx = a.nx, N = a.N;
  const size_t sbase = (size_t)s * N * nx;
  const double* blob = a.ffac + (size_t)s * L.doubles();
  if (threadIdx.x < W) {
    aw[threadIdx.x] = blob[L.aw_off() + threadIdx.x];
    sw[threadIdx.x] = blob[L.sw_off() + threadIdx.x];
  }
  double x[MR];
  const double hg = a.dt * a.g0;
  if (a.F_given == nullptr) {
    MwLane<MR> f;
    mw_load<MR>(f, blob, L, lane, nx);
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      const int row = lane * MR + j;
      x[j] = (row < nx) ? ((n == 0) ? a.u0[row] : a.U[sbase + (size_t)(n - 1) * nx + row]) + hg : 0.0;
    }
    __syncthreads();
    mw_steps<MR>(x, f, aw, sw, fw, bw, W, a.J, hg);
#pragma unroll
    for (int j = 0; j < MR; ++j) x[j] = (lane * MR + j < nx) ? x[j] - hg : 0.0;
  } else {
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      const int row = lane * MR + j;
      x[j] = (row < nx) ? a.F_given[sbase + (size_t)n * nx + row] : 0.0;
    }
  }
  if (a.F_out) {
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      const int row = lane * MR + j;
      if (row < nx) a.F_out[sbase + (size_t)n * nx + row] = x[j];
    }
  }
  // epilogue: R_n = scaling_n ((I + dT A) F_n - prev_n); neighbours across
  // lanes by shuffle, across warps through shared memory
  __shared__ double edge_lo[16], edge_hi[16];
  const int w = lane >> 5;
  if (k == 0) edge_lo[w] = x[0];
  if (k == 31) edge_hi[w] = x[MR - 1];
  __syncthreads();
  double left = __shfl_up_sync(KLE_FULL_MASK, x[MR - 1], 1);
  double right = __shfl_down_sync(KLE_FULL_MASK, x[0], 1);
  if (k == 0) left = (w > 0) ? edge_hi[w - 1] : 0.0;
  if (k == 31) right = (w + 1 < W) ? edge_lo[w + 1] : 0.0;
  const double* dd = a.dia + (size_t)s * nx;
  const double* ee = a.off + (size_t)s * nx;
  const double sc = a.scaling[n];
  const size_t prow = (n == 0) ? sbase + (size_t)(N - 1) * nx : sbase + (size_t)(n - 1) * nx;
  const double pmul = (n == 0) ? a.alpha : 1.0;
#pragma unroll
  for (int j = 0; j < MR; ++j) {
    const int row = lane * MR + j;
    if (row >= nx) continue;
    const double xm = (j > 0) ? x[j - 1] : left;
    const double xp = (j < MR - 1) ? x[j + 1] : right;
    const double em = (row > 0) ? ee[row - 1] : 0.0;
    const double ep = (row < nx - 1) ? ee[row] : 0.0;
    const double Ax = fma(em, xm, fma(dd[row], x[j], ep * xp));
    const double rhs = fma(a.dT, Ax, x[j]) - pmul * a.U[prow + row];
    a.Rout[sbase + (size_t)n * nx + row] = sc * rhs;
  }
}

template <int MR>
__global__ void __launch_bounds__(256, 2) sweep_mw_kernel(SweepArgs a, int W) {
  const MwLayout<MR> L(W);
  const int s = blockIdx.x, q = blockIdx.y;
  __shared__ double fw[16], bw[16], aw[16], sw[16];
  const int lane = threadIdx.x;
  const int nx = a.nx, Q = a.Q;
  const double* blob = a.fac + (size_t)s * L.doubles();
  if (threadIdx.x < W) {
    aw[threadIdx.x] = blob[L.aw_off() + threadIdx.x];
    sw[threadIdx.x] = blob[L.sw_off() + threadIdx.x];
  }
  MwLane<MR> f;
  mw_load<MR>(f, blob, L, lane, nx);
  const double hg = a.h * a.g0;
  double x[MR];
#pragma unroll
  for (int j = 0; j < MR; ++j) {
    const int row = lane * MR + j;
    x[j] = (row < nx) ? a.start[((size_t)s * Q + q) * nx + row] + hg : 0.0;
  }
  __syncthreads();
  for (int g = 0; g < a.nseg; ++g) {
    mw_steps<MR>(x, f, aw, sw, fw, bw, W, a.J, hg);
    double* o = a.out + (((size_t)s * Q + q) * a.nseg + g) * nx;
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      const int row = lane * MR + j;
      if (row < nx) o[row] = x[j] - hg;
    }
  }
}

// ---------------------------------------------------------------------------
// Fused F + CGC rhs, persistent over subintervals: CTA = (sample, group of G
// subintervals), R subintervals in flight per lane (R right-hand sides share
// the factor registers, the scans and the barriers), factors loaded once per
// CTA, the next group's start rows prefetched into shared memory (cp.async)
// while the current group sweeps; prev_n (= start_n for n >= 1) re-read from
// L2 in the epilogue.
// cfw[w][q] = prod_{q<p<w} aw[p] (q < w), cbw[w][q] = prod_{w<p<q} sw[p] (q > w):
// the weights of the warp composites, so each warp sums them in parallel
template <int MR, int R>
__device__ void mw_steps_r(double (&x)[R][MR], const MwLane<MR>& f, const double* __restrict__ cfw,
                           const double* __restrict__ cbw, double (*fw)[16], double (*bw)[16], int W, int J,
                           double hg) {
  const int k = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int it = 0; it < J; ++it) {
#pragma unroll
    for (int j = 1; j < MR; ++j)
#pragma unroll
      for (int r = 0; r < R; ++r) x[r][j] = fma(-f.l[j], x[r][j - 1], x[r][j]);
    double Y[R];
#pragma unroll
    for (int r = 0; r < R; ++r) Y[r] = x[r][MR - 1];
#pragma unroll
    for (int t = 0; t < 5; ++t)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double o = __shfl_up_sync(KLE_FULL_MASK, Y[r], 1 << t);
        Y[r] = fma(f.af[t], o, Y[r]);  // af = 0 for k < 2^t
      }
    if (k == 31)
#pragma unroll
      for (int r = 0; r < R; ++r) fw[r][w] = Y[r];
    __syncthreads();
    double Cin[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      // Yw = sum_{q<w} cfw[w][q] fw[q]: independent products, no serial chain
      double y0 = 0.0, y1 = 0.0;
#pragma unroll
      for (int q = 0; q < 16; q += 2) {
        if (q < w) y0 = fma(cfw[w * 16 + q], fw[r][q], y0);
        if (q + 1 < w) y1 = fma(cfw[w * 16 + q + 1], fw[r][q + 1], y1);
      }
      double Yex = __shfl_up_sync(KLE_FULL_MASK, Y[r], 1);
      if (k == 0) Yex = 0.0;
      Cin[r] = fma(f.aex, y0 + y1, Yex);
    }
    double pi = 1.0;
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      pi *= -f.l[j];
#pragma unroll
      for (int r = 0; r < R; ++r) x[r][j] = fma(pi, Cin[r], x[r][j]);
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
#pragma unroll
    for (int t = 0; t < 5; ++t)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double o = __shfl_down_sync(KLE_FULL_MASK, X[r], 1 << t);
        X[r] = fma(f.bb[t], o, X[r]);  // bb = 0 for k + 2^t >= 32
      }
    if (k == 0)
#pragma unroll
      for (int r = 0; r < R; ++r) bw[r][w] = X[r];
    __syncthreads();
    double Xin[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double x0 = 0.0, x1 = 0.0;
#pragma unroll
      for (int q = 0; q < 16; q += 2) {
        if (q > w && q < W) x0 = fma(cbw[w * 16 + q], bw[r][q], x0);
        if (q + 1 > w && q + 1 < W) x1 = fma(cbw[w * 16 + q + 1], bw[r][q + 1], x1);
      }
      double Xex = __shfl_down_sync(KLE_FULL_MASK, X[r], 1);
      if (k == 31) Xex = 0.0;
      Xin[r] = fma(f.sex, x0 + x1, Xex);
    }
    double sg = 1.0;
#pragma unroll
    for (int j = MR - 1; j >= 0; --j) {
      sg *= -((j + 1 < MR) ? f.l[j + 1] : f.lnx);
#pragma unroll
      for (int r = 0; r < R; ++r) x[r][j] = fma(sg, Xin[r], x[r][j]);
    }
  }
}

__device__ __forceinline__ void mw_cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}

// padded shared-memory row index: lane-owned MR-row chunks (stride MR + 1,
// odd) so the 32 lanes of a warp hit distinct banks
template <int MR>
__device__ __forceinline__ int mw_pidx(int row) { return row + row / MR; }

template <int MR, int R>
__global__ void __launch_bounds__(256, 1) fgr_mw2_kernel(FgrArgs a, int W, int G) {
  const MwLayout<MR> L(W);
  const int s = blockIdx.x;
  if (a.active && a.active[s] != KLE_SAMPLE_ACTIVE) return;
  const int LD = L.nxp + L.nxp / MR + 2;  // padded row length (+ guard for row nx)
  extern __shared__ __align__(16) double sm[];
  // [2][R][LD] start rows (double-buffered: the current group's rows are also
  // its prev rows in the epilogue), [R][LD] F ends
  double* ob = sm + 2 * R * LD;
  __shared__ double fw[R][16], bw[R][16], cfw[16 * 16], cbw[16 * 16];
  const int lane = threadIdx.x, tid = threadIdx.x;
  const int nx = a.nx, N = a.N, NT = 32 * W;
  const int nbeg = blockIdx.y * G, nend = min(N, nbeg + G);
  const size_t sbase = (size_t)s * N * nx;
  const double* blob = a.ffac + (size_t)s * L.doubles();
  if (tid < W) {  // composite weights of warp tid
    const int w = tid;
    double p = 1.0;
    for (int q = w - 1; q >= 0; --q) {
      cfw[w * 16 + q] = p;
      p *= blob[L.aw_off() + q];
    }
    p = 1.0;
    for (int q = w + 1; q < W; ++q) {
      cbw[w * 16 + q] = p;
      p *= blob[L.sw_off() + q];
    }
  }
  auto prefetch = [&](int n0, double* dst) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int n = n0 + r;
      if (n >= nend) break;
      const double* src = (n == 0) ? a.u0 : a.U + sbase + (size_t)(n - 1) * nx;
      for (int row = tid; row < nx; row += NT) mw_cp_async8(dst + r * LD + mw_pidx<MR>(row), src + row);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  prefetch(nbeg, sm);
  MwLane<MR> f;
  mw_load<MR>(f, blob, L, lane, nx);
  const double hg = a.dt * a.g0;
  const double* dd = a.dia + (size_t)s * nx;
  const double* ee = a.off + (size_t)s * nx;
  int cur = 0;
  for (int n0 = nbeg; n0 < nend; n0 += R, cur ^= 1) {
    double* buf = sm + cur * R * LD;
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    if (n0 + R < nend) prefetch(n0 + R, sm + (cur ^ 1) * R * LD);
    double x[R][MR];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int j = 0; j < MR; ++j) {
        const int row = lane * MR + j;
        x[r][j] = (row < nx && n0 + r < nend) ? buf[r * LD + mw_pidx<MR>(row)] + hg : 0.0;
      }
    mw_steps_r<MR, R>(x, f, cfw, cbw, fw, bw, W, a.J, hg);
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int j = 0; j < MR; ++j) {
        const int row = lane * MR + j;
        ob[r * LD + mw_pidx<MR>(row)] = (row < nx) ? x[r][j] - hg : 0.0;
      }
    if (tid == 0)
#pragma unroll
      for (int r = 0; r < R; ++r) ob[r * LD + mw_pidx<MR>(nx)] = 0.0;  // F_{nx} = 0 (Dirichlet)
    __syncthreads();
    // epilogue, rows strided over the threads (coalesced): R_n = scaling_n ((I + dT A) F_n - prev_n);
    // prev_n = start_n (buf) for n >= 1, alpha U_{N-1} for n = 0
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int n = n0 + r;
      if (n >= nend) break;
      const double* F = ob + r * LD;
      const double* pv = buf + r * LD;
      if (a.F_out)
        for (int row = tid; row < nx; row += NT) a.F_out[sbase + (size_t)n * nx + row] = F[mw_pidx<MR>(row)];
      if (!a.Rout) continue;
      const double sc = a.scaling[n];
      const double* p0 = a.U + sbase + (size_t)(N - 1) * nx;
      constexpr int EB = 8;
      for (int r0 = tid; r0 < nx; r0 += EB * NT) {
        double em[EB], dg[EB], ep[EB], pr[EB];
#pragma unroll
        for (int b = 0; b < EB; ++b) {
          const int row = r0 + b * NT;
          const bool in = row < nx;
          em[b] = (in && row > 0) ? __ldg(ee + row - 1) : 0.0;
          ep[b] = (in && row < nx - 1) ? __ldg(ee + row) : 0.0;
          dg[b] = in ? __ldg(dd + row) : 0.0;
          pr[b] = in ? ((n == 0) ? a.alpha * __ldg(p0 + row) : pv[mw_pidx<MR>(row)]) : 0.0;
        }
#pragma unroll
        for (int b = 0; b < EB; ++b) {
          const int row = r0 + b * NT;
          if (row >= nx) break;
          const double Fc = F[mw_pidx<MR>(row)];
          const double Fm = row > 0 ? F[mw_pidx<MR>(row - 1)] : 0.0;
          const double Fp = F[mw_pidx<MR>(row + 1)];
          const double Ax = fma(em[b], Fm, fma(dg[b], Fc, ep[b] * Fp));
          a.Rout[sbase + (size_t)n * nx + row] = sc * (fma(a.dT, Ax, Fc) - pr[b]);
        }
      }
    }
  }
}

int mw_warps(int nx) {
  const int W = (nx + 32 * MW_MR - 1) / (32 * MW_MR);
  return (W >= 1 && W <= 8) ? W : 0;
}

int mw_blob_doubles(int nx) {
  const int W = mw_warps(nx);
  return W ? MwLayout<MW_MR>(W).doubles() : 0;
}

int mw_factor(const double* dia, const double* off, double* blob, int M, int nx, double h, cudaStream_t st) {
  const int W = mw_warps(nx);
  if (!W) return set_error(KLE_ERR_UNSUPPORTED, "fine (multi-warp): nx too large");
  mw_factor_kernel<MW_MR><<<(M + 63) / 64, 64, 0, st>>>(dia, off, blob, M, nx, W, h);
  return check_launch("mw_factor_kernel");
}

template <int R>
static int launch_mw2(const FgrArgs& a, int W, cudaStream_t st) {
  const MwLayout<MW_MR> L(W);
  const int G = 16 * R;  // subintervals per CTA
  const size_t smem = sizeof(double) * 3 * R * (size_t)(L.nxp + L.nxp / MW_MR + 2);
  static PerDeviceOnce attr_once;
  if (int rc = once_per_device(attr_once, "kle_fine_mw: cudaFuncSetAttribute", [&] {
        return cudaFuncSetAttribute(fgr_mw2_kernel<MW_MR, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      }))
    return rc;
  fgr_mw2_kernel<MW_MR, R><<<dim3(a.M, (a.N + G - 1) / G), 32 * W, smem, st>>>(a, W, G);
  return check_launch("fgr_mw2_kernel");
}

int mw_fgr(const FgrArgs& a, cudaStream_t st) {
  const int W = mw_warps(a.nx);
  if (!W) return set_error(KLE_ERR_UNSUPPORTED, "fgr (multi-warp): nx too large");
  if (a.N > 65535) return set_error(KLE_ERR_UNSUPPORTED, "fgr (multi-warp): N too large");
  static const char* env = getenv("KLE_FINE_MW");  // 0: one CTA per subinterval (A/B); 1/2: R
  const int v = (env && *env) ? atoi(env) : 1;
  if (!a.F_given && v == 1) return launch_mw2<1>(a, W, st);
  if (!a.F_given && v == 2) return launch_mw2<2>(a, W, st);
  fgr_mw_kernel<MW_MR><<<dim3(a.M, a.N), 32 * W, 0, st>>>(a, W);
  return check_launch("fgr_mw_kernel");
}

int mw_sweep(const SweepArgs& a, cudaStream_t st) {
  const int W = mw_warps(a.nx);
  if (!W) return set_error(KLE_ERR_UNSUPPORTED, "sweep (multi-warp): nx too large");
  sweep_mw_kernel<MW_MR><<<dim3(a.M, a.Q), 32 * W, 0, st>>>(a, W);
  return check_launch("sweep_mw_kernel");
}

}  // namespace kle
