// 2D (5-point) path of the KLE-CGC hot path: BASELINE config 3.
//
// Reference counterparts (the same plugin surface as the 1D path):
//   LinearModel.linear_system     pintuq/models.py:114-116  (2D plugin: models.LogNormalKL2D)
//   _linear_factor / BE step      pintuq/propagators.py:25-39  (SuperLU of I + dt A)
//   propagate_fine / _coarse      pintuq/propagators.py:121-157
//   assemble_rhs_blocks, rhs      pintuq/pcgc.py:175-197, 233-237
//   factor_shifted (SuperLU / lambda, bandwidth > 1)  pintuq/pcgc.py:137-145
//   three_step_solve              pintuq/pcgc.py:148-172
//   pcgc_solve increment / stop   pintuq/pcgc.py:335-348
//
// The 5-point operator of an n x n grid (x fastest) has bandwidth n. Like the
// reference (SuperLU), every implicit solve is direct: each sample's
// T = I + dt A and the N/2+1 distinct shifted matrices B_f = lambda_f I + dT A
// (B_{N-f} = conj B_f) are factored once per solve as banded L D L^T without
// pivoting (T is SPD; B_f is complex symmetric with SPD real part, so no-pivot
// LDL^T is stable) and reused by every outer iteration.
//
// Kernels:
//   kl5pt_kernel       xi -> (dia, ex, ey) of A (cell-centre log a, face averages)
//   band_factor_kernel one CTA per matrix: right-looking band LDL^T with the
//                      (n+1) x (n+1) active window distributed over the CTA
//                      (entry (row slot, diagonal offset) per thread, real parts
//                      in shared memory, imaginary parts in registers); writes
//                      L by columns (Lt[i][t] = L(i+1+t, i)), read by both
//                      substitution directions
//   fine2d_kernel      one warp per (sample, 32 subintervals): J BE steps on 32
//                      right-hand sides in the lanes (dot-form banded solves, the
//                      last n solved rows in a shared-memory window), then the
//                      CGC right-hand side rhs_n = scaling_n ((I + dT A) F_n - prev_n)
//   dft_fwd_kernel     per (sample, DOF): p_f = fft(r)_f / sqrt(N), f <= N/2
//   band_solve_cplx    one warp per (sample, f): B_f q = p (column-form forward
//                      with a pending-update window, dot-form backward)
//   dft_inv_update     per (sample, DOF): u = Re ifft(q) / sqrt(N) / scaling
//                      (Hermitian completion), increment vs U, write U
//   status2d_kernel    per sample: stop test, status words, active count
#include <cmath>
#include <cstdlib>

#include "kle_common.cuh"
#include "kle_internal.h"

namespace kle {

// ---------------------------------------------------------------------------
// scalar helpers for the real / complex instantiations
// ---------------------------------------------------------------------------
template <bool C>
struct Sc;
template <>
struct Sc<false> {
  using T = double;
  __device__ static T mk(double r, double) { return r; }
  __device__ static T mul(T a, T b) { return a * b; }
  __device__ static T fms(T a, T b, T c) { return fma(-a, b, c); }  // c - a b
  __device__ static T fma_(T a, T b, T c) { return fma(a, b, c); }
  __device__ static T rcp(T a) { return 1.0 / a; }
  __device__ static T sub(T a, T b) { return a - b; }
  __device__ static T zero() { return 0.0; }
  __device__ static double re(T a) { return a; }
  __device__ static double im(T) { return 0.0; }
  __device__ static T shfl_xor(T a, int o) { return __shfl_xor_sync(KLE_FULL_MASK, a, o); }
  __device__ static T add(T a, T b) { return a + b; }
};
template <>
struct Sc<true> {
  using T = Cplx;
  __device__ static T mk(double r, double i) { return {r, i}; }
  __device__ static T mul(T a, T b) { return cmul(a, b); }
  __device__ static T fms(T a, T b, T c) {
    return {fma(-a.re, b.re, fma(a.im, b.im, c.re)), fma(-a.re, b.im, fma(-a.im, b.re, c.im))};
  }
  __device__ static T fma_(T a, T b, T c) {
    return {fma(a.re, b.re, fma(-a.im, b.im, c.re)), fma(a.re, b.im, fma(a.im, b.re, c.im))};
  }
  __device__ static T rcp(T a) { return crcp(a); }
  __device__ static T sub(T a, T b) { return {a.re - b.re, a.im - b.im}; }
  __device__ static T zero() { return {0.0, 0.0}; }
  __device__ static double re(T a) { return a.re; }
  __device__ static double im(T a) { return a.im; }
  __device__ static T shfl_xor(T a, int o) {
    return {__shfl_xor_sync(KLE_FULL_MASK, a.re, o), __shfl_xor_sync(KLE_FULL_MASK, a.im, o)};
  }
  __device__ static T add(T a, T b) { return {a.re + b.re, a.im + b.im}; }
};

// ---------------------------------------------------------------------------
// xi -> 5-point stencil. log a at the cell centres (p + 1/2, r + 1/2) h,
// p, r = 0..n, is kl_table^T xi (table [d][(n+1)^2], index r (n+1) + p);
// face coefficients are the averages of the two centres a face separates
// (models.LogNormalKL2D.stencil, same association of the sums).
// ---------------------------------------------------------------------------
__global__ void kl5pt_kernel(const double* __restrict__ xi, int M, int d, const double* __restrict__ table,
                             int n, double inv_h2, double* __restrict__ dia, double* __restrict__ ex,
                             double* __restrict__ ey) {
  const int nx = n * n, nc = n + 1;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)M * nx) return;
  const int s = (int)(t / nx), idx = (int)(t - (long long)s * nx);
  const int i = idx % n + 1, j = idx / n + 1;  // node (i h, j h)
  const double* v = xi + (size_t)s * d;
  auto a_at = [&](int p, int r) {
    const double* col = table + (size_t)r * nc + p;
    double acc = 0.0;
    for (int q = 0; q < d; ++q) acc = fma(col[(size_t)q * nc * nc], v[q], acc);
    return exp(acc);
  };
  const double a00 = a_at(i - 1, j - 1), a10 = a_at(i, j - 1), a01 = a_at(i - 1, j), a11 = a_at(i, j);
  const double axl = 0.5 * (a00 + a01), axr = 0.5 * (a10 + a11);
  const double ayd = 0.5 * (a00 + a10), ayu = 0.5 * (a01 + a11);
  const size_t o = (size_t)s * nx + idx;
  dia[o] = (((axl + axr) + ayd) + ayu) * inv_h2;
  ex[o] = (i < n) ? -axr * inv_h2 : 0.0;
  ey[o] = (j < n) ? -ayu * inv_h2 : 0.0;
}

// ---------------------------------------------------------------------------
// Banded L D L^T of B = shift I + c A, one CTA per matrix.
// Window entry (rho, delta): row r with r = rho (mod W), W = n+1, r in
// [i, i+n], column r - delta. Each thread owns two fixed diagonal offsets
// (delta, W-1-delta) in a set of row slots, real parts in shared memory,
// imaginary parts in registers. Step i:
// publish column i (the entry with delta == window position j), one barrier,
// eliminate W(r, c) -= (W(r,i) / d) W(c,i), emit Lt[i][t] = L(i+1+t, i) and
// Dinv[i], and load row i+n+1 into row i's slot from a shared-memory ring of
// operator values prefetched BF_AHEAD steps ahead (no global latency on the
// per-step critical path).
// ---------------------------------------------------------------------------
// NT threads per CTA, 16384 / NT window entries per thread (W <= 128); 1024
// for both (512 threads for the complex factor measured slower)
constexpr int BF_RING = 64;     // operator-row ring (rows i+W .. i+W+BF_AHEAD)
constexpr int BF_AHEAD = 32;

template <bool C, int NT>
__global__ void __launch_bounds__(NT, 1)
    band_factor_kernel(const double* __restrict__ dia, const double* __restrict__ ex,
                       const double* __restrict__ ey, int n, const double* __restrict__ lam, int NF,
                       double shift_re, double c, double* __restrict__ Lt, double* __restrict__ Dinv) {
  using S = Sc<C>;
  using T = typename S::T;
  constexpr int E = 16384 / NT;  // entries per thread (2 offsets x E/2 row slots)
  const int nx = n * n, W = n + 1;
  const int phi = blockIdx.x, s = phi / NF, f = phi - s * NF;
  const double* d_ = dia + (size_t)s * nx;
  const double* ex_ = ex + (size_t)s * nx;
  const double* ey_ = ey + (size_t)s * nx;
  const T shift = C ? S::mk(lam[2 * f], lam[2 * f + 1]) : S::mk(shift_re, 0.0);
  extern __shared__ __align__(16) double smem[];
  double* wre = smem;                                   // [E][NT]
  T* col = reinterpret_cast<T*>(wre + E * NT);    // [2][W]
  double* ring = reinterpret_cast<double*>(col + 2 * W);  // [BF_RING][3]: c*dia[r], c*ex[r-1], c*ey[r-n]
  const int tid = threadIdx.x;
  // balanced ownership: thread = (diagonal pair p, row group rho0); it holds the
  // offsets delta_a = p and delta_b = W-1-p in the row slots rho0 + Qr m, so
  // the active work per step (delta < window position) is even across threads
  const int H = (W + 1) / 2, Qr = NT / H, E2 = (W + Qr - 1) / Qr;
  const int pair = tid % H, rho0 = tid / H;
  const int dl[2] = {pair, W - 1 - pair};
  const bool two = dl[1] != dl[0];
  auto load_row = [&](int r) {  // operator values of row r (identity padding beyond nx)
    double* e = ring + 3 * (r % BF_RING);
    e[0] = (r < nx) ? c * d_[r] : 0.0;
    e[1] = (r < nx && r >= 1) ? c * ex_[r - 1] : 0.0;
    e[2] = (r < nx && r >= n) ? c * ey_[r - n] : 0.0;
  };
  auto entryB = [&](int r, int dlt, const double* e) -> T {  // B(r, r - dlt) from ring values e
    if (r >= nx) return dlt == 0 ? S::mk(1.0, 0.0) : S::zero();
    if (r - dlt < 0) return S::zero();
    if (dlt == 0) return S::add(shift, S::mk(e[0], 0.0));
    double v = 0.0;
    if (dlt == 1) v += e[1];
    if (dlt == n) v += e[2];
    return S::mk(v, 0.0);
  };
  for (int k = W + tid; k < W + BF_AHEAD; k += NT) load_row(k);
  double pre[3] = {0.0, 0.0, 0.0};  // thread NT-1: operator row in flight to the ring
  double wim[E];
#pragma unroll
  for (int m = 0; m < E / 2; ++m) {
    const int rho = rho0 + Qr * m;
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      T v = S::zero();
      if (m < E2 && rho < W && (w == 0 || two)) {  // rows 0..n in slots 0..n (operator from global memory)
        const double e[3] = {rho < nx ? c * d_[rho] : 0.0, (rho < nx && rho >= 1) ? c * ex_[rho - 1] : 0.0,
                             (rho < nx && rho >= n) ? c * ey_[rho - n] : 0.0};
        v = entryB(rho, dl[w], e);
      }
      wre[(2 * m + w) * NT + tid] = S::re(v);
      wim[2 * m + w] = S::im(v);
    }
  }
  __syncthreads();
  T* Lt_ = reinterpret_cast<T*>(Lt) + (size_t)phi * nx * n;
  T* Di_ = reinterpret_cast<T*>(Dinv) + (size_t)phi * nx;
  // window position of each owned row slot, (rho - i) mod W, advanced incrementally per row
  int jp[E / 2];
#pragma unroll
  for (int m = 0; m < E / 2; ++m) jp[m] = rho0 + Qr * m;
  for (int i = 0; i < nx; ++i) {
    T* cb = col + (i & 1) * W;
#pragma unroll
    for (int m = 0; m < E / 2; ++m) {
      const int rho = rho0 + Qr * m;
      if (m >= E2 || rho >= W) continue;
      const int jpos = jp[m];
#pragma unroll
      for (int w = 0; w < 2; ++w)
        if ((w == 0 || two) && dl[w] == jpos) cb[jpos] = S::mk(wre[(2 * m + w) * NT + tid], wim[2 * m + w]);
    }
    if (tid == NT - 1) {  // prefetch ring: store the row loaded last step, load the next one
      if (i > 0) {
        double* e = ring + 3 * ((i - 1 + W + BF_AHEAD) % BF_RING);
        e[0] = pre[0];
        e[1] = pre[1];
        e[2] = pre[2];
      }
      const int r = i + W + BF_AHEAD;
      pre[0] = (r < nx) ? c * d_[r] : 0.0;
      pre[1] = (r < nx && r >= 1) ? c * ex_[r - 1] : 0.0;
      pre[2] = (r < nx && r >= n) ? c * ey_[r - n] : 0.0;
    }
    __syncthreads();
    const T dinv = S::rcp(cb[0]);
    const double* e = ring + 3 * ((i + W) % BF_RING);
#pragma unroll
    for (int m = 0; m < E / 2; ++m) {
      const int rho = rho0 + Qr * m;
      if (m >= E2 || rho >= W) continue;
      const int jpos = jp[m];
      jp[m] = jpos == 0 ? W - 1 : jpos - 1;  // position at row i + 1
      if (jpos == 0) {  // row i leaves; row i + n + 1 enters its slot
#pragma unroll
        for (int w = 0; w < 2; ++w) {
          if (w == 1 && !two) continue;
          const T v = entryB(i + W, dl[w], e);
          wre[(2 * m + w) * NT + tid] = S::re(v);
          wim[2 * m + w] = S::im(v);
        }
        continue;
      }
      if (dl[0] >= jpos && (!two || dl[1] >= jpos)) continue;
      const T l = S::mul(cb[jpos], dinv);
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        if ((w == 1 && !two) || dl[w] >= jpos) continue;
        const T v = S::fms(l, cb[jpos - dl[w]], S::mk(wre[(2 * m + w) * NT + tid], wim[2 * m + w]));
        wre[(2 * m + w) * NT + tid] = S::re(v);
        wim[2 * m + w] = S::im(v);
      }
    }
    if (tid < n) {
      const int r = i + 1 + tid;
      const T l = (r < nx) ? S::mul(cb[tid + 1], dinv) : S::zero();
      Lt_[(size_t)i * n + tid] = l;
    }
    if (tid == 0) Di_[i] = dinv;
  }
}

// ---------------------------------------------------------------------------
// Panel (rank-PF_B) banded L D L^T of B = lam I + c A (complex shifts), one
// 512-thread CTA per matrix. The active window (rows i0 .. i0+n+PF_B-1, all
// columns >= i0 of the band) is kept complex in shared memory as diagonal
// rings: diagonal d (entries (r, r-d)) is a FIFO of NB - d entries, NB = n +
// PF_B, entry of column cc at roff(d) + cc mod (NB - d); eliminated columns
// free exactly the slots the rows entering next need. Per panel:
//   1. the first 160 threads (one window row each) factor the panel's PF_B
//      columns with one named barrier per column (rows' entries in registers,
//      the column's pivot rows published through shared memory), writing
//      PA[k][x] = W(x,k)/d_k and PB[k][x] = W(x,k); the other threads load the
//      PF_B operator rows that enter for the next panel;
//   2. all threads apply the rank-PF_B update W(r,c) -= sum_k PA[k][r] PB[k][c]
//      to the trailing triangle: 8 threads per folded row pair (r, n-1-r),
//      columns strided over them, each PB read feeding both rows.
// Each window entry is read and written once per PF_B rows instead of once
// per row (band_factor_kernel: ~4,400 shared-memory wavefronts per row).
// ---------------------------------------------------------------------------
#ifndef KLE_PF_B
#define KLE_PF_B 12
#endif
constexpr int PF_B = KLE_PF_B;  // panel width (columns per rank-PF_B update)
constexpr int PF_NT = 512;
constexpr int PF_PT = 160;  // panel threads (>= n + PF_B, a multiple of 32)
constexpr int PF_M = 16;    // trailing entries per thread (8 threads per folded row pair)

__host__ __device__ inline int pf_roff(int d, int NB) { return d * NB - d * (d - 1) / 2; }
__host__ inline size_t pf_smem_bytes(int n) {
  const int NB = n + PF_B;
  return sizeof(Cplx) * ((size_t)pf_roff(n + 1, NB) + 2 * (size_t)PF_B * NB + 2 * PF_B) + sizeof(int) * (n + 1);
}

__global__ void __launch_bounds__(PF_NT, 1)
    band_factor_panel_kernel(const double* __restrict__ dia, const double* __restrict__ ex,
                             const double* __restrict__ ey, int n, const double* __restrict__ lam, int NF, double c,
                             double* __restrict__ Lt, double* __restrict__ Dinv) {
  using S = Sc<true>;
  using T = Cplx;
  constexpr int B = PF_B;
  const int nx = n * n, NB = n + B;
  const int phi = blockIdx.x, s = phi / NF, f = phi - s * NF;
  const double* d_ = dia + (size_t)s * nx;
  const double* ex_ = ex + (size_t)s * nx;
  const double* ey_ = ey + (size_t)s * nx;
  const T shift = S::mk(lam[2 * f], lam[2 * f + 1]);
  extern __shared__ __align__(16) double smem[];
  T* ring = reinterpret_cast<T*>(smem);
  T* PA = ring + pf_roff(n + 1, NB);  // [B][NB]
  T* PB = PA + B * NB;                // [B][NB]
  T* pub = PB + B * NB;               // [2][B]
  int* rb = reinterpret_cast<int*>(pub + 2 * B);  // [n+1]: ring index of column i0+B on diagonal d
  const int tid = threadIdx.x;
  auto opB = [&](int r, int dd) -> T {  // B(r, r - dd): the operator (identity beyond nx)
    if (r >= nx) return dd == 0 ? S::mk(1.0, 0.0) : S::zero();
    if (r - dd < 0) return S::zero();
    if (dd == 0) return S::add(shift, S::mk(c * d_[r], 0.0));
    double v = 0.0;
    if (dd == 1) v += c * ex_[r - 1];
    if (dd == n) v += c * ey_[r - n];
    return S::mk(v, 0.0);
  };
  // initial window: rows 0 .. NB-1, column cc of ring d at index cc
  for (int dd = 0; dd <= n; ++dd)
    for (int idx = tid; idx < NB - dd; idx += PF_NT) ring[pf_roff(dd, NB) + idx] = opB(idx + dd, dd);
  // panel-thread state: row x, entries k with 0 <= x - k <= n; ring index of column i0 + k
  const int x = tid;
  int psl[B];
#pragma unroll
  for (int k = 0; k < B; ++k) {
    const int dd = x - k;
    psl[k] = (dd >= 0 && dd <= n) ? k % (NB - dd) : 0;
  }
  // trailing-thread state: folded pair p (rows p and n-1-p of the trailing triangle), lane g of 8
  const int p = tid >> 3, g = tid & 7;
  const int R1 = p, R2 = n - 1 - p;
  const bool pair_ok = R1 <= R2;
  __syncthreads();
  T* Lt_ = reinterpret_cast<T*>(Lt) + (size_t)phi * nx * n;
  T* Di_ = reinterpret_cast<T*>(Dinv) + (size_t)phi * nx;
  for (int i0 = 0; i0 < nx; i0 += B) {
    // ---- 1. panel: load the rows' panel entries, then factor the PF_B columns
    T e[B];
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int dd = x - k;
      e[k] = (x < NB && dd >= 0 && dd <= n) ? ring[pf_roff(dd, NB) + psl[k]] : S::zero();
    }
    __syncthreads();  // the panel columns' slots are free from here on
    if (tid < PF_PT) {
#pragma unroll
      for (int k = 0; k < B; ++k) {
        T* pb = pub + (k & 1) * B;
        if (x >= k && x < B) pb[x] = e[k];
        asm volatile("bar.sync 1, %0;\n" ::"r"(PF_PT) : "memory");
        const T di = S::rcp(pb[k]);
        if (x < NB) {
          const T ek = e[k];
          const T l = (x > k) ? S::mul(ek, di) : S::zero();
          PB[k * NB + x] = ek;
          PA[k * NB + x] = l;
#pragma unroll
          for (int k2 = k + 1; k2 < B; ++k2)
            if (x >= k2 && x - k2 <= n) e[k2] = S::fms(l, pb[k2], e[k2]);
          if (x == k && i0 + k < nx) Di_[i0 + k] = di;
        }
      }
    } else {  // rows entering for the next panel: i0+NB .. i0+NB+B-1 (operator values)
      for (int dd = tid - PF_PT; dd <= n; dd += PF_NT - PF_PT) rb[dd] = (i0 + B) % (NB - dd);
      for (int q = tid - PF_PT; q < B * (n + 1); q += PF_NT - PF_PT) {
        const int r = i0 + NB + q / (n + 1), dd = q % (n + 1), cc = r - dd;
        ring[pf_roff(dd, NB) + cc % (NB - dd)] = opB(r, dd);
      }
    }
    __syncthreads();
    for (int q = tid; q < B * n; q += PF_NT) {  // Lt[i][t] = L(i+1+t, i), i = i0 + k
      const int k = q / n, t = q - k * n, i = i0 + k;
      if (i < nx) Lt_[(size_t)i * n + t] = (i + 1 + t < nx) ? PA[k * NB + k + 1 + t] : S::zero();
    }
    // ---- 2. trailing rank-B update of rows/columns i0+B .. i0+NB-1
    if (pair_ok) {
      // columns C = g + 8 (4q + u) of both rows of the pair: the 8 lanes of a
      // pair read 8 consecutive PB entries and the warp's 4 pairs the same
      // ones (one wavefront); each PB value feeds both rows
#pragma unroll 1
      for (int q = 0; q < PF_M / 4; ++q) {
        const int c0 = g + 32 * q;
        if (c0 > R2) break;
        const bool do1 = c0 <= R1 && R1 != R2;
        T a1c[4], a2c[4];
        int w1[4], w2[4], C[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          C[u] = c0 + 8 * u;
          const int d2 = R2 - C[u], d1 = R1 - C[u];
          const int e2 = max(d2, 0), e1 = max(d1, 0);
          int i2 = rb[e2] + C[u];
          if (i2 >= NB - e2) i2 -= NB - e2;
          int i1 = rb[e1] + C[u];
          if (i1 >= NB - e1) i1 -= NB - e1;
          w2[u] = pf_roff(e2, NB) + i2;
          w1[u] = pf_roff(e1, NB) + i1;
          a2c[u] = d2 >= 0 ? ring[w2[u]] : S::zero();
          a1c[u] = (do1 && d1 >= 0) ? ring[w1[u]] : S::zero();
        }
        if (do1) {
#pragma unroll
          for (int k = 0; k < B; ++k) {
            const T x1 = PA[k * NB + B + R1], x2 = PA[k * NB + B + R2];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const T pbv = PB[k * NB + B + C[u]];
              a2c[u] = S::fms(x2, pbv, a2c[u]);
              a1c[u] = S::fms(x1, pbv, a1c[u]);
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < B; ++k) {
            const T x2 = PA[k * NB + B + R2];
#pragma unroll
            for (int u = 0; u < 4; ++u) a2c[u] = S::fms(x2, PB[k * NB + B + C[u]], a2c[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (C[u] <= R2) ring[w2[u]] = a2c[u];
          if (do1 && C[u] <= R1) ring[w1[u]] = a1c[u];
        }
      }
    }
    __syncthreads();
    // ---- advance the ring indices by one panel
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int dd = x - k;
      if (dd >= 0 && dd <= n) {
        psl[k] += B;
        if (psl[k] >= NB - dd) psl[k] -= NB - dd;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Fine sweeps, one warp per (sample, group of SB_R subintervals), the lanes
// are the right-hand sides; each BE step is a forward and a backward banded
// substitution (subst_pass), both reading the column-band factor Lt. State X and scratch Z: [slot][nx][SB_R].
// ---------------------------------------------------------------------------
struct Fine2dArgs {
  const double* start;   // mode 0: U [M][N][nx]; mode 1: start rows [M][Q][nx]
  const double* u0;      // mode 0: [nx]
  const double* F_given; // mode 0, optional [M][N][nx]: skip the sweep, take these F ends
  const double *dia, *ex, *ey;
  const double *Lt, *Dinv;         // per sample: [nx][n] (L(i+1+t, i)), [nx]
  const double* scaling;           // mode 0: [N]
  const int32_t* active;           // mode 0: [M] or null
  double* X;                       // [M * G][nx][SB_R]
  double* Z;                       // [M * G][nx][SB_R]
  double* out;                     // mode 0: R [M][N][nx]; mode 1: [M][Q][nseg][nx]
  int M, N, n, J, nseg, mode;      // mode 0: fgr, mode 1: sweep (N = Q)
  double dt, dT, g0, alpha;
};

// One banded substitution pass over the sequence positions p = 0..nx-1 (row
// p forward, row nx-1-p backward), 32 right-hand sides in the lanes:
//   v_p = b_p - sum_{q in [p-n, p)} c(p, q) v_q
// forward  c = L(i, k)     = Lt[k][i - k - 1]
// backward c = L(k, i)     = Lt[i][k - i - 1]   (k = row of position q)
// Positions are processed in blocks of RB: the far part (q < p0) is one
// register-blocked sweep over the window of the last n values (each window
// load feeds RB FMAs; the block's coefficients are staged skewed in shared
// memory, cst[qq][a] with qq = q - (p0 - n), straight from the registers the
// next block's rows are prefetched into), the near part (p0 <= q < p) a small
// triangular fix-up whose coefficients sit at cst[n + a2][a]. Window:
// [WP][SB_R], WP = 2^ceil(log2(n+1)), slot = q & (WP-1), zero for q < 0.
constexpr int SB_RB = 8;
constexpr int SB_PF = 4;   // ceil(127 / 32): coefficient values per lane and row
// SB_R: right-hand sides per warp, 32 (lanes), 16 or 8 (the lane groups split
// the window sweep: more coefficient traffic, more warps; chosen when the
// batch is too small to fill the SMs with 32-wide warps). A cp.async
// multi-stage pipeline for the coefficient / right-hand-side staging (instead
// of the register prefetch) measured slower (0.42-0.51 vs 0.33 s per c3 step).

template <bool BACK, int SB_R>
__device__ __forceinline__ void subst_pass(const double* __restrict__ Lc, const double* __restrict__ bsrc,
                                           double badd, const double* __restrict__ Di, double* __restrict__ out,
                                           double* win, double* cst, int n, int WP, int nx, int lane) {
  constexpr int RB = SB_RB;
  constexpr int SB_H = 32 / SB_R;
  const int wm = WP - 1;
  const int r = lane & (SB_R - 1), h = lane / SB_R;
  for (int q = lane; q < WP * SB_R; q += 32) win[q] = 0.0;
  for (int q = lane; q < (n + RB) * RB; q += 32) cst[q] = 0.0;
  auto row_of = [&](int p) { return BACK ? nx - 1 - p : p; };
  double pf[RB][SB_PF], pn = 0.0;
  // forward: cst[u][a] = L(p0+a, p0-n+u) = Lt[p0-n+u][n-1-u+a] (a <= u), near
  //          cst[n+a2][a] = L(p0+a, p0+a2) = Lt[p0+a2][a-a2-1] (a2 < a)
  // backward: cst[a+n-1-u][a] = Lt[row(p0+a)][u] (covers the near part too)
  auto fetch = [&](int p0) {
#pragma unroll
    for (int a = 0; a < RB; ++a)
#pragma unroll
      for (int m = 0; m < SB_PF; ++m) {
        const int u = lane + 32 * m;
        if (BACK) {
          pf[a][m] = (p0 + a < nx && u < n) ? __ldg(Lc + (size_t)row_of(p0 + a) * n + u) : 0.0;
        } else {
          const int k = p0 - n + u;
          pf[a][m] = (u < n && a <= u && k >= 0 && p0 + a < nx) ? __ldg(Lc + (size_t)k * n + (n - 1 - u + a)) : 0.0;
        }
      }
    if (!BACK) {
      const int a2 = (lane & 63) / RB, a = lane % RB;  // lanes 0..31 cover a2 < 4; second pass below
      pn = (a2 < a && p0 + a < nx) ? __ldg(Lc + (size_t)(p0 + a2) * n + (a - a2 - 1)) : 0.0;
    }
  };
  double pn2 = 0.0;
  auto fetch2 = [&](int p0) {  // forward near part, a2 >= 4
    if (!BACK) {
      const int a2 = 4 + lane / RB, a = lane % RB;
      pn2 = (a2 < a && p0 + a < nx) ? __ldg(Lc + (size_t)(p0 + a2) * n + (a - a2 - 1)) : 0.0;
    }
  };
  fetch(0);
  fetch2(0);
  for (int p0 = 0; p0 < nx; p0 += RB) {
    __syncwarp();
#pragma unroll
    for (int a = 0; a < RB; ++a)
#pragma unroll
      for (int m = 0; m < SB_PF; ++m) {
        const int u = lane + 32 * m;
        if (u < n) cst[(BACK ? a + n - 1 - u : u) * RB + a] = pf[a][m];
      }
    if (!BACK) {
      cst[(n + lane / RB) * RB + lane % RB] = pn;
      cst[(n + 4 + lane / RB) * RB + lane % RB] = pn2;
    }
    double bv[RB], dv[RB];  // loads in flight during the sweep (consumed in the near part)
#pragma unroll
    for (int a = 0; a < RB; ++a) {
      bv[a] = (p0 + a < nx) ? bsrc[(size_t)row_of(p0 + a) * SB_R + r] : 0.0;
      dv[a] = (Di && p0 + a < nx) ? __ldg(Di + row_of(p0 + a)) : 1.0;
    }
    __syncwarp();
    if (p0 + RB < nx) {  // in flight during the sweep
      fetch(p0 + RB);
      fetch2(p0 + RB);
    }
    double acc[RB];
#pragma unroll
    for (int a = 0; a < RB; ++a) acc[a] = 0.0;
    const int q0 = p0 - n;
#pragma unroll 4
    for (int qq = h; qq < n; qq += SB_H) {
      const double y = win[((q0 + qq) & wm) * SB_R + r];
#pragma unroll
      for (int a = 0; a < RB; a += 2) {
        const double2 c = *reinterpret_cast<const double2*>(cst + qq * RB + a);
        acc[a] = fma(c.x, y, acc[a]);
        acc[a + 1] = fma(c.y, y, acc[a + 1]);
      }
    }
#pragma unroll
    for (int o = SB_R; o < 32; o <<= 1)  // combine the lane groups' partial sweeps
#pragma unroll
      for (int a = 0; a < RB; ++a) acc[a] += __shfl_xor_sync(KLE_FULL_MASK, acc[a], o);
    double yv[RB];
#pragma unroll
    for (int a = 0; a < RB; ++a) {
      const int p = p0 + a;
      double v = (bv[a] + badd) - acc[a];
#pragma unroll
      for (int a2 = 0; a2 < a; ++a2) v = fma(-cst[(n + a2) * RB + a], yv[a2], v);
      yv[a] = v;
      if (p < nx && h == 0) {
        const int i = row_of(p);
        win[(p & wm) * SB_R + r] = v;
        out[(size_t)i * SB_R + r] = Di ? v * dv[a] : v;
      }
    }
  }
  __syncwarp();
}

__host__ __device__ inline int win_pow2(int n) {
  int w = 1;
  while (w < n + 1) w <<= 1;
  return w;
}

template <int SB_R>
__device__ __forceinline__ void fine2d_steps(const Fine2dArgs& a, int s, double* __restrict__ X,
                                             double* __restrict__ Z, double* win, double* cst, int lane) {
  const int n = a.n, nx = n * n, WP = win_pow2(n);
  const double* Lt = a.Lt + (size_t)s * nx * n;
  const double* Di = a.Dinv + (size_t)s * nx;
  const double hg = a.dt * a.g0;
  for (int step = 0; step < a.J; ++step) {
    subst_pass<false, SB_R>(Lt, X, hg, Di, Z, win, cst, n, WP, nx, lane);   // y = L^{-1}(x + h g); Z = D^{-1} y
    subst_pass<true, SB_R>(Lt, Z, 0.0, nullptr, X, win, cst, n, WP, nx, lane);  // x = L^{-T} Z
  }
}

template <int SB_R>
__global__ void __launch_bounds__(32, 5) fine2d_kernel(Fine2dArgs a) {
  constexpr int SB_H = 32 / SB_R;
  const int n = a.n, nx = n * n;
  const int G = (a.N + SB_R - 1) / SB_R;
  const int s = blockIdx.x / G, g = blockIdx.x % G;
  if (a.mode == 0 && a.active && a.active[s] != KLE_SAMPLE_ACTIVE) return;
  const int lane = threadIdx.x, rr = lane & (SB_R - 1), hh = lane / SB_R;
  const int q = g * SB_R + rr;  // subinterval (mode 0) / start row (mode 1)
  const bool live = q < a.N;
  extern __shared__ __align__(16) double sm2[];
  double* win = sm2;                       // [WP][SB_R]
  double* cst = win + win_pow2(n) * SB_R;  // [n + SB_RB][SB_RB]
  double* X = a.X + (size_t)blockIdx.x * nx * SB_R;
  double* Z = a.Z + (size_t)blockIdx.x * nx * SB_R;
  const double* src;
  if (a.mode == 0) src = (q == 0 || !live) ? a.u0 : a.start + ((size_t)s * a.N + (q - 1)) * nx;
  else src = a.start + ((size_t)s * a.N + (live ? q : 0)) * nx;
  const double* x0 = (a.mode == 0 && a.F_given) ? a.F_given + ((size_t)s * a.N + (live ? q : 0)) * nx : src;
  for (int i = hh; i < nx; i += SB_H) X[(size_t)i * SB_R + rr] = live ? x0[i] : 0.0;
  __syncwarp();
  if (a.mode == 1) {
    for (int sg = 0; sg < a.nseg; ++sg) {
      fine2d_steps<SB_R>(a, s, X, Z, win, cst, lane);
      if (live) {
        double* o = a.out + (((size_t)s * a.N + q) * a.nseg + sg) * nx;
        for (int i = hh; i < nx; i += SB_H) o[i] = X[(size_t)i * SB_R + rr];
      }
      __syncwarp();
    }
    return;
  }
  if (!a.F_given) fine2d_steps<SB_R>(a, s, X, Z, win, cst, lane);
  __syncwarp();
  if (!live) return;
  // rhs_n = scaling_n ((I + dT A) F_n - prev_n); prev_0 = alpha U_{N-1}
  const double* dd = a.dia + (size_t)s * nx;
  const double* ex = a.ex + (size_t)s * nx;
  const double* ey = a.ey + (size_t)s * nx;
  const double* pv = (q == 0) ? a.start + ((size_t)s * a.N + (a.N - 1)) * nx : src;
  const double pmul = (q == 0) ? a.alpha : 1.0;
  const double sc = a.scaling[q];
  double* o = a.out + ((size_t)s * a.N + q) * nx;
  const double* Xq = X + rr;
  for (int i = hh; i < nx; i += SB_H) {
    const double x = Xq[(size_t)i * SB_R];
    double Ax = dd[i] * x;
    if (i + 1 < nx) Ax = fma(ex[i], Xq[(size_t)(i + 1) * SB_R], Ax);
    if (i >= 1) Ax = fma(ex[i - 1], Xq[(size_t)(i - 1) * SB_R], Ax);
    if (i + n < nx) Ax = fma(ey[i], Xq[(size_t)(i + n) * SB_R], Ax);
    if (i >= n) Ax = fma(ey[i - n], Xq[(size_t)(i - n) * SB_R], Ax);
    const double rhs = fma(a.dT, Ax, x) - pmul * pv[i];
    o[i] = sc * rhs;
  }
}

// ---------------------------------------------------------------------------
// CGC: scaled DFT along time, per-frequency banded solves, inverse + update.
// P layout: [M][NF][nx] complex.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void load_twiddles(Cplx* tw, int N) {  // tw[j] = exp(-2 pi i j / N)
  for (int j = threadIdx.x; j < N; j += blockDim.x) {
    double sn, cs;
    sincospi(-2.0 * (double)j / (double)N, &sn, &cs);
    tw[j] = {cs, sn};
  }
  __syncthreads();
}

__global__ void dft_fwd_kernel(const double* __restrict__ R, const double* __restrict__ load_scale,
                               const int32_t* __restrict__ status, int M, int N, int nx,
                               Cplx* __restrict__ P) {
  __shared__ Cplx tw[1024];
  load_twiddles(tw, N);
  const int NF = N / 2 + 1;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)M * nx) return;
  const int s = (int)(t / nx), i = (int)(t - (long long)s * nx);
  if (status && status[s] != KLE_SAMPLE_ACTIVE) return;
  const double* r = R + (size_t)s * N * nx + i;
  const double rs = 1.0 / sqrt((double)N);
  for (int f = 0; f < NF; ++f) {
    double re = 0.0, im = 0.0;
    int w = 0;  // (f k) mod N
    for (int k = 0; k < N; ++k) {
      double v = r[(size_t)k * nx];
      if (load_scale) v *= load_scale[k];
      re = fma(v, tw[w].re, re);
      im = fma(v, tw[w].im, im);
      w += f;
      if (w >= N) w -= N;
    }
    P[((size_t)s * NF + f) * nx + i] = {re * rs, im * rs};
  }
}

// one warp per (sample, frequency): B_f q = p in place
// The factor rows are streamed PD rows ahead in registers (4 complex per lane
// and row for n <= 128) together with p_i and D_i^{-1}: the row recurrence
// only waits on shared memory, HBM latency is hidden PD rows deep.
constexpr int BS_PD = 4;

__global__ void __launch_bounds__(32) band_solve_cplx_kernel(Cplx* __restrict__ P, const double* __restrict__ Lt,
                                                             const double* __restrict__ Dinv,
                                                             const int32_t* __restrict__ status, int NF, int n) {
  constexpr int PD = BS_PD;
  const int nx = n * n, W = n + 1;
  const int phi = blockIdx.x, s = phi / NF;
  if (status && status[s] != KLE_SAMPLE_ACTIVE) return;
  const int lane = threadIdx.x;
  const Cplx* L = reinterpret_cast<const Cplx*>(Lt) + (size_t)phi * nx * n;
  const Cplx* Di = reinterpret_cast<const Cplx*>(Dinv) + (size_t)phi * nx;
  Cplx* p = P + (size_t)phi * nx;
  __shared__ Cplx win[128];
  Cplx lr[PD][4], pr[PD], dr[PD];
  auto fetch = [&](int u, int i, bool with_d) {
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int t = lane + 32 * m;
      lr[u][m] = (i >= 0 && i < nx && t < n) ? L[(size_t)i * n + t] : Cplx{0.0, 0.0};
    }
    pr[u] = (i >= 0 && i < nx) ? p[i] : Cplx{0.0, 0.0};
    if (with_d) dr[u] = (i >= 0 && i < nx) ? Di[i] : Cplx{0.0, 0.0};
  };
  for (int q = lane; q < W; q += 32) win[q] = {0.0, 0.0};
#pragma unroll
  for (int u = 0; u < PD; ++u) fetch(u, u, true);
  __syncwarp();
  // forward, column form: pending updates acc[(r) % W] for rows r in (i, i+n]
  for (int i0 = 0; i0 < nx; i0 += PD) {
#pragma unroll
    for (int u = 0; u < PD; ++u) {
      const int i = i0 + u;
      if (i < nx) {
        const int si = i % W;
        const Cplx acc = win[si];
        const Cplx y = {pr[u].re - acc.re, pr[u].im - acc.im};
        __syncwarp();
        if (lane == 0) {
          win[si] = {0.0, 0.0};
          p[i] = cmul(y, dr[u]);  // z_i = y_i / D_i
        }
        __syncwarp();
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int t = lane + 32 * m;
          if (t < n) {
            int sl = si + 1 + t;
            if (sl >= W) sl -= W;
            const Cplx l = lr[u][m];
            Cplx w = win[sl];
            w.re = fma(l.re, y.re, fma(-l.im, y.im, w.re));
            w.im = fma(l.re, y.im, fma(l.im, y.re, w.im));
            win[sl] = w;
          }
        }
        __syncwarp();
      }
      fetch(u, i + PD, true);
    }
  }
  for (int q = lane; q < W; q += 32) win[q] = {0.0, 0.0};
  __syncwarp();  // also orders the forward pass's p[] stores before the reloads below
#pragma unroll
  for (int u = 0; u < PD; ++u) fetch(u, nx - 1 - u, false);
  // backward, dot form: x_i = z_i - sum_t L(i+1+t, i) x_{i+1+t}
  for (int i0 = nx - 1; i0 >= 0; i0 -= PD) {
#pragma unroll
    for (int u = 0; u < PD; ++u) {
      const int i = i0 - u;
      if (i >= 0) {
        const int si = i % W;
        double re = 0.0, im = 0.0;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int t = lane + 32 * m;
          if (t < n) {
            int sl = si + 1 + t;
            if (sl >= W) sl -= W;
            const Cplx l = lr[u][m];
            const Cplx x = win[sl];
            re = fma(l.re, x.re, fma(-l.im, x.im, re));
            im = fma(l.re, x.im, fma(l.im, x.re, im));
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          re += __shfl_xor_sync(KLE_FULL_MASK, re, o);
          im += __shfl_xor_sync(KLE_FULL_MASK, im, o);
        }
        const Cplx z = pr[u];
        const Cplx x = {z.re - re, z.im - im};
        __syncwarp();
        if (lane == 0) {
          win[si] = x;
          p[i] = x;
        }
        __syncwarp();
      }
      fetch(u, i - PD, false);
    }
  }
}

// u_k = Re(ifft(q))_k / sqrt(N) / scaling_k with q_{N-f} = conj(q_f); the
// increment max |u - U| per sample into inc_bits (non-negative doubles and +NaN
// order like their bit patterns).
__global__ void dft_inv_update_kernel(const Cplx* __restrict__ P, const double* __restrict__ inv_scaling,
                                      const int32_t* __restrict__ status, int M, int N, int nx,
                                      double* __restrict__ U, double* __restrict__ Uout,
                                      unsigned long long* __restrict__ inc_bits) {
  __shared__ Cplx tw[1024];
  load_twiddles(tw, N);
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool in = t < (long long)M * nx;
  const int s = in ? (int)(t / nx) : 0, i = in ? (int)(t - (long long)s * nx) : 0;
  const bool act = in && !(status && status[s] != KLE_SAMPLE_ACTIVE);
  const int NF = N / 2 + 1;
  double incmax = 0.0;
  bool bad = false;
  if (act) {
    const Cplx* q = P + (size_t)s * NF * nx + i;
    const double rs = 1.0 / sqrt((double)N);
    double* out = (Uout ? Uout : U) + (size_t)s * N * nx + i;
    const double* old = (inc_bits && U) ? U + (size_t)s * N * nx + i : nullptr;
    for (int k = 0; k < N; ++k) {
      double re = 0.0;
      int w = 0;  // (f k) mod N; exp(+2 pi i f k / N) = conj tw
      for (int f = 0; f < N; ++f) {
        const int fe = f <= N / 2 ? f : N - f;
        const Cplx v = q[(size_t)fe * nx];
        const double vim = (f <= N / 2) ? v.im : -v.im;
        re = fma(v.re, tw[w].re, fma(vim, tw[w].im, re));  // Re(v conj(tw))
        w += k;
        if (w >= N) w -= N;
      }
      const double u = (re * rs) * inv_scaling[k];
      if (old) {
        const double dlt = fabs(u - old[(size_t)k * nx]);
        incmax = fmax(incmax, dlt);
        bad |= (dlt != dlt);
      }
      out[(size_t)k * nx] = u;
    }
  }
  if (inc_bits == nullptr) return;  // uniform
  if (bad) incmax = __longlong_as_double(0x7ff8000000000000LL);
  const int key = act ? s : -1;
  const int k0 = __shfl_sync(KLE_FULL_MASK, key, 0);
  if (__all_sync(KLE_FULL_MASK, key == k0)) {
    if (k0 < 0) return;
    double m = incmax;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = nanmax(m, __shfl_xor_sync(KLE_FULL_MASK, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(inc_bits + k0, (unsigned long long)__double_as_longlong(m));
  } else if (act) {
    atomicMax(inc_bits + s, (unsigned long long)__double_as_longlong(incmax));
  }
}

__global__ void status2d_kernel(unsigned long long* __restrict__ inc_bits, int M, int k, int max_iters,
                                double tol, int32_t* __restrict__ status, int32_t* __restrict__ iters,
                                double* __restrict__ inc_out, double* __restrict__ inc_hist,
                                int32_t* __restrict__ active_count) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= M) return;
  if (status[s] != KLE_SAMPLE_ACTIVE) return;
  const double inc = __longlong_as_double((long long)inc_bits[s]);
  inc_bits[s] = 0ULL;
  if (inc_out) inc_out[s] = inc;
  if (inc_hist) inc_hist[(size_t)s * max_iters + (k - 1)] = inc;
  int st = KLE_SAMPLE_ACTIVE;
  if (inc <= tol) st = KLE_SAMPLE_CONVERGED;
  else if (!isfinite(inc)) st = KLE_SAMPLE_NONFINITE;
  else if (k >= max_iters) st = KLE_SAMPLE_MAXITERS;
  if (st != KLE_SAMPLE_ACTIVE) {
    status[s] = st;
    if (iters) iters[s] = k;
  } else if (active_count) {
    atomicAdd(active_count, 1);
  }
}

}  // namespace kle

// ===========================================================================
// C ABI (declared in include/kle_b200.h)
// ===========================================================================
using namespace kle;
#define KLE2D_STREAM(s) (reinterpret_cast<cudaStream_t>(s))

extern "C" int kle_2d_kl5pt_f64(const double* xi, int M, int d, const double* kl_table, int n, double inv_h2,
                               double* dia, double* ex, double* ey, void* stream) {
  if (M < 0 || d < 1 || n < 1) return set_error(KLE_ERR_INVALID, "kl5pt: bad dims");
  const long long tot = (long long)M * n * n;
  if (tot == 0) return KLE_OK;
  kl5pt_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, KLE2D_STREAM(stream)>>>(xi, M, d, kl_table, n, inv_h2,
                                                                                  dia, ex, ey);
  return check_launch("kl5pt_kernel");
}

extern "C" int kle_2d_factor_f64(const double* dia, const double* ex, const double* ey, int M, int n,
                                 const double* lam, int NF, double shift, double c, double* Lt, double* Dinv,
                                 void* stream) {
  if (M < 0 || n < 1 || n > 127 || (lam && NF < 1))
    return set_error(KLE_ERR_INVALID, "factor2d: bad dims (n <= 127)");
  if (M == 0) return KLE_OK;
  const int W = n + 1;
  static const bool panel = [] {
    const char* e = getenv("KLE_2D_FACTOR_PANEL");
    return !(e && e[0] == '0');
  }();
  if (lam && panel && (n + 1) / 2 * 8 <= PF_NT && n + PF_B <= PF_PT && n + 1 <= 8 * PF_M) {
    const size_t smem = pf_smem_bytes(n);
    cudaFuncSetAttribute(band_factor_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    band_factor_panel_kernel<<<(unsigned)(M * NF), PF_NT, smem, KLE2D_STREAM(stream)>>>(dia, ex, ey, n, lam, NF, c,
                                                                                       Lt, Dinv);
    return check_launch("band_factor_panel_kernel");
  }
  if (lam) {
    const size_t smem = sizeof(double) * 16384 + 2 * W * sizeof(Cplx) + sizeof(double) * 3 * BF_RING;
    cudaFuncSetAttribute(band_factor_kernel<true, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    band_factor_kernel<true, 1024><<<(unsigned)(M * NF), 1024, smem, KLE2D_STREAM(stream)>>>(
        dia, ex, ey, n, lam, NF, 0.0, c, Lt, Dinv);
  } else {
    const size_t smem = sizeof(double) * 16384 + 2 * W * sizeof(double) + sizeof(double) * 3 * BF_RING;
    cudaFuncSetAttribute(band_factor_kernel<false, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    band_factor_kernel<false, 1024><<<(unsigned)M, 1024, smem, KLE2D_STREAM(stream)>>>(dia, ex, ey, n, nullptr, 1, shift,
                                                                                  c, Lt, Dinv);
  }
  return check_launch("band_factor_kernel");
}

extern "C" size_t kle_2d_fine_work_doubles(int M, int N, int n) {
  return (M <= 0 || N <= 0 || n <= 0) ? 0 : 2 * (size_t)M * ((N + 31) / 32) * n * n * 32;  // covers SB_R = 16
}

template <int SB_R>
static int fine2d_launch_r(Fine2dArgs& a, void* stream) {
  const int G = (a.N + SB_R - 1) / SB_R;
  const size_t smem = sizeof(double) * ((size_t)win_pow2(a.n) * SB_R + (size_t)(a.n + SB_RB) * SB_RB);
  cudaFuncSetAttribute(fine2d_kernel<SB_R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  fine2d_kernel<SB_R><<<(unsigned)(a.M * G), 32, smem, KLE2D_STREAM(stream)>>>(a);
  return check_launch("fine2d_kernel");
}

static int fine2d_launch(Fine2dArgs& a, void* stream) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  // narrowest warps (more warps per sample, more coefficient traffic) only as
  // far as needed to put ~4 warps on every SM
  const long long want = 4LL * sms;
  if (a.N > 16 && (long long)a.M * ((a.N + 31) / 32) < want) {
    if (a.N > 8 && (long long)a.M * ((a.N + 15) / 16) < want) return fine2d_launch_r<8>(a, stream);
    return fine2d_launch_r<16>(a, stream);
  }
  return fine2d_launch_r<32>(a, stream);
}

extern "C" int kle_2d_fgr_f64(const double* U, const double* u0, const double* F_given, const double* dia,
                              const double* ex, const double* ey, const double* Lt, const double* Dinv,
                              const double* scaling, const int32_t* active, int M, int N, int n, int J,
                             double dt, double dT, double g0, double alpha, double* work, size_t work_doubles,
                             double* Rout, void* stream) {
  if (M < 0 || N < 1 || n < 1 || n > 127 || J < 1) return set_error(KLE_ERR_INVALID, "fgr2d: bad dims");
  if (M == 0) return KLE_OK;
  const size_t need = kle_2d_fine_work_doubles(M, N, n);
  if (work_doubles < need) return set_error(KLE_ERR_WORKSPACE, "fgr2d: workspace too small");
  Fine2dArgs a{U, u0, F_given, dia, ex, ey, Lt, Dinv, scaling, active, work, work + need / 2, Rout,
               M, N, n, J, 1, 0, dt, dT, g0, alpha};
  return fine2d_launch(a, stream);
}

extern "C" int kle_2d_sweep_f64(const double* start, const double* dia, const double* ex, const double* ey,
                                const double* Lt, const double* Dinv, int M, int Q, int n,
                               int J, int nseg, double h, double g0, double* work, size_t work_doubles,
                               double* out, void* stream) {
  if (M < 0 || Q < 1 || n < 1 || n > 127 || J < 1 || nseg < 1) return set_error(KLE_ERR_INVALID, "sweep2d: bad dims");
  if (M == 0) return KLE_OK;
  const size_t need = kle_2d_fine_work_doubles(M, Q, n);
  if (work_doubles < need) return set_error(KLE_ERR_WORKSPACE, "sweep2d: workspace too small");
  Fine2dArgs a{start, nullptr, nullptr, dia, ex, ey, Lt, Dinv, nullptr, nullptr, work, work + need / 2, out,
               M, Q, n, J, nseg, 1, h, 0.0, g0, 0.0};
  return fine2d_launch(a, stream);
}

extern "C" size_t kle_2d_cgc_work_doubles(int M, int N, int n) {
  return (M <= 0 || N <= 0 || n <= 0) ? 0 : 2 * (size_t)M * (N / 2 + 1) * n * n + (size_t)M;
}

extern "C" int kle_2d_cgc_f64(const double* R, const double* load_scale, double* U, double* Uout,
                             const double* Lt, const double* Dinv, const double* inv_scaling, int M, int N, int n,
                             int k, int max_iters, double tol, int32_t* status, int32_t* iters, double* inc,
                             double* inc_hist, int32_t* active_count, double* work, size_t work_doubles,
                             void* stream) {
  if (M < 0 || N < 2 || (N & 1) || n < 1 || n > 127) return set_error(KLE_ERR_INVALID, "cgc2d: bad dims (N even)");
  if (M == 0) return KLE_OK;
  if (work_doubles < kle_2d_cgc_work_doubles(M, N, n)) return set_error(KLE_ERR_WORKSPACE, "cgc2d: workspace");
  const int nx = n * n, NF = N / 2 + 1;
  cudaStream_t st = KLE2D_STREAM(stream);
  Cplx* P = reinterpret_cast<Cplx*>(work);
  unsigned long long* bits = reinterpret_cast<unsigned long long*>(work + 2 * (size_t)M * NF * nx);
  const long long tot = (long long)M * nx;
  dft_fwd_kernel<<<(unsigned)((tot + 127) / 128), 128, 0, st>>>(R, load_scale, status, M, N, nx, P);
  if (int e = check_launch("dft_fwd_kernel")) return e;
  band_solve_cplx_kernel<<<(unsigned)(M * NF), 32, 0, st>>>(P, Lt, Dinv, status, NF, n);
  if (int e = check_launch("band_solve_cplx_kernel")) return e;
  const bool track = status != nullptr && U != nullptr && Uout == nullptr;
  dft_inv_update_kernel<<<(unsigned)((tot + 127) / 128), 128, 0, st>>>(P, inv_scaling, status, M, N, nx, U, Uout,
                                                                         track ? bits : nullptr);
  if (int e = check_launch("dft_inv_update_kernel")) return e;
  if (!track) return KLE_OK;
  status2d_kernel<<<(unsigned)((M + 127) / 128), 128, 0, st>>>(bits, M, k, max_iters, tol, status, iters, inc,
                                                                inc_hist, active_count);
  return check_launch("status2d_kernel");
}

// ---------------------------------------------------------------------------
// Matrix-free Krylov variants (kle_2d_krylov.cu): PCG fine sweeps and COCG
// shifted solves in place of the banded factors.
// ---------------------------------------------------------------------------
extern "C" int kle_2d_fgr_krylov_f64(const double* U, const double* u0, const double* F_given, const double* dia,
                                     const double* ex, const double* ey, const double* scaling,
                                     const int32_t* status, int M, int N, int n, int J, double dt, double dT,
                                     double g0, double alpha, double rtol, int max_its, double* R, double* F_out,
                                     long long* its, void* stream) {
  if (M < 0 || N < 1 || n < 1 || n > 128 || J < 1 || !(rtol > 0) || max_its < 1)
    return set_error(KLE_ERR_INVALID, "fgr2d_krylov: bad arguments");
  Kry2dArgs a{U, u0, F_given, dia, ex, ey, scaling, status, F_out, R, its, M, N, n, J, max_its, 1, dt, dT, g0, alpha,
              rtol};
  return kry2d_fine(a, KLE2D_STREAM(stream));
}

extern "C" int kle_2d_sweep_krylov_f64(const double* start, const double* dia, const double* ex, const double* ey,
                                       int M, int Q, int n, int J, double h, double g0, double rtol, int max_its,
                                       double* out, long long* its, void* stream) {
  if (M < 0 || Q < 1 || n < 1 || n > 128 || J < 1 || !(rtol > 0) || max_its < 1)
    return set_error(KLE_ERR_INVALID, "sweep2d_krylov: bad arguments");
  Kry2dArgs a{start, nullptr, nullptr, dia, ex, ey, nullptr, nullptr, out, nullptr, its, M, Q, n, J, max_its, 0, h,
              0.0, g0, 0.0, rtol};
  return kry2d_fine(a, KLE2D_STREAM(stream));
}

extern "C" size_t kle_2d_cgc_krylov_work_doubles(int M, int N, int n) {
  return (M <= 0 || N <= 0 || n <= 0) ? 0 : 6 * (size_t)M * (N / 2 + 1) * n * n + (size_t)M;
}

extern "C" int kle_2d_cgc_krylov_f64(const double* R, const double* load_scale, double* U, double* Uout,
                                     const double* dia, const double* ex, const double* ey, const double* lam,
                                     const double* inv_scaling, int M, int N, int n, int k, int max_iters,
                                     double tol, int32_t* status, int32_t* iters, double* inc, double* inc_hist,
                                     int32_t* active_count, double dT, double rtol, int max_its, double* work,
                                     size_t work_doubles, long long* its, void* stream) {
  if (M < 0 || N < 2 || (N & 1) || n < 1 || n > 128 || !(rtol > 0) || max_its < 1)
    return set_error(KLE_ERR_INVALID, "cgc2d_krylov: bad arguments (N even)");
  if (M == 0) return KLE_OK;
  if (work_doubles < kle_2d_cgc_krylov_work_doubles(M, N, n)) return set_error(KLE_ERR_WORKSPACE, "cgc2d_krylov: workspace");
  const int nx = n * n, NF = N / 2 + 1;
  cudaStream_t st = KLE2D_STREAM(stream);
  Cplx* P = reinterpret_cast<Cplx*>(work);
  unsigned long long* bits = reinterpret_cast<unsigned long long*>(work + 2 * (size_t)M * NF * nx);
  Cplx* kw = reinterpret_cast<Cplx*>(work + 2 * (size_t)M * NF * nx + M);
  const long long tot = (long long)M * nx;
  dft_fwd_kernel<<<(unsigned)((tot + 127) / 128), 128, 0, st>>>(R, load_scale, status, M, N, nx, P);
  if (int e = check_launch("dft_fwd_kernel")) return e;
  if (int e = kry2d_shift_solve(P, dia, ex, ey, lam, status, M, NF, n, dT, rtol, max_its, kw, its, st)) return e;
  const bool track = status != nullptr && U != nullptr && Uout == nullptr;
  dft_inv_update_kernel<<<(unsigned)((tot + 127) / 128), 128, 0, st>>>(P, inv_scaling, status, M, N, nx, U, Uout,
                                                                         track ? bits : nullptr);
  if (int e = check_launch("dft_inv_update_kernel")) return e;
  if (!track) return KLE_OK;
  status2d_kernel<<<(unsigned)((M + 127) / 128), 128, 0, st>>>(bits, M, k, max_iters, tol, status, iters, inc,
                                                                inc_hist, active_count);
  return check_launch("status2d_kernel");
}
