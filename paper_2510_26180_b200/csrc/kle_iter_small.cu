// Fused PCGC outer iteration for small blocks (nx <= 128, N = 2..16 a power
// of two: configs 1 and 4): one CTA per sample runs the whole iteration on
// chip —
//   1. the J-step backward-Euler fine sweeps of all N subintervals
//      (pintuq/propagators.py:121-145 via pcgc.py:321-330), the partitioned
//      register-resident LDL^T solve of kle_fine.cuh (8 lanes x 16 rows per
//      system, one system per 8-lane group: 16 groups = the CTA's 128 threads);
//   2. the CGC right-hand side rhs_n = scaling_n ((I + dT A) F_n - prev_n)
//      (assemble_rhs_blocks + cgc_correct, pcgc.py:175-243), the same
//      expression as fgr_kernel, written two-for-one packed into a complex
//      [N][64] tile (rows c and c + 64 as re / im);
//   3. the diagonalised three-step solve (three_step_solve, pcgc.py:148-172):
//      four-step FFT along time, one 8-lane group per frequency f <= N/2
//      solving (lambda_f I + dT A) q = p_f with the batch's precomputed shift
//      pivots (8 lanes x 16 rows, stitched by 3-stage lane scans; the whole
//      system is inside the CTA, no cluster), Hermitian pack, inverse FFT;
//   4. the U update, increment max|U_new - U| and stop test (pcgc.py:335-348).
// HBM per sample-iteration: U read and written (16 B per (n, i)), the fine
// factor blob (6.4 KB) and the shift pivots (16 (N/2+1) nx B); the CGC
// right-hand side never leaves shared memory, and the CTA's CGC phases
// (latency-bound) overlap the other resident CTAs' sweeps (FP64-bound).
#include <cstdlib>

#include "kle_fine.cuh"
#include "kle_internal.h"

namespace kle {
namespace itsmall {

constexpr int NT = 128;               // 4 warps
constexpr int MR = 16, P = 8;         // fine layout: 8 lanes x 16 rows (nxp = 128)
constexpr int RB = 128, HC = 64;      // rows, packed complex columns
constexpr int CLN = 8;                // lanes per frequency group in the CGC

// start / old-U rows: element j of lane-chunk k at k*16 + (j ^ sw), sw mixing
// the chunk and the subinterval parity, so the 8 lanes (and two slots) of a
// warp reading "row k*16+j" of their systems fall into distinct banks
__device__ __forceinline__ int rsw(int n, int row) { return row ^ (((row >> 4) & 7) | ((n & 1) << 3)); }
// packed tile [N][HC] complex: column XOR-swizzled by its 16-column group so the
// CGC's lanes (columns 16 apart) spread over the banks
__device__ __forceinline__ int tix(int n, int c) { return n * HC + (c ^ ((c >> 4) & 3)); }
// pivot slice [NF][RB] complex: lanes 16 rows apart in distinct banks
__device__ __forceinline__ int pix(int r) { return r ^ ((r >> 4) & 7); }

__device__ __forceinline__ Cplx cadd2(Cplx a, Cplx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ Cplx csub2(Cplx a, Cplx b) { return {a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ Cplx cfma(Cplx a, Cplx b, Cplx c) {  // a*b + c
  return {fma(a.re, b.re, fma(-a.im, b.im, c.re)), fma(a.re, b.im, fma(a.im, b.re, c.im))};
}
__device__ __forceinline__ Cplx cneg_mul(Cplx a, Cplx b) {  // -(a*b)
  return {fma(-a.re, b.re, a.im * b.im), fma(-a.re, b.im, -a.im * b.re)};
}
__device__ __forceinline__ Cplx shfl_up_c(Cplx v, int d) {
  return {__shfl_up_sync(KLE_FULL_MASK, v.re, d, CLN), __shfl_up_sync(KLE_FULL_MASK, v.im, d, CLN)};
}
__device__ __forceinline__ Cplx shfl_down_c(Cplx v, int d) {
  return {__shfl_down_sync(KLE_FULL_MASK, v.re, d, CLN), __shfl_down_sync(KLE_FULL_MASK, v.im, d, CLN)};
}
__device__ __forceinline__ Cplx shfl_xor_c(Cplx v, int d) {
  return {__shfl_xor_sync(KLE_FULL_MASK, v.re, d), __shfl_xor_sync(KLE_FULL_MASK, v.im, d)};
}
template <int S>
__device__ __forceinline__ Cplx mul_si(Cplx z) {  // z * (S i)
  return S > 0 ? Cplx{-z.im, z.re} : Cplx{z.im, -z.re};
}

template <int NS, int S>
struct Dft;
template <int S>
struct Dft<1, S> {
  __device__ __forceinline__ static void run(Cplx (&)[1]) {}
};
template <int S>
struct Dft<2, S> {
  __device__ __forceinline__ static void run(Cplx (&v)[2]) {
    const Cplx a = v[0], b = v[1];
    v[0] = cadd2(a, b);
    v[1] = csub2(a, b);
  }
};
template <int S>
struct Dft<4, S> {
  __device__ __forceinline__ static void run(Cplx (&v)[4]) {
    const Cplx s02 = cadd2(v[0], v[2]), d02 = csub2(v[0], v[2]);
    const Cplx s13 = cadd2(v[1], v[3]), d13 = mul_si<S>(csub2(v[1], v[3]));
    v[0] = cadd2(s02, s13);
    v[2] = csub2(s02, s13);
    v[1] = cadd2(d02, d13);
    v[3] = csub2(d02, d13);
  }
};

// Four-step FFT over the HC columns of the [N][HC] tile, natural order in and
// out (N = N1 N2, N1 = 2^ceil(LOGN/2) <= 4). S = -1: forward (np.fft.fft sign),
// S = +1: inverse (unnormalised). tw[j] = exp(-2 pi i j / N).
template <int LOGN, int S>
__device__ void fft4(Cplx* t, const Cplx* tw) {
  constexpr int N = 1 << LOGN;
  constexpr int N1 = 1 << ((LOGN + 1) / 2), N2 = N / N1;
  for (int task = threadIdx.x; task < N1 * HC; task += NT) {
    const int n1 = task / HC, c = task % HC;
    Cplx v[N2];
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) v[n2] = t[tix(n1 + N1 * n2, c)];
    Dft<N2, S>::run(v);
#pragma unroll
    for (int k2 = 1; k2 < N2; ++k2) {
      Cplx w = tw[(n1 * k2) & (N - 1)];
      if (S > 0) w.im = -w.im;
      v[k2] = cmul(v[k2], w);
    }
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) t[tix(n1 + N1 * k2, c)] = v[k2];
  }
  __syncthreads();
  constexpr int ROUNDS = (N2 * HC + NT - 1) / NT;
  Cplx w[ROUNDS][N1];
#pragma unroll
  for (int r = 0; r < ROUNDS; ++r) {
    const int task = threadIdx.x + r * NT;
    if (task < N2 * HC) {
      const int k2 = task / HC, c = task % HC;
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) w[r][n1] = t[tix(n1 + N1 * k2, c)];
      Dft<N1, S>::run(w[r]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < ROUNDS; ++r) {
    const int task = threadIdx.x + r * NT;
    if (task < N2 * HC) {
      const int k2 = task / HC, c = task % HC;
#pragma unroll
      for (int k1 = 0; k1 < N1; ++k1) t[tix(k2 + N2 * k1, c)] = w[r][k1];
    }
  }
  __syncthreads();
}

// (lambda_f I + dT A) q = p for one frequency, partitioned over an 8-lane group
// (lane k owns rows r0 .. r0 + MR - 1, r0 = 16 k): chunk-local LDL^T passes
// with the precomputed pivots 1/beta (piv(jj) = pivot of row r0 + jj, jj >= -1),
// stitched by 3-stage affine lane scans (the cluster kernel's recurrences with
// the whole system inside one group). off[jj] = dT * A[r0+jj-1][r0+jj].
template <class PivFn>
__device__ __forceinline__ void freq_solve(Cplx (&y)[MR], int k, const double* off, PivFn piv) {
  auto lj = [&](int j) -> Cplx {  // l_r = dT off_{r-1} / beta_{r-1}
    const double E = off[j];
    const Cplx ip = piv(j - 1);
    return {E * ip.re, E * ip.im};
  };
  Cplx A = {1.0, 0.0};
#pragma unroll
  for (int j = 0; j < MR; ++j) {
    const Cplx l = lj(j);
    if (j > 0) y[j] = cfma({-l.re, -l.im}, y[j - 1], y[j]);
    A = cneg_mul(l, A);
  }
  Cplx B = y[MR - 1];
#pragma unroll
  for (int d = 1; d < CLN; d <<= 1) {
    const Cplx Ao = shfl_up_c(A, d), Bo = shfl_up_c(B, d);
    if (k >= d) {
      B = cfma(A, Bo, B);
      A = cmul(A, Ao);
    }
  }
  Cplx Be = shfl_up_c(B, 1);
  if (k == 0) Be = {0.0, 0.0};
  {
    Cplx pi = {1.0, 0.0};
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      pi = cneg_mul(lj(j), pi);
      y[j] = cmul(cfma(pi, Be, y[j]), piv(j));
    }
  }
  const double En = off[MR];
  const Cplx ibl = piv(MR - 1);
  const Cplx lnext = {En * ibl.re, En * ibl.im};
  Cplx S = {1.0, 0.0};
#pragma unroll
  for (int j = MR - 1; j >= 0; --j) {
    const Cplx ln = (j == MR - 1) ? lnext : lj(j + 1);
    if (j < MR - 1) y[j] = cfma({-ln.re, -ln.im}, y[j + 1], y[j]);
    S = cneg_mul(ln, S);
  }
  Cplx T = y[0];
#pragma unroll
  for (int d = 1; d < CLN; d <<= 1) {
    const Cplx So = shfl_down_c(S, d), To = shfl_down_c(T, d);
    if (k + d < CLN) {
      T = cfma(S, To, T);
      S = cmul(S, So);
    }
  }
  Cplx Te = shfl_down_c(T, 1);
  if (k == CLN - 1) Te = {0.0, 0.0};
  Cplx sg = {1.0, 0.0};
#pragma unroll
  for (int j = MR - 1; j >= 0; --j) {
    const Cplx ln = (j == MR - 1) ? lnext : lj(j + 1);
    sg = cneg_mul(ln, sg);
    y[j] = cfma(sg, Te, y[j]);
  }
}

template <int LOGN, bool FUSE>
struct Shape {
  static constexpr int N = 1 << LOGN, NF = N / 2 + 1;
  static_assert(NF * CLN <= NT, "one 8-lane group per frequency: N <= 16");
  // shared memory (doubles); the CGC-only variant (FUSE = false) keeps neither
  // the old U rows (re-read from global in the update) nor the operator rows
  static constexpr int O_UST = 0;                    // [N][RB] old U rows (rsw)
  static constexpr int O_TILE = O_UST + (FUSE ? N * RB : 0);  // [N][HC] complex
  static constexpr int O_PIV = O_TILE + 2 * N * HC;  // [NF][RB] complex (pix)
  static constexpr int O_DD = O_PIV + 2 * NF * RB;   // [RB] dia (rsw with n = 0)
  static constexpr int O_EE = O_DD + (FUSE ? RB : 0);               // [RB + 16]: ee[rsw(0, i)] couples rows i-1 and i
  static constexpr int O_OFS = O_EE + (FUSE ? RB + 16 : 0);         // [RB + 2]: dT * off[row - 1]
  static constexpr int O_TW = O_OFS + RB + 2;        // [N] complex
  static constexpr int O_ISC = O_TW + 2 * N;         // [N]
  static constexpr int O_RED = O_ISC + N;            // [4]
  static constexpr size_t BYTES = sizeof(double) * (size_t)(O_RED + 4);
};

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}

#ifndef KLE_ITS_MINB
#define KLE_ITS_MINB 3
#endif
#ifndef KLE_CGS_MINB
#define KLE_CGS_MINB 3
#endif
// FUSE = true: the whole iteration; FUSE = false: the CGC update only, from the
// right-hand side R written by fgr_kernel (a drop-in for the cluster CGC at
// small N: one CTA per sample, no cluster barriers or cross-CTA reductions)
template <int LOGN, bool FUSE>
__global__ void __launch_bounds__(NT, FUSE ? KLE_ITS_MINB : KLE_CGS_MINB) iter_small_kernel(IterSmallArgs a) {
  using K = Shape<LOGN, FUSE>;
  using L = FineLayout<MR, P>;
  constexpr int N = K::N, NF = K::NF;
  const int s = blockIdx.x;
  if (a.status && a.status[s] != KLE_SAMPLE_ACTIVE) return;
  extern __shared__ __align__(16) double sm[];
  double* ust = sm + K::O_UST;
  Cplx* tile = reinterpret_cast<Cplx*>(sm + K::O_TILE);
  Cplx* piv = reinterpret_cast<Cplx*>(sm + K::O_PIV);
  double* dd = sm + K::O_DD;
  double* ee = sm + K::O_EE;
  double* offs = sm + K::O_OFS;
  Cplx* tw = reinterpret_cast<Cplx*>(sm + K::O_TW);
  double* isc = sm + K::O_ISC;
  double* red = sm + K::O_RED;
  const int tid = threadIdx.x, nx = a.nx;
  const size_t sb = (size_t)s * N * nx;

  // ---- phase 0: stage U, the operator and (second group) the shift pivots --
  if constexpr (FUSE) {
    for (int e = tid; e < N * RB; e += NT) {
      const int n = e / RB, row = e % RB;
      double* dst = ust + n * RB + rsw(n, row);
      if (row < nx) cp_async8(dst, a.U + sb + (size_t)n * nx + row);
      else *dst = 0.0;
    }
    for (int i = tid; i < RB; i += NT) {  // ee[rsw(0, i)] = A[i-1][i] (0 for i = 0 and i >= nx)
      if (i < nx) cp_async8(dd + rsw(0, i), a.dia + (size_t)s * nx + i);
      else dd[rsw(0, i)] = 0.0;
      if (i >= 1 && i < nx) cp_async8(ee + rsw(0, i), a.off + (size_t)s * nx + i - 1);
      else ee[rsw(0, i)] = 0.0;
    }
  } else {  // the right-hand side, packed two-for-one into the tile
    for (int e = tid; e < N * RB; e += NT) {
      const int n = e / RB, row = e % RB;
      double* dst = reinterpret_cast<double*>(&tile[tix(n, row & (HC - 1))]) + (row >> 6);
      if (row < nx) cp_async8(dst, a.R + sb + (size_t)n * nx + row);
      else *dst = 0.0;
    }
  }
  asm volatile("cp.async.commit_group;\n" ::);
  {
    const Cplx* src = reinterpret_cast<const Cplx*>(a.sfac) + (size_t)s * NF * nx;
    for (int e = tid; e < NF * RB; e += NT) {
      const int f = e / RB, r = e % RB;
      Cplx* dst = &piv[f * RB + pix(r)];
      if (r < nx) cp_async16(dst, src + (size_t)f * nx + r);
      else *dst = {1.0, 0.0};
    }
  }
  asm volatile("cp.async.commit_group;\n" ::);
  for (int e = tid; e < RB + 2; e += NT) {
    const int row = e - 1;  // offs[e] couples rows e-1 and e
    offs[e] = (row >= 0 && row + 1 < nx) ? a.dT * a.off[(size_t)s * nx + row] : 0.0;
  }
  for (int j = tid; j < N; j += NT) {
    double sn, cs;
    sincospi(-2.0 * (double)j / (double)N, &sn, &cs);
    tw[j] = {cs, sn};
    isc[j] = a.inv_scaling[j];
  }

  const int lane = tid & 31, k = lane & 7;
  if constexpr (FUSE) {
  // ---- phase 1: fine sweeps, one subinterval per 8-lane group -------------
  const int g = tid >> 3;  // group = subinterval
  const bool live = g < N;
  LaneFactors<MR, P> fac;
  fac.load(a.ffac + (size_t)s * L::DOUBLES, k, nx);
  const double hg = a.dt * a.g0;
  asm volatile("cp.async.wait_group 1;\n" ::);
  __syncthreads();
  double x[1][MR];
#pragma unroll
  for (int j = 0; j < MR; ++j) {
    const int row = k * MR + j;
    double v = 0.0;
    if (row < nx && live) v = (g == 0) ? __ldg(a.u0 + row) : ust[(g - 1) * RB + rsw(g - 1, row)];
    x[0][j] = (row < nx) ? v + hg : 0.0;
  }
  be_steps<MR, P, 1>(x, fac, k, a.J, hg);
#pragma unroll
  for (int j = 0; j < MR; ++j) x[0][j] = (k * MR + j < nx) ? x[0][j] - hg : 0.0;

  // ---- phase 2: rhs_n = scaling_n ((I + dT A) F_n - prev_n) into the tile --
  {
    const double left = __shfl_up_sync(KLE_FULL_MASK, x[0][MR - 1], 1, P);
    const double right = __shfl_down_sync(KLE_FULL_MASK, x[0][0], 1, P);
    const int n = live ? g : 0;
    const double sc = live ? a.scaling[n] : 0.0;
    const double pmul = (n == 0) ? a.alpha : 1.0;
    const int pn = (n == 0) ? N - 1 : n - 1;
    double xl = k > 0 ? left : 0.0;
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      const int row = k * MR + j;
      const double dj = dd[rsw(0, row)], em = ee[rsw(0, row)], ep = (row + 1 < RB) ? ee[rsw(0, row + 1)] : 0.0;
      const double xc = x[0][j];
      const double xp = (j < MR - 1) ? x[0][j + 1] : (k < P - 1 ? right : 0.0);
      const double Ax = fma(em, xl, fma(dj, xc, ep * xp));
      const double rhs = fma(a.dT, Ax, xc) - pmul * ust[pn * RB + rsw(pn, row)];
      xl = xc;
      x[0][j] = (row < nx) ? sc * rhs : 0.0;
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);  // the pivots (group 2)
  if (live) {
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      const int row = k * MR + j;
      reinterpret_cast<double*>(&tile[tix(g, row & (HC - 1))])[row >> 6] = x[0][j];
    }
  }
  } else {
    asm volatile("cp.async.wait_group 0;\n" ::);
  }
  __syncthreads();
  fft4<LOGN, -1>(tile, tw);

  // ---- phase 3: (lambda_f I + dT A) q = p_f, one 8-lane group per f --------
  {
    const int fsys = tid >> 3;
    const bool valid = fsys < NF;
    const int f = valid ? fsys : NF - 1;
    const int r0 = k * MR;
    const Cplx* pf = piv + f * RB;
    const double hs = 0.5 / sqrt((double)N);  // two-for-one unpacking x 1/sqrt(N)
    Cplx y[MR];
    const int fm = (N - f) & (N - 1);
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      const int col = r0 + j;
      const Cplx zf = tile[tix(f, col & (HC - 1))], zm = tile[tix(fm, col & (HC - 1))];
      if (col < HC) y[j] = {(zf.re + zm.re) * hs, (zf.im - zm.im) * hs};  // (Z_f + conj Z_-f)/2
      else y[j] = {(zf.im + zm.im) * hs, (zm.re - zf.re) * hs};           // (Z_f - conj Z_-f)/(2i)
    }
    freq_solve(y, k, offs + r0, [&](int jj) -> Cplx {  // pivot of row r0 + jj (jj >= -1)
      return (r0 + jj >= 0) ? pf[pix(r0 + jj)] : Cplx{0.0, 0.0};
    });
    __syncthreads();  // every group has read its p_f, p_{N-f} from the tile
    // pack W_f = q(col) + i q(col + HC) (and the mirror W_{N-f}): lanes k < 4 hold the first half
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      const Cplx qb = shfl_xor_c(y[j], CLN / 2);
      if (valid && k < CLN / 2) {
        const int col = r0 + j;
        tile[tix(f, col)] = {y[j].re - qb.im, y[j].im + qb.re};
        if (f > 0 && 2 * f < N) tile[tix(N - f, col)] = {y[j].re + qb.im, qb.re - y[j].im};
      }
    }
  }
  // CGC-only variant: the column's old values, loaded while the inverse FFT runs
  double uold[FUSE ? 1 : N];
  if constexpr (!FUSE) {
#pragma unroll
    for (int n = 0; n < N; ++n) uold[n] = (tid < nx) ? a.U[sb + (size_t)n * nx + tid] : 0.0;
  }
  __syncthreads();
  fft4<LOGN, +1>(tile, tw);

  // ---- phase 4: U update, increment, stop test --------------------------------
  const double rsN = 1.0 / sqrt((double)N);
  double incmax = 0.0;
  bool bad = false;
  {
    const int row = tid;  // NT == RB: one column per thread
    if (row < nx) {
      double* out = a.U + sb + row;
      const double* uo = uold;
#pragma unroll 4
      for (int n = 0; n < N; ++n) {
        const Cplx z = tile[tix(n, row & (HC - 1))];
        const double u = ((row < HC ? z.re : z.im) * rsN) * isc[n];
        const double d = fabs(u - (FUSE ? ust[n * RB + rsw(n, row)] : uo[n]));
        incmax = fmax(incmax, d);
        bad |= (d != d);
        out[(size_t)n * nx] = u;
      }
    }
  }
  if (__syncthreads_or(bad)) incmax = __longlong_as_double(0x7ff8000000000000LL);
  incmax = warp_max(incmax);
  if (lane == 0) red[tid >> 5] = incmax;
  __syncthreads();
  if (tid == 0) {
    double inc = red[0];
    for (int i = 1; i < NT / 32; ++i) inc = nanmax(inc, red[i]);
    if (a.inc_hist) a.inc_hist[(size_t)s * a.max_iters + (a.k - 1)] = inc;
    if (a.status) {
      int st = KLE_SAMPLE_ACTIVE;
      if (inc <= a.tol) st = KLE_SAMPLE_CONVERGED;
      else if (!isfinite(inc)) st = KLE_SAMPLE_NONFINITE;
      else if (a.k >= a.max_iters) st = KLE_SAMPLE_MAXITERS;
      if (st != KLE_SAMPLE_ACTIVE) {
        a.status[s] = st;
        if (a.iters) a.iters[s] = a.k;
      } else if (a.active_count) {
        atomicAdd(a.active_count, 1);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// One WARP per sample (N = 16): the whole iteration warp-synchronous (only
// __syncwarp), so the latency-bound FFT / shifted-solve phases of one warp
// overlap the FP64-bound sweeps of the other warps on the SM:
//   sweeps: 4 slots x R = 4 subintervals, 8 lanes x 16 rows each (the
//           fgr_kernel<16, 8, 4, 32> step with shared-memory chunk products);
//   rhs:    into the warp's packed tile [16][64];
//   FFT:    four-step over the tile, 8 tasks per lane and pass;
//   solve:  3 rounds of 4 frequency groups (f = 4 rho + lane / 8 <= 8), the
//           lane's 17 pivots in registers (from global: 16 B x 17);
//   update: lane = packed columns lane and lane + 32, old U from global.
// ---------------------------------------------------------------------------
namespace wv {
constexpr int N = 16, LOGN = 4, NF = 9, R = 4;
__device__ __forceinline__ void syncw() { __syncwarp(KLE_FULL_MASK); }

// four-step FFT over the [N][HC] tile by one warp (same DFTs/twiddles/order as fft4)
template <int S>
__device__ void fft_warp(Cplx* t, const Cplx* tw, int lane) {
  constexpr int N1 = 4, N2 = 4;
  for (int task = lane; task < N1 * HC; task += 32) {
    const int n1 = task / HC, c = task % HC;
    Cplx v[N2];
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) v[n2] = t[tix(n1 + N1 * n2, c)];
    Dft<N2, S>::run(v);
#pragma unroll
    for (int k2 = 1; k2 < N2; ++k2) {
      Cplx w = tw[(n1 * k2) & (N - 1)];
      if (S > 0) w.im = -w.im;
      v[k2] = cmul(v[k2], w);
    }
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) t[tix(n1 + N1 * k2, c)] = v[k2];
  }
  syncw();
  // pass 2: every lane reads all 8 of its tasks' inputs before any store (the
  // stores permute rows: k2 + N2 k1 overwrites inputs of other tasks)
  Cplx w[8][N1];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int task = lane + 32 * r;
    const int k2 = task / HC, c = task % HC;
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) w[r][n1] = t[tix(n1 + N1 * k2, c)];
    Dft<N1, S>::run(w[r]);
  }
  syncw();
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int task = lane + 32 * r;
    const int k2 = task / HC, c = task % HC;
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) t[tix(k2 + N2 * k1, c)] = w[r][k1];
  }
  syncw();
}
}  // namespace wv

struct WarpSmem {  // doubles, per warp (one warp per CTA)
  static constexpr int O_TILE = 0;                        // [16][64] complex
  static constexpr int O_CS = O_TILE + 2 * 16 * HC;       // [3][16][8] chunk products
  static constexpr int O_OFS = O_CS + 3 * MR * P;         // [RB + 2]: dT * off[row - 1]
  static constexpr int O_TW = O_OFS + RB + 2;             // [16] complex
  static constexpr int O_ISC = O_TW + 2 * 16;             // [16]
  static constexpr size_t BYTES = sizeof(double) * (size_t)(O_ISC + 16);
};

__global__ void __launch_bounds__(32, 8) iter_warp_kernel(IterSmallArgs a) {
  using L = FineLayout<MR, P>;
  constexpr int N = wv::N, NF = wv::NF, R = wv::R;
  const int s = blockIdx.x;
  if (a.status[s] != KLE_SAMPLE_ACTIVE) return;
  extern __shared__ __align__(16) double sm[];
  Cplx* tile = reinterpret_cast<Cplx*>(sm + WarpSmem::O_TILE);
  double* cs = sm + WarpSmem::O_CS;
  double* offs = sm + WarpSmem::O_OFS;
  Cplx* tw = reinterpret_cast<Cplx*>(sm + WarpSmem::O_TW);
  double* isc = sm + WarpSmem::O_ISC;
  const int lane = threadIdx.x, k = lane & 7, slot = lane >> 3, nx = a.nx;
  const size_t sb = (size_t)s * N * nx;
  const double* dia = a.dia + (size_t)s * nx;
  const double* off = a.off + (size_t)s * nx;

  // ---- stage: factors, chunk products, start rows ---------------------------
  LaneFactors<MR, P> fac;
  fac.load(a.ffac + (size_t)s * L::DOUBLES, k, nx);
  const double hg = a.dt * a.g0;
  if (slot == 0) chunk_products<MR, P>(cs, fac, k, hg);
  for (int e = lane; e < RB + 2; e += 32) {
    const int row = e - 1;
    offs[e] = (row >= 0 && row + 1 < nx) ? a.dT * off[row] : 0.0;
  }
  if (lane < N) {
    double sn, c;
    sincospi(-2.0 * (double)lane / (double)N, &sn, &c);
    tw[lane] = {c, sn};
    isc[lane] = a.inv_scaling[lane];
  }
  double x[R][MR];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int n = slot * R + r;
    const double* src = (n == 0) ? a.u0 : a.U + sb + (size_t)(n - 1) * nx;
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      const int row = k * MR + j;
      x[r][j] = row < nx ? __ldg(src + row) + hg : 0.0;
    }
  }
  wv::syncw();
  // ---- the J-step sweeps ------------------------------------------------------
  be_steps_cs<MR, P, R>(x, fac, k, a.J, cs);
  // ---- rhs_n = scaling_n ((I + dT A) F_n - prev_n) into the tile ---------------
  {
    double left[R], right[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int j = 0; j < MR; ++j) x[r][j] = (k * MR + j < nx) ? x[r][j] - hg : 0.0;
      left[r] = __shfl_up_sync(KLE_FULL_MASK, x[r][MR - 1], 1, P);
      right[r] = __shfl_down_sync(KLE_FULL_MASK, x[r][0], 1, P);
      if (k == 0) left[r] = 0.0;
      if (k == P - 1) right[r] = 0.0;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int n = slot * R + r;
      const double sc = a.scaling[n];
      const double pmul = (n == 0) ? a.alpha : 1.0;
      const double* prev = a.U + sb + (size_t)(n == 0 ? N - 1 : n - 1) * nx;
      double xl = left[r];
#pragma unroll
      for (int j = 0; j < MR; ++j) {
        const int row = k * MR + j;
        double rhs = 0.0;
        const double xc = x[r][j];
        if (row < nx) {
          const double dj = __ldg(dia + row);
          const double em = row > 0 ? __ldg(off + row - 1) : 0.0;
          const double ep = row + 1 < nx ? __ldg(off + row) : 0.0;
          const double xp = (j < MR - 1) ? x[r][j + 1] : right[r];
          const double Ax = fma(em, xl, fma(dj, xc, ep * xp));
          rhs = sc * (fma(a.dT, Ax, xc) - pmul * __ldg(prev + row));
        }
        xl = xc;
        reinterpret_cast<double*>(&tile[tix(n, row & (HC - 1))])[row >> 6] = rhs;
      }
    }
  }
  wv::syncw();
  wv::fft_warp<-1>(tile, tw, lane);
  // ---- three rounds of 4 frequency groups -------------------------------------
  const double hs = 0.5 / sqrt((double)N);
  const int r0 = k * MR;
#pragma unroll 1
  for (int rho = 0; rho < 3; ++rho) {
    const int fr = rho * 4 + slot;
    const bool valid = fr < NF;
    const int f = valid ? fr : NF - 1;
    const int fm = (N - f) & (N - 1);
    const Cplx* src = reinterpret_cast<const Cplx*>(a.sfac) + ((size_t)s * NF + f) * nx;
    Cplx preg[MR + 1];  // pivots of rows r0 - 1 .. r0 + MR - 1
#pragma unroll
    for (int jj = 0; jj <= MR; ++jj) {
      const int row = r0 + jj - 1;
      preg[jj] = row < 0 ? Cplx{0.0, 0.0} : (row < nx ? src[row] : Cplx{1.0, 0.0});
    }
    Cplx y[MR];
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      const int col = r0 + j;
      const Cplx zf = tile[tix(f, col & (HC - 1))], zm = tile[tix(fm, col & (HC - 1))];
      if (col < HC) y[j] = {(zf.re + zm.re) * hs, (zf.im - zm.im) * hs};
      else y[j] = {(zf.im + zm.im) * hs, (zm.re - zf.re) * hs};
    }
    freq_solve(y, k, offs + r0, [&](int jj) -> Cplx { return preg[jj + 1]; });
    wv::syncw();  // the groups have read their p_f, p_{N-f}
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      const Cplx qb = shfl_xor_c(y[j], CLN / 2);
      if (valid && k < CLN / 2) {
        const int col = r0 + j;
        tile[tix(f, col)] = {y[j].re - qb.im, y[j].im + qb.re};
        if (f > 0 && 2 * f < N) tile[tix(N - f, col)] = {y[j].re + qb.im, qb.re - y[j].im};
      }
    }
    wv::syncw();
  }
  wv::fft_warp<+1>(tile, tw, lane);
  // ---- update: packed columns lane and lane + 32 -------------------------------
  const double rsN = 1.0 / sqrt((double)N);
  double incmax = 0.0;
  bool bad = false;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int c = lane + 32 * h;
    const int ra = c, rb = c + HC;
#pragma unroll 4
    for (int n = 0; n < N; ++n) {
      const Cplx z = tile[tix(n, c)];
      if (ra < nx) {
        const double u = (z.re * rsN) * isc[n];
        const double d = fabs(u - a.U[sb + (size_t)n * nx + ra]);
        incmax = fmax(incmax, d);
        bad |= (d != d);
        a.U[sb + (size_t)n * nx + ra] = u;
      }
      if (rb < nx) {
        const double u = (z.im * rsN) * isc[n];
        const double d = fabs(u - a.U[sb + (size_t)n * nx + rb]);
        incmax = fmax(incmax, d);
        bad |= (d != d);
        a.U[sb + (size_t)n * nx + rb] = u;
      }
    }
  }
  if (__any_sync(KLE_FULL_MASK, bad)) incmax = __longlong_as_double(0x7ff8000000000000LL);
  incmax = warp_max(incmax);
  if (lane == 0) {
    const double inc = incmax;
    if (a.inc_hist) a.inc_hist[(size_t)s * a.max_iters + (a.k - 1)] = inc;
    int st = KLE_SAMPLE_ACTIVE;
    if (inc <= a.tol) st = KLE_SAMPLE_CONVERGED;
    else if (!isfinite(inc)) st = KLE_SAMPLE_NONFINITE;
    else if (a.k >= a.max_iters) st = KLE_SAMPLE_MAXITERS;
    if (st != KLE_SAMPLE_ACTIVE) {
      a.status[s] = st;
      if (a.iters) a.iters[s] = a.k;
    } else if (a.active_count) {
      atomicAdd(a.active_count, 1);
    }
  }
}

static int launch_warp(const IterSmallArgs& a, cudaStream_t st) {
  static PerDeviceOnce attr_once;
  if (int rc = once_per_device(attr_once, "kle_iter_warp: cudaFuncSetAttribute", [&] {
        const cudaError_t e = cudaFuncSetAttribute(iter_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)WarpSmem::BYTES);
        return e != cudaSuccess ? e : cudaFuncSetAttribute(iter_warp_kernel,
                                                           cudaFuncAttributePreferredSharedMemoryCarveout,
                                                           cudaSharedmemCarveoutMaxShared);
      }))
    return rc;
  iter_warp_kernel<<<(unsigned)a.M, 32, WarpSmem::BYTES, st>>>(a);
  return check_launch("iter_warp_kernel");
}

template <int LOGN, bool FUSE>
static int launch(const IterSmallArgs& a, cudaStream_t st) {
  using K = Shape<LOGN, FUSE>;
  static PerDeviceOnce attr_once;
  if (int rc = once_per_device(attr_once, "kle_iter_small: cudaFuncSetAttribute", [&] {
        const cudaError_t e = cudaFuncSetAttribute(iter_small_kernel<LOGN, FUSE>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::BYTES);
        return e != cudaSuccess ? e : cudaFuncSetAttribute(iter_small_kernel<LOGN, FUSE>,
                                                           cudaFuncAttributePreferredSharedMemoryCarveout,
                                                           cudaSharedmemCarveoutMaxShared);
      }))
    return rc;
  iter_small_kernel<LOGN, FUSE><<<(unsigned)a.M, NT, K::BYTES, st>>>(a);
  return check_launch(FUSE ? "iter_small_kernel" : "iter_small_kernel(cgc)");
}

template <bool FUSE>
static int dispatch(const IterSmallArgs& a, cudaStream_t st) {
  if (a.M <= 0) return KLE_OK;
  switch (a.N) {
    case 2: return launch<1, FUSE>(a, st);
    case 4: return launch<2, FUSE>(a, st);
    case 8: return launch<3, FUSE>(a, st);
    case 16: return launch<4, FUSE>(a, st);
  }
  return set_error(KLE_ERR_UNSUPPORTED, "iter_small: N");
}

}  // namespace itsmall

static bool small_shape(int N, int nx) {
  const FineLayoutRT l = fine_layout(nx);
  return nx >= 2 && nx <= itsmall::RB && N >= 2 && N <= 16 && (N & (N - 1)) == 0 && l.MR == itsmall::MR &&
         l.P == itsmall::P && l.kind == 0 && l.W == 0;
}

bool iter_small_supported(int N, int nx) {
  // opt-in: KLE_FUSED=1 / 2 (read per call). Measured at c4 (131k samples, one full solve):
  // one CTA per sample 104 ms, one warp per sample 160 ms, against 96 ms for fgr_kernel
  // (one-warp R = 4 sweeps) + the 2-CTA cluster CGC. The CTA variant sweeps with R = 1 per
  // 8-lane group; the warp variant keeps the sweep's 255 registers allocated through its
  // long, latency-bound single-warp CGC phase, which the other warps do not fill
  const char* env = getenv("KLE_FUSED");  // 1: one CTA per sample; 2: one warp per sample (N = 16)
  return env && (env[0] == '1' || env[0] == '2') && small_shape(N, nx);
}

bool cgc_small_supported(int N, int nx) {
  // opt-in: KLE_CGC_SMALL=1 (read per call). Measured at c4 (131k samples): 4.03 ms per launch
  // against 3.55 ms for the 2-CTA cluster kernel, whose per-sample row parallelism is twice as
  // high (8 rows per lane instead of 16) at the same number of samples in flight per SM
  const char* env = getenv("KLE_CGC_SMALL");
  return env && env[0] == '1' && small_shape(N, nx);
}

int iter_small_run(const IterSmallArgs& a, cudaStream_t st) {
  const char* env = getenv("KLE_FUSED");
  if (env && env[0] == '2' && a.N == 16) return a.M > 0 ? itsmall::launch_warp(a, st) : KLE_OK;
  return itsmall::dispatch<true>(a, st);
}
int cgc_small_run(const IterSmallArgs& a, cudaStream_t st) { return itsmall::dispatch<false>(a, st); }

}  // namespace kle
