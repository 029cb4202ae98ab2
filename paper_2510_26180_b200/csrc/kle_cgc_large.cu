// Diagonalised CGC for large blocks (config 5: N = 1024 time slices of
// nx = 4095 rows per sample), where one sample's N x nx block no longer fits
// a thread-block cluster. Three streaming kernels per outer iteration:
//
//   cgcl_fwd_kernel    p = F*(R) / sqrt(N) along time (pintuq/pcgc.py:85-87,
//                      np.fft.fft norm="ortho"), R already alpha-scaled by the
//                      fused fine kernel. CTA = (sample, 8 spatial columns):
//                      the columns are packed two-for-one into 4 complex
//                      columns, a four-step FFT N = N1 x N2 runs in shared
//                      memory with the N1-/N2-point DFTs in registers (two
//                      passes, one barrier each), and the half spectrum
//                      f = 0..N/2 of every real column is written to
//                      P[s][i][f] (f fastest: coalesced for the solves).
//   cgcl_solve_kernel  q_f = (lambda_f I + dT A)^{-1} p_f (pcgc.py:112-135,
//                      factor_shifted banded branch + three_step_solve step
//                      (b)), one thread per (sample, frequency): the pivots
//                      of the pivot-free complex LDL^T are formed on the fly
//                      (Re lambda_f > 0, A an M-matrix), y overwrites p, the
//                      pivots go to a scratch array, the back substitution
//                      overwrites y with q. Rows are prefetched ahead of the
//                      dependent recurrence; lanes = consecutive f, so every
//                      load and store is a coalesced 512-byte row segment.
//   cgcl_inv_kernel    Hermitian completion (q_{N-f} = conj q_f), inverse
//                      four-step FFT, u = Re / sqrt(N) / scaling (pcgc.py:
//                      79-82, 170-172), U update, increment max |U_new - U|
//                      (pcgc.py:335) into a per-sample slot; cgcl_status_kernel
//                      then applies the stop test (pcgc.py:345-348).
//
// HBM per (n, i) and iteration: R 8 + U 8 read, U 8 written; per (f, i):
// p written once and read twice, y/q written twice, pivots written and read
// once (96 B per (f, i), f <= N/2, i.e. ~48 B per (n, i)).
#include <cmath>
#include <cstdlib>

#include "kle_common.cuh"
#include "kle_internal.h"

namespace kle {

namespace {

#ifndef KLE_CGCL_CP
#define KLE_CGCL_CP 4
#endif
constexpr int CL_CP = KLE_CGCL_CP;  // complex columns per FFT tile (2 CP real columns)
constexpr int CL_RC = 2 * CL_CP;

__device__ __forceinline__ Cplx ca(Cplx a, Cplx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ Cplx cs(Cplx a, Cplx b) { return {a.re - b.re, a.im - b.im}; }

template <int LOGN>
struct LShape {
  static constexpr int N = 1 << LOGN;
  static constexpr int LOG_N1 = (LOGN + 1) / 2;
  static constexpr int N1 = 1 << LOG_N1, N2 = N / N1;
  static constexpr int NF = N / 2 + 1;
  static constexpr int NT = (N1 > N2 ? N1 : N2) * CL_CP;
  // tile [N][CP] complex, padded by CP complex every N1 rows (pass-2 reads of
  // rows n1 + N1 k2 by threads with different k2 then fall on distinct banks)
  static constexpr int ROWS_PAD = CL_CP;
  static constexpr int TILE = N * CL_CP + (N / N1) * ROWS_PAD;
  __device__ __forceinline__ static int idx(int n, int j) { return n * CL_CP + j + (n >> LOG_N1) * ROWS_PAD; }
};

// in-register DFT of NS points (NS <= 32, power of two), natural order in and
// out; twiddles W_NS^k = tw[k * (N / NS)] with tw[j] = exp(-2 pi i j / N).
// S = -1: forward (np.fft.fft sign), S = +1: inverse (unnormalised).
template <int NS>
__device__ __forceinline__ constexpr int rbits(int v) {
  int r = 0;
  for (int b = 1; b < NS; b <<= 1) {
    r = (r << 1) | (v & 1);
    v >>= 1;
  }
  return r;
}

template <int NS, int S, int N>
__device__ __forceinline__ void reg_dft(Cplx (&v)[NS], const Cplx* __restrict__ tw) {
  // radix-2 decimation in frequency, in place: on return v[k] = X[rbits(k)]
#pragma unroll
  for (int len = NS; len >= 2; len >>= 1) {
    const int half = len >> 1;
#pragma unroll
    for (int g = 0; g < NS; g += len) {
#pragma unroll
      for (int j = 0; j < half; ++j) {
        const Cplx a = v[g + j], b = v[g + j + half];
        Cplx d = cs(a, b);
        v[g + j] = ca(a, b);
        if (j != 0) {
          if (4 * j == len) {  // W_len^{len/4} = -i (forward) / +i (inverse)
            d = S < 0 ? Cplx{d.im, -d.re} : Cplx{-d.im, d.re};
          } else {
            Cplx w = {__ldg(&tw[j * (N / len)].re), __ldg(&tw[j * (N / len)].im)};
            if (S > 0) w.im = -w.im;
            d = cmul(d, w);
          }
        }
        v[g + j + half] = d;
      }
    }
  }
}

// four-step FFT over the CP columns of a tile (natural order in and out)
template <int LOGN, int S>
__device__ __forceinline__ void tile_fft(Cplx* t, const Cplx* __restrict__ tw) {
  using K = LShape<LOGN>;
  constexpr int N = K::N, N1 = K::N1, N2 = K::N2;
  const int tid = threadIdx.x;
  // pass 1: task (n1, j): N2-point DFT over x[n1 + N1 n2], twiddle W_N^{n1 k2}
  if (tid < N1 * CL_CP) {
    const int j = tid % CL_CP, n1 = tid / CL_CP;
    Cplx v[N2];
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) v[n2] = t[K::idx(n1 + N1 * n2, j)];
    reg_dft<N2, S, N>(v, tw);  // v[q] = Y[rbits(q)]
#pragma unroll
    for (int q = 0; q < N2; ++q) {
      const int k2 = rbits<N2>(q);
      if (k2 != 0) {
        Cplx w = {__ldg(&tw[n1 * k2].re), __ldg(&tw[n1 * k2].im)};
        if (S > 0) w.im = -w.im;
        v[q] = cmul(v[q], w);
      }
      t[K::idx(n1 + N1 * k2, j)] = v[q];
    }
  }
  __syncthreads();
  // pass 2: task (k2, j): N1-point DFT over y[n1 + N1 k2] -> X[k2 + N2 k1]
  Cplx w[N1];
  const bool act = tid < N2 * CL_CP;
  const int j = tid % CL_CP, k2 = tid / CL_CP;
  if (act) {
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) w[n1] = t[K::idx(n1 + N1 * k2, j)];
    reg_dft<N1, S, N>(w, tw);
  }
  __syncthreads();
  if (act) {
#pragma unroll
    for (int q = 0; q < N1; ++q) t[K::idx(k2 + N2 * rbits<N1>(q), j)] = w[q];
  }
  __syncthreads();
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}

}  // namespace

// ---------------------------------------------------------------------------
template <int LOGN>
__global__ void __launch_bounds__(LShape<LOGN>::NT) cgcl_fwd_kernel(CgcArgs a, int m0, const Cplx* __restrict__ tw,
                                                                   Cplx* __restrict__ P) {
  using K = LShape<LOGN>;
  constexpr int N = K::N, NF = K::NF, NT = K::NT;
  const int s = m0 + blockIdx.y, sl = blockIdx.y;
  if (a.status && a.status[s] != KLE_SAMPLE_ACTIVE) return;
  extern __shared__ __align__(16) Cplx t[];
  const int nx = a.nx, c0 = blockIdx.x * CL_RC;
  const size_t sb = (size_t)s * N * nx;
  for (int e = threadIdx.x; e < N * CL_RC; e += NT) {
    const int n = e / CL_RC, col = e % CL_RC;
    double* dst = reinterpret_cast<double*>(&t[K::idx(n, col >> 1)]) + (col & 1);
    if (c0 + col < nx) cp_async8(dst, a.R + sb + (size_t)n * nx + c0 + col);
    else *dst = 0.0;
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
  __syncthreads();
  if (a.load_scale) {  // stand-alone three-step: r is not alpha-scaled yet
    for (int e = threadIdx.x; e < N * CL_CP; e += NT) {
      const int n = e / CL_CP, j = e % CL_CP;
      Cplx& z = t[K::idx(n, j)];
      z.re *= a.load_scale[n];
      z.im *= a.load_scale[n];
    }
    __syncthreads();
  }
  tile_fft<LOGN, -1>(t, tw);
  // two-for-one unpacking x 1/sqrt(N): column 2j <- (Z_f + conj Z_-f)/2,
  // column 2j+1 <- (Z_f - conj Z_-f)/(2i)
  const double hs = 0.5 / sqrt((double)N);
  Cplx* out = P + (size_t)sl * nx * NF;
  for (int e = threadIdx.x; e < CL_RC * NF; e += NT) {  // column fastest: conflict-free tile reads
    const int f = e / CL_RC, col = e % CL_RC;
    if (c0 + col >= nx) continue;
    const int j = col >> 1;
    const Cplx zf = t[K::idx(f, j)], zm = t[K::idx((N - f) & (N - 1), j)];
    Cplx y;
    if ((col & 1) == 0) y = {(zf.re + zm.re) * hs, (zf.im - zm.im) * hs};
    else y = {(zf.im + zm.im) * hs, (zm.re - zf.re) * hs};
    out[(size_t)(c0 + col) * NF + f] = y;
  }
}

// one thread per (sample, frequency); P, IB: [MB][nx][NF] complex
__global__ void __launch_bounds__(128) cgcl_solve_kernel(CgcArgs a, int m0, int MB, int NF, Cplx* __restrict__ P,
                                                         Cplx* __restrict__ IB) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)MB * NF) return;
  const int sl = (int)(t / NF), f = (int)(t - (long long)sl * NF), s = m0 + sl;
  if (a.status && a.status[s] != KLE_SAMPLE_ACTIVE) return;
  const int nx = a.nx;
  const double* __restrict__ dd = a.dia + (size_t)s * nx;
  const double* __restrict__ ee = a.off + (size_t)s * nx;
  Cplx* __restrict__ p = P + (size_t)sl * nx * NF + f;
  Cplx* __restrict__ ib = IB + (size_t)sl * nx * NF + f;
  const Cplx lam = {a.lam[2 * f], a.lam[2 * f + 1]};
  const double dT = a.dT;
  // forward: LDL^T pivots on the fly, y_i = p_i - l_i y_{i-1}
  constexpr int PF = 8;  // rows in flight ahead of the recurrence
  Cplx ring[PF];
#pragma unroll
  for (int q = 0; q < PF; ++q) ring[q] = q < nx ? p[(size_t)q * NF] : Cplx{0.0, 0.0};
  Cplx y = {0.0, 0.0}, ibp = {0.0, 0.0};
  for (int i0 = 0; i0 < nx; i0 += PF) {
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const int i = i0 + q;
      if (i < nx) {
        const Cplx pi = ring[q];
        if (i + PF < nx) ring[q] = p[(size_t)(i + PF) * NF];
        const Cplx D = {fma(dT, __ldg(dd + i), lam.re), lam.im};
        Cplx beta = D;
        if (i > 0) {
          const double E = dT * __ldg(ee + i - 1);
          const Cplx l = {E * ibp.re, E * ibp.im};
          beta = {fma(-l.re, E, D.re), fma(-l.im, E, D.im)};
          y = cs(pi, cmul(l, y));
        } else {
          y = pi;
        }
        ibp = crcp(beta);
        p[(size_t)i * NF] = y;
        ib[(size_t)i * NF] = ibp;
      }
    }
  }
  // backward: q_i = y_i / beta_i - l_{i+1} q_{i+1}
  Cplx ry[PF], rb[PF];
#pragma unroll
  for (int q = 0; q < PF; ++q) {
    const int i = nx - 1 - q;
    ry[q] = i >= 0 ? p[(size_t)i * NF] : Cplx{0.0, 0.0};
    rb[q] = i >= 0 ? ib[(size_t)i * NF] : Cplx{0.0, 0.0};
  }
  Cplx x = {0.0, 0.0};
  for (int r0 = 0; r0 < nx; r0 += PF) {
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const int i = nx - 1 - (r0 + q);
      if (i >= 0) {
        const Cplx yy = ry[q], bi = rb[q];
        if (i - PF >= 0) {
          ry[q] = p[(size_t)(i - PF) * NF];
          rb[q] = ib[(size_t)(i - PF) * NF];
        }
        const Cplx z = cmul(yy, bi);
        if (i < nx - 1) {
          const double E = dT * __ldg(ee + i);
          const Cplx ln = {E * bi.re, E * bi.im};
          x = cs(z, cmul(ln, x));
        } else {
          x = z;
        }
        p[(size_t)i * NF] = x;
      }
    }
  }
}

template <int LOGN>
__global__ void __launch_bounds__(LShape<LOGN>::NT) cgcl_inv_kernel(CgcArgs a, int m0, const Cplx* __restrict__ tw,
                                                                   const Cplx* __restrict__ Q,
                                                                   unsigned long long* __restrict__ inc_bits) {
  using K = LShape<LOGN>;
  constexpr int N = K::N, NF = K::NF, NT = K::NT;
  const int s = m0 + blockIdx.y, sl = blockIdx.y;
  if (a.status && a.status[s] != KLE_SAMPLE_ACTIVE) return;
  extern __shared__ __align__(16) Cplx t[];
  const int nx = a.nx, c0 = blockIdx.x * CL_RC;
  const Cplx* q = Q + (size_t)sl * nx * NF;
  // packed Hermitian spectra W_f = q_a(f) + i q_b(f), W_{N-f} = conj q_a + i conj q_b;
  // tasks j fastest (conflict-free tile writes), loads staged in batches of QB
  constexpr int QB = 4;
  for (int e0 = threadIdx.x; e0 < CL_CP * NF; e0 += QB * NT) {
    Cplx qa[QB], qb[QB];
#pragma unroll
    for (int r = 0; r < QB; ++r) {
      const int e = e0 + r * NT, f = e / CL_CP, j = e % CL_CP;
      const int ia = c0 + 2 * j;
      const bool ok = e < CL_CP * NF;
      qa[r] = (ok && ia < nx) ? q[(size_t)ia * NF + f] : Cplx{0.0, 0.0};
      qb[r] = (ok && ia + 1 < nx) ? q[(size_t)(ia + 1) * NF + f] : Cplx{0.0, 0.0};
    }
#pragma unroll
    for (int r = 0; r < QB; ++r) {
      const int e = e0 + r * NT, f = e / CL_CP, j = e % CL_CP;
      if (e >= CL_CP * NF) break;
      t[K::idx(f, j)] = {qa[r].re - qb[r].im, qa[r].im + qb[r].re};
      if (f > 0 && 2 * f < N) t[K::idx(N - f, j)] = {qa[r].re + qb[r].im, qb[r].re - qa[r].im};
    }
  }
  __syncthreads();
  tile_fft<LOGN, +1>(t, tw);
  const double rsN = 1.0 / sqrt((double)N);
  const size_t sb = (size_t)s * N * nx;
  double* __restrict__ out = a.Uout ? a.Uout : a.U;
  const bool track = a.U != nullptr && inc_bits != nullptr;
  double incmax = 0.0;
  bool bad = false;
  // old U staged in batches of UB registers: the loads of a batch are issued
  // before its stores (out may alias U)
  constexpr int UB = 16;
  static_assert((N * CL_RC) % NT == 0, "update tasks");
  for (int e0 = threadIdx.x; e0 < N * CL_RC; e0 += UB * NT) {
    double old[UB];
#pragma unroll
    for (int r = 0; r < UB; ++r) {
      const int e = e0 + r * NT, n = e / CL_RC, col = e % CL_RC;
      old[r] = (track && e < N * CL_RC && c0 + col < nx) ? a.U[sb + (size_t)n * nx + c0 + col] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < UB; ++r) {
      const int e = e0 + r * NT, n = e / CL_RC, col = e % CL_RC;
      if (e >= N * CL_RC || c0 + col >= nx) continue;
      const Cplx z = t[K::idx(n, col >> 1)];
      const double u = (((col & 1) ? z.im : z.re) * rsN) * __ldg(a.inv_scaling + n);
      if (track) {
        const double d = fabs(u - old[r]);
        incmax = fmax(incmax, d);
        bad |= (d != d);
      }
      out[sb + (size_t)n * nx + c0 + col] = u;
    }
  }
  if (!track) return;
  if (__syncthreads_or(bad)) incmax = __longlong_as_double(0x7ff8000000000000LL);
  incmax = warp_max(incmax);
  if ((threadIdx.x & 31) == 0) atomicMax(inc_bits + s, (unsigned long long)__double_as_longlong(incmax));
}

// per-sample stop test after the update (pintuq/pcgc.py:335-348)
__global__ void cgcl_status_kernel(CgcArgs a, unsigned long long* __restrict__ inc_bits) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.M) return;
  if (a.status && a.status[s] != KLE_SAMPLE_ACTIVE) return;
  const double inc = __longlong_as_double((long long)inc_bits[s]);
  inc_bits[s] = 0ULL;
  if (a.inc) a.inc[s] = inc;
  if (a.inc_hist) a.inc_hist[(size_t)s * a.max_iters + (a.k - 1)] = inc;
  if (!a.status) return;
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

// ---------------------------------------------------------------------------
// Streaming variant (N >= 256): one CTA per sample walks the rows in blocks of
// RB = 16 (8 packed complex columns). Forward kernel: per block, the R rows are
// loaded, the four-step FFT runs over the block's columns, and thread f (one
// per frequency f <= N/2) unpacks p_f of the block's rows and advances the
// forward LDL^T recurrence (pivots on the fly), writing y and 1/beta. Backward
// kernel: blocks in reverse, thread f runs the back substitution over the
// block's rows, the packed Hermitian spectra go into the tile, the inverse FFT
// runs, and the block's U rows are updated. The spectrum never round-trips
// through HBM between the FFTs and the solves: per (n, i) and iteration
// R 8 + U 8 read, U 8 written, y and 1/beta written and read once (32 B):
// 56 B against 88 B for the three-kernel path above. Same operations in the
// same order per element as the three-kernel path (bitwise equal results).
// Opt-in (KLE_CGCL_STREAM=1): measured 33.8 ms per 256-sample c5 launch against
// 31.6 ms for the three kernels — one 135 KB-tile CTA per SM walks 256 row
// blocks with load, FFT and recurrence phases serialised, so it is latency-
// bound at 1.8 TB/s of (smaller) traffic where the three kernels reach 2.8.
namespace {
template <int LOGN>
struct SShape {
  static constexpr int N = 1 << LOGN, NF = N / 2 + 1;
  static constexpr int LOG_N1 = (LOGN + 1) / 2;
  static constexpr int N1 = 1 << LOG_N1, N2 = N / N1;
#ifndef KLE_CGCS_CP
#define KLE_CGCS_CP 8  // 4: 68 KB tiles, 3 CTAs/SM, measured slower (36.3 vs 33.8 ms per 256-sample launch)
#endif
  static constexpr int CP = KLE_CGCS_CP, RB = 2 * CP;  // complex columns / real rows per block
  static constexpr int FT = (N1 > N2 ? N1 : N2) * CP;
  static constexpr int FPT = 2;                      // frequencies per thread (two independent recurrences)
  static constexpr int NS = ((NF + FPT - 1) / FPT + 31) / 32 * 32;
  static constexpr int NT = NS > FT ? NS : FT;
  // tile [CP][N] complex, n fastest, padded one slot per 32 (pass-2 strides) and
  // one extra slot per column (column starts fall on distinct banks)
  static constexpr int LD = N + N / 32 + 1;
  static constexpr int TILE = CP * LD;
  __device__ __forceinline__ static int idx(int n, int j) { return j * LD + n + (n >> 5); }
};

template <int LOGN, int S>
__device__ __forceinline__ void stile_fft(Cplx* t, const Cplx* __restrict__ tw) {
  using K = SShape<LOGN>;
  constexpr int N = K::N, N1 = K::N1, N2 = K::N2, CP = K::CP;
  const int tid = threadIdx.x;
  if (tid < N1 * CP) {  // pass 1: task (n1, j), n1 fastest
    const int n1 = tid % N1, j = tid / N1;
    Cplx v[N2];
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) v[n2] = t[K::idx(n1 + N1 * n2, j)];
    reg_dft<N2, S, N>(v, tw);
#pragma unroll
    for (int q = 0; q < N2; ++q) {
      const int k2 = rbits<N2>(q);
      if (k2 != 0) {
        Cplx w = {__ldg(&tw[n1 * k2].re), __ldg(&tw[n1 * k2].im)};
        if (S > 0) w.im = -w.im;
        v[q] = cmul(v[q], w);
      }
      t[K::idx(n1 + N1 * k2, j)] = v[q];
    }
  }
  __syncthreads();
  Cplx w[N1];
  const bool act = tid < N2 * CP;
  const int k2 = tid % N2, j = tid / N2;  // pass 2: task (k2, j), k2 fastest
  if (act) {
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) w[n1] = t[K::idx(n1 + N1 * k2, j)];
    reg_dft<N1, S, N>(w, tw);
  }
  __syncthreads();
  if (act) {
#pragma unroll
    for (int q = 0; q < N1; ++q) t[K::idx(k2 + N2 * rbits<N1>(q), j)] = w[q];
  }
  __syncthreads();
}
}  // namespace

template <int LOGN>
__global__ void __launch_bounds__(SShape<LOGN>::NT) cgcs_fwd_kernel(CgcArgs a, int m0, const Cplx* __restrict__ tw,
                                                                      Cplx* __restrict__ Y, Cplx* __restrict__ IB) {
  using K = SShape<LOGN>;
  constexpr int N = K::N, NF = K::NF, NT = K::NT, CP = K::CP, RB = K::RB;
  const int s = m0 + blockIdx.x, sl = blockIdx.x;
  if (a.status && a.status[s] != KLE_SAMPLE_ACTIVE) return;
  extern __shared__ __align__(16) Cplx t[];
  const int nx = a.nx, tid = threadIdx.x;
  const size_t sb = (size_t)s * N * nx;
  constexpr int FPT = K::FPT;
  int fr[FPT];
  bool ok[FPT];
  Cplx lam[FPT], y[FPT], ibp[FPT];
  Cplx* yo[FPT];
  Cplx* ibo[FPT];
#pragma unroll
  for (int q = 0; q < FPT; ++q) {
    fr[q] = tid + q * NT;
    ok[q] = fr[q] < NF;
    const int fq = ok[q] ? fr[q] : 0;
    lam[q] = {a.lam[2 * fq], a.lam[2 * fq + 1]};
    y[q] = {0.0, 0.0};
    ibp[q] = {0.0, 0.0};
    yo[q] = Y + (size_t)sl * nx * NF + fq;
    ibo[q] = IB + (size_t)sl * nx * NF + fq;
  }
  const double dT = a.dT;
  const double* __restrict__ dd = a.dia + (size_t)s * nx;
  const double* __restrict__ ee = a.off + (size_t)s * nx;
  const double hs = 0.5 / sqrt((double)N);
  for (int c0 = 0; c0 < nx; c0 += RB) {
    __syncthreads();  // the previous block's unpack has read the tile
    for (int e = tid; e < N * RB; e += NT) {  // rows fastest: coalesced 128-byte row segments, all in flight
      const int n = e / RB, col = e % RB;
      double* dst = reinterpret_cast<double*>(&t[K::idx(n, col >> 1)]) + (col & 1);
      if (c0 + col < nx) cp_async8(dst, a.R + sb + (size_t)n * nx + c0 + col);
      else *dst = 0.0;
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
    __syncthreads();
    if (a.load_scale) {  // stand-alone three-step: r is not alpha-scaled yet
      for (int e = tid; e < N * RB; e += NT) {
        const int n = e / RB, col = e % RB;
        reinterpret_cast<double*>(&t[K::idx(n, col >> 1)])[col & 1] *= a.load_scale[n];
      }
      __syncthreads();
    }
    stile_fft<LOGN, -1>(t, tw);
#pragma unroll 2
    for (int col = 0; col < RB; ++col) {
      const int i = c0 + col;
      if (i >= nx) break;
      const int j = col >> 1;
      const double E = i > 0 ? dT * __ldg(ee + i - 1) : 0.0;
#pragma unroll
      for (int q = 0; q < FPT; ++q) {
        if (!ok[q]) continue;
        const int f = fr[q], fm = (N - f) & (N - 1);
        const Cplx zf = t[K::idx(f, j)], zm = t[K::idx(fm, j)];
        Cplx pi;
        if ((col & 1) == 0) pi = {(zf.re + zm.re) * hs, (zf.im - zm.im) * hs};
        else pi = {(zf.im + zm.im) * hs, (zm.re - zf.re) * hs};
        const Cplx D = {fma(dT, __ldg(dd + i), lam[q].re), lam[q].im};
        Cplx beta = D;
        if (i > 0) {
          const Cplx l = {E * ibp[q].re, E * ibp[q].im};
          beta = {fma(-l.re, E, D.re), fma(-l.im, E, D.im)};
          y[q] = cs(pi, cmul(l, y[q]));
        } else {
          y[q] = pi;
        }
        ibp[q] = crcp(beta);
        yo[q][(size_t)i * NF] = y[q];
        ibo[q][(size_t)i * NF] = ibp[q];
      }
    }
  }
}

template <int LOGN>
__global__ void __launch_bounds__(SShape<LOGN>::NT) cgcs_bwd_kernel(CgcArgs a, int m0, const Cplx* __restrict__ tw,
                                                                      const Cplx* __restrict__ Y,
                                                                      const Cplx* __restrict__ IB,
                                                                      unsigned long long* __restrict__ inc_bits) {
  using K = SShape<LOGN>;
  constexpr int N = K::N, NF = K::NF, NT = K::NT, CP = K::CP, RB = K::RB;
  const int s = m0 + blockIdx.x, sl = blockIdx.x;
  if (a.status && a.status[s] != KLE_SAMPLE_ACTIVE) return;
  extern __shared__ __align__(16) Cplx t[];
  const int nx = a.nx, tid = threadIdx.x;
  const size_t sb = (size_t)s * N * nx;
  constexpr int FPT = K::FPT;
  int fr[FPT];
  bool ok[FPT];
  const Cplx* yi[FPT];
  const Cplx* ibi[FPT];
#pragma unroll
  for (int q = 0; q < FPT; ++q) {
    fr[q] = tid + q * NT;
    ok[q] = fr[q] < NF;
    const int fq = ok[q] ? fr[q] : 0;
    yi[q] = Y + (size_t)sl * nx * NF + fq;
    ibi[q] = IB + (size_t)sl * nx * NF + fq;
  }
  const double dT = a.dT;
  const double* __restrict__ ee = a.off + (size_t)s * nx;
  const double rsN = 1.0 / sqrt((double)N);
  double* __restrict__ out = a.Uout ? a.Uout : a.U;
  const bool track = a.U != nullptr && inc_bits != nullptr;
  double incmax = 0.0;
  bool bad = false;
  Cplx x[FPT];
#pragma unroll
  for (int q = 0; q < FPT; ++q) x[q] = {0.0, 0.0};
  const int nb = (nx + RB - 1) / RB;
  for (int b = nb - 1; b >= 0; --b) {
    const int c0 = b * RB;
    __syncthreads();  // the previous block's update has read the tile
    // back substitution q_i = y_i / beta_i - l_{i+1} q_{i+1} over the block's rows, descending, the
    // loads of a half-block issued together; each finished row pair (2j, 2j+1) is packed into the
    // tile as W_f = q_2j + i q_2j+1 (and the mirror W_{N-f})
#pragma unroll
    for (int h = 1; h >= 0; --h) {
      Cplx yy[FPT][CP], bb[FPT][CP];
#pragma unroll
      for (int q = 0; q < FPT; ++q)
#pragma unroll
        for (int u = 0; u < CP; ++u) {
          const int i = c0 + h * CP + u;
          const bool in = ok[q] && i < nx;
          yy[q][u] = in ? yi[q][(size_t)i * NF] : Cplx{0.0, 0.0};
          bb[q][u] = in ? ibi[q][(size_t)i * NF] : Cplx{0.0, 0.0};
        }
      Cplx hi[FPT];
#pragma unroll
      for (int u = CP - 1; u >= 0; --u) {
        const int i = c0 + h * CP + u;
        const double E = (i < nx - 1) ? dT * __ldg(ee + i) : 0.0;
#pragma unroll
        for (int q = 0; q < FPT; ++q) {
          Cplx qi = {0.0, 0.0};
          if (i < nx) {
            const Cplx z = cmul(yy[q][u], bb[q][u]);
            if (i < nx - 1) {
              const Cplx ln = {E * bb[q][u].re, E * bb[q][u].im};
              x[q] = cs(z, cmul(ln, x[q]));
            } else {
              x[q] = z;
            }
            qi = x[q];
          }
          if (u & 1) {
            hi[q] = qi;  // row 2j+1 of the pair
          } else if (ok[q]) {
            const int f = fr[q], j = (h * CP + u) >> 1;
            const Cplx qa = qi, qb = hi[q];
            t[K::idx(f, j)] = {qa.re - qb.im, qa.im + qb.re};
            if (f > 0 && 2 * f < N) t[K::idx(N - f, j)] = {qa.re + qb.im, qb.re - qa.im};
          }
        }
      }
    }
    __syncthreads();
    stile_fft<LOGN, +1>(t, tw);
    // the old values staged in batches of UB registers: a batch's loads are in flight together and
    // precede its stores (out may alias U)
    constexpr int UB = 16;
    for (int e0 = tid; e0 < N * RB; e0 += UB * NT) {
      double old[UB];
#pragma unroll
      for (int r = 0; r < UB; ++r) {
        const int e = e0 + r * NT, n = e / RB, col = e % RB;
        old[r] = (track && e < N * RB && c0 + col < nx) ? a.U[sb + (size_t)n * nx + c0 + col] : 0.0;
      }
#pragma unroll
      for (int r = 0; r < UB; ++r) {
        const int e = e0 + r * NT, n = e / RB, col = e % RB;
        if (e >= N * RB || c0 + col >= nx) continue;
        const Cplx z = t[K::idx(n, col >> 1)];
        const double u = (((col & 1) ? z.im : z.re) * rsN) * __ldg(a.inv_scaling + n);
        if (track) {
          const double d = fabs(u - old[r]);
          incmax = fmax(incmax, d);
          bad |= (d != d);
        }
        out[sb + (size_t)n * nx + c0 + col] = u;
      }
    }
  }
  if (!track) return;
  if (__syncthreads_or(bad)) incmax = __longlong_as_double(0x7ff8000000000000LL);
  incmax = warp_max(incmax);
  if ((threadIdx.x & 31) == 0) atomicMax(inc_bits + s, (unsigned long long)__double_as_longlong(incmax));
}

__global__ void cgcl_twiddle_kernel(Cplx* tw, int N) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  double sn, c;
  sincospi(-2.0 * (double)j / (double)N, &sn, &c);
  tw[j] = {c, sn};
}

// ---------------------------------------------------------------------------
static int log2_exact(int N) {
  if (N < 2 || (N & (N - 1))) return -1;
  int l = 0;
  while ((1 << l) < N) ++l;
  return l;
}

bool cgc_large_supported(int N, int nx) {
  const int l = log2_exact(N);
  return l >= 2 && l <= 10 && nx >= 1;
}

static int batch_of(int M) { return M < 256 ? M : 256; }

size_t cgc_large_scratch_bytes(int M, int N, int nx) {
  const size_t NF = (size_t)N / 2 + 1;
  const size_t MB = (size_t)batch_of(M);
  return 2 * MB * nx * NF * sizeof(Cplx) + (size_t)M * sizeof(unsigned long long) + (size_t)N * sizeof(Cplx) + 1024;
}

template <int LOGN>
static int run_large(const CgcArgs& a, cudaStream_t st) {
  using K = LShape<LOGN>;
  constexpr int N = K::N, NF = K::NF;
  const int MB = batch_of(a.M);
  char* ws = reinterpret_cast<char*>(a.scratch);
  Cplx* P = reinterpret_cast<Cplx*>(ws);
  Cplx* IB = P + (size_t)MB * a.nx * NF;
  unsigned long long* bits = reinterpret_cast<unsigned long long*>(IB + (size_t)MB * a.nx * NF);
  Cplx* tw = reinterpret_cast<Cplx*>(bits + a.M);
  cudaMemsetAsync(bits, 0, sizeof(unsigned long long) * a.M, st);
  cgcl_twiddle_kernel<<<(N + 127) / 128, 128, 0, st>>>(tw, N);
  const int tiles = (a.nx + CL_RC - 1) / CL_RC;
  constexpr size_t smem = sizeof(Cplx) * K::TILE;
  static PerDeviceOnce attr_once;
  if (int rc = once_per_device(attr_once, "kle_cgc_large: cudaFuncSetAttribute", [&] {
        const cudaError_t e = cudaFuncSetAttribute(cgcl_fwd_kernel<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        return e != cudaSuccess ? e : cudaFuncSetAttribute(cgcl_inv_kernel<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      }))
    return rc;
  // two sub-batch streams over the two halves of the scratch: one half's FFT
  // kernels overlap the other half's per-frequency solves
  static const char* env = getenv("KLE_CGCL_STREAMS");
  const bool two = !(env && env[0] == '1') && MB >= 2;
  AuxResources* res = two ? aux_resources() : nullptr;
  if (two && !res) return KLE_ERR_CUDA;
  cudaStream_t* ss = two ? res->cgcl : nullptr;
  cudaEvent_t* ev = two ? res->cgcl_ev : nullptr;
  const int HB = two ? MB / 2 : MB;  // samples per sub-batch
  if (two) {
    cudaEventRecord(ev[2], st);
    for (int q = 0; q < 2; ++q) cudaStreamWaitEvent(ss[q], ev[2], 0);
  }
  static const char* senv = getenv("KLE_CGCL_STREAM");  // 1: the streaming kernels (A/B)
  if constexpr (LOGN >= 8) {
    if (senv && senv[0] == '1') {
      using S = SShape<LOGN>;
      constexpr size_t ssm = sizeof(Cplx) * S::TILE;
      static PerDeviceOnce sattr;
      if (int rc = once_per_device(sattr, "kle_cgc_stream: cudaFuncSetAttribute", [&] {
            const cudaError_t e = cudaFuncSetAttribute(cgcs_fwd_kernel<LOGN>,
                                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
            return e != cudaSuccess ? e : cudaFuncSetAttribute(cgcs_bwd_kernel<LOGN>,
                                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
          }))
        return rc;
      for (int m0 = 0; m0 < a.M; m0 += MB) {
        const int mb = a.M - m0 < MB ? a.M - m0 : MB;
        cgcs_fwd_kernel<LOGN><<<(unsigned)mb, S::NT, ssm, st>>>(a, m0, tw, P, IB);
        cgcs_bwd_kernel<LOGN><<<(unsigned)mb, S::NT, ssm, st>>>(a, m0, tw, P, IB, a.U ? bits : nullptr);
      }
      if (a.U) cgcl_status_kernel<<<(a.M + 127) / 128, 128, 0, st>>>(a, bits);
      return check_launch("cgc_stream");
    }
  }
  int j = 0;
  for (int m0 = 0; m0 < a.M; m0 += HB, ++j) {
    const int mb = a.M - m0 < HB ? a.M - m0 : HB;
    const int h = two ? (j & 1) : 0;
    cudaStream_t sq = two ? ss[h] : st;
    Cplx* Ph = P + (size_t)h * HB * a.nx * NF;
    Cplx* IBh = IB + (size_t)h * HB * a.nx * NF;
    cgcl_fwd_kernel<LOGN><<<dim3(tiles, mb), K::NT, smem, sq>>>(a, m0, tw, Ph);
    const long long nth = (long long)mb * NF;
    cgcl_solve_kernel<<<(unsigned)((nth + 127) / 128), 128, 0, sq>>>(a, m0, mb, NF, Ph, IBh);
    cgcl_inv_kernel<LOGN><<<dim3(tiles, mb), K::NT, smem, sq>>>(a, m0, tw, Ph, a.U ? bits : nullptr);
  }
  if (two) {
    for (int q = 0; q < 2; ++q) {
      cudaEventRecord(ev[q], ss[q]);
      cudaStreamWaitEvent(st, ev[q], 0);
    }
  }
  if (a.U) cgcl_status_kernel<<<(a.M + 127) / 128, 128, 0, st>>>(a, bits);
  return check_launch("cgc_large");
}

int cgc_large_run(const CgcArgs& a, cudaStream_t st) {
  if (a.imag) cudaMemsetAsync(a.imag, 0, sizeof(double) * a.M, st);  // real by construction
  switch (log2_exact(a.N)) {
    case 2: return run_large<2>(a, st);
    case 3: return run_large<3>(a, st);
    case 4: return run_large<4>(a, st);
    case 5: return run_large<5>(a, st);
    case 6: return run_large<6>(a, st);
    case 7: return run_large<7>(a, st);
    case 8: return run_large<8>(a, st);
    case 9: return run_large<9>(a, st);
    case 10: return run_large<10>(a, st);
  }
  return set_error(KLE_ERR_UNSUPPORTED, "cgc_large: N");
}

}  // namespace kle
