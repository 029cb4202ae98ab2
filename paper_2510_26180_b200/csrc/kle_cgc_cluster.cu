// Cluster-resident diagonalised CGC (three-step solve), one thread-block
// cluster per sample.
//
// Reference: three_step_solve pintuq/pcgc.py:148-172, factor_shifted :90-145,
// the increment / stop test of pcgc_solve :335-348.
//
// The sample's N x nx block is split into CL row blocks of RB = 8*MR rows
// (MR = 8), one CTA each. Per CTA (NT = 8 (N/2+1) threads rounded to warps):
//   0. cp.async prefetch of the R rows, the old U rows (for the increment)
//      and the operator's off-diagonal into shared memory; each thread keeps
//      one column, so the address arithmetic is incremental. The pivots of
//      the thread's frequency are loaded into registers at the same time.
//   1. Two-for-one real FFT along time: rows c and c + RB/2 are packed as
//      z = r_c + i r_{c+RB/2} into an [N][RB/2] complex tile (four-step FFT,
//      natural order; columns XOR-swizzled against bank conflicts).
//      p_f of both rows follows from Z_f, Z_{N-f}.
//   2. All frequencies f = 0..N/2 at once, one 8-lane group each: the group
//      owns the CTA's RB rows (MR per lane, registers) and solves
//      (lambda_f I + dT A) q = p with the LDL^T pivots 1/beta precomputed once
//      per batch (shift_factor_kernel). Chunks are stitched by a 3-stage
//      affine lane scan and across the cluster's CTAs through distributed
//      shared memory: every CTA publishes its block composite; a consumer
//      loads those of the blocks before (after) it in parallel, one per lane,
//      and composes them with a 3-stage lane butterfly. Two cluster barriers
//      per iteration.
//   3. The packed Hermitian spectra W_f = q_c + i q_{c+RB/2} (and the mirror
//      W_{N-f}) are written in natural order, inverse four-step FFT,
//      u = Re / Im parts over scaling; increment vs the prefetched old U;
//      block max-reduction, cluster max through an atomic slot (the last CTA
//      finishes the sample's stop test).
// The two-for-one packing enforces the Hermitian symmetry of the real
// solution, so u is real by construction (imag residue reported as 0).
// HBM traffic per outer iteration and (n, i): R 8 B + U 8 B read, U 8 B
// written, pivots 16 (N/2+1)/N B read.
#include <cooperative_groups.h>
#include <cstdlib>

#include "kle_common.cuh"
#include "kle_internal.h"

namespace cg = cooperative_groups;

namespace kle {

#ifdef KLE_CGC_TIMING
// debug: per-CTA phase timestamps (SM clock cycles), CTAs [KLE_CGC_T0, KLE_CGC_T0 + 4096)
#ifndef KLE_CGC_T0
#define KLE_CGC_T0 100000
#endif
__device__ unsigned long long g_cgc_t[4096][10];
#define CGC_T(i)                                                                                  \
  do {                                                                                            \
    if (threadIdx.x == 0 && blockIdx.x >= KLE_CGC_T0 && blockIdx.x < KLE_CGC_T0 + 4096)           \
      g_cgc_t[blockIdx.x - KLE_CGC_T0][i] = (unsigned long long)clock64();                        \
  } while (0)
#else
#define CGC_T(i) \
  do {           \
  } while (0)
#endif

constexpr int CL_LANES = 8;

__device__ __forceinline__ Cplx cfma(Cplx a, Cplx b, Cplx c) {  // a*b + c
  return {fma(a.re, b.re, fma(-a.im, b.im, c.re)), fma(a.re, b.im, fma(a.im, b.re, c.im))};
}
__device__ __forceinline__ Cplx cneg_mul(Cplx a, Cplx b) {  // -(a*b)
  return {fma(-a.re, b.re, a.im * b.im), fma(-a.re, b.im, -a.im * b.re)};
}
__device__ __forceinline__ Cplx shfl_up_c(Cplx v, int d) {
  return {__shfl_up_sync(KLE_FULL_MASK, v.re, d, CL_LANES), __shfl_up_sync(KLE_FULL_MASK, v.im, d, CL_LANES)};
}
__device__ __forceinline__ Cplx shfl_down_c(Cplx v, int d) {
  return {__shfl_down_sync(KLE_FULL_MASK, v.re, d, CL_LANES), __shfl_down_sync(KLE_FULL_MASK, v.im, d, CL_LANES)};
}
__device__ __forceinline__ Cplx shfl_xor_c(Cplx v, int d) {
  return {__shfl_xor_sync(KLE_FULL_MASK, v.re, d), __shfl_xor_sync(KLE_FULL_MASK, v.im, d)};
}
#ifndef KLE_CGC_UPRE
#define KLE_CGC_UPRE 1  // prefetch the old U columns into the dead pivot space during the inverse FFT
#endif

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
}

// Cluster barrier for distributed-shared-memory exchanges only: the release is
// restricted to this CTA's shared memory and the acquire to shared::cluster, so
// it lowers to MEMBAR.ALL.CTA around UCGABAR instead of the MEMBAR.ALL.GPU of
// cluster.sync() (no global-memory data crosses these barriers; the sample's
// cross-CTA increment reduction uses its own acq_rel atomics).
__device__ __forceinline__ void cluster_sync_smem() {
  asm volatile(
      "fence.release.sync_restrict::shared::cta.cluster;\n"
      "barrier.cluster.arrive.relaxed;\n"
      "barrier.cluster.wait;\n"
      "fence.acquire.sync_restrict::shared::cluster.cluster;\n" ::: "memory");
}

template <int LOGN>
__device__ __forceinline__ int brev(int n) {
  return LOGN == 0 ? 0 : (int)(__brev((unsigned)n) >> (32 - LOGN));
}

// ---- tile layout: [N][HC] complex, the column index XOR-swizzled within
// aligned groups of 8 (tswz) so that the 8-lane solver groups, whose lanes
// read columns MR apart at 4 different frequency rows, spread over the banks;
// consecutive columns of one row stay a permutation (conflict-free sweeps).
template <int MR>
__device__ __forceinline__ int tswz(int n, int c) {
  if constexpr (MR == 8) return c ^ (((c >> 3) & 3) | ((n & 1) << 2));
  else return c ^ (((c >> 3) & 1) | ((n & 3) << 1));
}
template <int MR, int HC>
__device__ __forceinline__ int tix(int n, int c) { return n * HC + tswz<MR>(n, c); }

// ---- four-step FFT over the columns of an [N][TC] tile (natural order in and
// out). N = N1*N2: pass 1 does N2-point DFTs along stride-N1 subsequences and
// the twiddle W_N^{n1 k2}; pass 2 does N1-point DFTs and writes X[k2 + N2 k1].
// S = -1: forward (np.fft.fft sign), S = +1: inverse (unnormalised).
template <int S>
__device__ __forceinline__ Cplx mul_si(Cplx z) {  // z * (S i)
  return S > 0 ? Cplx{-z.im, z.re} : Cplx{z.im, -z.re};
}
__device__ __forceinline__ Cplx cadd2(Cplx a, Cplx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ Cplx csub2(Cplx a, Cplx b) { return {a.re - b.re, a.im - b.im}; }

template <int NS, int S>
struct SmallDft;
template <int S>
struct SmallDft<1, S> {
  __device__ __forceinline__ static void run(Cplx (&)[1]) {}
};
template <int S>
struct SmallDft<2, S> {
  __device__ __forceinline__ static void run(Cplx (&v)[2]) {
    const Cplx a = v[0], b = v[1];
    v[0] = cadd2(a, b);
    v[1] = csub2(a, b);
  }
};
template <int S>
struct SmallDft<4, S> {
  __device__ __forceinline__ static void run(Cplx (&v)[4]) {
    const Cplx s02 = cadd2(v[0], v[2]), d02 = csub2(v[0], v[2]);
    const Cplx s13 = cadd2(v[1], v[3]), d13 = mul_si<S>(csub2(v[1], v[3]));
    v[0] = cadd2(s02, s13);
    v[2] = csub2(s02, s13);
    v[1] = cadd2(d02, d13);
    v[3] = csub2(d02, d13);
  }
};
template <int S>
struct SmallDft<8, S> {
  __device__ __forceinline__ static void run(Cplx (&v)[8]) {
    Cplx e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
    SmallDft<4, S>::run(e);
    SmallDft<4, S>::run(o);
    constexpr double h = 0.70710678118654752440;
    const Cplx w1 = {h, S * h}, w3 = {-h, S * h};
    const Cplx t0 = o[0], t1 = cmul(o[1], w1), t2 = mul_si<S>(o[2]), t3 = cmul(o[3], w3);
    v[0] = cadd2(e[0], t0);
    v[4] = csub2(e[0], t0);
    v[1] = cadd2(e[1], t1);
    v[5] = csub2(e[1], t1);
    v[2] = cadd2(e[2], t2);
    v[6] = csub2(e[2], t2);
    v[3] = cadd2(e[3], t3);
    v[7] = csub2(e[3], t3);
  }
};

// tw[j] = exp(-2 pi i j / N), j < N
template <int LOGN, int TC, int S, int MR>
__device__ void fft4step(Cplx* t, const Cplx* tw) {
  constexpr int N = 1 << LOGN;
  constexpr int N1 = 1 << ((LOGN + 1) / 2), N2 = N / N1;
  // pass 1: tasks (n1, c)
  for (int task = threadIdx.x; task < N1 * TC; task += blockDim.x) {
    const int n1 = task / TC, c = task % TC;
    Cplx v[N2];
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) v[n2] = t[tix<MR, TC>(n1 + N1 * n2, c)];
    SmallDft<N2, S>::run(v);
#pragma unroll
    for (int k2 = 1; k2 < N2; ++k2) {
      Cplx w = tw[(n1 * k2) & (N - 1)];
      if (S > 0) w.im = -w.im;
      v[k2] = cmul(v[k2], w);
    }
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) t[tix<MR, TC>(n1 + N1 * k2, c)] = v[k2];
  }
  __syncthreads();
  // pass 2: tasks (k2, c); outputs go to natural positions after a barrier
  constexpr int TASKS = N2 * TC;
  constexpr int MAXR = 2;  // rounds held in registers (launcher guarantees blockDim * MAXR >= TASKS)
  Cplx w[MAXR][N1];
#pragma unroll
  for (int r = 0; r < MAXR; ++r) {
    const int task = threadIdx.x + r * blockDim.x;
    if (task < TASKS) {
      const int k2 = task / TC, c = task % TC;
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) w[r][n1] = t[tix<MR, TC>(n1 + N1 * k2, c)];
      SmallDft<N1, S>::run(w[r]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < MAXR; ++r) {
    const int task = threadIdx.x + r * blockDim.x;
    if (task < TASKS) {
      const int k2 = task / TC, c = task % TC;
#pragma unroll
      for (int k1 = 0; k1 < N1; ++k1) t[tix<MR, TC>(k2 + N2 * k1, c)] = w[r][k1];
    }
  }
  __syncthreads();
}

// The same four-step FFT as fft4step for one column held in registers (N <=
// 16): the same DFTs, twiddles and output order, so the results are bitwise
// those of the shared-memory tile passes; one shared-memory store (forward)
// or load (inverse) per element instead of four passes over the tile.
template <int LOGN, int S>
__device__ __forceinline__ void reg_fft(Cplx (&x)[1 << LOGN], const Cplx* tw) {
  constexpr int N = 1 << LOGN;
  constexpr int N1 = 1 << ((LOGN + 1) / 2), N2 = N / N1;
  Cplx y[N];
#pragma unroll
  for (int n1 = 0; n1 < N1; ++n1) {
    Cplx v[N2];
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) v[n2] = x[n1 + N1 * n2];
    SmallDft<N2, S>::run(v);
#pragma unroll
    for (int k2 = 1; k2 < N2; ++k2) {
      Cplx w = tw[(n1 * k2) & (N - 1)];
      if (S > 0) w.im = -w.im;
      v[k2] = cmul(v[k2], w);
    }
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) y[n1 + N1 * k2] = v[k2];
  }
#pragma unroll
  for (int k2 = 0; k2 < N2; ++k2) {
    Cplx w[N1];
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) w[n1] = y[n1 + N1 * k2];
    SmallDft<N1, S>::run(w);
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) x[k2 + N2 * k1] = w[k1];
  }
}

// pivots 1/beta_i of (lambda_f I + dT A), f = 0..N/2, layout [s][f][i].
// Thread (sample, f) runs the sequential complex recurrence (factor_shifted,
// pintuq/pcgc.py:112-135) over the rows in chunks of SF_CH; a CTA packs
// SPB = 128 / NF samples (N = 16: 14 samples x 9 frequencies on 126 of its 128
// threads, instead of one sample on 9 of 64) and stages each chunk in shared
// memory so the whole CTA stores it coalesced (rows contiguous per frequency).
constexpr int SF_CH = 16;
constexpr int SF_NT = 128;
__global__ void __launch_bounds__(SF_NT) shift_factor_kernel(const double* __restrict__ dia, const double* __restrict__ off,
                                                             const double* __restrict__ lam, int M, int NF, int nx,
                                                             double dT, double* __restrict__ sfac) {
  extern __shared__ __align__(16) Cplx stage[];  // [SPB][NF][SF_CH + 1]
  const int SPB = SF_NT / NF;
  const int sl = threadIdx.x / NF, f = threadIdx.x - sl * NF;
  const int s0 = blockIdx.x * SPB;
  const int s = s0 + sl;
  const bool act = sl < SPB && s < M;
  const double* d = dia + (size_t)(act ? s : 0) * nx;
  const double* e = off + (size_t)(act ? s : 0) * nx;
  const Cplx lm = act ? Cplx{lam[2 * f], lam[2 * f + 1]} : Cplx{1.0, 0.0};
  const int ns = min(SPB, M - s0);
  Cplx ib = {0.0, 0.0};
  for (int i0 = 0; i0 < nx; i0 += SF_CH) {
    const int nr = min(SF_CH, nx - i0);
    if (act) {
      // the chunk's operator rows first (all loads in flight), then the dependent recurrence
      double dv[SF_CH], ev[SF_CH];
#pragma unroll
      for (int r = 0; r < SF_CH; ++r) {
        const int i = i0 + r;
        dv[r] = r < nr ? __ldg(d + i) : 0.0;
        ev[r] = (r < nr && i > 0) ? __ldg(e + i - 1) : 0.0;
      }
#pragma unroll
      for (int r = 0; r < SF_CH; ++r) {
        if (r >= nr) break;
        const int i = i0 + r;
        Cplx beta = {fma(dT, dv[r], lm.re), lm.im};
        if (i > 0) {
          const double E = dT * ev[r];
          beta.re = fma(-E * E, ib.re, beta.re);
          beta.im = fma(-E * E, ib.im, beta.im);
        }
        ib = crcp(beta);
        stage[(sl * NF + f) * (SF_CH + 1) + r] = ib;
      }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < ns * NF * nr; q += SF_NT) {
      const int r = q % nr, sf = q / nr;  // sf = sample-local * NF + frequency
      const int ss = sf / NF, ff = sf - ss * NF;
      Cplx* out = reinterpret_cast<Cplx*>(sfac) + ((size_t)(s0 + ss) * NF + ff) * nx;
      out[i0 + r] = stage[sf * (SF_CH + 1) + r];
    }
    __syncthreads();
  }
}

template <int MR>
__device__ __forceinline__ void load_pivots(Cplx (&ib)[MR], Cplx& ibprev, const Cplx* __restrict__ src, int r0,
                                            int nx) {
  ibprev = (r0 > 0 && r0 - 1 < nx) ? src[r0 - 1] : Cplx{0.0, 0.0};
#pragma unroll
  for (int j = 0; j < MR; ++j) ib[j] = (r0 + j < nx) ? src[r0 + j] : Cplx{1.0, 0.0};
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}

// The lane's pivots 1/beta (rows r0 .. r0+MR-1 of its frequency, plus row
// r0-1): in registers (SP = false) or read from the CTA's shared-memory copy
// where used (SP = true: 32 fewer registers, 3 CTAs/SM).
template <int MR, bool SP>
struct PivSrc;
template <int MR>
struct PivSrc<MR, false> {
  Cplx v[MR], pv;
  __device__ __forceinline__ void init(const Cplx* g, const Cplx*, int, int r0, int nx) { load_pivots<MR>(v, pv, g, r0, nx); }
  __device__ __forceinline__ Cplx operator[](int j) const { return v[j]; }
  __device__ __forceinline__ Cplx prev(int j) const { return j == 0 ? pv : v[j - 1]; }
};
template <int MR>
struct PivSrc<MR, true> {
  const Cplx* sp;  // this frequency's [RB] row slice (swizzled)
  int r0l;
  Cplx pv;         // row r0 - 1
  __device__ __forceinline__ void init(const Cplx* g, const Cplx* s, int rl, int r0, int nx) {
    sp = s;
    r0l = rl;
    if (rl == 0) pv = (r0 > 0 && r0 - 1 < nx) ? g[r0 - 1] : Cplx{0.0, 0.0};
  }
  __device__ __forceinline__ Cplx at(int r) const { return sp[r ^ ((r >> 3) & 7)]; }
  __device__ __forceinline__ Cplx operator[](int j) const { return at(r0l + j); }
  __device__ __forceinline__ Cplx prev(int j) const { return (j == 0 && r0l == 0) ? pv : at(r0l + j - 1); }
};

// Composes the affine maps x -> A x + B held by the 8 lanes of a group
// (butterfly; every lane ends with the ordered composite). OUTER_HIGH: the
// higher lane's map is applied last.
template <bool OUTER_HIGH>
__device__ __forceinline__ void compose_lanes(Cplx& A, Cplx& B, int k) {
#pragma unroll
  for (int d = 1; d < CL_LANES; d <<= 1) {
    const Cplx Ao = shfl_xor_c(A, d), Bo = shfl_xor_c(B, d);
    const bool outer = OUTER_HIGH ? (k & d) != 0 : (k & d) == 0;
    B = outer ? cfma(A, Bo, B) : cfma(Ao, B, Bo);
    A = cmul(A, Ao);
  }
}

template <int LOGN, int MR>
struct ClShape {
  static constexpr int N = 1 << LOGN, NF = N / 2 + 1, RB = CL_LANES * MR, HC = RB / 2;
  static constexpr int NT = ((NF * CL_LANES + 31) / 32) * 32;  // one 8-lane group per frequency
  static constexpr int NSTEP = NT / RB;                         // column-fixed sweeps (0: generic loop)
#ifndef KLE_CGC_REGFFT
#define KLE_CGC_REGFFT 0  // 1: N <= 16 column FFTs in registers, one thread per packed column (A/B:
                          // bitwise equal, but 7.33 vs 3.39 ms per 131k c4 launch: 32 threads per CTA
                          // serialise the loads and FFTs that 96 share in the tile passes)
#endif
  static constexpr bool REGFFT = LOGN <= 4 && KLE_CGC_REGFFT && NT >= RB / 2;
#ifndef KLE_CGC_SP
#define KLE_CGC_SP 1  // pivots in shared memory, old U re-read from global: 3 CTAs/SM at 288 threads
#endif
  static constexpr bool SP = KLE_CGC_SP != 0;
#ifndef KLE_CGC_MINB
#define KLE_CGC_MINB 2  // 288 threads, pivots in registers: 2 CTAs/SM (measured; 1 CTA without spills is slower)
#endif
#ifndef KLE_CGC_MINB_SP
#define KLE_CGC_MINB_SP 3  // CTAs/SM bound for the shared-memory-pivot shapes (N = 64: 288 threads)
#endif
#ifndef KLE_CGC_MINB_SMALL
#define KLE_CGC_MINB_SMALL 8  // N <= 16 (<= 96 threads): 80 registers, 8 CTAs/SM (c4: 4.88 -> 3.55 ms / 131k samples)
#endif
  static constexpr int MINB = NT <= 96 ? KLE_CGC_MINB_SMALL : ((NT <= 160 || SP) ? KLE_CGC_MINB_SP : KLE_CGC_MINB);
  static constexpr size_t UOLD = SP ? 0 : (size_t)N * RB;           // doubles
  static constexpr size_t PIV = SP ? (size_t)2 * NF * RB : 0;       // doubles: [NF][RB] complex, swizzled rows
  static constexpr size_t SMEM = sizeof(double) * ((size_t)2 * N * HC + UOLD + PIV + RB + 2 + N + 2 * N +
                                                   8 * NF + 16);
};

template <int LOGN, int MR>
__global__ void __launch_bounds__(ClShape<LOGN, MR>::NT, ClShape<LOGN, MR>::MINB)
    cgc_cluster_kernel(CgcArgs a, const double* __restrict__ sfac_d) {
  using K = ClShape<LOGN, MR>;
  constexpr int N = K::N, NF = K::NF, RB = K::RB, HC = K::HC, NT = K::NT, NSTEP = K::NSTEP;
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks();
  const int c = (int)cluster.block_rank();
  const int s = blockIdx.x / CL;
  const int nx = a.nx;
  if (a.status && a.status[s] != KLE_SAMPLE_ACTIVE) return;  // uniform over the cluster

  extern __shared__ __align__(16) double smem[];
  Cplx* tile = reinterpret_cast<Cplx*>(smem);       // [N][HC] packed spectra (swizzled columns)
  double* uold = smem + 2 * N * HC;                 // [N][RB] (pivots in registers only)
  Cplx* piv = reinterpret_cast<Cplx*>(uold + K::UOLD);  // [NF][RB] pivots (SP), row r at r ^ ((r >> 3) & 7)
  double* offs = uold + K::UOLD + K::PIV;           // [RB + 2]: dT*off[row0-1 .. row0+RB]
  double* isc = offs + RB + 2;                      // [N]: inv_scaling
  Cplx* tw = reinterpret_cast<Cplx*>(isc + N);      // [N]
  Cplx* fwd = tw + N;                               // [NF][2]
  Cplx* bwd = fwd + 2 * NF;                         // [NF][2]
  double* red = reinterpret_cast<double*>(bwd + 2 * NF);  // [16]

  const int tid = threadIdx.x;
  const size_t sb = (size_t)s * N * nx;
  const int row0 = c * RB;
  CGC_T(0);
  // ---- phase 0: prefetch --------------------------------------------------
  Cplx zc[K::REGFFT ? N : 1];  // REGFFT: column tid of the packed block, rows row0+tid (re) and row0+tid+HC (im)
  if constexpr (K::REGFFT) {
    if (tid < HC) {
      const int ra = row0 + tid, rb = ra + HC;
#pragma unroll
      for (int n = 0; n < N; ++n) {
        zc[n].re = ra < nx ? a.R[sb + (size_t)n * nx + ra] : 0.0;
        zc[n].im = rb < nx ? a.R[sb + (size_t)n * nx + rb] : 0.0;
      }
    }
  } else if constexpr (NSTEP > 0) {  // each thread keeps one column; rows n = tid/RB + m*NSTEP
    if (tid < NSTEP * RB) {
      const int col = tid % RB, row = row0 + col, ci = col % HC, part = col / HC;
      for (int n = tid / RB; n < N; n += NSTEP) {
        double* dst = reinterpret_cast<double*>(&tile[tix<MR, HC>(n, ci)]) + part;
        if (row < nx) {
          cp_async8(dst, a.R + sb + (size_t)n * nx + row);
          if (!K::SP && a.U) cp_async8(uold + n * RB + col, a.U + sb + (size_t)n * nx + row);
        } else {
          *dst = 0.0;
        }
      }
    }
  } else {
    for (int e = tid; e < N * RB; e += NT) {
      const int n = e / RB, col = e % RB, row = row0 + col;
      double* dst = reinterpret_cast<double*>(&tile[tix<MR, HC>(n, col % HC)]) + (col / HC);
      if (row < nx) {
        cp_async8(dst, a.R + sb + (size_t)n * nx + row);
        if (!K::SP && a.U) cp_async8(uold + n * RB + col, a.U + sb + (size_t)n * nx + row);
      } else {
        *dst = 0.0;
      }
    }
  }
  if constexpr (K::SP) {  // the CTA's rows of every frequency's pivots, 16-byte copies
    const Cplx* src = reinterpret_cast<const Cplx*>(sfac_d) + (size_t)s * NF * nx;
    for (int e = tid; e < NF * RB; e += NT) {
      const int ff = e / RB, r = e % RB, row = row0 + r;
      Cplx* dst = &piv[ff * RB + (r ^ ((r >> 3) & 7))];
      if (row < nx) cp_async16(dst, src + (size_t)ff * nx + row);
      else *dst = {1.0, 0.0};
    }
  }
  for (int e = tid; e < RB + 2; e += NT) {
    const int row = row0 - 1 + e;  // offs[e] couples rows row and row+1
    offs[e] = (row >= 0 && row + 1 < nx) ? a.dT * a.off[(size_t)s * nx + row] : 0.0;
  }
  for (int j = tid; j < N; j += NT) {
    double sn, cs;
    sincospi(-2.0 * (double)j / (double)N, &sn, &cs);
    tw[j] = {cs, sn};
    isc[j] = a.inv_scaling[j];
  }
  const int fsys = tid / CL_LANES, k = tid % CL_LANES;
  const bool valid = fsys < NF;
  const int f = valid ? fsys : NF - 1;
  const int r0l = k * MR;  // local first row of this lane
  const int r0 = row0 + r0l;
  PivSrc<MR, K::SP> ib;
  ib.init(reinterpret_cast<const Cplx*>(sfac_d) + ((size_t)s * NF + f) * nx, piv + f * RB, r0l, r0, nx);
  cp_async_wait_all();
  __syncthreads();
  CGC_T(1);
  if constexpr (K::REGFFT) {
    if (tid < HC) {
      if (a.load_scale) {  // stand-alone three-step: r is not alpha-scaled yet
#pragma unroll
        for (int n = 0; n < N; ++n) {
          zc[n].re *= a.load_scale[n];
          zc[n].im *= a.load_scale[n];
        }
      }
      reg_fft<LOGN, -1>(zc, tw);
#pragma unroll
      for (int n = 0; n < N; ++n) tile[tix<MR, HC>(n, tid)] = zc[n];
    }
    __syncthreads();
  } else {
    if (a.load_scale) {  // stand-alone three-step: r is not alpha-scaled yet
      for (int e = tid; e < N * RB; e += NT) {
        const int n = e / RB, col = e % RB;
        reinterpret_cast<double*>(&tile[tix<MR, HC>(n, col % HC)])[col / HC] *= a.load_scale[n];
      }
      __syncthreads();
    }
    fft4step<LOGN, HC, -1, MR>(tile, tw);
  }
  CGC_T(2);

  // ---- one frequency per 8-lane group: (lambda_f I + dT A) q = p_f ---------
  const double hs = 0.5 / sqrt((double)N);  // two-for-one unpacking x 1/sqrt(N)
  Cplx y[MR];
  const int fm = (N - f) & (N - 1);
#pragma unroll
  for (int j = 0; j < MR; ++j) {
    const int col = r0l + j;
    const Cplx zf = tile[tix<MR, HC>(f, col % HC)], zm = tile[tix<MR, HC>(fm, col % HC)];
    if (col < HC) y[j] = {(zf.re + zm.re) * hs, (zf.im - zm.im) * hs};   // (Z_f + conj Z_-f)/2
    else y[j] = {(zf.im + zm.im) * hs, (zm.re - zf.re) * hs};            // (Z_f - conj Z_-f)/(2i)
  }
  // l_r = dT off_{r-1} / beta_{r-1}, formed where used (E from shared memory):
  // keeping all MR of them live as well as the pivots spills registers
  auto lj = [&](int j) -> Cplx {
    const double E = offs[r0l + j];  // couples rows r0+j-1 and r0+j
    const Cplx ip = ib.prev(j);
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
  for (int d = 1; d < CL_LANES; d <<= 1) {
    const Cplx Ao = shfl_up_c(A, d), Bo = shfl_up_c(B, d);
    if (k >= d) {
      B = cfma(A, Bo, B);
      A = cmul(A, Ao);
    }
  }
  Cplx Ae = shfl_up_c(A, 1), Be = shfl_up_c(B, 1);
  if (k == 0) {
    Ae = {1.0, 0.0};
    Be = {0.0, 0.0};
  }
  if (valid && k == CL_LANES - 1) {
    fwd[2 * f] = A;
    fwd[2 * f + 1] = B;
  }
  CGC_T(3);
  cluster_sync_smem();
  CGC_T(4);
  Cplx Yc;
  {  // composite of the blocks q < c, q = k (+ 8) per lane, then a lane butterfly
    Cplx A0 = {1.0, 0.0}, B0 = {0.0, 0.0}, A1 = {1.0, 0.0}, B1 = {0.0, 0.0};
    if (k < c) {
      const Cplx* rf = cluster.map_shared_rank(fwd, k);
      A0 = rf[2 * f];
      B0 = rf[2 * f + 1];
    }
    if (k + CL_LANES < c) {
      const Cplx* rf = cluster.map_shared_rank(fwd, k + CL_LANES);
      A1 = rf[2 * f];
      B1 = rf[2 * f + 1];
    }
    compose_lanes<true>(A0, B0, k);
    if (c > CL_LANES) compose_lanes<true>(A1, B1, k);
    Yc = cfma(A1, B0, B1);
  }
  const Cplx Cin = cfma(Ae, Yc, Be);
  {
    Cplx pi = {1.0, 0.0};
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      pi = cneg_mul(lj(j), pi);
      y[j] = cmul(cfma(pi, Cin, y[j]), ib[j]);
    }
  }
  const double En = offs[r0l + MR];  // couples the lane's last row and the next
  const Cplx lnext = {En * ib[MR - 1].re, En * ib[MR - 1].im};
  Cplx S = {1.0, 0.0};
#pragma unroll
  for (int j = MR - 1; j >= 0; --j) {
    const Cplx ln = (j == MR - 1) ? lnext : lj(j + 1);
    if (j < MR - 1) y[j] = cfma({-ln.re, -ln.im}, y[j + 1], y[j]);
    S = cneg_mul(ln, S);
  }
  Cplx T = y[0];
#pragma unroll
  for (int d = 1; d < CL_LANES; d <<= 1) {
    const Cplx So = shfl_down_c(S, d), To = shfl_down_c(T, d);
    if (k + d < CL_LANES) {
      T = cfma(S, To, T);
      S = cmul(S, So);
    }
  }
  Cplx Se = shfl_down_c(S, 1), Te = shfl_down_c(T, 1);
  if (k == CL_LANES - 1) {
    Se = {1.0, 0.0};
    Te = {0.0, 0.0};
  }
  if (valid && k == 0) {
    bwd[2 * f] = S;
    bwd[2 * f + 1] = T;
  }
  CGC_T(5);
  cluster_sync_smem();  // also: every thread has read its inputs from the tile
  CGC_T(6);
  Cplx Xc;
  {  // composite of the blocks q > c (the nearest block applied last)
    Cplx A0 = {1.0, 0.0}, B0 = {0.0, 0.0}, A1 = {1.0, 0.0}, B1 = {0.0, 0.0};
    if (c + 1 + k < CL) {
      const Cplx* rb = cluster.map_shared_rank(bwd, c + 1 + k);
      A0 = rb[2 * f];
      B0 = rb[2 * f + 1];
    }
    if (c + 1 + CL_LANES + k < CL) {
      const Cplx* rb = cluster.map_shared_rank(bwd, c + 1 + CL_LANES + k);
      A1 = rb[2 * f];
      B1 = rb[2 * f + 1];
    }
    compose_lanes<false>(A0, B0, k);
    if (c + 1 + CL_LANES < CL) compose_lanes<false>(A1, B1, k);
    Xc = cfma(A0, B1, B0);
  }
  const Cplx Xin = cfma(Se, Xc, Te);
  {
    Cplx sg = {1.0, 0.0};
#pragma unroll
    for (int j = MR - 1; j >= 0; --j) {
      const Cplx ln = (j == MR - 1) ? lnext : lj(j + 1);
      sg = cneg_mul(ln, sg);
      y[j] = cfma(sg, Xin, y[j]);
    }
  }
  // every CTA has done its last DSMEM read (completed before the relaxed arrive)
  asm volatile("fence.release.sync_restrict::shared::cta.cluster;\nbarrier.cluster.arrive.relaxed;\n" ::: "memory");
  // pack W_f = q(col) + i q(col + HC): lanes k < 4 hold the first half rows
#pragma unroll
  for (int j = 0; j < MR; ++j) {
    const Cplx qb = shfl_xor_c(y[j], CL_LANES / 2);
    if (valid && k < CL_LANES / 2) {
      const int col = r0l + j;
      tile[tix<MR, HC>(f, col)] = {y[j].re - qb.im, y[j].im + qb.re};
      if (f > 0 && 2 * f < N) tile[tix<MR, HC>(N - f, col)] = {y[j].re + qb.im, qb.re - y[j].im};
    }
  }
  __syncthreads();
  // the pivots are dead now: stream the column's old values into their space
  // while the inverse FFT runs (each thread loads exactly what it reads later)
  constexpr bool UPRE = K::SP && NSTEP > 0 && KLE_CGC_UPRE && !K::REGFFT;
  double* uold_p = reinterpret_cast<double*>(piv);  // [N][RB]
  if constexpr (UPRE) {
    if (a.U && tid < NSTEP * RB && row0 + tid % RB < nx) {
      const int col = tid % RB;
      for (int n = tid / RB; n < N; n += NSTEP) cp_async8(uold_p + n * RB + col, a.U + sb + (size_t)n * nx + row0 + col);
    }
  }
  if constexpr (!K::REGFFT) fft4step<LOGN, HC, +1, MR>(tile, tw);
  CGC_T(7);
  // ---- update ----------------------------------------------------------------
  const double rsN = 1.0 / sqrt((double)N);
  double incmax = 0.0;
  bool bad = false;  // fmax drops NaN; remember it separately (a NaN increment must not converge)
  double* __restrict__ out = a.Uout ? a.Uout : a.U;
  const bool track = a.U != nullptr;
  auto upd = [&](int n, int col, int row, double uo) {
    const Cplx z = tile[tix<MR, HC>(n, col % HC)];
    const double u = ((col < HC ? z.re : z.im) * rsN) * isc[n];
    if (track) {
      const double d = fabs(u - uo);
      incmax = fmax(incmax, d);
      bad |= (d != d);
    }
    out[sb + (size_t)n * nx + row] = u;
  };
  if constexpr (K::REGFFT) {  // inverse column FFT in registers, then the column's two rows
    if (tid < HC) {
      const int ra = row0 + tid, rb = ra + HC;
#pragma unroll
      for (int n = 0; n < N; ++n) zc[n] = tile[tix<MR, HC>(n, tid)];
      reg_fft<LOGN, +1>(zc, tw);
#pragma unroll
      for (int n = 0; n < N; ++n) {
        // the old values: each row's load precedes its store (out may alias U)
        const double uan = (track && ra < nx) ? a.U[sb + (size_t)n * nx + ra] : 0.0;
        const double ubn = (track && rb < nx) ? a.U[sb + (size_t)n * nx + rb] : 0.0;
        const double u0v = (zc[n].re * rsN) * isc[n], u1v = (zc[n].im * rsN) * isc[n];
        if (ra < nx) {
          if (track) {
            const double d = fabs(u0v - uan);
            incmax = fmax(incmax, d);
            bad |= (d != d);
          }
          out[sb + (size_t)n * nx + ra] = u0v;
        }
        if (rb < nx) {
          if (track) {
            const double d = fabs(u1v - ubn);
            incmax = fmax(incmax, d);
            bad |= (d != d);
          }
          out[sb + (size_t)n * nx + rb] = u1v;
        }
      }
    }
  } else if constexpr (NSTEP > 0) {
    if (tid < NSTEP * RB) {
      const int col = tid % RB, row = row0 + col;
      if (row < nx) {
        if constexpr (UPRE) {
          cp_async_wait_all();
          for (int n = tid / RB; n < N; n += NSTEP) upd(n, col, row, track ? uold_p[n * RB + col] : 0.0);
        } else if constexpr (K::SP) {
          // the column's old values, all loads issued before the stores (out may alias U)
          constexpr int NR = (N + NSTEP - 1) / NSTEP;
          constexpr int UB = NR < 8 ? NR : 8;  // loads in flight per batch
#pragma unroll
          for (int m0 = 0; m0 < NR; m0 += UB) {
            double uo[UB];
#pragma unroll
            for (int m = 0; m < UB; ++m) {
              const int n = tid / RB + (m0 + m) * NSTEP;
              uo[m] = (track && m0 + m < NR && n < N) ? a.U[sb + (size_t)n * nx + row] : 0.0;
            }
#pragma unroll
            for (int m = 0; m < UB; ++m) {
              const int n = tid / RB + (m0 + m) * NSTEP;
              if (m0 + m < NR && n < N) upd(n, col, row, uo[m]);
            }
          }
        } else {
          for (int n = tid / RB; n < N; n += NSTEP) upd(n, col, row, track ? uold[n * RB + col] : 0.0);
        }
      }
    }
  } else {
    for (int e = tid; e < N * RB; e += NT) {
      const int n = e / RB, col = e % RB, row = row0 + col;
      if (row < nx) upd(n, col, row, track ? (K::SP ? a.U[sb + (size_t)n * nx + row] : uold[n * RB + col]) : 0.0);
    }
  }
  if (__syncthreads_or(bad)) incmax = __longlong_as_double(0x7ff8000000000000LL);
  CGC_T(8);
  incmax = warp_max(incmax);
  const int lane = tid & 31, w = tid >> 5;
  constexpr int NW = NT / 32;
  if (lane == 0) red[w] = incmax;
  __syncthreads();
  if (tid == 0) {
    double r1 = 0.0;
    for (int i = 0; i < NW; ++i) r1 = nanmax(r1, red[i]);
    // cluster-wide max through a global slot; the last CTA to arrive finishes
    // the sample (no further cluster barrier needed). Non-negative doubles
    // (and +NaN) order like their bit patterns.
    unsigned long long* slot = a.red_slots + 2 * (size_t)s;
    atomicMax(slot, (unsigned long long)__double_as_longlong(r1));
    // the ticket is an acq_rel atomic: it releases this CTA's max (program order)
    // and, for the last arriver, acquires every other CTA's (no separate fences)
    unsigned long long ticket;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(ticket) : "l"(slot + 1), "l"(1ULL) : "memory");
    if ((ticket + 1) % (unsigned long long)CL == 0) {
      const double inc = __longlong_as_double((long long)atomicExch(slot, 0ULL));
      if (a.inc) a.inc[s] = inc;
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
  // every CTA arrived (after its last DSMEM read) before the pack; wait here
  // so no CTA's shared memory disappears under a remote reader
  asm volatile("barrier.cluster.wait;\n" ::: "memory");
  CGC_T(9);
}

// ---------------------------------------------------------------------------
static bool cluster_shape(int N, int nx, int* MR, int* CL, int* LOGN) {
  if (N < 2 || N > 64 || (N & (N - 1))) return false;
  int logn = 0;
  while ((1 << logn) < N) ++logn;
  // 64-row blocks: measured faster than 32-row blocks in clusters of up to 16
  // (c2: 2.97 vs 4.34 ms per 4096 samples; fewer, fatter CTAs per sample)
  static const char* env = getenv("KLE_CGC_MR");  // 4: 32-row blocks (A/B)
  const int mr = (env && atoi(env) == 4) ? 4 : 8;
  const int rb = CL_LANES * mr;
  const int cl = (nx + rb - 1) / rb;
  if (cl > 16) return false;
  *MR = mr;
  *CL = cl;
  *LOGN = logn;
  return true;
}

bool cgc_cluster_supported(int N, int nx) {
  int mr, cl, ln;
  return cluster_shape(N, nx, &mr, &cl, &ln);
}

size_t shift_factor_doubles(int M, int N, int nx) { return 2 * (size_t)M * (N / 2 + 1) * nx; }

int shift_factor(const double* dia, const double* off, const double* lam, int M, int N, int nx, double dT,
                 double* sfac, cudaStream_t st) {
  const int NF = N / 2 + 1;
  const long long nth = (long long)M * NF;
  if (nth == 0) return KLE_OK;
  if (NF > SF_NT) return set_error(KLE_ERR_UNSUPPORTED, "shift_factor: N > 254");
  const int spb = SF_NT / NF;
  const size_t smem = sizeof(Cplx) * (size_t)spb * NF * (SF_CH + 1);
  shift_factor_kernel<<<(unsigned)((M + spb - 1) / spb), SF_NT, smem, st>>>(dia, off, lam, M, NF, nx, dT, sfac);
  return check_launch("shift_factor_kernel");
}

template <int LOGN, int MR>
static int launch_cluster(const CgcArgs& a, const double* sfac, int CL, cudaStream_t st) {
  using K = ClShape<LOGN, MR>;
  constexpr int N2 = K::N / (1 << ((LOGN + 1) / 2));
  static_assert(K::NT * 2 >= N2 * K::HC, "cgc_cluster: FFT pass-2 tasks exceed 2 rounds");
  auto kern = cgc_cluster_kernel<LOGN, MR>;
  static PerDeviceOnce attr_once;
  if (int rc = once_per_device(attr_once, "kle_cgc_cluster: cudaFuncSetAttribute", [&] {
        const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::SMEM);
        return e != cudaSuccess ? e : cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      }))
    return rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a.M * CL), 1, 1);
  cfg.blockDim = dim3((unsigned)K::NT, 1, 1);
  cfg.dynamicSmemBytes = K::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = CL;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a, sfac);
  if (e != cudaSuccess) return set_error(KLE_ERR_CUDA, cudaGetErrorString(e));
  return check_launch("cgc_cluster_kernel");
}

template <int MR>
static int dispatch_logn(int logn, const CgcArgs& a, const double* sfac, int CL, cudaStream_t st) {
  switch (logn) {
    case 1: return launch_cluster<1, MR>(a, sfac, CL, st);
    case 2: return launch_cluster<2, MR>(a, sfac, CL, st);
    case 3: return launch_cluster<3, MR>(a, sfac, CL, st);
    case 4: return launch_cluster<4, MR>(a, sfac, CL, st);
    case 5: return launch_cluster<5, MR>(a, sfac, CL, st);
    case 6: return launch_cluster<6, MR>(a, sfac, CL, st);
  }
  return set_error(KLE_ERR_UNSUPPORTED, "cgc_cluster: N");
}

#ifdef KLE_CGC_TIMING
extern "C" int kle_debug_cgc_timing(unsigned long long* host) {
  return (int)cudaMemcpyFromSymbol(host, g_cgc_t, sizeof(g_cgc_t));
}
#endif

int cgc_cluster_run(const CgcArgs& a, const double* sfac, cudaStream_t st) {
  int MR, CL, LOGN;
  if (!cluster_shape(a.N, a.nx, &MR, &CL, &LOGN)) return set_error(KLE_ERR_UNSUPPORTED, "cgc_cluster: shape");
  if (a.M <= 0) return KLE_OK;
  if (cgc_row_supported(a.N, a.nx)) return cgc_row_run(a, sfac, st);  // same pivots, same arguments
  if (a.imag) cudaMemsetAsync(a.imag, 0, sizeof(double) * a.M, st);  // real by construction
  if (MR == 4) return dispatch_logn<4>(LOGN, a, sfac, CL, st);
  return dispatch_logn<8>(LOGN, a, sfac, CL, st);
}

}  // namespace kle
