// Diagonalised CGC (three-step solve) for small blocks: power-of-two N <= 16
// time points, nx <= 128 rows (BASELINE configs 1 and 4). One CTA per sample,
// no cluster, no shared-memory FFT passes.
//
// Reference: three_step_solve pintuq/pcgc.py:148-172, factor_shifted :90-145,
// the increment / stop test of pcgc_solve :335-348.
//
// Why a second kernel for these shapes: at c4 the cluster kernel
// (kle_cgc_cluster.cu) is bound by shared-memory wavefronts (85% of peak,
// tools/cgc_timing_c4.py: prefetch 18%, the two tile FFTs and the pack 36% of
// a CTA's life, 13 block barriers and 2 cluster barriers per CTA). Here
//   1. thread r < 128 owns row r: its N values of R come straight from
//      global memory (coalesced over the rows) into registers, and the
//      N-point real FFT along time runs in registers (one N/2-point complex
//      FFT of the even/odd packing plus the split);
//   2. the half spectrum P_f[r], f = 0..N/2, goes to shared memory once
//      ([f][r], rows XOR-swizzled within their 8-row chunk);
//   3. one 16-lane group per frequency solves (lambda_f I + dT A) q = p_f with
//      the precomputed pivots (8 rows per lane, a 4-stage affine lane scan
//      each way; the same recurrences as the cluster kernel, whose DSMEM
//      composites vanish because the block is the whole sample);
//   4. q goes back to the same shared slots, thread r runs the Hermitian
//      inverse FFT in registers and updates its N values of U (the old values
//      were requested before the barrier), block max-reduction, stop test.
// Shared-memory traffic per sample: 4 passes over the 18 KB spectrum plus the
// pivot reads, against 350 KB in the cluster kernel; 2 block barriers.
// u is real by construction (the inverse transform is Hermitian); the imag
// residue is reported as 0 like the cluster kernel.
#include <cstdlib>

#include "kle_common.cuh"
#include "kle_internal.h"

namespace kle {

namespace {

constexpr int RW_LANES = 16;  // lanes per frequency group
constexpr int RW_MR = 8;      // rows per lane
constexpr int RW_RB = RW_LANES * RW_MR;  // 128 rows

__device__ __forceinline__ Cplx cfma_(Cplx a, Cplx b, Cplx c) {  // a*b + c
  return {fma(a.re, b.re, fma(-a.im, b.im, c.re)), fma(a.re, b.im, fma(a.im, b.re, c.im))};
}
__device__ __forceinline__ Cplx cneg_mul_(Cplx a, Cplx b) {  // -(a*b)
  return {fma(-a.re, b.re, a.im * b.im), fma(-a.re, b.im, -a.im * b.re)};
}
__device__ __forceinline__ Cplx shfl_up16(Cplx v, int d) {
  return {__shfl_up_sync(KLE_FULL_MASK, v.re, d, RW_LANES), __shfl_up_sync(KLE_FULL_MASK, v.im, d, RW_LANES)};
}
__device__ __forceinline__ Cplx shfl_down16(Cplx v, int d) {
  return {__shfl_down_sync(KLE_FULL_MASK, v.re, d, RW_LANES), __shfl_down_sync(KLE_FULL_MASK, v.im, d, RW_LANES)};
}
__device__ __forceinline__ void cp_async16_(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ int rswz(int r) { return r ^ ((r >> 3) & 7); }

__device__ __forceinline__ Cplx cadd_(Cplx a, Cplx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ Cplx csub_(Cplx a, Cplx b) { return {a.re - b.re, a.im - b.im}; }
template <int S>
__device__ __forceinline__ Cplx mul_si_(Cplx z) {  // z * (S i)
  return S > 0 ? Cplx{-z.im, z.re} : Cplx{z.im, -z.re};
}

// in-place DFTs of length 1, 2, 4, 8 (natural order in and out); S = -1 forward, +1 inverse (unnormalised)
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
    v[0] = cadd_(a, b);
    v[1] = csub_(a, b);
  }
};
template <int S>
struct Dft<4, S> {
  __device__ __forceinline__ static void run(Cplx (&v)[4]) {
    const Cplx s02 = cadd_(v[0], v[2]), d02 = csub_(v[0], v[2]);
    const Cplx s13 = cadd_(v[1], v[3]), d13 = mul_si_<S>(csub_(v[1], v[3]));
    v[0] = cadd_(s02, s13);
    v[2] = csub_(s02, s13);
    v[1] = cadd_(d02, d13);
    v[3] = csub_(d02, d13);
  }
};
template <int S>
struct Dft<8, S> {
  __device__ __forceinline__ static void run(Cplx (&v)[8]) {
    Cplx e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
    Dft<4, S>::run(e);
    Dft<4, S>::run(o);
    constexpr double h = 0.70710678118654752440;
    const Cplx w1 = {h, S * h}, w3 = {-h, S * h};
    const Cplx t0 = o[0], t1 = cmul(o[1], w1), t2 = mul_si_<S>(o[2]), t3 = cmul(o[3], w3);
    v[0] = cadd_(e[0], t0);
    v[4] = csub_(e[0], t0);
    v[1] = cadd_(e[1], t1);
    v[5] = csub_(e[1], t1);
    v[2] = cadd_(e[2], t2);
    v[6] = csub_(e[2], t2);
    v[3] = cadd_(e[3], t3);
    v[7] = csub_(e[3], t3);
  }
};

// cos / sin of 2 pi k / 16, k = 0..8
__device__ __forceinline__ Cplx root16(int k) {  // exp(+2 pi i k / 16); k is a compile-time constant after unrolling
  constexpr double c1 = 0.92387953251128673848, s1 = 0.38268343236508978178, h = 0.70710678118654752440;
  switch (k) {
    case 0: return {1.0, 0.0};
    case 1: return {c1, s1};
    case 2: return {h, h};
    case 3: return {s1, c1};
    case 4: return {0.0, 1.0};
    case 5: return {-s1, c1};
    case 6: return {-h, h};
    case 7: return {-c1, s1};
    default: return {-1.0, 0.0};
  }
}

// Real FFT of x[N] along time, ortho-scaled half spectrum X[0..N/2]:
// X_k = (1/sqrt N) sum_n x_n exp(-2 pi i n k / N), through the N/2-point FFT of z_m = x_2m + i x_2m+1.
template <int LOGN>
__device__ __forceinline__ void rfft_fwd(const double (&x)[1 << LOGN], Cplx (&X)[(1 << LOGN) / 2 + 1], double hs) {
  constexpr int N = 1 << LOGN, M = N / 2;
  Cplx z[M];
#pragma unroll
  for (int m = 0; m < M; ++m) z[m] = {x[2 * m], x[2 * m + 1]};
  Dft<M, -1>::run(z);
  X[0] = {(z[0].re + z[0].im) * (2.0 * hs), 0.0};
  X[M] = {(z[0].re - z[0].im) * (2.0 * hs), 0.0};
#pragma unroll
  for (int k = 1; k < M; ++k) {
    const Cplx a = z[k], b = z[M - k];
    const Cplx E = {a.re + b.re, a.im - b.im};   // Z_k + conj Z_{M-k}
    const Cplx O = {a.im + b.im, b.re - a.re};   // (Z_k - conj Z_{M-k}) / i
    const Cplx w = root16(k * (16 / N));
    const Cplx W = {w.re, -w.im};                // exp(-2 pi i k / N)
    X[k] = {fma(W.re, O.re, fma(-W.im, O.im, E.re)) * hs, fma(W.re, O.im, fma(W.im, O.re, E.im)) * hs};
  }
}

// Inverse of rfft_fwd without the 1/sqrt N: x_n = sum over the full Hermitian spectrum of Q_k exp(+2 pi i n k / N)
template <int LOGN>
__device__ __forceinline__ void rfft_inv(const Cplx (&Q)[(1 << LOGN) / 2 + 1], double (&x)[1 << LOGN]) {
  constexpr int N = 1 << LOGN, M = N / 2;
  Cplx z[M];
#pragma unroll
  for (int k = 0; k < M; ++k) {
    const Cplx a = Q[k], b = {Q[M - k].re, -Q[M - k].im};  // conj Q_{M-k}
    const Cplx E = cadd_(a, b), D = csub_(a, b);
    const Cplx w = root16(k * (16 / N));                    // exp(+2 pi i k / N)
    const Cplx O = (k == 0) ? D : cmul(D, w);
    z[k] = {E.re - O.im, E.im + O.re};                      // E + i O
  }
  Dft<M, +1>::run(z);
#pragma unroll
  for (int m = 0; m < M; ++m) {
    x[2 * m] = z[m].re;
    x[2 * m + 1] = z[m].im;
  }
}

template <int LOGN>
struct RowShape {
  static constexpr int N = 1 << LOGN, NF = N / 2 + 1;
  static constexpr int NTS = ((NF * RW_LANES + 31) / 32) * 32;  // solver threads
  static constexpr int NT = NTS > RW_RB ? NTS : RW_RB;
#ifndef KLE_CGC_ROW_MINB
#define KLE_CGC_ROW_MINB 4  // N = 16 (160 threads): 96 registers, no spills: 1.63 ms per 131k c4 launch;
                            // 5 CTAs/SM (80 registers, 304 B spills): 2.22 ms
#endif
  static constexpr int MINB = NT > 128 ? KLE_CGC_ROW_MINB : 5;
  static constexpr size_t SMEM = sizeof(double) * ((size_t)4 * NF * RW_RB + RW_RB + 2 + N + 8);
};

template <int LOGN>
__global__ void __launch_bounds__(RowShape<LOGN>::NT, RowShape<LOGN>::MINB)
    cgc_row_kernel(CgcArgs a, const double* __restrict__ sfac_d) {
  using K = RowShape<LOGN>;
  constexpr int N = K::N, NF = K::NF, NT = K::NT, RB = RW_RB, MR = RW_MR;
  const int s = blockIdx.x;
  if (a.status && a.status[s] != KLE_SAMPLE_ACTIVE) return;
  extern __shared__ __align__(16) double smem[];
  Cplx* spec = reinterpret_cast<Cplx*>(smem);  // [NF][RB] half spectra, then the solutions
  Cplx* piv = spec + NF * RB;                  // [NF][RB] pivots 1/beta
  double* offs = reinterpret_cast<double*>(piv + NF * RB);  // [RB + 2]: dT*off[row-1 .. ]: offs[e] couples rows e-1, e
  double* isc = offs + RB + 2;                 // [N]
  double* red = isc + N;                       // [8]
  const int tid = threadIdx.x, nx = a.nx;
  const size_t sb = (size_t)s * N * nx;

  // ---- requests: this row's R values (registers), the pivots (cp.async), the off-diagonal ----
  double x[N];
  const bool rowt = tid < RB && tid < nx;
  if (rowt) {
#pragma unroll
    for (int n = 0; n < N; ++n) x[n] = a.R[sb + (size_t)n * nx + tid];
  } else {
#pragma unroll
    for (int n = 0; n < N; ++n) x[n] = 0.0;
  }
  {
    const Cplx* src = reinterpret_cast<const Cplx*>(sfac_d) + (size_t)s * NF * nx;
    for (int e = tid; e < NF * RB; e += NT) {
      const int ff = e / RB, r = e % RB;
      Cplx* dst = &piv[ff * RB + rswz(r)];
      if (r < nx) cp_async16_(dst, src + (size_t)ff * nx + r);
      else *dst = {1.0, 0.0};
    }
    asm volatile("cp.async.commit_group;\n" ::);
  }
  for (int e = tid; e < RB + 2; e += NT) {
    const int row = e - 1;  // offs[e] couples rows row and row + 1
    offs[e] = (row >= 0 && row + 1 < nx) ? a.dT * a.off[(size_t)s * nx + row] : 0.0;
  }
  if (tid < N) isc[tid] = a.inv_scaling[tid];
  // ---- forward real FFT in registers, half spectrum to shared memory ----
  if (tid < RB) {
    if (a.load_scale) {  // stand-alone three-step: r is not alpha-scaled yet
#pragma unroll
      for (int n = 0; n < N; ++n) x[n] *= a.load_scale[n];
    }
    Cplx X[NF];
    rfft_fwd<LOGN>(x, X, 0.5 / sqrt((double)N));
    const int pos = rswz(tid);
#pragma unroll
    for (int f = 0; f < NF; ++f) spec[f * RB + pos] = X[f];
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();

  // ---- one frequency per 16-lane group: (lambda_f I + dT A) q = p_f ----
  {
    const int fsys = tid / RW_LANES, k = tid % RW_LANES;
    const bool valid = fsys < NF;
    const int f = valid ? fsys : NF - 1;
    const int r0 = k * MR;
    const int kx = k & 7;
    Cplx* sp = spec + f * RB + r0;       // row r0 + j at sp[j ^ kx]
    const Cplx* pp = piv + f * RB + r0;  // pivot of row r0 + j at pp[j ^ kx]
    const Cplx pvm = (k > 0) ? piv[f * RB + rswz(r0 - 1)] : Cplx{0.0, 0.0};
    Cplx y[MR];
#pragma unroll
    for (int j = 0; j < MR; ++j) y[j] = sp[j ^ kx];
    // l_r = dT off_{r-1} / beta_{r-1}, formed where used
    auto lj = [&](int j) -> Cplx {
      const double E = offs[r0 + j];  // couples rows r0+j-1 and r0+j
      const Cplx ip = (j == 0) ? pvm : pp[(j - 1) ^ kx];
      return {E * ip.re, E * ip.im};
    };
    Cplx A = {1.0, 0.0};
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      const Cplx l = lj(j);
      if (j > 0) y[j] = cfma_({-l.re, -l.im}, y[j - 1], y[j]);
      A = cneg_mul_(l, A);
    }
    Cplx B = y[MR - 1];
#pragma unroll
    for (int d = 1; d < RW_LANES; d <<= 1) {
      const Cplx Ao = shfl_up16(A, d), Bo = shfl_up16(B, d);
      if (k >= d) {
        B = cfma_(A, Bo, B);
        A = cmul(A, Ao);
      }
    }
    Cplx Cin = shfl_up16(B, 1);  // true y of the row before this chunk
    if (k == 0) Cin = {0.0, 0.0};
    {
      Cplx pi = {1.0, 0.0};
#pragma unroll
      for (int j = 0; j < MR; ++j) {
        pi = cneg_mul_(lj(j), pi);
        y[j] = cmul(cfma_(pi, Cin, y[j]), pp[j ^ kx]);
      }
    }
    const double En = offs[r0 + MR];  // couples the lane's last row and the next
    const Cplx ibl = pp[(MR - 1) ^ kx];
    const Cplx lnext = {En * ibl.re, En * ibl.im};
    Cplx S = {1.0, 0.0};
#pragma unroll
    for (int j = MR - 1; j >= 0; --j) {
      const Cplx ln = (j == MR - 1) ? lnext : lj(j + 1);
      if (j < MR - 1) y[j] = cfma_({-ln.re, -ln.im}, y[j + 1], y[j]);
      S = cneg_mul_(ln, S);
    }
    Cplx T = y[0];
#pragma unroll
    for (int d = 1; d < RW_LANES; d <<= 1) {
      const Cplx So = shfl_down16(S, d), To = shfl_down16(T, d);
      if (k + d < RW_LANES) {
        T = cfma_(S, To, T);
        S = cmul(S, So);
      }
    }
    Cplx Xin = shfl_down16(T, 1);  // true q of the row after this chunk
    if (k == RW_LANES - 1) Xin = {0.0, 0.0};
    {
      Cplx sg = {1.0, 0.0};
#pragma unroll
      for (int j = MR - 1; j >= 0; --j) {
        const Cplx ln = (j == MR - 1) ? lnext : lj(j + 1);
        sg = cneg_mul_(ln, sg);
        y[j] = cfma_(sg, Xin, y[j]);
      }
    }
    if (valid) {
#pragma unroll
      for (int j = 0; j < MR; ++j) sp[j ^ kx] = y[j];
    }
  }
  // the old values of this row, requested before the barrier (out may alias U: loads precede the stores)
  const bool track = a.U != nullptr;
  double uo[N];
  if (rowt && track) {
#pragma unroll
    for (int n = 0; n < N; ++n) uo[n] = a.U[sb + (size_t)n * nx + tid];
  } else {
#pragma unroll
    for (int n = 0; n < N; ++n) uo[n] = 0.0;
  }
  __syncthreads();

  // ---- inverse FFT in registers, update, increment ----
  double incmax = 0.0;
  bool bad = false;  // fmax drops NaN; remember it separately (a NaN increment must not converge)
  if (rowt) {
    Cplx Q[NF];
    const int pos = rswz(tid);
#pragma unroll
    for (int f = 0; f < NF; ++f) Q[f] = spec[f * RB + pos];
    rfft_inv<LOGN>(Q, x);
    const double rsN = 1.0 / sqrt((double)N);
    double* __restrict__ out = a.Uout ? a.Uout : a.U;
#pragma unroll
    for (int n = 0; n < N; ++n) {
      const double u = (x[n] * rsN) * isc[n];
      if (track) {
        const double d = fabs(u - uo[n]);
        incmax = fmax(incmax, d);
        bad |= (d != d);
      }
      out[sb + (size_t)n * nx + tid] = u;
    }
  }
  if (__syncthreads_or(bad)) incmax = __longlong_as_double(0x7ff8000000000000LL);
  incmax = warp_max(incmax);
  const int lane = tid & 31, w = tid >> 5;
  constexpr int NW = NT / 32;
  if (lane == 0) red[w] = incmax;
  __syncthreads();
  if (tid == 0) {
    double inc = 0.0;
    for (int i = 0; i < NW; ++i) inc = nanmax(inc, red[i]);
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

template <int LOGN>
int launch_row(const CgcArgs& a, const double* sfac, cudaStream_t st) {
  using K = RowShape<LOGN>;
  auto kern = cgc_row_kernel<LOGN>;
  static PerDeviceOnce attr_once;
  if (int rc = once_per_device(attr_once, "kle_cgc_row: cudaFuncSetAttribute", [&] {
        return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::SMEM);
      }))
    return rc;
  kern<<<(unsigned)a.M, K::NT, K::SMEM, st>>>(a, sfac);
  return check_launch("cgc_row_kernel");
}

}  // namespace

bool cgc_row_supported(int N, int nx) {
  const char* env = getenv("KLE_CGC_ROW");  // 0: keep the cluster kernel for these shapes (A/B; read per call)
  if (env && *env && atoi(env) == 0) return false;
  return N >= 2 && N <= 16 && (N & (N - 1)) == 0 && nx >= 1 && nx <= RW_RB;
}

int cgc_row_run(const CgcArgs& a, const double* sfac, cudaStream_t st) {
  if (a.M <= 0) return KLE_OK;
  if (a.imag) cudaMemsetAsync(a.imag, 0, sizeof(double) * a.M, st);  // real by construction
  switch (a.N) {
    case 2: return launch_row<1>(a, sfac, st);
    case 4: return launch_row<2>(a, sfac, st);
    case 8: return launch_row<3>(a, sfac, st);
    case 16: return launch_row<4>(a, sfac, st);
  }
  return set_error(KLE_ERR_UNSUPPORTED, "cgc_row: N");
}

}  // namespace kle
