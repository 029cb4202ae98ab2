// Diagonalised coarse-grid correction (alpha-circulant three-step solve).
//
// Reference counterparts:
//   three_step_solve   pintuq/pcgc.py:148-172
//   factor_shifted     pintuq/pcgc.py:90-145 (banded branch 112-135)
//   forward/inverse_dft pintuq/pcgc.py:79-87   (np.fft, norm="ortho")
//   pcgc_solve stop    pintuq/pcgc.py:335-348  (increment = max|U_new - U|)
//
// One CTA processes one sample at a time (persistent loop over samples):
//   phase 1  p = F*(R) along the time axis for every spatial column
//            (R is already alpha-scaled by the fused F kernel), keeping the
//            non-redundant half spectrum f = 0..N/2 (R is real, so
//            p_{N-f} = conj(p_f) and lambda_{N-f} = conj(lambda_f) give
//            q_{N-f} = conj(q_f): half the shifted solves);
//   phase 2  q_f = (lambda_f I + dT A)^{-1} p_f, one thread per frequency,
//            pivot-free complex LDL^T factorised on the fly (Re lambda_f >=
//            1 - alpha^{1/N} > 0 and A is an M-matrix);
//   phase 3  u = diag(1/scaling) F(q) (Hermitian completion), U^{k+1} = Re u,
//            increment / imaginary-residue reductions, per-sample stop test.
#include <cmath>
#include <cstdlib>

#include "kle_common.cuh"
#include "kle_internal.h"

namespace kle {

constexpr int CGC_NT = 256;

__device__ __forceinline__ Cplx cadd(Cplx a, Cplx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ Cplx csub(Cplx a, Cplx b) { return {a.re - b.re, a.im - b.im}; }

// In-place radix-2 DIT over a [N][TC] tile whose rows were loaded in
// bit-reversed order; tw[j] = exp(-2 pi i j / N). inverse: conjugate twiddles.
__device__ void fft_tile(Cplx* t, const Cplx* tw, int N, int TC, bool inverse) {
  for (int len = 2; len <= N; len <<= 1) {
    const int half = len >> 1, step = N / len;
    const int nbf = (N >> 1) * TC;
    for (int b = threadIdx.x; b < nbf; b += CGC_NT) {
      const int c = b % TC, bf = b / TC;
      const int g = bf / half, j = bf - g * half;
      const int i0 = g * len + j, i1 = i0 + half;
      Cplx w = tw[j * step];
      if (inverse) w.im = -w.im;
      const Cplx x0 = t[i0 * TC + c];
      const Cplx v = cmul(t[i1 * TC + c], w);
      t[i0 * TC + c] = cadd(x0, v);
      t[i1 * TC + c] = csub(x0, v);
    }
    __syncthreads();
  }
}

// Bluestein's chirp-z transform for N that is not a power of two (the
// reference's np.fft handles every N, pintuq/pcgc.py:79-87): with the chirp
// c_n = exp(-i pi n^2 / N),
//   sum_n x_n exp(-2 pi i n k / N) = c_k (a * b)_k,   a_n = x_n c_n,  b_m = conj(c_m),
// a circular convolution of length Mb = 2^ceil(log2(2N - 1)) done with radix-2
// FFTs of size Mb (B^ = FFT(b) precomputed per CTA); the inverse sign uses the
// conjugate chirps, whose kernel transform is conj(B^[-k]). On entry the tile
// ([Mb][TC]) holds a in bit-reversed row order, zero padded; on exit it holds
// Mb (a * b) in natural order. O(N log N) per column instead of the O(N^2)
// direct sum.
__device__ void bluestein_conv(Cplx* t, const Cplx* twM, const Cplx* Bhat, int Mb, int log2Mb, int TC,
                               bool inverse) {
  fft_tile(t, twM, Mb, TC, false);
  for (int e = threadIdx.x; e < Mb * TC; e += CGC_NT) {  // pointwise product with the kernel transform
    const int k = e / TC;
    Cplx b = Bhat[inverse ? ((Mb - k) & (Mb - 1)) : k];
    if (inverse) b.im = -b.im;
    t[e] = cmul(t[e], b);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < Mb * TC; e += CGC_NT) {  // in-place bit reversal of the rows
    const int k = e / TC, c = e - k * TC;
    const int r = (int)(__brev((unsigned)k) >> (32 - log2Mb));
    if (k < r) {
      const Cplx u = t[k * TC + c];
      t[k * TC + c] = t[r * TC + c];
      t[r * TC + c] = u;
    }
  }
  __syncthreads();
  fft_tile(t, twM, Mb, TC, true);
}

__device__ __forceinline__ double block_max(double v, double* red) {
  v = warp_max(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) red[w] = v;
  __syncthreads();
  double r = red[0];
  for (int i = 1; i < CGC_NT / 32; ++i) r = nanmax(r, red[i]);
  __syncthreads();
  return r;
}

// a.full (the max_imag_residue diagnostic of three_step_solve, pintuq/pcgc.py:
// 170-172): the transform keeps all N frequencies, all N shifted systems are
// solved independently and u = diag(1/scaling) F q is formed without Hermitian
// completion, as the reference does; the rounding asymmetry between f and N - f
// (amplified up to cond(V) = alpha^{-(N-1)/N} by the unscaling) is what
// max|Im u| measures. Only imag is written.
__global__ void __launch_bounds__(CGC_NT) cgc_kernel(CgcArgs a, int TC, int log2N) {
  extern __shared__ double sm[];
  const int N = a.N, nx = a.nx, NF = a.full ? N : N / 2 + 1;
  const bool pow2 = log2N >= 0;
  const bool direct = log2N == -2;  // other N whose Bluestein tables do not fit: O(N^2) direct DFT
  const bool blue = !pow2 && !direct;
  // non-power-of-two N: Bluestein with transforms of size Mb (tile rows)
  int log2Mb = 0;
  while ((1 << log2Mb) < 2 * N - 1) ++log2Mb;
  const int Mb = blue ? (1 << log2Mb) : N, TR = Mb;
  Cplx* tw = reinterpret_cast<Cplx*>(sm);
  Cplx* tile = tw + N;
  Cplx* twM = tile + (size_t)TR * TC;        // [Mb] (Bluestein)
  Cplx* chirp = twM + (blue ? Mb : 0);       // [N]
  Cplx* Bhat = chirp + (blue ? N : 0);       // [Mb]
  double* red = reinterpret_cast<double*>(Bhat + (blue ? Mb : 0));
  for (int j = threadIdx.x; j < N; j += CGC_NT) {
    double sn, cs;
    sincospi(-2.0 * (double)j / (double)N, &sn, &cs);
    tw[j] = {cs, sn};
  }
  if (blue) {
    for (int j = threadIdx.x; j < Mb; j += CGC_NT) {
      double sn, cs;
      sincospi(-2.0 * (double)j / (double)Mb, &sn, &cs);
      twM[j] = {cs, sn};
    }
    for (int n = threadIdx.x; n < N; n += CGC_NT) {  // c_n = exp(-i pi n^2 / N), n^2 reduced mod 2N
      double sn, cs;
      sincospi(-(double)(((long long)n * n) % (2LL * N)) / (double)N, &sn, &cs);
      chirp[n] = {cs, sn};
    }
    __syncthreads();
    // B^ = FFT_Mb(b), b_m = conj(c_|m|) for |m| < N (circular), computed once in column 0 of the tile
    for (int e = threadIdx.x; e < Mb * TC; e += CGC_NT) tile[e] = {0.0, 0.0};
    __syncthreads();
    for (int m = threadIdx.x; m < Mb; m += CGC_NT) {
      const int d = m < N ? m : (Mb - m < N ? Mb - m : -1);
      const Cplx v = d >= 0 ? Cplx{chirp[d].re, -chirp[d].im} : Cplx{0.0, 0.0};
      tile[(int)(__brev((unsigned)m) >> (32 - log2Mb)) * TC] = v;
    }
    __syncthreads();
    fft_tile(tile, twM, Mb, TC, false);
    for (int k = threadIdx.x; k < Mb; k += CGC_NT) Bhat[k] = tile[k * TC];
  }
  __syncthreads();
  const double rMb = 1.0 / (double)Mb;
  const double rsN = 1.0 / sqrt((double)N);
  Cplx* pbuf = reinterpret_cast<Cplx*>(a.scratch + (size_t)blockIdx.x * a.scratch_doubles_per_cta);
  Cplx* ibuf = pbuf + (size_t)nx * NF;

  for (int s = blockIdx.x; s < a.M; s += gridDim.x) {
    if (a.status && a.status[s] != KLE_SAMPLE_ACTIVE) continue;
    const size_t sb = (size_t)s * N * nx;
    // ---------------- phase 1: forward transform --------------------------
    for (int c0 = 0; c0 < nx; c0 += TC) {
      const int tc = min(TC, nx - c0);
      if (blue)
        for (int e = threadIdx.x; e < TR * TC; e += CGC_NT) tile[e] = {0.0, 0.0};
      __syncthreads();
      for (int idx = threadIdx.x; idx < N * TC; idx += CGC_NT) {
        const int n = idx / TC, c = idx - n * TC;
        double v = 0.0;
        if (c < tc) {
          v = a.R[sb + (size_t)n * nx + c0 + c];
          if (a.load_scale) v *= a.load_scale[n];
        }
        if (!blue) {
          const int pos = log2N > 0 ? (int)(__brev((unsigned)n) >> (32 - log2N)) : n;
          tile[pos * TC + c] = {v, 0.0};
        } else {  // a_n = x_n c_n, bit-reversed over Mb rows
          tile[(int)(__brev((unsigned)n) >> (32 - log2Mb)) * TC + c] = {v * chirp[n].re, v * chirp[n].im};
        }
      }
      __syncthreads();
      if (pow2 && N > 1) fft_tile(tile, tw, N, TC, false);
      if (blue) bluestein_conv(tile, twM, Bhat, Mb, log2Mb, TC, false);
      for (int idx = threadIdx.x; idx < tc * NF; idx += CGC_NT) {
        const int c = idx / NF, f = idx - c * NF;
        Cplx v = tile[f * TC + c];
        if (blue) {  // X_f = c_f (a * b)_f
          v = cmul(chirp[f], v);
          v = {v.re * rMb, v.im * rMb};
        } else if (direct) {
          v = {0.0, 0.0};
          for (int n = 0; n < N; ++n) v = cadd(v, cmul(tile[n * TC + c], tw[(int)(((long long)n * f) % N)]));
        }
        pbuf[(size_t)(c0 + c) * NF + f] = {v.re * rsN, v.im * rsN};
      }
      __syncthreads();
    }
    // ---------------- phase 2: shifted tridiagonal solves -----------------
    const double* dd = a.dia + (size_t)s * nx;
    const double* ee = a.off + (size_t)s * nx;
    for (int f = threadIdx.x; f < NF; f += CGC_NT) {
      const Cplx lam = {a.lam[2 * f], a.lam[2 * f + 1]};
      Cplx y = {0.0, 0.0}, ib = {0.0, 0.0};
      for (int i = 0; i < nx; ++i) {
        const Cplx D = {fma(a.dT, dd[i], lam.re), lam.im};
        const Cplx p = pbuf[(size_t)i * NF + f];
        Cplx beta = D;
        if (i > 0) {
          const double E = a.dT * ee[i - 1];
          const Cplx l = {E * ib.re, E * ib.im};
          beta = {fma(-l.re, E, D.re), fma(-l.im, E, D.im)};
          y = csub(p, cmul(l, y));
        } else {
          y = p;
        }
        ib = crcp(beta);
        pbuf[(size_t)i * NF + f] = y;
        ibuf[(size_t)i * NF + f] = ib;
      }
      Cplx x = {0.0, 0.0};
      for (int i = nx - 1; i >= 0; --i) {
        const Cplx yy = pbuf[(size_t)i * NF + f];
        const Cplx bi = ibuf[(size_t)i * NF + f];
        const Cplx z = cmul(yy, bi);
        if (i < nx - 1) {
          const double E = a.dT * ee[i];
          const Cplx ln = {E * bi.re, E * bi.im};
          x = csub(z, cmul(ln, x));
        } else {
          x = z;
        }
        pbuf[(size_t)i * NF + f] = x;
      }
    }
    __syncthreads();
    // ---------------- phase 3: inverse transform + update -----------------
    double incmax = 0.0, immax = 0.0;
    for (int c0 = 0; c0 < nx; c0 += TC) {
      const int tc = min(TC, nx - c0);
      if (blue)
        for (int e = threadIdx.x; e < TR * TC; e += CGC_NT) tile[e] = {0.0, 0.0};
      __syncthreads();
      for (int idx = threadIdx.x; idx < N * TC; idx += CGC_NT) {
        const int c = idx / N, n = idx - c * N;
        Cplx v = {0.0, 0.0};
        if (c < tc) {
          if (a.full || n < NF) {
            v = pbuf[(size_t)(c0 + c) * NF + n];
          } else {
            const Cplx w = pbuf[(size_t)(c0 + c) * NF + (N - n)];
            v = {w.re, -w.im};
          }
        }
        if (!blue) {
          const int pos = log2N > 0 ? (int)(__brev((unsigned)n) >> (32 - log2N)) : n;
          tile[pos * TC + c] = v;
        } else {  // inverse sign: a_f = V_f conj(c_f)
          tile[(int)(__brev((unsigned)n) >> (32 - log2Mb)) * TC + c] = cmul(v, Cplx{chirp[n].re, -chirp[n].im});
        }
      }
      __syncthreads();
      if (pow2 && N > 1) fft_tile(tile, tw, N, TC, true);
      if (blue) bluestein_conv(tile, twM, Bhat, Mb, log2Mb, TC, true);
      for (int idx = threadIdx.x; idx < N * TC; idx += CGC_NT) {
        const int n = idx / TC, c = idx - n * TC;
        if (c >= tc) continue;
        Cplx v = tile[n * TC + c];
        if (blue) {  // X_n = conj(c_n) (a * conj b)_n
          v = cmul(Cplx{chirp[n].re, -chirp[n].im}, v);
          v = {v.re * rMb, v.im * rMb};
        } else if (direct) {
          v = {0.0, 0.0};
          for (int f = 0; f < N; ++f) {
            Cplx w = tw[(int)(((long long)n * f) % N)];
            w.im = -w.im;
            v = cadd(v, cmul(tile[f * TC + c], w));
          }
        }
        const double isc = a.inv_scaling[n];
        const double u = (v.re * rsN) * isc;
        const double ui = (v.im * rsN) * isc;
        const size_t g = sb + (size_t)n * nx + c0 + c;
        if (a.full) {
          immax = nanmax(immax, fabs(ui));
          continue;
        }
        if (a.Uout) {
          if (a.U) incmax = nanmax(incmax, fabs(u - a.U[g]));
          a.Uout[g] = u;
        } else {
          incmax = nanmax(incmax, fabs(u - a.U[g]));
          a.U[g] = u;
        }
        immax = nanmax(immax, fabs(ui));
      }
      __syncthreads();
    }
    incmax = block_max(incmax, red);
    immax = block_max(immax, red);
    if (a.full) {
      if (threadIdx.x == 0 && a.imag) a.imag[s] = nanmax(a.imag[s], immax);
      continue;
    }
    if (threadIdx.x == 0) {
      if (a.inc) a.inc[s] = incmax;
      if (a.inc_hist) a.inc_hist[(size_t)s * a.max_iters + (a.k - 1)] = incmax;
      if (a.imag) a.imag[s] = nanmax(a.imag[s], immax);
      if (a.status) {
        int st = KLE_SAMPLE_ACTIVE;
        if (incmax <= a.tol) st = KLE_SAMPLE_CONVERGED;
        else if (!isfinite(incmax)) st = KLE_SAMPLE_NONFINITE;
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
}

static bool is_pow2(int N) { return N > 0 && (N & (N - 1)) == 0; }

static int bluestein_len(int N) {
  int m = 1;
  while (m < 2 * N - 1) m <<= 1;
  return m;
}

// Bluestein for N that is not a power of two, unless its tables (size-Mb
// twiddles and kernel transform, the chirp) and a one-column tile exceed the
// shared-memory budget (N > 1024): then the direct O(N^2) DFT
static bool use_bluestein(int N) {
  if (is_pow2(N)) return false;
  const size_t Mb = bluestein_len(N);
  return (size_t)N * sizeof(Cplx) + (3 * Mb + N) * sizeof(Cplx) + 32 * sizeof(double) <= 200 * 1024;
}

static int tile_rows(int N) { return use_bluestein(N) ? bluestein_len(N) : N; }

static int tile_cols(int N) {
  int tc = (use_bluestein(N) ? 4096 : 2048) / tile_rows(N);
  if (tc > 64) tc = 64;
  if (tc < 1) tc = 1;
  return tc;
}

static size_t cgc_smem_bytes(int N) {
  const size_t extra = use_bluestein(N) ? (size_t)(2 * tile_rows(N) + N) * sizeof(Cplx) : 0;  // twM, chirp, B^
  return (size_t)N * sizeof(Cplx) + (size_t)tile_rows(N) * tile_cols(N) * sizeof(Cplx) + extra +
         32 * sizeof(double);
}

// kernel transform mode: log2 N (power of two), -1 Bluestein, -2 direct DFT
static int transform_mode(int N) {
  if (is_pow2(N)) {
    int l = 0;
    while ((1 << l) < N) ++l;
    return l;
  }
  return use_bluestein(N) ? -1 : -2;
}

int cgc_grid(int M, int N, int nx) {
  int g = 148 * 4;
  // keep the per-CTA scratch slabs within a modest footprint for huge blocks
  const size_t slab = cgc_scratch_doubles_per_cta(N, nx) * sizeof(double);
  while (g > 148 && (size_t)g * slab > (size_t)8 << 30) g /= 2;
  return M < g ? (M > 0 ? M : 1) : g;
}

static bool use_large(int N, int nx) {
  static const char* env = getenv("KLE_CGC_LARGE");  // 0: on-the-fly kernel (A/B)
  return cgc_large_supported(N, nx) && !(env && env[0] == '0');
}

size_t cgc_scratch_doubles_per_cta(int N, int nx) {
  const size_t NF = (size_t)N / 2 + 1;
  return 4 * (size_t)nx * NF;  // p/y/q (complex) + inverse pivots (complex)
}

// The diagnostic keeps all N frequencies per sample: its slabs are twice the
// size, so it runs on as many CTAs as fit a 256 MB scratch budget (<= 148 * 4).
static int imag_grid(int M, int N, int nx) {
  const size_t slab = 4 * (size_t)nx * N * sizeof(double);
  size_t g = ((size_t)256 << 20) / (slab ? slab : 1);
  if (g > 148 * 4) g = 148 * 4;
  if (g < 1) g = 1;
  return M < (int)g ? (M > 0 ? M : 1) : (int)g;
}

size_t imag_residue_scratch_bytes(int M, int N, int nx) {
  if (M <= 0 || N <= 0 || nx <= 0) return 0;
  return (size_t)imag_grid(M, N, nx) * 4 * (size_t)nx * N * sizeof(double);
}

int cgc_run(const CgcArgs& a, cudaStream_t st) {
  if (a.N < 1 || a.nx < 1) return set_error(KLE_ERR_INVALID, "cgc: bad dims");
  if (use_large(a.N, a.nx)) return cgc_large_run(a, st);
  const int log2N = transform_mode(a.N);
  const int TC = tile_cols(a.N);
  const size_t smem = cgc_smem_bytes(a.N);
  static PerDeviceOnce attr_once;
  if (int rc = once_per_device(attr_once, "kle_cgc: cudaFuncSetAttribute", [&] {
        return cudaFuncSetAttribute(cgc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      }))
    return rc;
  const int grid = cgc_grid(a.M, a.N, a.nx);
  cgc_kernel<<<grid, CGC_NT, smem, st>>>(a, TC, log2N);
  return check_launch("cgc_kernel");
}

int imag_residue_run(const CgcArgs& a0, cudaStream_t st) {
  if (a0.N < 1 || a0.nx < 1) return set_error(KLE_ERR_INVALID, "imag_residue: bad dims");
  if (a0.M <= 0 || !a0.imag) return KLE_OK;
  CgcArgs a = a0;
  a.full = 1;
  a.U = nullptr;
  a.Uout = nullptr;
  // a.status, if given, only selects the active samples (full mode never writes it)
  const int log2N = transform_mode(a.N);
  a.scratch_doubles_per_cta = 4 * (size_t)a.nx * a.N;
  static PerDeviceOnce attr_once;
  if (int rc = once_per_device(attr_once, "kle_cgc(imag): cudaFuncSetAttribute", [&] {
        return cudaFuncSetAttribute(cgc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      }))
    return rc;
  cgc_kernel<<<imag_grid(a.M, a.N, a.nx), CGC_NT, cgc_smem_bytes(a.N), st>>>(a, tile_cols(a.N), log2N);
  return check_launch("cgc_kernel(imag residue)");
}

}  // namespace kle
