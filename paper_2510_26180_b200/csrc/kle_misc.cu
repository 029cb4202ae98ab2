// Coefficient field, Hermite gPC basis, moments and small element-wise ops.
#include "kle_common.cuh"
#include "kle_internal.h"

namespace kle {

// a(m_j) = exp(sum_k table[k][j] xi_k) on the nx+1 midpoints, then the
// tridiagonal A (models.py LogNormalKL1D.tridiagonal; the reference plugin
// contract is pintuq/models.py:114-116). One CTA per sample.
__global__ void kl_tridiag_kernel(const double* __restrict__ xi, int d, const double* __restrict__ table,
                                  int nx, double inv_h2, double* __restrict__ dia, double* __restrict__ off) {
  extern __shared__ double a[];
  const int s = blockIdx.x;
  const double* x = xi + (size_t)s * d;
  for (int j = threadIdx.x; j <= nx; j += blockDim.x) {
    double la = 0.0;
    for (int k = 0; k < d; ++k) la = fma(table[(size_t)k * (nx + 1) + j], x[k], la);
    a[j] = exp(la);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nx; i += blockDim.x) {
    dia[(size_t)s * nx + i] = (a[i] + a[i + 1]) * inv_h2;
    off[(size_t)s * nx + i] = (i < nx - 1) ? -a[i + 1] * inv_h2 : 0.0;
  }
}

int kl_tridiag(const double* xi, int M, int d, const double* table, int nx, double inv_h2, double* dia,
               double* off, cudaStream_t st) {
  if (M <= 0) return KLE_OK;
  const size_t smem = (size_t)(nx + 1) * sizeof(double);
  if (smem > 200 * 1024) return set_error(KLE_ERR_UNSUPPORTED, "kl_tridiag: nx too large");
  static PerDeviceOnce attr_once;
  if (int rc = once_per_device(attr_once, "kle_misc: cudaFuncSetAttribute", [&] {
        return cudaFuncSetAttribute(kl_tridiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      }))
    return rc;
  kl_tridiag_kernel<<<M, 256, smem, st>>>(xi, d, table, nx, inv_h2, dia, off);
  return check_launch("kl_tridiag_kernel");
}

// Psi[s][col] = prod_d phi_{k_d}(map_d(xi_{s,d})) in gpc_multi_indices order:
// gpc_basis_matrix + _legendre_table / _hermite_table + ParameterMap.apply
// (pintuq/surrogate.py:208-248, pintuq/models.py:39-45), the same recurrences,
// normalisation and product order, every operation rounded separately (no FMA
// contraction) so the Hermite/Legendre tables and the affine map are
// bit-identical to numpy's. maps: optional [d][3] (kind, lo, hi), kind 0 =
// identity, 1 = affine onto [-1, 1], 2 = cos(2 pi v) (the device cos can differ
// from numpy's in the last bit).
constexpr int GPC_MAXDEG = 8;
constexpr int GPC_MAXDIM = 32;

__global__ void gpc_basis_kernel(const double* __restrict__ xi, int M, int d, int degree, int family,
                                 const double* __restrict__ maps, const int32_t* __restrict__ midx, int P,
                                 const double* __restrict__ norms, double* __restrict__ Psi) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= M) return;
  double T[GPC_MAXDIM][GPC_MAXDEG + 1];
  for (int k = 0; k < d; ++k) {
    double x = xi[(size_t)s * d + k];
    if (maps) {
      const int kind = (int)maps[3 * k];
      const double lo = maps[3 * k + 1], hi = maps[3 * k + 2];
      if (kind == 1) x = __dsub_rn(__ddiv_rn(__dmul_rn(2.0, __dsub_rn(x, lo)), __dsub_rn(hi, lo)), 1.0);
      else if (kind == 2) x = cos(__dmul_rn(2.0 * 3.141592653589793, x));
    }
    T[k][0] = 1.0;
    if (degree >= 1) T[k][1] = x;
    if (family == 0) {  // probabilists' Hermite: He_{q+1} = x He_q - q He_{q-1}
      for (int q = 1; q < degree; ++q)
        T[k][q + 1] = __dsub_rn(__dmul_rn(x, T[k][q]), __dmul_rn((double)q, T[k][q - 1]));
    } else {  // Legendre: P_{q+1} = ((2q+1) x P_q - q P_{q-1}) / (q+1)
      for (int q = 1; q < degree; ++q)
        T[k][q + 1] = __ddiv_rn(__dsub_rn(__dmul_rn(__dmul_rn((double)(2 * q + 1), x), T[k][q]),
                                          __dmul_rn((double)q, T[k][q - 1])),
                                (double)(q + 1));
    }
    for (int q = 0; q <= degree; ++q) T[k][q] = __dmul_rn(T[k][q], norms[q]);
  }
  for (int col = 0; col < P; ++col) {
    double b = 1.0;
    for (int k = 0; k < d; ++k) {
      const int kd = midx[col * d + k];
      if (kd) b = __dmul_rn(b, T[k][kd]);
    }
    Psi[(size_t)s * P + col] = b;
  }
}

int gpc_basis(const double* xi, int M, int d, int degree, int family, const double* maps, const int32_t* midx, int P,
              const double* norms, double* Psi, cudaStream_t st) {
  if (d > GPC_MAXDIM || degree > GPC_MAXDEG || degree < 0)
    return set_error(KLE_ERR_UNSUPPORTED, "gpc_basis: degree/dimension too large");
  if (family != 0 && family != 1) return set_error(KLE_ERR_INVALID, "gpc_basis: family must be 0 (Hermite) or 1 (Legendre)");
  if (M <= 0) return KLE_OK;
  gpc_basis_kernel<<<(M + 127) / 128, 128, 0, st>>>(xi, M, d, degree, family, maps, midx, P, norms, Psi);
  return check_launch("gpc_basis_kernel");
}

// Deterministic column sums over samples: out[l] = sum_s (U[s][l] - c[l])^p,
// p = 1 without a center, p = 2 with one (two-pass variance).
constexpr int CS_CHUNKS = 128;

// per (column l, chunk): four interleaved partial sums (samples s0 + 4 q + u go
// to accumulator u), so four loads per thread are in flight; combined in a
// fixed order, so the result is deterministic
__global__ void col_sum_partial_kernel(const double* __restrict__ U, int M, int L,
                                       const double* __restrict__ center, double* __restrict__ partial) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L) return;
  const int chunk = blockIdx.y, nch = gridDim.y;
  const int s0 = (int)(((long long)M * chunk) / nch), s1 = (int)(((long long)M * (chunk + 1)) / nch);
  const double c = center ? center[l] : 0.0;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  int s = s0;
  for (; s + 4 <= s1; s += 4) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldg(U + (size_t)(s + u) * L + l);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (center) {
        const double dv = v[u] - c;
        acc[u] = fma(dv, dv, acc[u]);
      } else {
        acc[u] += v[u];
      }
    }
  }
  for (int u = 0; s < s1; ++s, ++u) {
    const double v = __ldg(U + (size_t)s * L + l);
    if (center) {
      const double dv = v - c;
      acc[u] = fma(dv, dv, acc[u]);
    } else {
      acc[u] += v;
    }
  }
  partial[(size_t)chunk * L + l] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

__global__ void col_sum_final_kernel(const double* __restrict__ partial, int nch, int L, double* __restrict__ out) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L) return;
  double acc = 0.0;
  for (int c = 0; c < nch; ++c) acc += partial[(size_t)c * L + l];
  out[l] = acc;
}

size_t col_sum_partial_doubles(int M, int L) {
  const int nch = M < CS_CHUNKS ? (M > 0 ? M : 1) : CS_CHUNKS;
  return (size_t)nch * L;
}

int col_sum(const double* U, int M, int L, const double* center, double* out, double* partial, cudaStream_t st) {
  if (L <= 0) return KLE_OK;
  const int nch = M < CS_CHUNKS ? (M > 0 ? M : 1) : CS_CHUNKS;
  dim3 g1((L + 255) / 256, nch);
  col_sum_partial_kernel<<<g1, 256, 0, st>>>(U, M, L, center, partial);
  col_sum_final_kernel<<<(L + 255) / 256, 256, 0, st>>>(partial, nch, L, out);
  return check_launch("col_sum");
}

__global__ void axpby_kernel(const double* __restrict__ x, const double* __restrict__ y, double* __restrict__ o,
                             double a, double b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    o[i] = a * x[i] + b * y[i];
}

int axpby(const double* x, const double* y, double* out, double a, double b, size_t n, cudaStream_t st) {
  if (n == 0) return KLE_OK;
  size_t blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  axpby_kernel<<<(unsigned)blocks, 256, 0, st>>>(x, y, out, a, b, n);
  return check_launch("axpby_kernel");
}

// Error of the iterate against the serial fine reference, per subinterval
// (_error_record, pintuq/parareal.py:87-91: err_n = max_x |U_n - ref_n|,
// max_err = max_n err_n), and the stop_on="reference" test of pcgc_solve
// (pintuq/pcgc.py:312-316 for k = 0, :343-348 for k >= 1). One CTA per
// sample. A sample takes part at iteration k if it was active during it:
// status ACTIVE, or it terminated at this k (iters == k). With stop_ref the
// CGC ran with tol < 0 (the increment never stops a sample), and this kernel
// converges the samples whose max_err <= tol (fixing the active count).
__global__ void err_ref_kernel(const double* __restrict__ U, const double* __restrict__ ref, int N, int nx, int k,
                               int max_iters, double tol, int stop_ref, int32_t* __restrict__ status,
                               int32_t* __restrict__ iters, int32_t* __restrict__ active_count,
                               double* __restrict__ err_hist, double* __restrict__ max_err) {
  const int s = blockIdx.x;
  const int st0 = status[s];
  if (k > 0 && st0 != KLE_SAMPLE_ACTIVE && iters[s] != k) return;
  __shared__ double wmax[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const size_t base = (size_t)s * N * nx;
  double mine = 0.0;
  for (int n = w; n < N; n += nw) {
    const double* u = U + base + (size_t)n * nx;
    const double* r = ref + base + (size_t)n * nx;
    double e = 0.0;
    for (int i = lane; i < nx; i += 32) e = nanmax(e, fabs(__ldg(u + i) - __ldg(r + i)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e = nanmax(e, __shfl_xor_sync(KLE_FULL_MASK, e, o));
    if (lane == 0 && err_hist) err_hist[((size_t)s * (max_iters + 1) + k) * N + n] = e;
    mine = nanmax(mine, e);
  }
  if (lane == 0) wmax[w] = mine;
  __syncthreads();
  if (threadIdx.x != 0) return;
  double me = 0.0;
  for (int i = 0; i < nw; ++i) me = nanmax(me, wmax[i]);
  if (max_err) max_err[s] = me;
  if (!stop_ref) return;
  if (me <= tol) {  // NaN compares false
    status[s] = KLE_SAMPLE_CONVERGED;
    iters[s] = k;
    if (k > 0 && st0 == KLE_SAMPLE_ACTIVE && active_count) atomicSub(active_count, 1);
  } else if (k == 0) {
    if (me != me) {
      status[s] = KLE_SAMPLE_NONFINITE;
      iters[s] = 0;
    } else if (active_count) {
      atomicAdd(active_count, 1);
    }
  }
}

int err_ref(const double* U, const double* ref, int M, int N, int nx, int k, int max_iters, double tol, int stop_ref,
            int32_t* status, int32_t* iters, int32_t* active_count, double* err_hist, double* max_err,
            cudaStream_t st) {
  if (M <= 0) return KLE_OK;
  err_ref_kernel<<<M, 256, 0, st>>>(U, ref, N, nx, k, max_iters, tol, stop_ref, status, iters, active_count,
                                    err_hist, max_err);
  return check_launch("err_ref_kernel");
}

// ---------------------------------------------------------------------------
// Block DFT along the first axis (forward_dft / inverse_dft, pintuq/pcgc.py:
// 79-87): out[k][l] = sum_n in[n][l] exp(sign 2 pi i n k / N) / sqrt(N),
// sign = +1 for F (x) I (np.fft.ifft, norm="ortho"), -1 for F* (x) I
// (np.fft.fft). Direct O(N^2) per column (API utility, not the hot path:
// the CGC kernels fuse their own FFTs).
__global__ void block_dft_kernel(const Cplx* __restrict__ in, Cplx* __restrict__ out, int N, int L, int sign) {
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (t >= (size_t)N * L) return;
  const int k = (int)(t / L), l = (int)(t - (size_t)k * L);
  double re = 0.0, im = 0.0;
  for (int n = 0; n < N; ++n) {
    double sn, cs;
    sincospi((double)sign * 2.0 * (double)(((long long)n * k) % N) / (double)N, &sn, &cs);
    const Cplx v = in[(size_t)n * L + l];
    re += v.re * cs - v.im * sn;
    im += v.re * sn + v.im * cs;
  }
  const double r = 1.0 / sqrt((double)N);
  out[t] = {re * r, im * r};
}

int block_dft(const double* in, double* out, int N, int L, int sign, cudaStream_t st) {
  const size_t tot = (size_t)N * L;
  if (tot == 0) return KLE_OK;
  block_dft_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(reinterpret_cast<const Cplx*>(in),
                                                                  reinterpret_cast<Cplx*>(out), N, L, sign);
  return check_launch("block_dft_kernel");
}

// (lam I - dT J) q = p for nrhs right-hand sides, J = tridiag(sub, dia, sup)
// real (sub[i] = J[i+1][i], sup[i] = J[i][i+1]): the banded shifted solvers of
// factor_shifted (pintuq/pcgc.py:112-135), pivot-free complex Thomas, one
// thread per right-hand side. status[r] = 1 for a zero or non-finite pivot
// (the reference's SingularShiftError).
__global__ void shifted_tridiag_kernel(const double* __restrict__ sub, const double* __restrict__ dia,
                                       const double* __restrict__ sup, double lre, double lim, double dT,
                                       const Cplx* __restrict__ p, Cplx* __restrict__ q, Cplx* __restrict__ cwork,
                                       int nx, int nrhs, int32_t* __restrict__ status) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrhs) return;
  const Cplx* pr = p + (size_t)r * nx;
  Cplx* qr = q + (size_t)r * nx;
  Cplx* cp = cwork + (size_t)r * nx;
  bool bad = false;
  Cplx cprev = {0.0, 0.0}, dprev = {0.0, 0.0};
  for (int i = 0; i < nx; ++i) {
    const double a = i > 0 ? -dT * sub[i - 1] : 0.0;  // coupling to row i-1
    const double c = i < nx - 1 ? -dT * sup[i] : 0.0;  // coupling to row i+1
    const Cplx den = {lre - dT * dia[i] - a * cprev.re, lim - a * cprev.im};
    const double m2 = den.re * den.re + den.im * den.im;
    if (!(m2 > 0.0) || !isfinite(m2)) bad = true;
    const Cplx iden = crcp(den);
    const Cplx num = {pr[i].re - a * dprev.re, pr[i].im - a * dprev.im};
    dprev = cmul(num, iden);
    cprev = {c * iden.re, c * iden.im};
    cp[i] = cprev;
    qr[i] = dprev;
  }
  Cplx x = qr[nx - 1];
  for (int i = nx - 2; i >= 0; --i) {
    const Cplx cc = cp[i];
    x = {qr[i].re - (cc.re * x.re - cc.im * x.im), qr[i].im - (cc.re * x.im + cc.im * x.re)};
    qr[i] = x;
  }
  if (status) status[r] = bad ? 1 : 0;
}

int shifted_tridiag(const double* sub, const double* dia, const double* sup, double lre, double lim, double dT,
                    const double* p, double* q, double* cwork, int nx, int nrhs, int32_t* status, cudaStream_t st) {
  if (nx <= 0 || nrhs <= 0) return KLE_OK;
  shifted_tridiag_kernel<<<(nrhs + 127) / 128, 128, 0, st>>>(sub, dia, sup, lre, lim, dT,
                                                             reinterpret_cast<const Cplx*>(p),
                                                             reinterpret_cast<Cplx*>(q),
                                                             reinterpret_cast<Cplx*>(cwork), nx, nrhs, status);
  return check_launch("shifted_tridiag_kernel");
}

// Harness aggregation (pintuq/experiments.py:314-334): over the "good"
// samples (every recorded error vector finite), each sample's error vectors
// err_hist[s][0..K_s][:] (K_s = iters[s], records past the stop are NaN) are
// padded with their last record to k_max + 1 rows and averaged over samples.
// The sums run over samples in id order per (k, n) entry; divided once by
// n_good (by the caller) they are numpy's stack.mean(axis=0), bit for bit.
__global__ void err_good_kernel(const double* __restrict__ err, const int32_t* __restrict__ iters, int M, int N,
                                int K1, int32_t* __restrict__ good, int32_t* __restrict__ counts) {
  const int s = blockIdx.x * blockDim.y + threadIdx.y;
  if (s >= M) return;
  int K = iters[s];
  K = K < 0 ? 0 : (K >= K1 ? K1 - 1 : K);
  const double* e = err + (size_t)s * K1 * N;
  bool ok = true;
  for (int j = threadIdx.x; j < (K + 1) * N; j += 32) ok = ok && isfinite(e[j]);
  ok = __all_sync(KLE_FULL_MASK, ok);
  if (threadIdx.x == 0) {
    good[s] = ok ? 1 : 0;
    if (ok) {
      atomicAdd(&counts[0], 1);
      atomicMax(&counts[1], K);
    }
  }
}

__global__ void err_sum_kernel(const double* __restrict__ err, const int32_t* __restrict__ iters,
                               const int32_t* __restrict__ good, const int32_t* __restrict__ counts, int M, int N,
                               int K1, int k_pad, double* __restrict__ sums) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= K1 * N) return;
  const int k = j / N, n = j - k * N;
  const int kp = k_pad >= 0 ? k_pad : counts[1];
  if (k > kp) {
    sums[j] = __longlong_as_double(0x7ff8000000000000LL);
    return;
  }
  double acc = 0.0;
  for (int s = 0; s < M; ++s) {
    if (!good[s]) continue;
    int K = iters[s];
    K = K < 0 ? 0 : (K >= K1 ? K1 - 1 : K);
    acc += err[((size_t)s * K1 + (k < K ? k : K)) * N + n];
  }
  sums[j] = acc;
}

int err_aggregate(const double* err, const int32_t* iters, int M, int N, int max_iters, int k_pad, int32_t* good,
                  int32_t* counts, double* sums, cudaStream_t st) {
  const int K1 = max_iters + 1;
  cudaMemsetAsync(counts, 0, 2 * sizeof(int32_t), st);
  if (M > 0) err_good_kernel<<<(M + 7) / 8, dim3(32, 8), 0, st>>>(err, iters, M, N, K1, good, counts);
  err_sum_kernel<<<(K1 * N + 127) / 128, 128, 0, st>>>(err, iters, good, counts, M, N, K1, k_pad, sums);
  return check_launch("err_aggregate");
}

}  // namespace kle
