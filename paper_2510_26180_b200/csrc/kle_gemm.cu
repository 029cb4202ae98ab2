// FP64 tensor-core GEMM for the gPC surrogate evaluation:
//   U0[M][L] = bias[L] + Psi[M][K] * C[K][L]
// (surrogate_predict, pintuq/surrogate.py:321-333, batched over samples:
//  pred = mean + (sqrt(lam) * (H psi)) @ modes  ==  mean + psi @ (H^T diag(sqrt lam) G)).
//
// sm_100a has no tcgen05 kind::f64 (ptxas rejects it), so FP64 MMA is the
// DMMA path: mma.sync.aligned.m8n8k4.row.col.f64. CTA tile 64 x 128, 8 warps
// of 32 x 32 (4 x 4 DMMA tiles), K staged through shared memory in chunks of
// 8 with cp.async double buffering.
#include "kle_common.cuh"
#include "kle_internal.h"

namespace kle {

constexpr int GB_M = 64, GB_N = 128, GB_K = 8, G_NT = 256;
constexpr int AS_LD = GB_M + 4, BS_LD = GB_N + 4;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

// TB: B is given transposed, [L][K] row-major (C = bias + A B^T: Gram and
// projection products of the surrogate build, pintuq/surrogate.py:153, 183)
template <bool TB>
__global__ void __launch_bounds__(G_NT) gemm_bias_kernel(const double* __restrict__ A, const double* __restrict__ B,
                                                         const double* __restrict__ bias, double* __restrict__ C,
                                                         int M, int K, int L) {
  __shared__ double As[2][GB_K][AS_LD];
  __shared__ double Bs[2][GB_K][BS_LD];
  const int m0 = blockIdx.y * GB_M, n0 = blockIdx.x * GB_N;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 2) * 32, wn = (warp & 3) * 32;
  const int g = lane >> 2, t = lane & 3;

  auto load_stage = [&](int stage, int k0) {
    // A tile: GB_M x GB_K, stored transposed As[k][m]
    for (int idx = tid; idx < GB_M * GB_K; idx += G_NT) {
      const int m = idx / GB_K, kk = idx % GB_K;
      const int gm = m0 + m, gk = k0 + kk;
      const bool ok = gm < M && gk < K;
      cp_async8(&As[stage][kk][m], A + (ok ? (size_t)gm * K + gk : 0), ok);
    }
    for (int idx = tid; idx < GB_K * GB_N; idx += G_NT) {
      const int kk = TB ? idx % GB_K : idx / GB_N, n = TB ? idx / GB_K : idx % GB_N;
      const int gk = k0 + kk, gn = n0 + n;
      const bool ok = gk < K && gn < L;
      const size_t off = TB ? (size_t)gn * K + gk : (size_t)gk * L + gn;
      cp_async8(&Bs[stage][kk][n], B + (ok ? off : 0), ok);
    }
    cp_async_commit();
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = (K + GB_K - 1) / GB_K;
  load_stage(0, 0);
  for (int kc = 0; kc < nk; ++kc) {
    const int cur = kc & 1;
    cp_async_wait_all();
    __syncthreads();
    if (kc + 1 < nk) load_stage(cur ^ 1, (kc + 1) * GB_K);
#pragma unroll
    for (int k4 = 0; k4 < GB_K; k4 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[cur][k4 + t][wm + i * 8 + g];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bs[cur][k4 + t][wn + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
    __syncthreads();
  }
  // epilogue: C = bias + acc ; d0,d1 at (row g, cols 2t, 2t+1)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + wm + i * 8 + g;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = n0 + wn + j * 8 + 2 * t;
      const size_t o = (size_t)row * L + col;
      if (col + 1 < L && (o & 1) == 0) {  // the pair as one 16-byte store: full 64-byte row segments per warp
        const double2 bv = bias ? *reinterpret_cast<const double2*>(bias + col) : make_double2(0.0, 0.0);
        *reinterpret_cast<double2*>(C + o) = make_double2(bv.x + acc[i][j][0], bv.y + acc[i][j][1]);
      } else {
        if (col < L) C[o] = (bias ? bias[col] : 0.0) + acc[i][j][0];
        if (col + 1 < L) C[o + 1] = (bias ? bias[col + 1] : 0.0) + acc[i][j][1];
      }
    }
  }
}

int gemm_bias(const double* A, const double* B, const double* bias, double* C, int M, int K, int L,
              cudaStream_t st, bool trans_b) {
  if (M <= 0 || L <= 0) return KLE_OK;
  if (K <= 0) return set_error(KLE_ERR_INVALID, "gemm: K must be > 0");
  dim3 grid((L + GB_N - 1) / GB_N, (M + GB_M - 1) / GB_M);
  if (grid.y > 65535) return set_error(KLE_ERR_UNSUPPORTED, "gemm: M too large for one launch");
  if (trans_b) gemm_bias_kernel<true><<<grid, G_NT, 0, st>>>(A, B, bias, C, M, K, L);
  else gemm_bias_kernel<false><<<grid, G_NT, 0, st>>>(A, B, bias, C, M, K, L);
  return check_launch("gemm_bias_kernel");
}

// out[s][l] = X[s][l] - v[l] (snapshot fluctuations, pintuq/surrogate.py:63)
__global__ void sub_row_kernel(const double* __restrict__ X, const double* __restrict__ v, double* __restrict__ out,
                               int M, int L) {
  const size_t n = (size_t)M * L;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = X[i] - v[i % L];
}

int sub_row(const double* X, const double* v, double* out, int M, int L, cudaStream_t st) {
  if (M <= 0 || L <= 0) return KLE_OK;
  size_t blocks = ((size_t)M * L + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  sub_row_kernel<<<(unsigned)blocks, 256, 0, st>>>(X, v, out, M, L);
  return check_launch("sub_row_kernel");
}

}  // namespace kle
