// Microbenchmark: DFMA pipe utilisation of the fine step's phases (register layout of fgr_kernel<16, 8, 4, 32>:
// x[4][16], l[16], inv[16] per lane), one-warp CTAs, 8 per SM. Variants of the loop order test how much the
// operand-reuse cache recovers (a DFMA with three distinct register operands takes 3 cycles, tools/fp64_ops.cu).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int MR = 16, R = 4;

template <int PH>
__global__ void __launch_bounds__(32, 8) k(double* out, const double* in, int iters) {
  double x[R][MR], l[MR], inv[MR], Y[R];
#pragma unroll
  for (int j = 0; j < MR; ++j) {
    l[j] = in[j] * 1e-3;
    inv[j] = 1.0 + in[j + 16] * 1e-3;
#pragma unroll
    for (int r = 0; r < R; ++r) x[r][j] = in[32 + r * 16 + j + threadIdx.x];
  }
#pragma unroll
  for (int r = 0; r < R; ++r) Y[r] = in[100 + r] * 1e-3;
  for (int it = 0; it < iters; ++it) {
    if (PH == 0) {  // forward chain, r inner
#pragma unroll
      for (int j = 1; j < MR; ++j)
#pragma unroll
        for (int r = 0; r < R; ++r) x[r][j] = fma(-l[j], x[r][j - 1], x[r][j]);
    }
    if (PH == 1) {  // stitch, r inner
#pragma unroll
      for (int j = 0; j < MR; ++j)
#pragma unroll
        for (int r = 0; r < R; ++r) x[r][j] = fma(l[j], Y[r], x[r][j]);
    }
    if (PH == 2) {  // stitch, boustrophedon over r: every DFMA shares an operand with its predecessor
#pragma unroll
      for (int j = 0; j < MR; ++j)
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          const int r = (j & 1) ? R - 1 - rr : rr;
          x[r][j] = fma(l[j], Y[r], x[r][j]);
        }
    }
    if (PH == 3) {  // stitch, j inner (Y[r] shared by 16 consecutive)
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int j = 0; j < MR; ++j) x[r][j] = fma(l[j], Y[r], x[r][j]);
    }
    if (PH == 4) {  // backward: scale + chain, r inner
#pragma unroll
      for (int j = MR - 1; j >= 0; --j)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          double z = fma(x[r][j], inv[j], Y[0]);
          if (j + 1 < MR) z = fma(-l[j], x[r][j + 1], z);
          x[r][j] = z;
        }
    }
    if (PH == 5) {  // backward: all scales of a row first, then its chain FMAs
#pragma unroll
      for (int j = MR - 1; j >= 0; --j) {
#pragma unroll
        for (int r = 0; r < R; ++r) x[r][j] = fma(x[r][j], inv[j], Y[0]);
        if (j + 1 < MR) {
#pragma unroll
          for (int r = 0; r < R; ++r) x[r][j] = fma(-l[j], x[r][j + 1], x[r][j]);
        }
      }
    }
    if (PH == 6) {  // forward chain with the accumulator as the multiplicand slot: x_j = fma(x_{j-1}, -l_j, x_j)
#pragma unroll
      for (int j = 1; j < MR; ++j)
#pragma unroll
        for (int r = 0; r < R; ++r) x[r][j] = fma(x[r][j - 1], -l[j], x[r][j]);
    }
  }
  double s = 0;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int j = 0; j < MR; ++j) s += x[r][j];
  if (s == 1234.5) out[0] = s;
}

template <int PH>
void run(const char* name, int ndfma, int sms, double ghz, double* d, const double* in) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2000, blocks = sms * 8 * 4;
  k<PH><<<blocks, 32>>>(d, in, 10);
  cudaEventRecord(e0);
  k<PH><<<blocks, 32>>>(d, in, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double cyc = ms * 1e-3 * ghz * 1e9;
  const double per = cyc / ((double)blocks / (sms * 4) * iters * ndfma);
  printf("{\"phase\":\"%s\",\"dfma_per_iter\":%d,\"cycles_per_dfma_per_subpartition\":%.3f,\"dfma_pipe_util\":%.3f}\n", name, ndfma, per, 2.0 / per);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  const double ghz = p.clockRate / 1e6;
  double *d, *in;
  cudaMalloc(&d, 64);
  cudaMalloc(&in, 4096);
  cudaMemset(in, 0, 4096);
  run<0>("fwd chain (r inner)", 60, sms, ghz, d, in);
  run<6>("fwd chain (accumulator first)", 60, sms, ghz, d, in);
  run<1>("stitch (r inner)", 64, sms, ghz, d, in);
  run<2>("stitch (boustrophedon)", 64, sms, ghz, d, in);
  run<3>("stitch (j inner)", 64, sms, ghz, d, in);
  run<4>("bwd (r inner, fused)", 124, sms, ghz, d, in);
  run<5>("bwd (scales then chain)", 124, sms, ghz, d, in);
  return 0;
}
