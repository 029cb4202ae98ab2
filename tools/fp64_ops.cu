// Microbenchmark: DFMA pipe utilisation on B200 as a function of operand pattern, chain ILP and warps per SM
// sub-partition (one-warp CTAs). 100% = one warp-DFMA per 2 cycles per sub-partition.
#include <cstdio>
#include <cuda_runtime.h>

// MODE 0: acc = fma(acc, a, b) with a, b loop constants (two operands from the reuse cache)
// MODE 1: acc[i] = fma(x[i], y[i], acc[i]) with 3 distinct register operands per DFMA
// MODE 2: chain: acc[i] = fma(c[j], acc[i], x[i][j]) over 16 "rows" like the forward recurrence (ILP = chains)
template <int MODE, int ILP>
__global__ void __launch_bounds__(32) k(double* out, int iters, double a, double b) {
  double acc[ILP], x[ILP][4], y[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) {
    acc[i] = threadIdx.x * 1e-3 + i;
    y[i] = 1.0 + 1e-9 * (threadIdx.x + i);
#pragma unroll
    for (int j = 0; j < 4; ++j) x[i][j] = 1e-9 * (i + j + threadIdx.x);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 64 / ILP; ++q) {
#pragma unroll
      for (int i = 0; i < ILP; ++i) {
        if (MODE == 0) acc[i] = fma(acc[i], a, b);
        if (MODE == 1) acc[i] = fma(x[i][q & 3], y[i], acc[i]);
        if (MODE == 2) acc[i] = fma(y[(i + q) % ILP], acc[i], x[i][q & 3]);
        if (MODE == 3) acc[i] = fma(y[q % ILP], x[i][q & 3], acc[i]);   // operand A shared by ILP consecutive DFMAs
        if (MODE == 4) acc[i] = fma(x[i][q & 3], y[q % ILP], acc[i]);   // operand B shared
        if (MODE == 5) acc[i] = fma(y[q % ILP], acc[i], x[i][q & 3]);   // shared multiplier, accumulator in slot B (chain form)
        if (MODE == 6) acc[i] = fma(acc[i], y[q % ILP], y[(q + 1) % ILP]);  // two shared operands (scale + shift form)
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 1234.5) out[0] = s;
}

template <int MODE, int ILP>
void run(const char* name, int sms, double ghz, double* d, int warps_per_sm) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000, blocks = sms * warps_per_sm * 4;
  // occupancy limit through dynamic shared memory: 227 KB / warps_per_sm
  const int smem = warps_per_sm >= 16 ? 0 : (220 * 1024) / warps_per_sm - 1024;
  cudaFuncSetAttribute(k<MODE, ILP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<MODE, ILP><<<blocks, 32, smem>>>(d, 10, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  k<MODE, ILP><<<blocks, 32, smem>>>(d, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double pipe_cycles = (double)blocks / (sms * 4) * iters * 64 * 2;
  printf("{\"mode\":\"%s\",\"ilp\":%d,\"warps_per_sm\":%d,\"ms\":%.3f,\"dfma_pipe_util\":%.3f}\n", name, ILP, warps_per_sm, ms,
         pipe_cycles / (ms * 1e-3 * ghz * 1e9));
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  const double ghz = p.clockRate / 1e6;
  double* d;
  cudaMalloc(&d, 64);
  for (int w : {4, 8}) {
    run<0, 8>("const_operands", sms, ghz, d, w);
    run<1, 8>("three_registers", sms, ghz, d, w);
    run<1, 4>("three_registers", sms, ghz, d, w);
    run<2, 4>("chain", sms, ghz, d, w);
    run<2, 8>("chain", sms, ghz, d, w);
    run<3, 4>("shared_A", sms, ghz, d, w);
    run<3, 8>("shared_A", sms, ghz, d, w);
    run<4, 4>("shared_B", sms, ghz, d, w);
    run<5, 4>("shared_mult_chain", sms, ghz, d, w);
    run<5, 8>("shared_mult_chain", sms, ghz, d, w);
    run<6, 4>("two_shared", sms, ghz, d, w);
  }
  return 0;
}
