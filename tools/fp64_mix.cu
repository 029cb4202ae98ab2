// Microbenchmark: what does a SHFL / LDS / STS cost next to a DFMA stream on B200?
// One-warp CTAs, 8 per SM (the c4 fgr occupancy). Each loop iteration issues 64 independent-enough
// DFMAs (8 accumulators) and K "other" instructions on independent registers.
// Prints the DFMA pipe utilisation (2 cycles per warp-DFMA per SM sub-partition = 100%).
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND, int K>  // KIND 0: SHFL.32, 1: LDS.64, 2: STS.64 + LDS.64 pairs, 3: SHFL dependent on the DFMA results
__global__ void __launch_bounds__(32) mix(double* out, int iters, double a, double b) {
  __shared__ double sm[64];
  sm[threadIdx.x] = threadIdx.x;
  sm[threadIdx.x + 32] = 1.0;
  __syncwarp();
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  int sv[K > 0 ? K : 1];
#pragma unroll
  for (int j = 0; j < K; ++j) sv[j] = threadIdx.x + j;
  double lv[K > 0 ? K : 1] = {};
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sm) + 8 * threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
      // K others spread over the 8 groups
#pragma unroll
      for (int j = q; j < K; j += 8) {
        if (KIND == 0) sv[j] = __shfl_xor_sync(0xffffffffu, sv[j], 1 + (j & 3));
        if (KIND == 1) asm volatile("ld.shared.f64 %0, [%1];" : "=d"(lv[j]) : "r"(sa));
        if (KIND == 2) {
          asm volatile("st.shared.f64 [%0], %1;" ::"r"(sa), "d"(lv[j]));
          asm volatile("ld.shared.f64 %0, [%1];" : "=d"(lv[j]) : "r"(sa ^ 8));
        }
        if (KIND == 3) {
          const int lo = __shfl_xor_sync(0xffffffffu, __double2loint(acc[j & 7]), 1);
          sv[j] += lo;
        }
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
#pragma unroll
  for (int j = 0; j < K; ++j) s += sv[j] + lv[j];
  if (s == 1234.5) out[0] = s;
}

template <int KIND, int K>
void run(const char* name, int sms, double ghz, double* d) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000, blocks = sms * 8 * 4;
  mix<KIND, K><<<blocks, 32>>>(d, 10, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  mix<KIND, K><<<blocks, 32>>>(d, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  // per SM sub-partition: blocks/(sms*4) warps, each iters*64 DFMAs of 2 cycles
  const double pipe_cycles = (double)blocks / (sms * 4) * iters * 64 * 2;
  const double cycles = ms * 1e-3 * ghz * 1e9;
  printf("{\"kind\":\"%s\",\"others_per_64_dfma\":%d,\"ms\":%.3f,\"dfma_pipe_util\":%.3f,\"extra_cycles_per_other\":%.2f}\n", name, K, ms,
         pipe_cycles / cycles, K ? (cycles - pipe_cycles / 0.9) / ((double)blocks / (sms * 4) * iters * K) : 0.0);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  const double ghz = p.clockRate / 1e6;
  double* d;
  cudaMalloc(&d, 64);
  run<0, 0>("none", sms, ghz, d);
  run<0, 4>("shfl", sms, ghz, d);
  run<0, 8>("shfl", sms, ghz, d);
  run<0, 16>("shfl", sms, ghz, d);
  run<0, 32>("shfl", sms, ghz, d);
  run<3, 8>("shfl_of_dfma_result", sms, ghz, d);
  run<3, 16>("shfl_of_dfma_result", sms, ghz, d);
  run<1, 8>("lds", sms, ghz, d);
  run<1, 16>("lds", sms, ghz, d);
  run<1, 32>("lds", sms, ghz, d);
  run<2, 8>("sts+lds", sms, ghz, d);
  run<2, 16>("sts+lds", sms, ghz, d);
  return 0;
}
