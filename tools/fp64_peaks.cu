// Microbenchmark: FP64 DFMA throughput/latency, DMMA (mma.sync m8n8k4 f64) throughput,
// SHFL throughput on B200 (sm_100a). Prints JSON lines. Used to ground the
// FP64 roofline denominators (MEASURED_PEAKS.json has no FP64 entry).
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void dfma_tput(double* out, int iters, double a, double b) {
  double acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 1234.5) out[0] = s;
}

__global__ void dfma_lat(double* out, long long* cyc, int iters, double a, double b) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) x = fma(x, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[1] = x; }
}

__global__ void dmma_tput(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[4][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
  if (s == 1234.5) out[0] = s;
}

__global__ void shfl_tput(double* out, int iters) {
  double x = threadIdx.x, y = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { y += __shfl_xor_sync(0xffffffffu, x, 1 << (j & 3)); x += 1e-9; }
  }
  if (y == 1234.5) out[0] = y;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int sms = p.multiProcessorCount;
  double* d; long long* c; cudaMalloc(&d, 64); cudaMalloc(&c, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // DFMA throughput
  {
    int iters = 20000; int blocks = sms * 8, threads = 256;
    dfma_tput<8><<<blocks, threads>>>(d, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_tput<8><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * (double)iters * blocks * threads;
    printf("{\"what\":\"dfma_tflops\",\"value\":%.3f,\"ms\":%.3f}\n", fl / ms / 1e9, ms);
  }
  {
    dfma_lat<<<1, 32>>>(d, c, 1000, 1.0000001, 1e-9);
    dfma_lat<<<1, 32>>>(d, c, 100000, 1.0000001, 1e-9);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("{\"what\":\"dfma_latency_cycles\",\"value\":%.2f}\n", h / 100000.0);
  }
  {
    int iters = 20000; int blocks = sms * 8, threads = 256;
    dmma_tput<<<blocks, threads>>>(d, 100);
    cudaEventRecord(e0);
    dmma_tput<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * 8 * 4 * 4 * (double)iters * blocks * (threads / 32);
    printf("{\"what\":\"dmma_tflops\",\"value\":%.3f,\"ms\":%.3f}\n", fl / ms / 1e9, ms);
  }
  {
    int iters = 20000; int blocks = sms * 8, threads = 256;
    shfl_tput<<<blocks, threads>>>(d, 100);
    cudaEventRecord(e0);
    shfl_tput<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double n = 2.0 * 8 * (double)iters * blocks * threads;  // 32-bit lane-shuffles
    printf("{\"what\":\"shfl32_lane_per_clk_per_sm\",\"value\":%.2f,\"assume_ghz\":%.3f}\n",
           n / (ms * 1e-3) / sms / (p.clockRate * 1e3), p.clockRate / 1e6);
  }
  printf("{\"what\":\"device\",\"name\":\"%s\",\"sms\":%d,\"clock_mhz\":%d,\"smem_optin\":%zu}\n",
         p.name, sms, p.clockRate / 1000, p.sharedMemPerBlockOptin);
  return 0;
}
