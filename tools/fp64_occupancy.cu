// DFMA throughput vs resident warps per SM and independent chains per thread,
// plus the same with a 5-stage shuffle scan interleaved (the fine-sweep shape).
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void chains(double* out, int iters, double a, double b) {
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

template <int ILP, int ROWS>
__global__ void chains_scan(double* out, int iters, double a, double b) {
  double acc[ILP];
  const int k = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int rr = 0; rr < ROWS; ++rr)
#pragma unroll
      for (int i = 0; i < ILP; ++i) acc[i] = fma(acc[i], a, b);
#pragma unroll
    for (int t = 0; t < 5; ++t)
#pragma unroll
      for (int i = 0; i < ILP; ++i) {
        const double o = __shfl_up_sync(0xffffffffu, acc[i], 1 << t);
        if (k >= (1 << t)) acc[i] = fma(a, o, acc[i]);
      }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 1234.5) out[0] = s;
}

template <class F>
float timeit(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaEventRecord(e0);
  f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  double* d;
  cudaMalloc(&d, 64);
  const int sms = 148, iters = 4000;
  for (int wps : {4, 8, 12, 16, 32}) {
    const int threads = 32 * wps;  // one CTA per SM
#define RUN(ILP)                                                                                  \
  {                                                                                               \
    float ms = timeit([&] { chains<ILP><<<sms, threads>>>(d, iters, 1.0000001, 1e-9); });       \
    double fl = 2.0 * ILP * (double)iters * sms * threads;                                        \
    printf("{\"kind\":\"chains\",\"warps_per_sm\":%d,\"ilp\":%d,\"tflops\":%.2f}\n", wps, ILP, fl / ms / 1e9); \
  }
    RUN(1) RUN(2) RUN(3) RUN(4) RUN(8)
#define RUNS(ILP, ROWS)                                                                           \
  {                                                                                               \
    float ms = timeit([&] { chains_scan<ILP, ROWS><<<sms, threads>>>(d, iters / 4, 1.0000001, 1e-9); }); \
    double fl = 2.0 * ILP * (ROWS + 5) * (double)(iters / 4) * sms * threads;                    \
    printf("{\"kind\":\"chains+scan\",\"warps_per_sm\":%d,\"ilp\":%d,\"rows\":%d,\"tflops\":%.2f}\n", wps, ILP, ROWS, fl / ms / 1e9); \
  }
    RUNS(2, 16) RUNS(3, 16) RUNS(4, 16) RUNS(2, 32)
  }
  return 0;
}
