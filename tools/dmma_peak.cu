// FP64 tensor-core (mma.sync m8n8k4 f64 -> DMMA) throughput probe on B200, alone
// and concurrently with an FP64 FMA stream in the same warps.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int NT, int NF>
__global__ void __launch_bounds__(256) k_mix(double* out, int iters, double a, double b) {
  double acc[2 * NT + 2], f[NF + 1];
#pragma unroll
  for (int i = 0; i < 2 * NT; ++i) acc[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < NF; ++i) f[i] = threadIdx.x * 1e-4 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < NT; ++t) dmma(acc[2 * t], acc[2 * t + 1], a, b);
#pragma unroll
    for (int i = 0; i < NF; ++i) f[i] = fma(f[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 2 * NT; ++i) s += acc[i];
#pragma unroll
  for (int i = 0; i < NF; ++i) s += f[i];
  if (s == 1.2345) out[0] = s;
}

template <int NT, int NF>
void run(const char* name) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 2048, blocks = sms * 8, threads = 256;
  for (int r = 0; r < 2; ++r) k_mix<NT, NF><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) k_mix<NT, NF><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = (double)blocks * threads / 32 * iters * reps;
  const double tc = warps * NT * 512.0;          // 8x8x4 MACs x 2 flop per DMMA
  const double fm = warps * 32 * NF * 2.0;
  printf("{\"probe\": \"%s\", \"ms\": %.3f, \"dmma_tflops\": %.2f, \"dfma_tflops\": %.2f, \"total_tflops\": %.2f}\n", name, ms,
         tc / (ms * 1e-3) / 1e12, fm / (ms * 1e-3) / 1e12, (tc + fm) / (ms * 1e-3) / 1e12);
  cudaFree(out);
}

int main() {
  run<8, 0>("dmma_only");
  run<0, 8>("dfma_only");
  run<8, 8>("dmma8+dfma8");
  run<8, 16>("dmma8+dfma16");
  run<4, 16>("dmma4+dfma16");
  return 0;
}
