// FP64 FMA throughput probe for B200 (sm_100a): many independent DFMA chains
// per thread at full occupancy; reports achieved TFLOP/s (2 flop per DFMA),
// timed with CUDA events. Used for the "alu" roofline peak.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 1.2345) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 4096, blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) k_dfma<8><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int rep = 0; rep < reps; ++rep) k_dfma<8><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 8 * iters * (double)blocks * threads * reps;
  printf("{\"fp64_tflops\": %.3f, \"sms\": %d, \"clock_mhz_attr\": %.0f, \"per_sm_per_clk_at_attr\": %.2f}\n",
         flops / (ms * 1e-3) / 1e12, sms, clk / 1e3, flops / (ms * 1e-3) / sms / (clk * 1e3));
  return 0;
}
