// FP64 roofline denominator for this repo: measured DFMA and DDIV throughput
// on the box's B200 (MEASURED_PEAKS.json carries no FP64 figure).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void ddiv_loop(double* out, int iters, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = 1.0 + threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = b / acc[c];
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 256, blocks = sms * 8;
  // DFMA
  const int it = 20000;
  for (int w = 0; w < 3; ++w) dfma_loop<8><<<blocks, threads>>>(out, it, 0.999999, 1e-7);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dfma_loop<8><<<blocks, threads>>>(out, it, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double flops = 2.0 * 8 * (double)it * threads * blocks;
  double tf = flops / (best * 1e-3) / 1e12;
  // DDIV
  const int itd = 2000;
  for (int w = 0; w < 3; ++w) ddiv_loop<8><<<blocks, threads>>>(out, itd, 3.0);
  float bestd = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    ddiv_loop<8><<<blocks, threads>>>(out, itd, 3.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < bestd) bestd = ms;
  }
  double divs = 8.0 * itd * threads * blocks;
  double gdiv = divs / (bestd * 1e-3) / 1e9;
  printf("{\"fp64_fma_tflops\": %.3f, \"fp64_div_gops\": %.2f, \"dfma_ms\": %.3f, "
         "\"ddiv_ms\": %.3f, \"sms\": %d, \"clock_khz_attr\": %d, "
         "\"how\": \"%d blocks x %d threads, 8 independent chains/thread, best of 5, CUDA events\"}\n",
         tf, gdiv, best, bestd, sms, clk, blocks, threads);
  return 0;
}
