// Dependent-chain latency of the FP64 instructions the search kernel is made
// of (DFMA, DMUL, DADD, MUFU.RCP64H, a full IEEE division, a double compare
// feeding a select), one warp, clock64 around a chain of 1024 ops.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fp64_latency tools/fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kN = 1024;

__global__ void lat(double x, double y, long long* cyc, double* sink) {
  double a = x, b = y;
  long long t0, t1;
  // DFMA
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < kN; ++i) a = fma(a, b, 0.5);
  t1 = clock64();
  cyc[0] = t1 - t0;
  // DMUL
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < kN; ++i) a = __dmul_rn(a, b);
  t1 = clock64();
  cyc[1] = t1 - t0;
  // DADD
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < kN; ++i) a = __dadd_rn(a, b);
  t1 = clock64();
  cyc[2] = t1 - t0;
  // MUFU.RCP64H
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < kN; ++i) {
    double r;
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
    a = r;
  }
  t1 = clock64();
  cyc[3] = t1 - t0;
  // IEEE division
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < kN; ++i) a = __ddiv_rn(b, a);
  t1 = clock64();
  cyc[4] = t1 - t0;
  // compare -> select
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < kN; ++i) a = (a < b) ? b : a + 1e-300;
  t1 = clock64();
  cyc[5] = t1 - t0;
  // int -> double
  long long k = (long long)x;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < kN; ++i) {
    double d = (double)k;
    k = __double_as_longlong(d) & 0xff;
  }
  t1 = clock64();
  cyc[6] = t1 - t0;
  sink[threadIdx.x] = a + b + (double)k;
}

// Throughput: 8 independent chains per thread, full GPU.
template <int OP>
__global__ void thr(double x, double y, double* sink) {
  double a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = x + j * 1e-3;
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) a[j] = fma(a[j], y, 0.5);
      if (OP == 1) a[j] = __dmul_rn(a[j], y);
      if (OP == 2) a[j] = __dadd_rn(a[j], y);
      if (OP == 3) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a[j])); a[j] = r; }
      if (OP == 4) a[j] = (a[j] < y) ? a[j] + 1.0 : a[j] - 1.0;
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int OP>
double run_thr(double* sink) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  thr<OP><<<1184, 256>>>(1.0000001, 0.9999999, sink);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    thr<OP><<<1184, 256>>>(1.0000001, 0.9999999, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  int sms = 0, khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const double warp_inst = 1184.0 * 8 * 256 * 8;  // warps x iterations x chains
  return warp_inst / (best * 1e-3) / (sms * 4.0 * khz * 1e3);  // warp-inst / cycle / SMSP
}

int main() {
  long long* dc;
  double* ds;
  cudaMalloc(&dc, 8 * sizeof(long long));
  cudaMalloc(&ds, 32 * sizeof(double));
  lat<<<1, 32>>>(1.0000001, 0.9999999, dc, ds);
  lat<<<1, 32>>>(1.0000001, 0.9999999, dc, ds);
  long long h[8];
  cudaMemcpy(h, dc, 7 * sizeof(long long), cudaMemcpyDeviceToHost);
  const char* names[] = {"DFMA", "DMUL", "DADD", "MUFU.RCP64H", "ddiv_rn", "DSETP+select", "I2F.F64"};
  printf("{");
  for (int i = 0; i < 7; ++i) printf("%s\"%s\": %.2f", i ? ", " : "", names[i], (double)h[i] / kN);
  printf("}\n");
  double* sink;
  cudaMalloc(&sink, 1184 * 256 * sizeof(double));
  printf("{\"thr_DFMA\": %.3f, \"thr_DMUL\": %.3f, \"thr_DADD\": %.3f, \"thr_RCP64H\": %.3f, \"thr_DSETP_sel\": %.3f, \"unit\": \"warp-inst/cycle/SMSP at the attribute clock\"}\n",
         run_thr<0>(sink), run_thr<1>(sink), run_thr<2>(sink), run_thr<3>(sink), run_thr<4>(sink));
  return 0;
}
