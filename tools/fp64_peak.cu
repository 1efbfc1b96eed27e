// FP64 peak microbenchmark for B200 (sm_100a): DMMA.8x8x4 (mma.sync m8n8k4 f64) and DFMA.
// Measures the roofline denominator for the FP64 phases (MEASURED_PEAKS.json has no FP64 entry).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ITER>
__global__ void dmma_loop(const double* a, double* c) {
  double x = a[threadIdx.x & 31], y = a[(threadIdx.x + 7) & 31];
  double d[8][2];
#pragma unroll
  for (int i = 0; i < 8; i++) d[i][0] = d[i][1] = 0.0;
  for (int it = 0; it < ITER; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(x), "d"(y));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += d[i][0] + d[i][1];
  if (s == 12345.678) c[threadIdx.x] = s;
}

template <int ITER>
__global__ void dfma_loop(const double* a, double* c) {
  double x = a[threadIdx.x & 31], y = a[(threadIdx.x + 3) & 31];
  double d[16];
#pragma unroll
  for (int i = 0; i < 16; i++) d[i] = a[(threadIdx.x + i) & 31];
  for (int it = 0; it < ITER; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) d[i] = fma(d[i], x, y);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += d[i];
  if (s == 12345.678) c[threadIdx.x] = s;
}

int main() {
  int dev = 0, nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  double *a, *c;
  cudaMalloc(&a, 1024 * 8);
  cudaMalloc(&c, 1 << 20);
  cudaMemset(a, 0, 1024 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int ITER = 4096;
  for (int warps = 4; warps <= 32; warps *= 2) {
    for (int rep = 0; rep < 2; rep++) {
      int blocks = nsm * 2, threads = warps * 32;
      dmma_loop<ITER><<<blocks, threads>>>(a, c);
      cudaEventRecord(e0);
      dmma_loop<ITER><<<blocks, threads>>>(a, c);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 8 * (double)ITER * blocks * warps;
      if (rep) printf("{\"kind\":\"dmma_m8n8k4\",\"warps_per_cta\":%d,\"ctas\":%d,\"tflops\":%.3f}\n", warps, blocks, flops / ms / 1e9);
      dfma_loop<ITER><<<blocks, threads>>>(a, c);
      cudaEventRecord(e0);
      dfma_loop<ITER><<<blocks, threads>>>(a, c);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 32 * 16 * (double)ITER * blocks * warps;
      if (rep) printf("{\"kind\":\"dfma\",\"warps_per_cta\":%d,\"ctas\":%d,\"tflops\":%.3f}\n", warps, blocks, flops / ms / 1e9);
    }
  }
  printf("sms=%d err=%s\n", nsm, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
