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

// sm_90+ FP64 shapes: m16n8k4 (A 2, B 1, C 4 doubles per lane), m16n8k8 (A 4, B 2), m16n8k16 (A 8, B 4)
template <int ITER, int K>
__global__ void dmma16_loop(const double* a, double* c) {
  double x[8], y[4];
#pragma unroll
  for (int i = 0; i < 8; i++) x[i] = a[(threadIdx.x + i) & 31];
#pragma unroll
  for (int i = 0; i < 4; i++) y[i] = a[(threadIdx.x + 5 + i) & 31];
  double d[8][4];
#pragma unroll
  for (int i = 0; i < 8; i++) d[i][0] = d[i][1] = d[i][2] = d[i][3] = 0.0;
  for (int it = 0; it < ITER; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      if constexpr (K == 4)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(d[i][0]), "+d"(d[i][1]), "+d"(d[i][2]), "+d"(d[i][3]) : "d"(x[0]), "d"(x[1]), "d"(y[0]));
      else if constexpr (K == 8)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+d"(d[i][0]), "+d"(d[i][1]), "+d"(d[i][2]), "+d"(d[i][3])
                     : "d"(x[0]), "d"(x[1]), "d"(x[2]), "d"(x[3]), "d"(y[0]), "d"(y[1]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
                     "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                     : "+d"(d[i][0]), "+d"(d[i][1]), "+d"(d[i][2]), "+d"(d[i][3])
                     : "d"(x[0]), "d"(x[1]), "d"(x[2]), "d"(x[3]), "d"(x[4]), "d"(x[5]), "d"(x[6]), "d"(x[7]),
                       "d"(y[0]), "d"(y[1]), "d"(y[2]), "d"(y[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += d[i][0] + d[i][1] + d[i][2] + d[i][3];
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
  for (int warps = 4; warps <= 16; warps *= 2) {
    const int blocks = nsm * 2, threads = warps * 32;
    float ms;
    auto run = [&](auto kern, int k, const char* name) {
      kern<<<blocks, threads>>>(a, c);
      cudaEventRecord(e0);
      kern<<<blocks, threads>>>(a, c);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double flops = 2.0 * 16 * 8 * k * 8 * (double)ITER * blocks * warps;
      printf("{\"kind\":\"%s\",\"warps_per_cta\":%d,\"ctas\":%d,\"tflops\":%.3f}\n", name, warps, blocks, flops / ms / 1e9);
    };
    run(dmma16_loop<ITER, 4>, 4, "dmma_m16n8k4");
    run(dmma16_loop<ITER, 8>, 8, "dmma_m16n8k8");
    run(dmma16_loop<ITER, 16>, 16, "dmma_m16n8k16");
  }
  printf("sms=%d err=%s\n", nsm, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
