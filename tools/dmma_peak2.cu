// DMMA throughput vs operand-register pattern (B200 microbenchmark).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
template <int CH, int MODE>
__global__ void k(double* out, int iters) {
  double a[CH], b[CH], c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) { a[i] = 1.0 + threadIdx.x * 1e-9 + i; b[i] = 1.0 - i * 1e-3; c[i][0] = c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (MODE == 0) dmma(c[i], a[0], b[0]);          // all share a,b
      else if (MODE == 1) dmma(c[i], a[i], b[i]);     // distinct
      else if (MODE == 2) dmma(c[i], a[i], b[i / 2]); // pairs share b
      else dmma(c[i], a[i / 2], b[i % 4]);           // gemm-like reuse
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}
template <int CH, int MODE>
void run(const char* name, int warps) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4000;
  k<CH, MODE><<<sms, 32 * warps>>>(d, 100);
  cudaEventRecord(e0);
  k<CH, MODE><<<sms, 32 * warps>>>(d, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 256 * CH * (double)iters * warps * sms;
  printf("%-28s warps=%2d chains=%2d %.2f TFLOP/s\n", name, warps, CH, fl / ms / 1e9);
  cudaFree(d);
}
int main() {
  run<4, 1>("distinct a,b", 16);
  run<4, 1>("distinct a,b", 12);
  run<8, 1>("distinct a,b", 12);
  run<4, 1>("distinct a,b", 8);
  run<2, 1>("distinct a,b", 16);
  run<8, 0>("shared a,b", 8);
  run<8, 1>("distinct a,b", 8);
  run<16, 1>("distinct a,b", 8);
  run<8, 2>("pairs share b", 8);
  run<16, 2>("pairs share b", 8);
  run<16, 3>("gemm-like", 8);
  run<16, 1>("distinct a,b", 4);
  run<16, 1>("distinct a,b", 16);
  run<8, 1>("distinct a,b", 16);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
