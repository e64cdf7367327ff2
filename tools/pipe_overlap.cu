// Do DMMA and DFMA share hardware? Run both in different warps of one CTA.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__global__ void k(double* out, int iters, int mode, int dfma_iters) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  const bool do_dmma = (mode == 0 || mode == 2) ? (warp < 8) : false;
  const bool do_dfma = (mode == 1 || mode == 2) ? (warp >= 8) : false;
  if (do_dmma) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0, c[8][2];
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(c[i], a, b);
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  }
  if (do_dfma) {
    double c[8];
    for (int i = 0; i < 8; ++i) c[i] = i;
    const double a = 1.0 + threadIdx.x * 1e-12, b = 1e-9;
    for (int it = 0; it < dfma_iters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) c[i] = fma(c[i], a, b);
    for (int i = 0; i < 8; ++i) s += c[i];
  }
  if (s == 1.2345) out[0] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* nm[] = {"DMMA only (8 warps)", "DFMA only (8 warps)", "both (8+8 warps)"};
  int iters = 8000, dfi = 8000 * 4;
  for (int mode = 0; mode < 3; ++mode) {
    k<<<sms, 512>>>(d, 100, mode, 400);
    cudaEventRecord(e0);
    k<<<sms, 512>>>(d, iters, mode, dfi);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double dm = 2.0 * 256 * 8 * (double)iters * 8 * sms;
    double df = 2.0 * 32 * 8 * (double)dfi * 8 * sms;
    printf("%-22s %.3f ms  DMMA %.1f TF  DFMA %.1f TF\n", nm[mode], ms,
           mode != 1 ? dm / ms / 1e9 : 0.0, mode != 0 ? df / ms / 1e9 : 0.0);
  }
}
