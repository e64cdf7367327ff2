// Microbenchmark of the fused64 GEMM building blocks (steady state).
#include <cstdio>
#include "../paper_2010_00465_b200/csrc/k0_select.cu"
#include "../paper_2010_00465_b200/csrc/fused64.cu"

using namespace csm;
using namespace csm::f64k;

__global__ void __launch_bounds__(256, 1) micro(int iters, int mode, double* out) {
  extern __shared__ __align__(16) double smem[];
  for (int p = threadIdx.x; p < 6 * SLOT; p += 256) smem[p] = 1e-3 * ((p * 7) % 13);
  __syncthreads();
  Lane ln;
  make_lane(ln);
  Acc acc, acc2, keep;
  zero(keep);
  double sink = 0;
  for (int it = 0; it < iters; ++it) {
    double* L = smem + SLOT * (1 + (it & 1));
    double* R = smem + SLOT * 3;
    if (mode == 3 || mode == 4) gemm<true>(L, smem, R, acc, acc2, ln);
    else gemm<false>(L, nullptr, R, acc, acc2, ln);
    if (mode == 2 || mode == 4) {
      EpiArgs E; E.o[0] = smem + 4 * SLOT; E.scale = 1.0;
      epilogue(E_SCALED, E, acc, acc2, keep, ln);
    }
    if (mode >= 1) __syncthreads();
    sink += acc[0][0][0] + acc[1][3][1];
    if (mode >= 3) sink += acc2[1][2][0];
  }
  if (sink == 1.2345) out[0] = sink;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d; cudaMalloc(&d, 8);
  size_t smem = 6 * SLOT * 8;
  cudaFuncSetAttribute(micro, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"gemm1 nosync", "gemm1+sync", "gemm1+epi+sync", "gemm2 nosync", "gemm2+epi+sync"};
  for (int mode = 0; mode < 5; ++mode) {
    int iters = 2000;
    micro<<<sms, 256, smem>>>(100, mode, d);
    cudaEventRecord(e0);
    micro<<<sms, 256, smem>>>(iters, mode, d);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double prods = (mode >= 3 ? 2.0 : 1.0) * iters * sms;
    double fl = prods * 2.0 * 64 * 64 * 64;
    printf("%-18s %.2f TFLOP/s  %.0f cycles/product/SM\n", names[mode], fl / ms / 1e9,
           ms * 1e-3 * 1.965e9 / (prods / sms));
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
