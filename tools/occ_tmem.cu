// Does a tcgen05.alloc in a kernel cap its occupancy at one CTA per SM?
// nvcc -gencode arch=compute_100a,code=sm_100a -o occ_tmem occ_tmem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 2) with_tmem(unsigned* out, int cols) {
  __shared__ uint32_t base;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(
        static_cast<unsigned>(__cvta_generic_to_shared(&base))));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  __syncthreads();
  long long t0 = clock64();
  while (clock64() - t0 < 2000000) { }
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0) { out[2 * blockIdx.x] = smid; out[2 * blockIdx.x + 1] = (unsigned)(t0 & 0xffffffff); }
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(base));
}
__global__ void __launch_bounds__(256, 2) without_tmem(unsigned* out) {
  long long t0 = clock64();
  while (clock64() - t0 < 2000000) { }
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0) { out[2 * blockIdx.x] = smid; out[2 * blockIdx.x + 1] = (unsigned)(t0 & 0xffffffff); }
}
int main() {
  int o = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, with_tmem, 256, 0);
  printf("occupancy API with tcgen05.alloc: %d\n", o);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, without_tmem, 256, 0);
  printf("occupancy API without: %d\n", o);
  unsigned* d; cudaMalloc(&d, 296 * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int which = 0; which < 2; ++which) {
    cudaEventRecord(a);
    if (which == 0) with_tmem<<<296, 256>>>(d, 256); else without_tmem<<<296, 256>>>(d);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%s: 296 CTAs x 2M-cycle spin: %.3f ms (%s) err=%s\n", which ? "without" : "with tmem", ms,
           ms > 1.6 ? "two waves: 1 CTA/SM" : "one wave: 2 CTAs/SM", cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
