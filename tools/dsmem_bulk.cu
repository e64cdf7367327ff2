// DSMEM push bandwidth with cp.async.bulk shared::cta -> shared::cluster
// (cluster of 4, each CTA pushes into its right neighbour); bytes/clk/SM.
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int CHUNK>
__global__ void __cluster_dims__(4, 1, 1) push_kernel(int rounds, long long* cyc) {
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char* src = sm;            // CHUNK bytes
  unsigned char* dst = sm + CHUNK;    // CHUNK bytes
  __shared__ __align__(8) unsigned long long bar;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned me = cl.block_rank(), right = (me + 1) % 4;
  for (int i = threadIdx.x; i < CHUNK; i += blockDim.x) src[i] = (unsigned char)i;
  const int per_phase = (1 << 19) / CHUNK;  // 512 KB per phase
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  cl.sync();
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                   "r"(per_phase * CHUNK));
    }
    cl.sync();  // every destination armed before pushes start
    if (threadIdx.x < per_phase) {
      // remote addresses of the right neighbour's dst buffer and barrier
      uint32_t rdst, rbar;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rdst) : "r"(smem_u32(dst)), "r"(right));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(smem_u32(&bar)), "r"(right));
      asm volatile(
          "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
          ::"r"(rdst), "r"(smem_u32(src)), "r"(CHUNK), "r"(rbar) : "memory");
    }
    if (threadIdx.x == 0) {
      uint32_t done = 0;
      while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done) : "r"(smem_u32(&bar)), "r"(r & 1));
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  cl.sync();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int CHUNK>
void run() {
  long long* cyc; cudaMalloc(&cyc, 148 * 8);
  auto k = push_kernel<CHUNK>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * CHUNK);
  k<<<148, 128, 2 * CHUNK>>>(2, cyc);
  cudaDeviceSynchronize();
  const int rounds = 40;
  k<<<148, 128, 2 * CHUNK>>>(rounds, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mean = 0; for (int i = 0; i < 148; ++i) mean += h[i]; mean /= 148;
  printf("chunk=%d err=%s cycles=%.0f bytes/clk/SM=%.2f\n", CHUNK, cudaGetErrorString(e), mean,
         double(rounds) * (1 << 19) / mean);
  cudaFree(cyc);
}

int main() { run<4096>(); run<8192>(); run<16384>(); run<32768>(); return 0; }
