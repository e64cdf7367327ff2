// DSMEM read bandwidth / latency probe (cluster of 4 CTAs, one per SM).
// Each thread streams 8- or 16-byte ld.shared::cluster loads from a peer
// CTA's shared memory; reports bytes per clock per SM.
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

template <int VEC, int PEER>
__global__ void __cluster_dims__(4, 1, 1) bw_kernel(double* out, int iters, long long* cyc) {
  __shared__ double buf[4096];  // 32 KB
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = i * 1e-3;
  cl.sync();
  const unsigned me = cl.block_rank();
  const unsigned peer = PEER ? (me + 1) % 4 : me;
  double* rb = cl.map_shared_rank(buf, peer);
  double acc = 0.0;
  long long t0 = clock64();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int j = 0; j < 8; ++j) {
      const int idx = ((it * 8 + j) * 32 * (blockDim.x / 32) + w * 32 + lane) * VEC & (4096 - VEC);
      if (VEC == 2) {
        double2 v = *reinterpret_cast<const double2*>(rb + idx);
        acc += v.x + v.y;
      } else {
        acc += rb[idx];
      }
    }
  }
  long long t1 = clock64();
  cl.sync();
  if (acc == 12345.0) out[0] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int VEC, int PEER>
void run(int threads) {
  double* out; long long* cyc; cudaMalloc(&out, 8); cudaMalloc(&cyc, 148 * 8);
  int blocks = 148;
  int iters = 2000;
  bw_kernel<VEC, PEER><<<blocks, threads>>>(out, 10, cyc);
  cudaDeviceSynchronize();
  bw_kernel<VEC, PEER><<<blocks, threads>>>(out, iters, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mean = 0; for (int i = 0; i < blocks; ++i) mean += h[i]; mean /= blocks;
  double bytes = double(iters) * 8 * threads * 8 * VEC;
  printf("vec=%d peer=%d threads=%d err=%s cycles=%.0f bytes/clk/SM=%.2f\n", VEC, PEER, threads,
         cudaGetErrorString(e), mean, bytes / mean);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int th : {256, 512, 1024}) {
    run<1, 1>(th); run<2, 1>(th); run<1, 0>(th); run<2, 0>(th);
  }
  return 0;
}
