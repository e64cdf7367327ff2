// DMMA (mma.sync m8n8k4 f64) dependent-chain latency and 1-warp throughput.
#include <cstdio>
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
template <int CHAINS>
__global__ void k(double* out, long long* cyc, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[CHAINS][2];
  for (int i = 0; i < CHAINS; ++i) c[i][0] = c[i][1] = 0.0;
  __syncwarp();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) dmma(c[i], a, b);
  // consume results so the timing includes the last completion
  double s = 0;
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  long long t1 = clock64();
  if (s == 1234.5) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int C>
void run(int warps) {
  double* o; long long* cy; cudaMalloc(&o, 8); cudaMalloc(&cy, 8 * 8);
  const int iters = 4096;
  k<C><<<1, 32 * warps>>>(o, cy, 16);
  k<C><<<1, 32 * warps>>>(o, cy, iters);
  long long h; cudaMemcpy(&h, cy, 8, cudaMemcpyDeviceToHost);
  printf("chains=%d warps/SM=%d: %.1f cycles per DMMA per warp (%.2f DMMA/clk/SM)\n", C, warps,
         double(h) / (iters * C), double(iters) * C * warps / h);
}
int main() {
  run<1>(1); run<2>(1); run<4>(1); run<8>(1); run<8>(4); run<8>(8); run<8>(16);
  return 0;
}
