// Prototype: one tcgen05.mma.kind::i8 GEMM tile (M=128, N=128, K=256) with
// the operands in the canonical K-major no-swizzle smem layout, int32
// accumulators in TMEM, read back with tcgen05.ld.  Checks against the CPU
// and times a repeated-MMA loop for the per-SM int8 rate.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

constexpr int M = 128, N = 128, K = 128, UK = 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// K-major, no swizzle: core matrix = 8 rows x 16 B; rows of one 16-B K chunk
// are contiguous (16 B apart); chunk c of all R rows starts at c * R * 16 B.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version = 1 (sm100)
  // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
  return d;
}
__host__ __device__ constexpr uint32_t make_idesc_i8(int m, int n) {
  return (2u << 4)            // c_format = S32
       | (1u << 7)            // a_format = signed int8
       | (1u << 10)           // b_format = signed int8
       | (0u << 15)           // a K-major
       | (0u << 16)           // b K-major
       | ((uint32_t)(n >> 3) << 17)
       | ((uint32_t)(m >> 4) << 24);
}

__global__ void __launch_bounds__(128) tile_kernel(const int8_t* A, const int8_t* B, int32_t* C,
                                                   int reps, long long* cyc) {
  // A: M x K row-major (K-major); B: N x K row-major (K-major)
  __shared__ __align__(128) int8_t sA[M * K];
  __shared__ __align__(128) int8_t sB[N * K];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // canonical layout: byte (r, k) -> (k / 16) * R * 16 + r * 16 + (k % 16)
  for (int i = tid; i < M * K / 16; i += 128) {
    const int r = i / (K / 16), c = i % (K / 16);
    *reinterpret_cast<int4*>(sA + c * M * 16 + r * 16) = *reinterpret_cast<const int4*>(A + r * K + c * 16);
  }
  for (int i = tid; i < N * K / 16; i += 128) {
    const int r = i / (K / 16), c = i % (K / 16);
    *reinterpret_cast<int4*>(sB + c * N * 16 + r * 16) = *reinterpret_cast<const int4*>(B + r * K + c * 16);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
  }
  asm volatile("fence.proxy.async.shared::cta;\n");  // smem writes visible to the async (tensor) proxy
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = make_idesc_i8(M, N);
  long long t0 = clock64();
  if (tid == 0) {
    for (int rep = 0; rep < reps; ++rep)
      for (int kk = 0; kk < K / UK; ++kk) {
        const uint64_t da = make_desc(smem_u32(sA) + kk * 2 * M * 16, M * 16, 128);
        const uint64_t db = make_desc(smem_u32(sB) + kk * 2 * N * 16, N * 16, 128);
        const uint32_t acc = (rep > 0 || kk > 0) ? 1u : 0u;
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)));
  }
  // wait for the MMAs
  asm volatile(
      "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar)));
  long long t1 = clock64();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  // each warp reads its 32 lanes (rows 32w..32w+31), 32 columns at a time
  for (int cb = 0; cb < N; cb += 32) {
    uint32_t v[32];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + cb;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    const int row = warp * 32 + lane;
    for (int j = 0; j < 32; ++j) C[row * N + cb + j] = static_cast<int32_t>(v[j]);
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(128));
  if (tid == 0) *cyc = t1 - t0;
}

int main() {
  std::vector<int8_t> A(M * K), B(N * K);
  srand(1);
  for (auto& x : A) x = (int8_t)(rand() % 255 - 127);
  for (auto& x : B) x = (int8_t)(rand() % 255 - 127);
  int8_t *dA, *dB; int32_t* dC; long long* dcyc;
  cudaMalloc(&dA, A.size()); cudaMalloc(&dB, B.size()); cudaMalloc(&dC, M * N * 4); cudaMalloc(&dcyc, 8);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  for (int reps : {1, 200}) {
    tile_kernel<<<1, 128>>>(dA, dB, dC, reps, dcyc);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<int32_t> C(M * N);
    long long cyc = 0;
    cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
    long long bad = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        long long s = 0;
        for (int k = 0; k < K; ++k) s += (long long)A[i * K + k] * B[j * K + k];
        s *= reps;
        if ((int32_t)s != C[i * N + j]) ++bad;
      }
    printf("reps=%d err=%s mismatches=%lld cycles=%lld  int8 ops/clk/SM=%.1f\n", reps, cudaGetErrorString(e), bad, cyc,
           2.0 * M * N * K * reps / (double)cyc);
  }
  return 0;
}
