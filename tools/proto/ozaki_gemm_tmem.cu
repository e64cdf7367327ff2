// Prototype: fp64 GEMM emulated on the int8 tensor cores (Ozaki scheme,
// S = 8 signed 7-bit slices per operand, row / column power-of-two scaling,
// products with i + j <= S + 1 accumulated exactly in int32, one TMEM
// accumulator per level i + j).  Research code for round 2 -- not on the
// product path.  Usage: ozaki_gemm N  (square N x N, N multiple of 128).
//
// Kernels
//   slice_rows   A (M x K, fp64 row-major) -> S int8 planes [s][M][K]
//                + per-row exponent; B is sliced the same way after a
//                transpose (B^T rows = B columns), giving K-major operands.
//   ozaki_gemm   128 x 64 output tile per CTA (128 threads).  Per 32-deep
//                K block: cp.async stages the 8 A planes (128 x 32) and the
//                8 B planes (64 x 32) into the canonical K-major no-swizzle
//                UMMA layout (4-stage ring, 48 KiB per stage); thread 0
//                issues 36 tcgen05.mma.kind::i8 into the 8 level
//                accumulators (8 x 64 TMEM columns = all 512) and commits
//                to the stage's mbarrier; the stage is refilled with K
//                block kb + 3 once those MMAs are done, while the next
//                block's MMAs are already queued.  Epilogue: tcgen05.ld
//                each level, combine in fp64 with 2^-7L and the row /
//                column scales.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int S = 8;              // slices
constexpr int TM = 128, TN = 32;  // CTA tile (A planes staged in TMEM next to 8 x 32 accumulators)
constexpr int BK = 32;            // K block (1 MMA of K = 32 per slice pair)
constexpr int THREADS = 128;
constexpr int A_PLANE = TM * BK, B_PLANE = TN * BK;      // bytes per plane per stage
constexpr int STAGE = S * (A_PLANE + B_PLANE);           // 40 KiB
constexpr int NSTAGE = 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) |
         (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (static_cast<uint64_t>(1) << 46);
}
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src));
}

// rows of X (R x K fp64, row-major) -> S int8 planes, exponent e[r] with
// |x| < 2^e[r] for the whole row.  Plane layout is tile-major and already
// the canonical K-major no-swizzle UMMA layout: for a tile of TR rows and a
// 32-deep K block, one contiguous 32 TR-byte block [chunk 0..1][row][16 B],
// so the GEMM brings each (plane, tile, K block) with ONE bulk copy.
//   offset(s, r, k) = (((s * (R / TR) + r / TR) * (K / 32) + k / 32) * 2
//                      + (k % 32) / 16) * TR * 16 + (r % TR) * 16 + k % 16
__global__ void slice_rows(const double* X, int R, int K, int TR, int8_t* planes, int* ex) {
  const int r = blockIdx.x;
  const double* row = X + static_cast<size_t>(r) * K;
  __shared__ double red[32];
  double m = 0.0;
  for (int k = threadIdx.x; k < K; k += blockDim.x) m = fmax(m, fabs(row[k]));
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (int)(blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) red[0] = m;
  }
  __syncthreads();
  int e = 0;
  frexp(red[0], &e);  // max < 2^e
  if (red[0] == 0.0) e = 0;
  if (threadIdx.x == 0) ex[r] = e;
  const size_t tiles = R / TR, kbs = K / 32;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    // 56-bit fixed point relative to 2^e, split into 8 x 7-bit digits
    const long long q = llrint(ldexp(row[k], 7 * S - e));
    const long long a = q < 0 ? -q : q;
    const size_t in_tile = static_cast<size_t>((k % 32) / 16) * TR * 16 + (r % TR) * 16 + k % 16;
    for (int s2 = 0; s2 < S; ++s2) {
      const int d = static_cast<int>((a >> (7 * (S - 1 - s2))) & 127);
      const size_t blk = (static_cast<size_t>(s2) * tiles + r / TR) * kbs + k / 32;
      planes[blk * 32 * TR + in_tile] = static_cast<int8_t>(q < 0 ? -d : d);
    }
  }
}

__global__ void transpose(const double* X, double* Y, int R, int C) {  // Y = X^T
  __shared__ double t[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) t[i][threadIdx.x] = X[(size_t)(by + i) * C + bx + threadIdx.x];
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) Y[(size_t)(bx + i) * R + by + threadIdx.x] = t[threadIdx.x][i];
}

__global__ void __launch_bounds__(THREADS, 1)
ozaki_gemm(const int8_t* Ap, const int8_t* Bp, const int* ea, const int* eb, double* C, int M,
           int N, int K) {
  extern __shared__ __align__(1024) int8_t sm[];
  __shared__ __align__(8) uint64_t bar_free[NSTAGE];
  __shared__ __align__(8) uint64_t bar_full[NSTAGE];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int i = 0; i < NSTAGE; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar_free[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar_full[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;

  const int nk = K / BK;
  const uint32_t idesc = idesc_i8(TM, TN);
  const size_t a_tiles = M / TM, b_tiles = N / TN;
  // ONE thread runs the whole pipeline: bulk copies (TMA engine) fill a
  // 4-stage ring, MMAs are queued as soon as a stage is full, and a stage is
  // refilled once the tensor core has finished reading it.
  if (tid == 0) {
    auto fill = [&](int stage, int kb) {
      const uint32_t bar = smem_u32(&bar_full[stage]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(STAGE));
      int8_t* base = sm + stage * STAGE;
      for (int s2 = 0; s2 < S; ++s2) {
        const int8_t* a = Ap + ((static_cast<size_t>(s2) * a_tiles + blockIdx.y) * nk + kb) * A_PLANE;
        const int8_t* b = Bp + ((static_cast<size_t>(s2) * b_tiles + blockIdx.x) * nk + kb) * B_PLANE;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                     ::"r"(smem_u32(base + s2 * A_PLANE)), "l"(a), "r"(A_PLANE), "r"(bar) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                     ::"r"(smem_u32(base + S * A_PLANE + s2 * B_PLANE)), "l"(b), "r"(B_PLANE), "r"(bar) : "memory");
      }
    };
    uint32_t ph_full[NSTAGE] = {}, ph_free[NSTAGE] = {};
    for (int p = 0; p < NSTAGE - 1 && p < nk; ++p) fill(p, p);
    for (int kb = 0; kb < nk; ++kb) {
      const int st = kb % NSTAGE;
      asm volatile("{\n.reg .pred p;\nWF:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WF;\n}\n" ::"r"(smem_u32(&bar_full[st])), "r"(ph_full[st]));
      ph_full[st] ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const uint64_t da0 = make_desc(smem_u32(sm + st * STAGE), TM * 16, 128);
      const uint64_t db0 = make_desc(smem_u32(sm + st * STAGE + S * A_PLANE), TN * 16, 128);
      // A planes of this K block: smem -> TMEM columns 256 + 64 st + 8 i
      // (tcgen05 ops run in issue order, so the MMAs below see them)
      const uint32_t a_t0 = tmem + 256 + st * 64;
#pragma unroll
      for (int i = 0; i < S; ++i) {
        const uint64_t da = da0 + ((i * A_PLANE) >> 4);
        asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;\n" ::"r"(a_t0 + i * 8), "l"(da));
      }
#pragma unroll
      for (int i = 0; i < S; ++i)
#pragma unroll
        for (int j = 0; j < S; ++j) {
          const int lvl = i + j;
          if (lvl >= S) continue;
          const uint64_t db = db0 + ((j * B_PLANE) >> 4);
          const uint32_t acc = (kb > 0 || i > 0) ? 1u : 0u;  // first write: (0, lvl) in block 0
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + lvl * TN),
                       "r"(a_t0 + i * 8), "l"(db), "r"(idesc), "r"(acc));
        }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar_free[st])));
      const int nxt = kb + NSTAGE - 1;
      if (nxt < nk) {
        const int rst = nxt % NSTAGE;
        if (kb >= 1) {  // K block kb-1 read this stage
          asm volatile("{\n.reg .pred p;\nWR:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WR;\n}\n" ::"r"(smem_u32(&bar_free[rst])), "r"(ph_free[rst]));
          ph_free[rst] ^= 1;
        }
        fill(rst, nxt);
      }
    }
    // tcgen05.commit tracks every earlier MMA of this thread
    const int st = (nk - 1) % NSTAGE;
    asm volatile("{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}\n" ::"r"(smem_u32(&bar_free[st])), "r"(ph_free[st]));
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  // epilogue: row (warp*32 + lane) of the tile, 64 columns per level
  const int row = m0 + warp * 32 + lane;
  double out[TN];
#pragma unroll
  for (int c = 0; c < TN; ++c) out[c] = 0.0;
  for (int lvl = S - 1; lvl >= 0; --lvl) {
    for (int cb = 0; cb < TN; cb += 32) {
      uint32_t v[32];
      const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + lvl * TN + cb;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
            "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
            "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(ta));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n");
      const double sc = ldexp(1.0, -7 * (lvl + 2));
#pragma unroll
      for (int j = 0; j < 32; ++j) out[cb + j] = fma(static_cast<double>(static_cast<int32_t>(v[j])), sc, out[cb + j]);
    }
  }
  const int e_r = ea[row];
#pragma unroll
  for (int c = 0; c < TN; ++c)
    C[static_cast<size_t>(row) * N + n0 + c] = ldexp(out[c], e_r + eb[n0 + c]);
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

__global__ void dgemm_ref(const double* A, const double* B, double* C, int N) {  // naive check
  const int i = blockIdx.y * 16 + threadIdx.y, j = blockIdx.x * 16 + threadIdx.x;
  double s = 0.0;
  for (int k = 0; k < N; ++k) s = fma(A[(size_t)i * N + k], B[(size_t)k * N + j], s);
  C[(size_t)i * N + j] = s;
}

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 1024;
  const size_t nn = (size_t)N * N;
  std::vector<double> hA(nn), hB(nn);
  srand(7);
  for (auto& x : hA) x = (rand() / (double)RAND_MAX - 0.5) * pow(10.0, (rand() % 7) - 3);
  for (auto& x : hB) x = (rand() / (double)RAND_MAX - 0.5);
  double *A, *B, *Bt, *C, *Cref;
  int8_t *Ap, *Bp;
  int *ea, *eb;
  cudaMalloc(&A, nn * 8); cudaMalloc(&B, nn * 8); cudaMalloc(&Bt, nn * 8);
  cudaMalloc(&C, nn * 8); cudaMalloc(&Cref, nn * 8);
  cudaMalloc(&Ap, nn * S); cudaMalloc(&Bp, nn * S); cudaMalloc(&ea, N * 4); cudaMalloc(&eb, N * 4);
  cudaMemcpy(A, hA.data(), nn * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB.data(), nn * 8, cudaMemcpyHostToDevice);
  const int smem = NSTAGE * STAGE;
  cudaFuncSetAttribute(ozaki_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  auto run = [&]() {
    slice_rows<<<N, 256>>>(A, N, N, TM, Ap, ea);
    transpose<<<dim3(N / 32, N / 32), dim3(32, 8)>>>(B, Bt, N, N);
    slice_rows<<<N, 256>>>(Bt, N, N, TN, Bp, eb);
    ozaki_gemm<<<dim3(N / TN, N / TM), THREADS, smem>>>(Ap, Bp, ea, eb, C, N, N, N);
  };
  run();
  cudaError_t e = cudaDeviceSynchronize();
  printf("run: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int reps = 5;
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) run();
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i)
    ozaki_gemm<<<dim3(N / TN, N / TM), THREADS, smem>>>(Ap, Bp, ea, eb, C, N, N, N);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms_g = 0; cudaEventElapsedTime(&ms_g, e0, e1); ms_g /= reps;
  dgemm_ref<<<dim3(N / 16, N / 16), dim3(16, 16)>>>(A, B, Cref, N);
  cudaDeviceSynchronize();
  std::vector<double> hC(nn), hR(nn);
  cudaMemcpy(hC.data(), C, nn * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hR.data(), Cref, nn * 8, cudaMemcpyDeviceToHost);
  double num = 0, den = 0;
  for (size_t i = 0; i < nn; ++i) { num = fmax(num, fabs(hC[i] - hR[i])); den = fmax(den, fabs(hR[i])); }
  const double fl = 2.0 * N * N * (double)N;
  printf("N=%d max|C-Cref|/max|Cref| = %.3e  total %.3f ms (%.1f TF/s fp64-equiv)  gemm only %.3f ms (%.1f TF/s)\n",
         N, num / den, ms, fl / ms / 1e9, ms_g, fl / ms_g / 1e9);
  return 0;
}
