// Prototype: fp64 GEMM emulated on the int8 tensor cores with the Ozaki
// scheme II (Chinese remainder theorem over int8 moduli).  Research code --
// not on the product path.  Usage: ozaki2_gemm N [NM]  (square N x N, N a
// multiple of 256, NM moduli <= 15).
//
//   A (row scaled) and B (column scaled) are rounded to integers A', B' of
//   at most P bits (P from NM and K so that |A'B'| < M/4, M = prod m_t).
//   For each modulus m_t <= 256: C_t = (A' mod m_t)(B' mod m_t) is ONE exact
//   int8 GEMM (int32 accumulation, |C_t| <= K 2^14), reduced mod m_t.  The
//   CRT then rebuilds A'B' = sum_t r_t W_t mod M in three exact fp64 levels.
//   So the tensor work is NM int8 GEMMs (vs S(S+1)/2 = 36 for the slice
//   scheme at S = 8), each an ordinary GEMM with its own operands.
//
// Kernels
//   scale_rows / scale_cols  per-row / per-column power-of-two shift
//   residues                 operand -> NM int8 planes in the canonical
//                            K-major no-swizzle UMMA layout, tile-major
//   gemm_mod                 128 x 256 tile per CTA, one modulus per CTA
//                            (grid z); thread 0 drives a 4-stage ring of
//                            bulk copies (one A and one B copy per 128-deep
//                            K stage) and 4 tcgen05.mma.kind::i8 per stage
//                            into a 256-column TMEM accumulator; epilogue
//                            tcgen05.ld -> mod m_t -> int8 residue tile
//   crt                      residues -> fp64 product
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int TM = 128, TN = 256;
constexpr int KS = 128;  // K bytes per pipeline stage (4 MMAs of K = 32)
constexpr int A_ST = TM * KS, B_ST = TN * KS, STAGE = A_ST + B_ST;  // 48 KiB
constexpr int NSTAGE = 4;
constexpr int THREADS = 128;
constexpr int MAXM = 15;
constexpr int LV = 3;          // CRT levels of 40 bits
constexpr int LVB = 40;

__constant__ int c_mod[MAXM];
__constant__ float c_inv[MAXM];
__constant__ double c_w[MAXM][LV];  // W_t in 40-bit digits, most significant first
__constant__ double c_M[LV];
__constant__ double c_invM;

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

// shift[r] = P - e with max_k |x(r, k)| < 2^e: |x 2^shift| < 2^P
__global__ void scale_rows(const double* X, int R, int K, int P, int* shift) {
  const int r = blockIdx.x;
  __shared__ double red[32];
  double m = 0.0;
  for (int k = threadIdx.x; k < K; k += blockDim.x) m = fmax(m, fabs(X[(size_t)r * K + k]));
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) m = fmax(m, red[i]);
    m = fmax(m, red[0]);
    int e = 0;
    frexp(m, &e);
    shift[r] = m == 0.0 ? 0 : P - e;
  }
}
__global__ void scale_cols(const double* X, int K, int N, int P, int* shift) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  double m = 0.0;
  for (int k = 0; k < K; ++k) m = fmax(m, fabs(X[(size_t)k * N + c]));
  int e = 0;
  frexp(m, &e);
  shift[c] = m == 0.0 ? 0 : P - e;
}

__device__ __forceinline__ size_t plane_off(int t, int r, int k, int R, int K, int TR) {
  return ((((size_t)t * (R / TR) + r / TR) * (K / 32) + k / 32) * 2 + (k % 32) / 16) * TR * 16 +
         (r % TR) * 16 + k % 16;
}

__device__ __forceinline__ int8_t resid(double v, int t) {
  // v an integer with |v| < 2^53; symmetric residue in [-128, 127]
  const double m = (double)c_mod[t];
  const double q = rint(v * (1.0 / m));
  int r = (int)fma(-q, m, v);
  if (r > 127) r -= c_mod[t];
  if (r < -128) r += c_mod[t];
  return (int8_t)r;
}

// A (M x K row-major) -> planes with rows = M (TR = TM); element (i, k)
__global__ void residues_rows(const double* X, int R, int K, const int* shift, int NM,
                              int8_t* planes, int TR) {
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)R * K) return;
  const int r = idx / K, k = idx % K;
  const double v = rint(ldexp(X[idx], shift[r]));
  for (int t = 0; t < NM; ++t) planes[plane_off(t, r, k, R, K, TR)] = resid(v, t);
}
// B (K x N row-major), column scaled -> planes with rows = N (K-major B^T)
__global__ void residues_cols(const double* X, int K, int N, const int* shift, int NM,
                              int8_t* planes, int TR) {
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (size_t)K * N) return;
  const int k = idx / N, c = idx % N;
  const double v = rint(ldexp(X[idx], shift[c]));
  for (int t = 0; t < NM; ++t) planes[plane_off(t, c, k, N, K, TR)] = resid(v, t);
}

// Coalesced conversion.  Max |x| per row / column as the bit pattern of a
// non-negative double (atomicMax on u64 orders them like the values).
__global__ void absmax_rows(const double* X, int R, int K, unsigned long long* mx) {
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= R) return;
  double m = 0.0;
  for (int k = lane * 2; k < K; k += 64) {
    const double2 v = *reinterpret_cast<const double2*>(X + (size_t)r * K + k);
    m = fmax(m, fmax(fabs(v.x), fabs(v.y)));
  }
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) mx[r] = __double_as_longlong(m);
}
__global__ void absmax_cols(const double* X, int K, int N, int kchunk, unsigned long long* mx) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int k0 = blockIdx.y * kchunk;
  if (c >= N) return;
  double m = 0.0;
  for (int k = k0; k < min(K, k0 + kchunk); ++k) m = fmax(m, fabs(X[(size_t)k * N + c]));
  atomicMax(mx + c, (unsigned long long)__double_as_longlong(m));
}
__global__ void shifts(const unsigned long long* mx, int R, int P, int* shift) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const double m = __longlong_as_double((long long)mx[r]);
  int e = 0;
  frexp(m, &e);
  shift[r] = m == 0.0 ? 0 : P - e;
}
__device__ __forceinline__ uint4 pack16(const int8_t (&b)[16]) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    w[i] = (uint32_t)(uint8_t)b[4 * i] | ((uint32_t)(uint8_t)b[4 * i + 1] << 8) |
           ((uint32_t)(uint8_t)b[4 * i + 2] << 16) | ((uint32_t)(uint8_t)b[4 * i + 3] << 24);
  return make_uint4(w[0], w[1], w[2], w[3]);
}
// one thread = 16 K-consecutive elements of one plane row (= 16 output bytes
// per modulus); consecutive threads take consecutive plane rows, so every
// modulus' stores of a warp are one contiguous 512-byte run.
// rows: X is R x K row-major (plane row r = X row r)
__global__ void conv_rows(const double* X, int R, int K, const int* shift, int NM,
                          int8_t* planes, int TR) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x, k0 = blockIdx.y * 16;
  if (r >= R) return;
  const int sh = shift[r];
  double v[16];
#pragma unroll
  for (int i = 0; i < 16; i += 2) {
    const double2 x = *reinterpret_cast<const double2*>(X + (size_t)r * K + k0 + i);
    v[i] = rint(ldexp(x.x, sh));
    v[i + 1] = rint(ldexp(x.y, sh));
  }
  for (int t = 0; t < NM; ++t) {
    int8_t b[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) b[i] = resid(v[i], t);
    *reinterpret_cast<uint4*>(planes + plane_off(t, r, k0, R, K, TR)) = pack16(b);
  }
}
// cols: X is K x N row-major (plane row c = X column c)
__global__ void conv_cols(const double* X, int K, int N, const int* shift, int NM,
                          int8_t* planes, int TR) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x, k0 = blockIdx.y * 16;
  if (c >= N) return;
  const int sh = shift[c];
  double v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = rint(ldexp(X[(size_t)(k0 + i) * N + c], sh));
  for (int t = 0; t < NM; ++t) {
    int8_t b[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) b[i] = resid(v[i], t);
    *reinterpret_cast<uint4*>(planes + plane_off(t, c, k0, N, K, TR)) = pack16(b);
  }
}

__global__ void __launch_bounds__(THREADS, 1)
gemm_mod(const int8_t* Ap, const int8_t* Bp, int8_t* Rout, int M, int N, int K) {
  extern __shared__ __align__(1024) int8_t sm[];
  __shared__ __align__(8) uint64_t bar_free[NSTAGE];
  __shared__ __align__(8) uint64_t bar_full[NSTAGE];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t = blockIdx.z;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)), "r"(TN));
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
  const int nk = K / KS;
  const uint32_t idesc = idesc_i8(TM, TN);
  const size_t kb32 = K / 32;
  const int8_t* abase = Ap + (((size_t)t * (M / TM) + blockIdx.y) * kb32) * 32 * TM;
  const int8_t* bbase = Bp + (((size_t)t * (N / TN) + blockIdx.x) * kb32) * 32 * TN;
  if (tid == 0) {
    auto fill = [&](int stage, int kb) {
      const uint32_t bar = smem_u32(&bar_full[stage]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(STAGE));
      int8_t* base = sm + stage * STAGE;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                   ::"r"(smem_u32(base)), "l"(abase + (size_t)kb * A_ST), "r"(A_ST), "r"(bar) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                   ::"r"(smem_u32(base + A_ST)), "l"(bbase + (size_t)kb * B_ST), "r"(B_ST), "r"(bar) : "memory");
    };
    uint32_t ph_full[NSTAGE] = {}, ph_free[NSTAGE] = {};
    for (int p = 0; p < NSTAGE - 1 && p < nk; ++p) fill(p, p);
    for (int kb = 0; kb < nk; ++kb) {
      const int st = kb % NSTAGE;
      asm volatile("{\n.reg .pred p;\nWF:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WF;\n}\n" ::"r"(smem_u32(&bar_full[st])), "r"(ph_full[st]));
      ph_full[st] ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;\n");
#pragma unroll
      for (int j = 0; j < KS / 32; ++j) {
        const uint64_t da = make_desc(smem_u32(sm + st * STAGE + j * 32 * TM), TM * 16, 128);
        const uint64_t db = make_desc(smem_u32(sm + st * STAGE + A_ST + j * 32 * TN), TN * 16, 128);
        const uint32_t acc = (kb > 0 || j > 0) ? 1u : 0u;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                     "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar_free[st])));
      const int nxt = kb + NSTAGE - 1;
      if (nxt < nk) {
        const int rst = nxt % NSTAGE;
        if (kb >= 1) {
          asm volatile("{\n.reg .pred p;\nWR:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WR;\n}\n" ::"r"(smem_u32(&bar_free[rst])), "r"(ph_free[rst]));
          ph_free[rst] ^= 1;
        }
        fill(rst, nxt);
      }
    }
    const int st = (nk - 1) % NSTAGE;
    // the last stage's final commit is the only one never waited on, and
    // tcgen05.commit tracks every earlier MMA of this thread
    asm volatile("{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}\n" ::"r"(smem_u32(&bar_free[st])), "r"(ph_free[st]));
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const int row = m0 + warp * 32 + lane;
  const int mod = c_mod[t];
  const float inv = c_inv[t];
  int8_t* dst = Rout + ((size_t)t * M + row) * N + n0;
#pragma unroll 1
  for (int cb = 0; cb < TN; cb += 32) {
    uint32_t v[32];
    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + cb;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    uint32_t packed[8];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int x = (int)v[j];
      int r = x - __float2int_rn(__int2float_rn(x) * inv) * mod;
      if (r > 127) r -= mod;
      if (r < -128) r += mod;
      const uint32_t b = (uint32_t)(r & 0xff);
      if ((j & 3) == 0) packed[j >> 2] = b;
      else packed[j >> 2] |= b << (8 * (j & 3));
    }
    uint4* d4 = reinterpret_cast<uint4*>(dst + cb);
    d4[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
    d4[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TN));
}


// Cluster (1, 2, 1) variant: the two CTAs of a cluster take vertically
// adjacent 128 x 256 tiles, so they need the same B stage; each loads its
// own A stage and HALF of the B stage, multicast into both CTAs' shared
// memory (cp.async.bulk ... .multicast::cluster).  A stage is refilled only
// when both CTAs' MMAs have read it: each MMA commit is multicast to both
// CTAs' free barriers (count 2).  Producer and MMA issuer are separate
// warps.
template <int CM>
__global__ void __launch_bounds__(THREADS, 1)
gemm_mod_mc(const int8_t* Ap, const int8_t* Bp, int8_t* Rout, int M, int N, int K) {
  extern __shared__ __align__(1024) int8_t sm[];
  __shared__ __align__(8) uint64_t bar_free[NSTAGE];
  __shared__ __align__(8) uint64_t bar_full[NSTAGE];
  __shared__ __align__(8) uint64_t bar_done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
  const int t = blockIdx.z;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)), "r"(TN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int i = 0; i < NSTAGE; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&bar_free[i])), "r"(CM));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar_full[i])));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar_done)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  const int nk = K / KS;
  const size_t kb32 = K / 32;
  const int8_t* abase = Ap + (((size_t)t * (M / TM) + blockIdx.y) * kb32) * 32 * TM;
  const int8_t* bbase = Bp + (((size_t)t * (N / TN) + blockIdx.x) * kb32) * 32 * TN;
  constexpr int BH = B_ST / CM;
  const unsigned short cmask = (unsigned short)((1 << CM) - 1);
  if (warp == 0 && lane == 0) {
    for (int kb = 0; kb < nk; ++kb) {
      const int st = kb % NSTAGE;
      if (kb >= NSTAGE) {
        const uint32_t par = ((kb / NSTAGE) - 1) & 1;
        asm volatile("{\n.reg .pred p;\nWR:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WR;\n}\n" ::"r"(smem_u32(&bar_free[st])), "r"(par) : "memory");
      }
      const uint32_t bar = smem_u32(&bar_full[st]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(STAGE));
      int8_t* base = sm + st * STAGE;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                   ::"r"(smem_u32(base)), "l"(abase + (size_t)kb * A_ST), "r"(A_ST), "r"(bar) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;\n"
                   ::"r"(smem_u32(base + A_ST + rank * BH)), "l"(bbase + (size_t)kb * B_ST + rank * BH), "r"(BH), "r"(bar), "h"(cmask) : "memory");
    }
  } else if (warp == 1 && lane == 0) {
    const uint32_t idesc = idesc_i8(TM, TN);
    for (int kb = 0; kb < nk; ++kb) {
      const int st = kb % NSTAGE;
      const uint32_t par = (kb / NSTAGE) & 1;
      asm volatile("{\n.reg .pred p;\nWF:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WF;\n}\n" ::"r"(smem_u32(&bar_full[st])), "r"(par) : "memory");
      asm volatile("tcgen05.fence::after_thread_sync;\n");
#pragma unroll
      for (int j = 0; j < KS / 32; ++j) {
        const uint64_t da = make_desc(smem_u32(sm + st * STAGE + j * 32 * TM), TM * 16, 128);
        const uint64_t db = make_desc(smem_u32(sm + st * STAGE + A_ST + j * 32 * TN), TN * 16, 128);
        const uint32_t acc = (kb > 0 || j > 0) ? 1u : 0u;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                     "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
                   ::"r"(smem_u32(&bar_free[st])), "h"(cmask));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar_done)));
  }
  __syncwarp();
  asm volatile("{\n.reg .pred p;\nWD:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra WD;\n}\n" ::"r"(smem_u32(&bar_done)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const int row = m0 + warp * 32 + lane;
  const int mod = c_mod[t];
  const float inv = c_inv[t];
  int8_t* dst = Rout + ((size_t)t * M + row) * N + n0;
#pragma unroll 1
  for (int cb = 0; cb < TN; cb += 32) {
    uint32_t v[32];
    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + cb;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    uint32_t packed[8];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int x = (int)v[j];
      int r = x - __float2int_rn(__int2float_rn(x) * inv) * mod;
      if (r > 127) r -= mod;
      if (r < -128) r += mod;
      const uint32_t b = (uint32_t)(r & 0xff);
      if ((j & 3) == 0) packed[j >> 2] = b;
      else packed[j >> 2] |= b << (8 * (j & 3));
    }
    uint4* d4 = reinterpret_cast<uint4*>(dst + cb);
    d4[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
    d4[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TN));
}

// 2-CTA variant (cta_group::2): a cluster pair computes a 256 x 256 tile;
// CTA rank r holds A rows [128 r, +128) and B^T rows [128 r, +128) of the
// pair's tile (planes with 128-row tiles for both operands) and receives
// D rows [128 r, +128) x 256 in its own TMEM.  The leader (rank 0) issues
// tcgen05.mma.cta_group::2 (M = 256, N = 256); each CTA's thread 0 fills its
// own stages; the peer forwards "my stage landed" to the leader's full
// barrier by a remote arrive; the leader's commit frees the stage in both
// CTAs (multicast).
constexpr int P_ST = 2 * 128 * KS;  // 32 KiB per stage per CTA
template <int NST>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
gemm_mod2(const int8_t* Ap, const int8_t* Bp, int8_t* Rout, int M, int N, int K) {
  extern __shared__ __align__(1024) int8_t sm[];
  __shared__ __align__(8) uint64_t bar_free[NST];
  __shared__ __align__(8) uint64_t bar_full[NST];
  __shared__ __align__(8) uint64_t bar_done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
  const int t = blockIdx.z;
  const int nx = blockIdx.x >> 1, my = blockIdx.y;
  const int atile = 2 * my + rank, btile = 2 * nx + rank;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar_free[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&bar_full[i])), "r"(rank == 0 ? 2 : 1));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar_done)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  const int nk = K / KS;
  const size_t kb32 = K / 32;
  const int8_t* abase = Ap + (((size_t)t * (M / 128) + atile) * kb32) * 32 * 128;
  const int8_t* bbase = Bp + (((size_t)t * (N / 128) + btile) * kb32) * 32 * 128;
  // warp 0 / lane 0: producer (this CTA's halves of each stage)
  // warp 1 / lane 0: leader -> MMA issuer; peer -> forwards "landed" to the leader
  if (warp == 0 && lane == 0) {
    for (int kb = 0; kb < nk; ++kb) {
      const int st = kb % NST;
      if (kb >= NST) {
        const uint32_t par = ((kb / NST) - 1) & 1;
        asm volatile("{\n.reg .pred p;\nWR:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WR;\n}\n" ::"r"(smem_u32(&bar_free[st])), "r"(par) : "memory");
      }
      const uint32_t bar = smem_u32(&bar_full[st]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(P_ST));
      int8_t* base = sm + st * P_ST;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                   ::"r"(smem_u32(base)), "l"(abase + (size_t)kb * 128 * KS), "r"(128 * KS), "r"(bar) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                   ::"r"(smem_u32(base + 128 * KS)), "l"(bbase + (size_t)kb * 128 * KS), "r"(128 * KS), "r"(bar) : "memory");
    }
  } else if (warp == 1 && lane == 0) {
    uint32_t leader_full0;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;\n" : "=r"(leader_full0) : "r"(smem_u32(&bar_full[0])));
    const uint32_t idesc = idesc_i8(256, 256);
    for (int kb = 0; kb < nk; ++kb) {
      const int st = kb % NST;
      const uint32_t par = (kb / NST) & 1;
      asm volatile("{\n.reg .pred p;\nWF:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WF;\n}\n" ::"r"(smem_u32(&bar_full[st])), "r"(par) : "memory");
      if (rank != 0) {
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(leader_full0 + st * 8) : "memory");
        continue;
      }
      asm volatile("tcgen05.fence::after_thread_sync;\n");
#pragma unroll
      for (int j = 0; j < KS / 32; ++j) {
        const uint64_t da = make_desc(smem_u32(sm + st * P_ST + j * 32 * 128), 128 * 16, 128);
        const uint64_t db = make_desc(smem_u32(sm + st * P_ST + 128 * KS + j * 32 * 128), 128 * 16, 128);
        const uint32_t acc = (kb > 0 || j > 0) ? 1u : 0u;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                     "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
                   ::"r"(smem_u32(&bar_free[st])), "h"((unsigned short)3));
    }
    if (rank == 0)
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
                   ::"r"(smem_u32(&bar_done)), "h"((unsigned short)3));
  }
  __syncwarp();
  // every thread: the pair's MMAs are complete (this CTA's TMEM is final)
  asm volatile("{\n.reg .pred p;\nWD:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra WD;\n}\n" ::"r"(smem_u32(&bar_done)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const int row = 256 * my + 128 * rank + warp * 32 + lane;
  const int n0 = 256 * nx;
  const int mod = c_mod[t];
  const float inv = c_inv[t];
  int8_t* dst = Rout + ((size_t)t * M + row) * N + n0;
#pragma unroll 1
  for (int cb = 0; cb < 256; cb += 32) {
    uint32_t v[32];
    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + cb;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    uint32_t packed[8];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int x = (int)v[j];
      int r = x - __float2int_rn(__int2float_rn(x) * inv) * mod;
      if (r > 127) r -= mod;
      if (r < -128) r += mod;
      const uint32_t b = (uint32_t)(r & 0xff);
      if ((j & 3) == 0) packed[j >> 2] = b;
      else packed[j >> 2] |= b << (8 * (j & 3));
    }
    uint4* d4 = reinterpret_cast<uint4*>(dst + cb);
    d4[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
    d4[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(256));
}

// residues -> C = (sum_t r_t W_t mod M) 2^-(sa_i + sb_j); 8 columns per thread
__global__ void crt(const int8_t* Rr, int NM, int M, int N, const int* sa, const int* sb, double* C) {
  const size_t idx = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (idx >= (size_t)M * N) return;
  const int i = idx / N, j = idx % N;
  double s[8][LV];
#pragma unroll
  for (int e = 0; e < 8; ++e)
#pragma unroll
    for (int l = 0; l < LV; ++l) s[e][l] = 0.0;
  for (int t = 0; t < NM; ++t) {
    const uint2 w = *reinterpret_cast<const uint2*>(Rr + (size_t)t * M * N + idx);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int8_t r = (int8_t)(((e < 4 ? w.x : w.y) >> (8 * (e & 3))) & 0xff);
      const double rd = (double)r;
#pragma unroll
      for (int l = 0; l < LV; ++l) s[e][l] = fma(rd, c_w[t][l], s[e][l]);
    }
  }
  const double two40 = ldexp(1.0, LVB), two80 = ldexp(1.0, 2 * LVB);
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const double approx = fma(s[e][0], two80, fma(s[e][1], two40, s[e][2]));
    const double q = rint(approx * c_invM);
    const double d0 = fma(-q, c_M[0], s[e][0]);
    const double d1 = fma(-q, c_M[1], s[e][1]);
    const double d2 = fma(-q, c_M[2], s[e][2]);
    const double v = fma(d0, two80, fma(d1, two40, d2));
    C[idx + e] = ldexp(v, -(sa[i] + sb[j + e]));
  }
}

__global__ void dgemm_ref(const double* A, const double* B, double* C, int N) {
  __shared__ double As[16][16], Bs[16][17];
  const int i = blockIdx.y * 16 + threadIdx.y, j = blockIdx.x * 16 + threadIdx.x;
  double s = 0.0;
  for (int k0 = 0; k0 < N; k0 += 16) {
    As[threadIdx.y][threadIdx.x] = A[(size_t)i * N + k0 + threadIdx.x];
    Bs[threadIdx.y][threadIdx.x] = B[(size_t)(k0 + threadIdx.y) * N + j];
    __syncthreads();
    for (int k = 0; k < 16; ++k) s = fma(As[threadIdx.y][k], Bs[k][threadIdx.x], s);
    __syncthreads();
  }
  C[(size_t)i * N + j] = s;
}

typedef unsigned __int128 u128;

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 1024;
  const int NM = argc > 2 ? atoi(argv[2]) : 15;
  const int spread = argc > 3 ? atoi(argv[3]) : 6;
  const int mods_all[MAXM] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197};
  // CRT constants
  u128 Mp = 1;
  for (int t = 0; t < NM; ++t) Mp *= (u128)mods_all[t];
  double log2M = 0;
  for (int t = 0; t < NM; ++t) log2M += log2((double)mods_all[t]);
  const int P = (int)floor((log2M - 2.0 - log2((double)N)) / 2.0);
  int hmod[MAXM];
  float hinv[MAXM];
  double hw[MAXM][LV], hM[LV];
  const u128 mask = (((u128)1) << LVB) - 1;
  for (int t = 0; t < NM; ++t) {
    const int m = mods_all[t];
    hmod[t] = m;
    hinv[t] = 1.0f / (float)m;
    const u128 Mt = Mp / (u128)m;
    const int a = (int)(Mt % (u128)m);
    int inv = 0;
    for (int x = 1; x < m; ++x)
      if ((a * x) % m == 1) { inv = x; break; }
    const u128 W = (Mt * (u128)inv) % Mp;
    for (int l = 0; l < LV; ++l) hw[t][l] = (double)(uint64_t)((W >> (LVB * (LV - 1 - l))) & mask);
  }
  for (int l = 0; l < LV; ++l) hM[l] = (double)(uint64_t)((Mp >> (LVB * (LV - 1 - l))) & mask);
  const double hinvM = 1.0 / ((double)(uint64_t)(Mp >> 64) * 18446744073709551616.0 + (double)(uint64_t)Mp);
  cudaMemcpyToSymbol(c_mod, hmod, sizeof(hmod));
  cudaMemcpyToSymbol(c_inv, hinv, sizeof(hinv));
  cudaMemcpyToSymbol(c_w, hw, sizeof(hw));
  cudaMemcpyToSymbol(c_M, hM, sizeof(hM));
  cudaMemcpyToSymbol(c_invM, &hinvM, sizeof(hinvM));
  printf("N=%d NM=%d log2M=%.2f P=%d\n", N, NM, log2M, P);

  const size_t nn = (size_t)N * N;
  std::vector<double> hA(nn), hB(nn);
  srand(7);
  for (auto& x : hA) x = (rand() / (double)RAND_MAX - 0.5) * pow(10.0, (rand() % (spread + 1)) - spread / 2);
  for (auto& x : hB) x = (rand() / (double)RAND_MAX - 0.5);
  double *A, *B, *C, *Cref;
  int8_t *Ap, *Bp, *Rr;
  int *sa, *sb;
  cudaMalloc(&A, nn * 8); cudaMalloc(&B, nn * 8);
  cudaMalloc(&C, nn * 8); cudaMalloc(&Cref, nn * 8);
  cudaMalloc(&Ap, nn * NM); cudaMalloc(&Bp, nn * NM); cudaMalloc(&Rr, nn * NM);
  cudaMalloc(&sa, N * 4); cudaMalloc(&sb, N * 4);
  cudaMemcpy(A, hA.data(), nn * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB.data(), nn * 8, cudaMemcpyHostToDevice);
  const int smem = NSTAGE * STAGE;
  cudaFuncSetAttribute(gemm_mod, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int eb = 256;
  const unsigned ge = (unsigned)((nn + eb - 1) / eb);
  unsigned long long *mxa, *mxb;
  cudaMalloc(&mxa, N * 8); cudaMalloc(&mxb, N * 8);
  const bool slow = getenv("OZ_SLOWCONV") != nullptr;
  const int pair = getenv("OZ_PAIR") ? atoi(getenv("OZ_PAIR")) : 0;
  cudaFuncSetAttribute(gemm_mod2<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * P_ST);
  cudaFuncSetAttribute(gemm_mod_mc<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(gemm_mod_mc<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int mc = getenv("OZ_MC") ? atoi(getenv("OZ_MC")) : 0;
  cudaFuncSetAttribute(gemm_mod2<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * P_ST);
  auto conv = [&]() {
    if (slow) {
      scale_rows<<<N, 256>>>(A, N, N, P, sa);
      scale_cols<<<(N + 255) / 256, 256>>>(B, N, N, P, sb);
      residues_rows<<<ge, eb>>>(A, N, N, sa, NM, Ap, TM);
      residues_cols<<<ge, eb>>>(B, N, N, sb, NM, Bp, TN);
      return;
    }
    cudaMemsetAsync(mxb, 0, N * 8);
    absmax_rows<<<(N + 7) / 8, 256>>>(A, N, N, mxa);
    absmax_cols<<<dim3((N + 255) / 256, (N + 255) / 256), 256>>>(B, N, N, 256, mxb);
    shifts<<<(N + 255) / 256, 256>>>(mxa, N, P, sa);
    shifts<<<(N + 255) / 256, 256>>>(mxb, N, P, sb);
    conv_rows<<<dim3((N + 127) / 128, N / 16), 128>>>(A, N, N, sa, NM, Ap, TM);
    conv_cols<<<dim3((N + 127) / 128, N / 16), 128>>>(B, N, N, sb, NM, Bp, pair ? 128 : TN);
  };
  auto gemm = [&]() {
    if (mc) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = mc; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      cfg.gridDim = dim3(N / TN, N / TM, NM); cfg.blockDim = dim3(THREADS); cfg.dynamicSmemBytes = smem;
      cudaError_t le = mc == 4 ? cudaLaunchKernelEx(&cfg, gemm_mod_mc<4>, (const int8_t*)Ap, (const int8_t*)Bp, Rr, N, N, N)
                              : cudaLaunchKernelEx(&cfg, gemm_mod_mc<2>, (const int8_t*)Ap, (const int8_t*)Bp, Rr, N, N, N);
      if (le != cudaSuccess) printf("launch: %s\n", cudaGetErrorString(le));
    }
    else if (pair == 6) gemm_mod2<6><<<dim3(2 * (N / 256), N / 256, NM), THREADS, 6 * P_ST>>>(Ap, Bp, Rr, N, N, N);
    else if (pair) gemm_mod2<4><<<dim3(2 * (N / 256), N / 256, NM), THREADS, 4 * P_ST>>>(Ap, Bp, Rr, N, N, N);
    else gemm_mod<<<dim3(N / TN, N / TM, NM), THREADS, smem>>>(Ap, Bp, Rr, N, N, N);
  };
  auto rec = [&]() { crt<<<(unsigned)((nn / 8 + 255) / 256), 256>>>(Rr, NM, N, N, sa, sb, C); };
  conv(); gemm(); rec();
  cudaError_t e = cudaDeviceSynchronize();
  printf("run: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  cudaEvent_t e0, e1, e2, e3;
  cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2); cudaEventCreate(&e3);
  const int reps = 5;
  float tc = 0, tg = 0, tr = 0;
  for (int i = 0; i < reps; ++i) {
    cudaEventRecord(e0); conv(); cudaEventRecord(e1); gemm(); cudaEventRecord(e2); rec(); cudaEventRecord(e3);
    cudaEventSynchronize(e3);
    float a, b, c;
    cudaEventElapsedTime(&a, e0, e1); cudaEventElapsedTime(&b, e1, e2); cudaEventElapsedTime(&c, e2, e3);
    tc += a; tg += b; tr += c;
  }
  tc /= reps; tg /= reps; tr /= reps;
  dgemm_ref<<<dim3(N / 16, N / 16), dim3(16, 16)>>>(A, B, Cref, N);
  cudaDeviceSynchronize();
  std::vector<double> hC(nn), hR(nn);
  cudaMemcpy(hC.data(), C, nn * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hR.data(), Cref, nn * 8, cudaMemcpyDeviceToHost);
  // normwise (1-norm) and max-entry relative differences
  std::vector<double> cs(N, 0.0), cr(N, 0.0);
  double num = 0, den = 0;
  for (size_t i = 0; i < nn; ++i) {
    num = fmax(num, fabs(hC[i] - hR[i])); den = fmax(den, fabs(hR[i]));
    cs[i % N] += fabs(hC[i] - hR[i]); cr[i % N] += fabs(hR[i]);
  }
  double n1d = 0, n1r = 0;
  for (int j = 0; j < N; ++j) { n1d = fmax(n1d, cs[j]); n1r = fmax(n1r, cr[j]); }
  const double fl = 2.0 * N * N * (double)N;
  printf("N=%d NM=%d  max|C-Cref|/max|Cref| = %.3e  rel 1-norm diff = %.3e\n", N, NM, num / den, n1d / n1r);
  printf("  conv %.3f ms  gemm %.3f ms (%.1f TF/s fp64-equiv, %.0f int8 TOPS)  crt %.3f ms  total %.3f ms = %.1f TF/s\n",
         tc, tg, fl / tg / 1e9, NM * fl / tg / 1e9, tr, tc + tg + tr, fl / (tc + tg + tr) / 1e9);
  return 0;
}
