// ozaki.cuh -- the Ozaki-II product engine of the tiled chain (included by
// tiled.cu inside namespace csm::tk; selected by csm_set_engine).
//
// One chain op's product acc = L R (FP64, NP x NP, K = NP) is computed
// exactly on integers and rebuilt by the Chinese remainder theorem:
//   * L's rows and R's columns are scaled by powers of two so that
//     |L'|, |R'| < 2^P and rounded to integers (oz_rowmax / oz_colmax give
//     the per-row / per-column max, oz_conv_* the scaled integers' residues
//     modulo nm pairwise coprime moduli m_t <= 256, as int8 planes in the
//     canonical K-major UMMA layout, tile-major);
//   * each modulus is ONE 8-bit GEMM on the 5th-generation tensor cores
//     (oz_gemm_p: tcgen05.mma.kind::i8 on unsigned residues in [0, m_t),
//     int32 accumulators in TMEM, exact because sum <= K 255^2 < 2^31 for
//     K <= 33025), reduced mod m_t to an int8 residue in [-128, 127];
//   * oz_crt_epi rebuilds L'R' = sum_t r_t W_t mod M (M = prod m_t) in three
//     42-bit fp64 levels, undoes the scaling, and runs the op's
//     epilogue (the same epilogue_tile as the DMMA kernel).
// P is the largest value with K 2^(2P) <= M / 4, so the integer product is
// exact and the only error is the rounding of L and R to P bits relative to
// their row / column maxima: P = 55..57 for nm = 16 (fp64 results), 30 for
// nm = 9 (float32 results).  Tensor work per product: nm int8 GEMMs.
// Residues: v mod G for groups of moduli with G < 2^24 (fp64 FMA pipe),
// then each modulus by integer multiply-high (no conversion instructions).
//
// Reference: the products are matcore.py:90-97 (`a @ b`, ledger +1); the
// engine changes how each product is computed, not the chain.

constexpr int OZ_MAXM = 16, OZ_LV = 3, OZ_LVB = 42;
constexpr int OZ_MAXG = 6;  // moduli groups with products below 2^24
constexpr int OZ_TM = 128, OZ_TN = 256, OZ_KS = 128, OZ_NSTAGE = 4;
constexpr int OZ_A_ST = OZ_TM * OZ_KS, OZ_B_ST = OZ_TN * OZ_KS, OZ_STAGE = OZ_A_ST + OZ_B_ST;
constexpr size_t OZ_SMEM = static_cast<size_t>(OZ_NSTAGE) * OZ_STAGE;  // 192 KiB
// one-CTA-per-tile oz_gemm (CSM_OZ_GEMM=tile) for NP <= 1024: 2 stages
// (96 KiB) so two CTAs share an SM and one's epilogue overlaps the other's
constexpr int OZ_NSTAGE_SMALL = 2;
constexpr int OZ_THREADS = 128;
// oz_crt_epi: the 64 x 64 product tile in the epilogue's padded layout only
constexpr size_t OZ_CRT_SMEM = static_cast<size_t>(BM) * LDE * sizeof(double);

struct OzConst {
  int nm, P;
  int mod[OZ_MAXM];
  uint32_t cdiv[OZ_MAXM];    // floor(2^32 / m_t): x / m_t by multiply-high
  double gmod[OZ_MAXG];      // product of moduli 3g .. 3g + 2 (< 2^24)
  double ginv[OZ_MAXG];      // 1 / gmod
  double w[OZ_MAXM][OZ_LV];  // W_t = (M/m_t) ((M/m_t)^-1 mod m_t) in 42-bit digits, high first
  double M[OZ_LV];
  double invM;
};

struct OzArgs {
  int item0, nitems;
  unsigned long long* mxL;  // [nitems][M]  max |L| per row (u64 bits of a double >= 0)
  unsigned long long* mxR;  // [nitems][NP] max |R| per column
  int8_t* pL;               // [nitems][nm][M x NP]  residue planes of L'
  int8_t* pR;               // [nitems][nm][NP x NP] residue planes of R'^T
  int8_t* res;              // [nitems][nm][M x NP]  residues of L'R'
  unsigned* bad;            // [nitems] nonzero: L or R holds a non-finite entry
  // accuracy guard (oz_guard): sums over the real n x n block only
  double* rsumL;            // [nitems][M]           sum_k |L_rk| per row
  double* csumR;            // [nitems][NP/64][NP]   sum_k |R_kc| per 64-row chunk
  double* csumC;            // [nitems][M/64][NP]    sum_r |C_rc| per 64-row tile
  unsigned* flag;           // [nitems] 1: rerun this item's product on DMMA
};

__device__ __forceinline__ void oz_item(const LaunchArgs& a, int item, int& opi, int& b) {
  Seg sg = a.seg[0];
#pragma unroll
  for (int i = 1; i < MAXSEG; ++i)
    if (i < a.nseg && item >= a.seg[i].start) sg = a.seg[i];
  opi = sg.op;
  b = a.idx[sg.idx_off + item - sg.start];
}
__device__ __forceinline__ const double* oz_lhs(const LaunchArgs& a, int item) {
  int opi, b;
  oz_item(a, item, opi, b);
  return slot_ptr(a, b, a.ops[opi].lhs);
}
__device__ __forceinline__ const double* oz_rhs(const LaunchArgs& a, int item) {
  int opi, b;
  oz_item(a, item, opi, b);
  return a.rhs_full ? a.rhs_full : slot_ptr(a, b, a.ops[opi].rhs);
}
// Chunk-local item whose right-operand residues item ci uses.  A doubling
// launch pairs S C and C C per group (consecutive segments with the same
// matrices, doubling_ops): the second op's items take the first's planes of
// C when those are in the same chunk, so C is converted once per step.
__device__ __forceinline__ int oz_rsrc(const LaunchArgs& a, const OzArgs& oz, int ci) {
  if (a.dbl_step < 0) return ci;
  const int item = oz.item0 + ci;
  int k = 0;
#pragma unroll
  for (int i = 1; i < MAXSEG; ++i)
    if (i < a.nseg && item >= a.seg[i].start) k = i;
  if ((k & 1) == 0) return ci;
  const int partner = item - (a.seg[k].start - a.seg[k - 1].start);
  return partner >= oz.item0 ? partner - oz.item0 : ci;
}
// |x| for the maxima, with NaN mapped to +Inf (fmax would drop it): a row or
// column holding a non-finite entry gets max +Inf, and every product entry
// it touches is NaN (oz_crt_epi), as an fp64 GEMM would make it non-finite
__device__ __forceinline__ double oz_absmax(double m, double x) {
  const double a = fabs(x);
  return a <= 1.7976931348623157e308 ? fmax(m, a) : __longlong_as_double(0x7ff0000000000000ll);
}
constexpr unsigned long long OZ_INF_BITS = 0x7ff0000000000000ull;
// 2^shift scales a row (column) whose max |x| has bits mx below 2^P
__device__ __forceinline__ int oz_shift(unsigned long long mx, int P) {
  if (mx >= OZ_INF_BITS) return 0;  // non-finite row / column: result is NaN anyway
  const double m = __longlong_as_double(static_cast<long long>(mx));
  int e = 0;
  frexp(m, &e);
  return m == 0.0 ? 0 : P - e;
}
// K-major canonical layout, tile-major: plane t of R rows x K, tile rows TR
__device__ __forceinline__ size_t oz_off(int r, int k, int K, int TR) {
  return ((static_cast<size_t>(r / TR) * (K / 32) + k / 32) * 2 + (k % 32) / 16) * TR * 16 +
         (r % TR) * 16 + k % 16;
}
// v: an integer-valued double, |v| <= 2^57.  x = (v mod G) + G in [0, 2G)
// for a group's product of moduli G < 2^24, without the conversion pipe:
// the quotient is rounded by the 1.5 2^52 trick (|v / G| < 2^51), the fma
// remainder is exact, and the same trick hands its integer bits over.
// Then each modulus of the group: floor(x / m) by multiply-high with
// floor(2^32 / m) (x < 2^25: at most one short) and one correction: the
// residue in [0, m) (the GEMM runs unsigned 8-bit operands).  Integer / FMA
// pipes only.
__device__ __forceinline__ uint32_t oz_mod_group(double v, double G, double invG) {
  const double M52 = 6755399441055744.0;  // 1.5 * 2^52
  const double q = fma(v, invG, M52) - M52;
  const double r = fma(-q, G, v);  // |r| < G
  return static_cast<uint32_t>(__double2loint(r + M52)) + static_cast<uint32_t>(G);
}
__device__ __forceinline__ int oz_mod_small(uint32_t x, const OzConst& C, int t) {
  const uint32_t m = static_cast<uint32_t>(C.mod[t]);
  uint32_t r = x - __umulhi(x, C.cdiv[t]) * m;  // in [0, 2m)
  if (r >= m) r -= m;
  return static_cast<int>(r);
}
// C_t (0 <= C_t <= K 255^2 < 2^31) mod m_t as a representative in
// [-128, 127] for the CRT: multiply-high quotient (C_t < 2^32: at most one
// short), one correction, then the symmetric range.
__device__ __forceinline__ int oz_mod_acc(uint32_t x, uint32_t m, uint32_t cdiv) {
  uint32_t r = x - __umulhi(x, cdiv) * m;
  if (r >= m) r -= m;
  return r > 127u ? static_cast<int>(r) - static_cast<int>(m) : static_cast<int>(r);
}

// grid (M / 8, nitems), 256 threads: one warp per row of L
__global__ void oz_rowmax(const LaunchArgs la, const OzArgs oz) {
  const int ci = blockIdx.y;
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  const int NP = la.NP;
  const double* L = oz_lhs(la, oz.item0 + ci) + static_cast<size_t>(r) * NP;
  double m = 0.0, sum = 0.0;
  for (int k = lane * 2; k < NP; k += 64) {
    const double2 v = *reinterpret_cast<const double2*>(L + k);
    m = oz_absmax(oz_absmax(m, v.x), v.y);
    sum += fabs(v.x) + fabs(v.y);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
  }
  if (lane == 0) {
    oz.mxL[static_cast<size_t>(ci) * la.M + r] = __double_as_longlong(m);
    // row sums of the real block only (row0 + r < n in slab mode: n == NP)
    oz.rsumL[static_cast<size_t>(ci) * la.M + r] = r < la.n ? sum : 0.0;
    if (!(m <= 1.7976931348623157e308)) atomicOr(oz.bad + ci, 1u);
  }
}
// grid (NP / 256, NP / 64, nitems), 256 threads: column maxima of R over
// 64-row chunks, combined by atomicMax (mxR zeroed beforehand); the chunk's
// column sums (real block) go to csumR for the accuracy guard
__global__ void oz_colmax(const LaunchArgs la, const OzArgs oz) {
  const int ci = blockIdx.z, NP = la.NP;
  if (oz_rsrc(la, oz, ci) != ci) return;  // shares an earlier item's right operand
  const int c = blockIdx.x * 256 + threadIdx.x, k0 = blockIdx.y * 64;
  const double* R = oz_rhs(la, oz.item0 + ci);
  double m = 0.0, sum = 0.0;
#pragma unroll 8
  for (int k = k0; k < k0 + 64; ++k) {
    const double x = R[static_cast<size_t>(k) * NP + c];
    m = oz_absmax(m, x);
    sum += k < la.n ? fabs(x) : 0.0;
  }
  atomicMax(oz.mxR + static_cast<size_t>(ci) * NP + c,
            static_cast<unsigned long long>(__double_as_longlong(m)));
  oz.csumR[(static_cast<size_t>(ci) * (NP / 64) + blockIdx.y) * NP + c] = c < la.n ? sum : 0.0;
  if (!(m <= 1.7976931348623157e308)) atomicOr(oz.bad + ci, 1u);
}

__device__ __forceinline__ uint4 oz_pack16(const int (&b)[16]) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    w[i] = (static_cast<uint32_t>(b[4 * i]) & 0xffu) |
           ((static_cast<uint32_t>(b[4 * i + 1]) & 0xffu) << 8) |
           ((static_cast<uint32_t>(b[4 * i + 2]) & 0xffu) << 16) |
           ((static_cast<uint32_t>(b[4 * i + 3]) & 0xffu) << 24);
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// 16 entries -> 16 residue bytes per modulus at out + t * plane.  Moduli
// are grouped in threes (products < 2^24, host oz_const) in table order.
template <int NM>
__device__ __forceinline__ void oz_store_residues(const double (&v)[16], const OzConst& C,
                                                  int8_t* out, size_t plane) {
#pragma unroll
  for (int g = 0; g < (NM + 2) / 3; ++g) {
    uint32_t x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = oz_mod_group(v[i], C.gmod[g], C.ginv[g]);
#pragma unroll
    for (int t = 3 * g; t < 3 * g + 3 && t < NM; ++t) {
      int b[16];
#pragma unroll
      for (int i = 0; i < 16; ++i)  // m_0 = 256 divides G_0: its residue is the low byte
        b[i] = t == 0 ? static_cast<int>(x[i] & 255u) : oz_mod_small(x[i], C, t);
      *reinterpret_cast<uint4*>(out + t * plane) = oz_pack16(b);
    }
  }
}

// One thread = 16 K-consecutive entries of one plane row, i.e. 16 output
// bytes per modulus; consecutive threads take consecutive plane rows, so a
// warp's stores for one modulus are one contiguous 512-byte run.
// grid (M / 128, NP / 16, nitems), 128 threads.  L rows are plane rows.
template <int NM>
__global__ void oz_conv_rows(const LaunchArgs la, const OzArgs oz, const OzConst C) {
  const int ci = blockIdx.z, NP = la.NP, M = la.M;
  const int r = blockIdx.x * 128 + threadIdx.x, k0 = blockIdx.y * 16;
  const double* L = oz_lhs(la, oz.item0 + ci) + static_cast<size_t>(r) * NP + k0;
  const int sh = oz_shift(oz.mxL[static_cast<size_t>(ci) * M + r], C.P);
  double v[16];
#pragma unroll
  for (int i = 0; i < 16; i += 2) {
    const double2 x = *reinterpret_cast<const double2*>(L + i);
    v[i] = rint(ldexp(x.x, sh));
    v[i + 1] = rint(ldexp(x.y, sh));
  }
  const size_t plane = static_cast<size_t>(M) * NP;
  oz_store_residues<NM>(v, C, oz.pL + static_cast<size_t>(ci) * NM * plane + oz_off(r, k0, NP, OZ_TM),
                    plane);
}
// grid (NP / 128, NP / 16, nitems), 128 threads.  R columns are plane rows.
template <int NM>
__global__ void oz_conv_cols(const LaunchArgs la, const OzArgs oz, const OzConst C) {
  const int ci = blockIdx.z, NP = la.NP;
  if (oz_rsrc(la, oz, ci) != ci) return;
  const int c = blockIdx.x * 128 + threadIdx.x, k0 = blockIdx.y * 16;
  const double* R = oz_rhs(la, oz.item0 + ci) + static_cast<size_t>(k0) * NP + c;
  const int sh = oz_shift(oz.mxR[static_cast<size_t>(ci) * NP + c], C.P);
  double v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = rint(ldexp(R[static_cast<size_t>(i) * NP], sh));
  const size_t plane = static_cast<size_t>(NP) * NP;
  oz_store_residues<NM>(v, C, oz.pR + static_cast<size_t>(ci) * NM * plane + oz_off(c, k0, NP, OZ_TN),
                    plane);
}

__device__ __forceinline__ uint32_t oz_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t oz_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  // canonical K-major, no swizzle: start, leading (K-adjacent core matrix)
  // and stride (8-row group) byte offsets, >> 4; bit 46: sm_100 descriptor
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) |
         (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (static_cast<uint64_t>(1) << 46);
}
// instruction descriptor: kind::i8, s32 accumulator, unsigned 8-bit A and B
// (residues in [0, m_t)), K-major
__host__ __device__ constexpr uint32_t oz_idesc(int m, int n) {
  return (2u << 4) | (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}
__device__ __forceinline__ void oz_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nOZW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra OZW_%=;\n}\n" ::"r"(oz_smem(bar)),
      "r"(parity)
      : "memory");
}

// C_t = L'_t R'_t (mod m_t) for one 128 x 256 tile of one item and modulus.
// grid (NP / 256, M / 128, nitems * nm), clusters of 2 along y, 128
// threads, NST x 48 KiB dynamic shared memory.  The two CTAs of a cluster
// take vertically adjacent tiles and so need the same B stage: each loads
// its own A stage and HALF of the B stage, multicast into both CTAs' shared
// memory (cp.async.bulk ... .multicast::cluster), which cuts the L2->SM
// operand traffic from 384 to 256 bytes per K row (measured +22% at
// NP = 8192; clusters of 4 gained nothing more).  Warp 0 lane 0 is the
// producer; warp 1 lane 0 issues four tcgen05.mma.kind::i8 (K = 32) per
// 128-deep stage into one 256-column TMEM accumulator and multicasts each
// commit to both CTAs' free barriers (count 2: a stage is refilled once
// both CTAs have read it).  Then each warp reads its 32 TMEM lanes (rows)
// 32 columns at a time, reduces mod m_t and stores the int8 residues.
template <int NST>
__global__ void __launch_bounds__(OZ_THREADS, 1) oz_gemm(const LaunchArgs la, const OzArgs oz,
                                                         const OzConst C) {
  extern __shared__ __align__(128) int8_t osm[];
  __shared__ __align__(8) uint64_t bar_free[NST];
  __shared__ __align__(8) uint64_t bar_full[NST];
  __shared__ __align__(8) uint64_t bar_done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NP = la.NP, M = la.M;
  const int ci = blockIdx.z / C.nm, t = blockIdx.z - ci * C.nm;
  const int m0 = blockIdx.y * OZ_TM, n0 = blockIdx.x * OZ_TN;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     oz_smem(&tmem_base)),
                 "r"(OZ_TN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;\n" ::"r"(oz_smem(&bar_free[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(oz_smem(&bar_full[i])));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(oz_smem(&bar_done)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  const int nk = NP / OZ_KS;
  const size_t kb32 = NP / 32;
  const size_t lplane = static_cast<size_t>(M) * NP, rplane = static_cast<size_t>(NP) * NP;
  const int8_t* abase = oz.pL + (static_cast<size_t>(ci) * C.nm + t) * lplane +
                        static_cast<size_t>(blockIdx.y) * kb32 * 32 * OZ_TM;
  const int8_t* bbase = oz.pR + (static_cast<size_t>(oz_rsrc(la, oz, ci)) * C.nm + t) * rplane +
                        static_cast<size_t>(blockIdx.x) * kb32 * 32 * OZ_TN;
  constexpr int BH = OZ_B_ST / 2;
  if (warp == 0 && lane == 0) {
    for (int kb = 0; kb < nk; ++kb) {
      const int st = kb % NST;
      if (kb >= NST) oz_wait(&bar_free[st], ((kb / NST) - 1) & 1);
      const uint32_t bar = oz_smem(&bar_full[st]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar),
                   "r"(OZ_STAGE));
      int8_t* base = osm + st * OZ_STAGE;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
              oz_smem(base)),
          "l"(abase + static_cast<size_t>(kb) * OZ_A_ST), "r"(OZ_A_ST), "r"(bar)
          : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
          "[%0], [%1], %2, [%3], %4;\n" ::"r"(oz_smem(base + OZ_A_ST + rank * BH)),
          "l"(bbase + static_cast<size_t>(kb) * OZ_B_ST + rank * BH), "r"(BH), "r"(bar),
          "h"(static_cast<unsigned short>(3))
          : "memory");
    }
  } else if (warp == 1 && lane == 0) {
    const uint32_t idesc = oz_idesc(OZ_TM, OZ_TN);
    for (int kb = 0; kb < nk; ++kb) {
      const int st = kb % NST;
      oz_wait(&bar_full[st], (kb / NST) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
#pragma unroll
      for (int j = 0; j < OZ_KS / 32; ++j) {
        const uint64_t da = oz_desc(oz_smem(osm + st * OZ_STAGE + j * 32 * OZ_TM), OZ_TM * 16, 128);
        const uint64_t db =
            oz_desc(oz_smem(osm + st * OZ_STAGE + OZ_A_ST + j * 32 * OZ_TN), OZ_TN * 16, 128);
        const uint32_t acc = (kb > 0 || j > 0) ? 1u : 0u;
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
          "[%0], %1;\n" ::"r"(oz_smem(&bar_free[st])),
          "h"(static_cast<unsigned short>(3)));
    }
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            oz_smem(&bar_done)));
  }
  __syncwarp();
  oz_wait(&bar_done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const int row = m0 + warp * 32 + lane;
  const int mod = C.mod[t];
  const uint32_t cdiv = C.cdiv[t];
  int8_t* dst = oz.res + (static_cast<size_t>(ci) * C.nm + t) * lplane +
                static_cast<size_t>(row) * NP + n0;
#pragma unroll 1
  for (int cb = 0; cb < OZ_TN; cb += 32) {
    uint32_t v[32];
    const uint32_t ta = tmem + (static_cast<uint32_t>(warp * 32) << 16) + cb;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
          "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
          "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    uint32_t packed[8];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      // |x| <= K 2^14 <= 2^27: the float quotient is within 0.1 of x / m, so
      // one correction lands in [-128, 127]
      const int r = oz_mod_acc(v[j], static_cast<uint32_t>(mod), cdiv);
      const uint32_t bb = static_cast<uint32_t>(r) & 0xffu;
      packed[j >> 2] = (j & 3) == 0 ? bb : (packed[j >> 2] | (bb << (8 * (j & 3))));
    }
    uint4* d4 = reinterpret_cast<uint4*>(dst + cb);
    d4[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
    d4[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  // no CTA leaves while its cluster peer may still multicast into it or
  // arrive on its barriers
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(OZ_TN));
}

// Persistent form of oz_gemm: one cluster pair per two SMs walks the pair
// tiles (x, y pair, item x modulus) round-robin, with warp roles --
// warp 0: producer (the stage ring runs on across tiles), warp 1: MMA
// issuer, warps 2..9: epilogue, two per TMEM lane quarter -- and two
// 256-column TMEM accumulators, so
// a tile's TMEM drain / residue epilogue overlaps the next tile's MMAs and
// the set-up is paid once per CTA.  grid = 2 x clusters, 320 threads,
// NST x 48 KiB dynamic shared memory.
constexpr int OZ_PEPI = 8;  // epilogue warps: two per TMEM lane quarter, 128 columns each
constexpr int OZ_PTHREADS = 32 * (2 + OZ_PEPI);
template <int NST>
__global__ void __launch_bounds__(OZ_PTHREADS, 1) oz_gemm_p(const LaunchArgs la, const OzArgs oz,
                                                            const OzConst C, int pair_tiles,
                                                            int gx) {
  extern __shared__ __align__(128) int8_t osm[];
  __shared__ __align__(8) uint64_t bar_free[NST];
  __shared__ __align__(8) uint64_t bar_full[NST];
  __shared__ __align__(8) uint64_t tm_full[2];
  __shared__ __align__(8) uint64_t tm_empty[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NP = la.NP, M = la.M;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const int nx = NP / OZ_TN, nyp = M / (2 * OZ_TM);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     oz_smem(&tmem_base)),
                 "r"(2 * OZ_TN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;\n" ::"r"(oz_smem(&bar_free[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(oz_smem(&bar_full[i])));
    }
    for (int i = 0; i < 2; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(oz_smem(&tm_full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(oz_smem(&tm_empty[i])),
                   "r"(OZ_PEPI));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  const int nk = NP / OZ_KS;
  const size_t kb32 = NP / 32;
  const size_t lplane = static_cast<size_t>(M) * NP, rplane = static_cast<size_t>(NP) * NP;
  // pair tile T -> x fastest inside a group of gx column tiles, then y pair,
  // then the next column group, then item x modulus.  The co-resident
  // clusters then share gx right-operand panels (gx x 256 x NP bytes: 16 MiB
  // at NP = 8192, gx = 8) that stay in L2 while the y pairs stream past,
  // instead of cycling through the whole 64 MiB residue plane per y pair.
  // gx = nx is the plain row-major walk.
  auto decode = [&](int T, int& x, int& y, int& z) {
    const int per_z = nx * nyp;
    z = T / per_z;
    const int t = T - z * per_z;
    const int band = gx * nyp;
    const int g = t / band, r = t - g * band;
    const int yy = r / gx;
    x = g * gx + (r - yy * gx);
    y = 2 * yy + static_cast<int>(rank);
  };
  constexpr int BH = OZ_B_ST / 2;
  if (warp == 0) {
    if (lane == 0) {
      int g = 0;  // k-block counter across tiles (the stage ring)
      for (int T = cluster; T < pair_tiles; T += nclusters) {
        int x, y, z;
        decode(T, x, y, z);
        const int ci = z / C.nm, t = z - ci * C.nm;
        const int8_t* abase = oz.pL + (static_cast<size_t>(ci) * C.nm + t) * lplane +
                              static_cast<size_t>(y) * kb32 * 32 * OZ_TM;
        const int8_t* bbase = oz.pR + (static_cast<size_t>(oz_rsrc(la, oz, ci)) * C.nm + t) * rplane +
                              static_cast<size_t>(x) * kb32 * 32 * OZ_TN;
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int st = g % NST;
          if (g >= NST) oz_wait(&bar_free[st], ((g / NST) - 1) & 1);
          const uint32_t bar = oz_smem(&bar_full[st]);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar),
                       "r"(OZ_STAGE));
          int8_t* base = osm + st * OZ_STAGE;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                  oz_smem(base)),
              "l"(abase + static_cast<size_t>(kb) * OZ_A_ST), "r"(OZ_A_ST), "r"(bar)
              : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
              "[%0], [%1], %2, [%3], %4;\n" ::"r"(oz_smem(base + OZ_A_ST + rank * BH)),
              "l"(bbase + static_cast<size_t>(kb) * OZ_B_ST + rank * BH), "r"(BH), "r"(bar),
              "h"(static_cast<unsigned short>(3))
              : "memory");
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = oz_idesc(OZ_TM, OZ_TN);
      int g = 0, i = 0;
      for (int T = cluster; T < pair_tiles; T += nclusters, ++i) {
        const int acc_i = i & 1;
        if (i >= 2) oz_wait(&tm_empty[acc_i], ((i >> 1) - 1) & 1);  // epilogue drained it
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const uint32_t dacc = tmem + acc_i * OZ_TN;
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int st = g % NST;
          oz_wait(&bar_full[st], (g / NST) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n");
#pragma unroll
          for (int j = 0; j < OZ_KS / 32; ++j) {
            const uint64_t da =
                oz_desc(oz_smem(osm + st * OZ_STAGE + j * 32 * OZ_TM), OZ_TM * 16, 128);
            const uint64_t db =
                oz_desc(oz_smem(osm + st * OZ_STAGE + OZ_A_ST + j * 32 * OZ_TN), OZ_TN * 16, 128);
            const uint32_t acc = (kb > 0 || j > 0) ? 1u : 0u;
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(dacc),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
          }
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
              "[%0], %1;\n" ::"r"(oz_smem(&bar_free[st])),
              "h"(static_cast<unsigned short>(3)));
        }
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                oz_smem(&tm_full[acc_i])));
      }
    }
  } else {  // epilogue warps 2..9: TMEM lane quarter (warp % 4), column half
    const int q = warp & 3, half = (warp - 2) >> 2;  // lane quarter, column half
    int i = 0;
    for (int T = cluster; T < pair_tiles; T += nclusters, ++i) {
      int x, y, z;
      decode(T, x, y, z);
      const int ci = z / C.nm, t = z - ci * C.nm;
      const int acc_i = i & 1;
      oz_wait(&tm_full[acc_i], (i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const int row = y * OZ_TM + q * 32 + lane;
      const int mod = C.mod[t];
      const uint32_t cdiv = C.cdiv[t];
      int8_t* dst = oz.res + (static_cast<size_t>(ci) * C.nm + t) * lplane +
                    static_cast<size_t>(row) * NP + x * OZ_TN;
#pragma unroll 1
      for (int cb = half * (OZ_TN / 2); cb < (half + 1) * (OZ_TN / 2); cb += 32) {
        uint32_t v[32];
        const uint32_t ta = tmem + (static_cast<uint32_t>(q * 32) << 16) + acc_i * OZ_TN + cb;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
              "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
              "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
              "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n");
        uint32_t packed[8];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int r = oz_mod_acc(v[j], static_cast<uint32_t>(mod), cdiv);
          const uint32_t bb = static_cast<uint32_t>(r) & 0xffu;
          packed[j >> 2] = (j & 3) == 0 ? bb : (packed[j >> 2] | (bb << (8 * (j & 3))));
        }
        uint4* d4 = reinterpret_cast<uint4*>(dst + cb);
        d4[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
        d4[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(oz_smem(&tm_empty[acc_i]))
                     : "memory");
    }
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  // no CTA leaves while its cluster peer may still multicast into it or
  // arrive on its barriers
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(2 * OZ_TN));
}

// Product tile (CRT + unscaling) into shared memory, then the op's epilogue.
// grid (tiles of 64 x 64, nitems), 128 threads, tk::SMEM dynamic.
template <int NM>
__global__ void __launch_bounds__(THREADS, 3) oz_crt_epi(const LaunchArgs la, const OzArgs oz,
                                                      const OzConst C) {
  extern __shared__ __align__(16) double sm[];
  __shared__ Op op;
  __shared__ int sh_b;
  const int tid = threadIdx.x;
  const int ci = blockIdx.y, item = oz.item0 + ci;
  if (tid == 0) {
    int opi, b;
    oz_item(la, item, opi, b);
    sh_b = b;
  }
  {
    int opi, b;
    oz_item(la, item, opi, b);
    for (int i = tid; i < static_cast<int>(sizeof(Op) / 4); i += THREADS)
      reinterpret_cast<int*>(&op)[i] = reinterpret_cast<const int*>(la.ops + opi)[i];
  }
  const int NP = la.NP, M = la.M;
  const int tiles_n = NP / BN;
  const int tm = blockIdx.x / tiles_n, tn = blockIdx.x - tm * tiles_n;
  const int rs = oz_rsrc(la, oz, ci);  // item holding this product's right operand
  // 64 x 64 tile: thread -> columns 4 (tid & 15) .. +4 of rows (tid >> 4) + 8 g,
  // g = 0..7, so a warp's residue loads are two contiguous 64-byte row runs
  const int c4 = (tid & 15) * 4, rbase = tid >> 4;
  const size_t plane = static_cast<size_t>(M) * NP;
  const int8_t* res = oz.res + static_cast<size_t>(ci) * NM * plane +
                      static_cast<size_t>(tm * BM) * NP + tn * BN + c4;
  int sb[4];
  {
    const unsigned long long* mxr = oz.mxR + static_cast<size_t>(rs) * NP + tn * BN + c4;
#pragma unroll
    for (int e = 0; e < 4; ++e) sb[e] = oz_shift(mxr[e], C.P);
  }
  const unsigned long long* mxl = oz.mxL + static_cast<size_t>(ci) * M + tm * BM;
  double* E = sm;
  const double d1s = ldexp(1.0, OZ_LVB), d2s = ldexp(1.0, 2 * OZ_LVB);
  // residue loads run one group ahead of the reconstruction (the kernel is
  // bound by their latency at 12 warps per SM)
  uint32_t w4[NM];
#pragma unroll
  for (int t = 0; t < NM; ++t)
    w4[t] = *reinterpret_cast<const uint32_t*>(res + t * plane + static_cast<size_t>(rbase) * NP);
  for (int g = 0; g < 8; ++g) {
    const int rr = rbase + 8 * g;
    const int sa = oz_shift(mxl[rr], C.P);
    double s[4][OZ_LV];
#pragma unroll
    for (int e = 0; e < 4; ++e)
#pragma unroll
      for (int l = 0; l < OZ_LV; ++l) s[e][l] = 0.0;
    uint32_t wn[NM];
    const int rn = g < 7 ? rr + 8 : rr;
#pragma unroll
    for (int t = 0; t < NM; ++t)
      wn[t] = *reinterpret_cast<const uint32_t*>(res + t * plane + static_cast<size_t>(rn) * NP);
#pragma unroll
    for (int t = 0; t < NM; ++t) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const double rd = static_cast<double>(static_cast<int8_t>((w4[t] >> (8 * e)) & 0xffu));
#pragma unroll
        for (int l = 0; l < OZ_LV; ++l) s[e][l] = fma(rd, C.w[t][l], s[e][l]);
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      // S = s0 2^84 + s1 2^42 + s2 exactly (16 terms below 2^7 2^42: each
      // |s_l| < 2^53); q = round(S / M); s0 - q M0 is exact (|result| <
      // 2^40), the two lower levels may round by an ulp (<= 2^44 absolute,
      // far below the P-bit truncation); only those and the final sum round
      const double approx = fma(s[e][0], d2s, fma(s[e][1], d1s, s[e][2]));
      const double q = rint(approx * C.invM);
      const double e0 = fma(-q, C.M[0], s[e][0]);
      const double e1 = fma(-q, C.M[1], s[e][1]);
      const double e2 = fma(-q, C.M[2], s[e][2]);
      const double v = fma(e0, d2s, fma(e1, d1s, e2));
      E[rr * LDE + c4 + e] = ldexp(v, -(sa + sb[e]));
    }
#pragma unroll
    for (int t = 0; t < NM; ++t) w4[t] = wn[t];
  }
  {
    // a row of L or a column of R with a non-finite entry (max +Inf): the
    // product entries it touches are NaN, as an fp64 GEMM would make them
    // non-finite (rare: the max kernels flag the item, a fix-up pass then)
    const unsigned long long* mxr = oz.mxR + static_cast<size_t>(rs) * NP + tn * BN;
    __syncthreads();
    if (oz.bad[ci] | oz.bad[rs]) {
      for (int p = tid; p < BM * BN; p += THREADS) {
        const int rr = p / BN, cc = p % BN;
        if (mxl[rr] >= OZ_INF_BITS || mxr[cc] >= OZ_INF_BITS)
          E[rr * LDE + cc] = __longlong_as_double(0x7ff8000000000000ll);
      }
    }
  }
  __syncthreads();
  if (tid < BN) {  // the tile's column sums of |C| (real block) for oz_guard
    const int c = tn * BN + tid;
    double sum = 0.0;
    if (c < la.n)
      for (int rr = 0; rr < BM && tm * BM + rr < la.n; ++rr) sum += fabs(E[rr * LDE + tid]);
    oz.csumC[(static_cast<size_t>(ci) * (M / BM) + tm) * NP + c] = sum;
  }
  epilogue_tile<THREADS>(la, op, sh_b, tm, tn, E);
}

// Accuracy guard of one product item (grid (nitems), 256 threads).  The
// integer product is exact; the only error is the rounding of row i of L
// (column j of R) to the integer grid 2^-shift, |dL_ik| <= d_i = 2^(e_i-P-1)
// with max_k |L_ik| in [2^(e_i-1), 2^e_i) (and |dR_kj| <= f_j likewise), so
//   || C~ - L R ||_1 <= max_j [ (sum_i d_i) colsum_j(|R|)
//                               + f_j (sum_ik |L_ik| + K sum_i d_i) ] =: E.
// The fp64 GEMM the reference runs (matcore.py:97) is bounded by
// gamma_n || |L||R| ||_1 >= n u ||L R||_1.  The item is flagged for a DMMA
// rerun unless E <= n u ||C~||_1: the Ozaki bound then never exceeds the
// fp64 one.  Row / column maxima make the rounding relative to whole rows
// and columns, not entries; badly scaled operands (graded rows, Pascal-like
// matrices) fail the test and take the DMMA path.  Items with a non-finite
// entry keep their NaN-propagating CRT result.
__global__ void __launch_bounds__(256) oz_guard(const LaunchArgs la, const OzArgs oz,
                                                const OzConst C) {
  const int ci = blockIdx.x, tid = threadIdx.x;
  const int NP = la.NP, M = la.M, n = la.n;
  const int rs = oz_rsrc(la, oz, ci);
  __shared__ double red[2][8];
  double sd = 0.0, sl = 0.0;
  for (int r = tid; r < M && r < n; r += 256) {
    const unsigned long long mx = oz.mxL[static_cast<size_t>(ci) * M + r];
    if (mx != 0ull && mx < OZ_INF_BITS) {
      int e = 0;
      frexp(__longlong_as_double(static_cast<long long>(mx)), &e);
      sd += ldexp(1.0, e - C.P - 1);
    }
    sl += oz.rsumL[static_cast<size_t>(ci) * M + r];
  }
  for (int o = 16; o; o >>= 1) {
    sd += __shfl_xor_sync(0xffffffffu, sd, o);
    sl += __shfl_xor_sync(0xffffffffu, sl, o);
  }
  if ((tid & 31) == 0) { red[0][tid >> 5] = sd; red[1][tid >> 5] = sl; }
  __syncthreads();
  sd = sl = 0.0;
  for (int w = 0; w < 8; ++w) { sd += red[0][w]; sl += red[1][w]; }
  __syncthreads();
  const double lterm = sl + static_cast<double>(NP) * sd;
  double emax = 0.0, cmax = 0.0;
  for (int j = tid; j < NP && j < n; j += 256) {
    double cs = 0.0;
    for (int ch = 0; ch < NP / 64; ++ch) cs += oz.csumR[(static_cast<size_t>(rs) * (NP / 64) + ch) * NP + j];
    const unsigned long long mx = oz.mxR[static_cast<size_t>(rs) * NP + j];
    double fj = 0.0;
    if (mx != 0ull && mx < OZ_INF_BITS) {
      int e = 0;
      frexp(__longlong_as_double(static_cast<long long>(mx)), &e);
      fj = ldexp(1.0, e - C.P - 1);
    }
    emax = fmax(emax, fma(sd, cs, fj * lterm));
    double cc = 0.0;
    for (int tm = 0; tm < M / BM; ++tm) cc += oz.csumC[(static_cast<size_t>(ci) * (M / BM) + tm) * NP + j];
    cmax = fmax(cmax, cc);
  }
  for (int o = 16; o; o >>= 1) {
    emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
    cmax = fmax(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
  }
  if ((tid & 31) == 0) { red[0][tid >> 5] = emax; red[1][tid >> 5] = cmax; }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < 8; ++w) { emax = fmax(emax, red[0][w]); cmax = fmax(cmax, red[1][w]); }
    emax = fmax(emax, red[0][0]);
    cmax = fmax(cmax, red[1][0]);
    const bool bad = (oz.bad[ci] | oz.bad[rs]) != 0u;
    const double gamma = static_cast<double>(n) * 0x1p-53;
    // !(E <= gamma C) also flags a NaN bound (never expected: bad items skip)
    oz.flag[ci] = (!bad && !(emax <= gamma * cmax)) ? 1u : 0u;
#ifdef CSM_OZ_GUARD_DEBUG
    printf("oz_guard item %d rs %d: E %.3e ||C|| %.3e gamma %.3e sd %.3e sl %.3e bad %d flag %u\n",
           oz.item0 + ci, rs, emax, cmax, gamma, sd, sl, (int)bad, oz.flag[ci]);
#endif
  }
}

