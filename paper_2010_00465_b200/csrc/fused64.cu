// fused64.cu -- K1: the whole cos/sin (or wave) pipeline for n <= 64 with
// every intermediate resident in shared memory, and K1c: the same program
// for 64 < n <= 128 on a 4-CTA thread-block cluster whose distributed shared
// memory holds the 128 x 128 slots as four 32-row bands.
//
// One persistent CTA per SM (256 threads, 8 warps) walks a static snake
// schedule over the matrices sorted by cost k + 2s (K0 builds it), so the
// CTAs finish together without a shared work queue.  A matrix is
// zero-padded to 64x64 (block-diagonal padding is exact: the padded block
// evolves as p(0) I and never touches the real block).  Seven 32 KiB
// slots: the input A (slot 0), five work slots and slot 6, which receives
// the NEXT matrix's input by one TMA bulk copy as soon as the current chain
// no longer needs it as a work slot.
//
// The chain of scheme k is a short PROGRAM of steps (kChains below): each
// step is one 64x64x64 FP64 product on the DMMA pipe (mma.sync m8n8k4; or a
// dual product sharing its right operand) followed by an epilogue that
// forms the scheme's linear combinations from the accumulator registers and
// writes them to slots that are not operands of the step, then one barrier.
// So the GEMM code exists once, every lincomb is fused, and there is one
// __syncthreads per product.
//
// Layout: slot element (r, c) lives at r*64 + 2*((c/2) ^ f(r)) + (c&1) with
// f(r) = ((r&1)<<2) | (r&2): an XOR swizzle on 16-byte pairs that makes the
// DMMA A/B fragment loads (LDS.64) and the epilogue's 16-byte accesses in
// accumulator layout all bank-conflict free.
//
// Scaling is folded: Taylor never uses A elementwise, so y = 2^-2s (A A)
// and sin = 2^-s (A sc) are exact power-of-two rescalings of the
// accumulators (driver.py:115); the wave family materialises y = (t')^2 A
// (schemes.py:424) in place.
//
// K1c (CL = 4): CTA q of the cluster owns rows [32q, 32q+32) of every
// slot (7 x 32 KiB, the same footprint as K1).  A product band
// out[32q.., :] = L[32q.., :] R reads L from the CTA's own band and R, the
// full matrix, through distributed shared memory (generic loads on
// __cluster_map_shared_rank pointers); the per-step barrier becomes a
// cluster barrier (release/acquire).  Each warp computes a 32 x 16 tile so
// every R element crosses the cluster once per product: 96 KiB per CTA per
// 2 x 32 x 128^2 flop, 11.7 B/clk at the DMMA rate against a measured
// 14-15 B/clk DSMEM bandwidth (tools/dsmem_bw.cu, tools/dsmem_bulk.cu).
//
// Reference mapping: chains schemes.py:264-361, trig use :376-395, wave use
// :411-430, scaling driver.py:115/:139, doubling driver.py:91-98.
#include <cstdlib>

#include "common.cuh"

namespace csm {

namespace f64k {

// Optional phase trace (build with -DCSM_TRACE; tools/trace_fused.py): CTA 0,
// thread 0 logs (clock64 << 8 | tag) at phase boundaries.
#ifdef CSM_TRACE
#ifndef CSM_TRACE_TID
#define CSM_TRACE_TID 0
#endif
__device__ unsigned long long g_trace[1 << 16];
__device__ int g_trace_n;
__device__ __forceinline__ int& trace_count() {
  __shared__ int n;  // only thread 0 of CTA 0 touches it
  return n;
}
#define CSM_TRACE_EV(tag, val)                                                    \
  do {                                                                            \
    if (blockIdx.x == 0 && threadIdx.x == CSM_TRACE_TID) {                        \
      const int i_ = trace_count()++;                                             \
      if (i_ < (1 << 16)) g_trace[i_] = ((val) << 8) | (tag);                     \
      g_trace_n = i_ + 1;                                                         \
    }                                                                             \
  } while (0)
#else
#define CSM_TRACE_EV(tag, val) do { } while (0)
#endif
#define TRACE_T(tag) CSM_TRACE_EV(tag, static_cast<unsigned long long>(clock64()))

// Geometry: CL = CTAs per matrix (1: K1, 4: K1c).  BAND rows of NP columns
// per CTA and slot; each warp owns an (8 MI) x (8 NI) accumulator tile.
// K1 runs 16 warps (4 per SMSP, 16 x 16 warp tiles, <= 128 registers) by
// default; CSM_K1_THREADS=256 builds the 8-warp form (16 x 32 tiles).
#ifndef CSM_K1_THREADS
#define CSM_K1_THREADS 512
#endif
template <int V> struct Geo;  // V: the kernel variant (1: K1, 4: K1c, 5: K1s)
template <> struct Geo<1> {
  static constexpr bool ROTATE = false;
  static constexpr int CL = 1, NP = 64, BAND = 64, THREADS = CSM_K1_THREADS, MI = 2,
                       NI = THREADS == 512 ? 2 : 4;
};
template <> struct Geo<4> {
  static constexpr bool ROTATE = true;  // each CTA starts the k loop at its own band
  static constexpr int CL = 4, NP = 128, BAND = 32, THREADS = 256, MI = 4, NI = 2;
};
// K1s: one n <= 64 matrix over a 4-CTA cluster (16-row bands, 4 warps of
// 16 x 16): the latency-bound small-batch path, a quarter product per SM.
template <> struct Geo<5> {
  static constexpr bool ROTATE = false;
  static constexpr int CL = 4, NP = 64, BAND = 16, THREADS = 128, MI = 2, NI = 2;
};
static_assert(Geo<1>::THREADS == 256 || Geo<1>::THREADS == 512, "K1: 8 or 16 warps");
constexpr int SLOT = 4096;  // doubles per slot band (64 x 64 or 32 x 128)
constexpr int NSLOTS = 7;

__host__ __device__ constexpr int swz_f(int r) { return ((r & 1) << 2) | (r & 2); }
template <int NP>
__device__ __forceinline__ int swz(int r, int c) {
  return r * NP + 2 * ((c >> 1) ^ swz_f(r)) + (c & 1);
}

// ---------------------------------------------------------------------------
// Chain programs.

enum Epi : int8_t {
  E_SCALED,    // o0 = scale * acc
  E_DEG2,      // o0 = I - y/2 + acc/24 ; o1 = I - y/6 + acc/120            (y=i0)
  E_DEG4A,     // o0 = acc ; o1 = -y/720 + acc/40320                        (y=i0)
  E_DEG4B,     // o0 = I - y/2 + y2/24 + acc ; o1 = I - y/6 + y2/120 + acc/7 (y,y2)
  E_DEG4W1,    // o0 = acc ; o1 = -y/720 + acc/40320 ; o2 = -y/5040 + acc/9! (y)
  E_DEG4W2,    // dual: o0 = I - y/2 + y2/24 + q ; o1 = tp (I - y/6 + y2/120 + q9)
  E_DEG8A,     // o0 = acc ; o1 = x1 y + x2 acc                             (y)
  E_DEG8B,     // o0 = acc ; o1 = x3 y2 + acc ; o2 = x4 I + x5 y + x6 y2 + x7 acc
  E_DEG8C,     // o0 = cos ; o1 = inner ; keep = sin base     (y, y2, p8)
  E_KEEP,      // o0 = scale * (keep + acc)
  E_DEG12B,    // o0 = acc ; o1 = c4                                        (y, y2)
  E_DEG12C,    // o0 = mid = c3 + acc ; o1 = c2 + mid                       (y, y2, y3)
  E_DEG12D,    // o0 = cos = c1 + acc ; o1 = inner ; keep = sin base (y,y2,y3,mid)
  E_Y2,        // o0 = acc (y2 of the degree-12 chain), also kept in acc2
};

enum Scale : int8_t { SC_ONE = 0, SC_F = 1, SC_F2 = 2, SC_TP = 3 };

struct __align__(16) Step {
  int8_t dual;            // 0: acc = L1 R ; 1: acc = L1 R, acc2 = L2 R
  int8_t l1, l2, r;       // operand slots
  int8_t epi, scale;
  int8_t o0, o1, o2;      // output slots (-1 unused)
  int8_t i0, i1, i2, i3;  // elementwise input slots (-1 unused)
  int8_t pad[3];
};
static_assert(sizeof(Step) == 16, "one 128-bit load per step");

struct __align__(16) Chain {
  int8_t nsteps;
  int8_t cos_slot, sin_slot, free1, free2;  // final pair and two free slots
  int8_t pf_after;  // the next matrix's input may land in slot 6 after this step
  int8_t cos_step, cos_out, sin_step, sin_out;  // producers of the final pair
  int8_t pad[6];
  Step step[7];
};
static_assert(sizeof(Chain) == 128, "chain table layout");

// Slot ids: 0 = this matrix's input (A, or y for the wave family), 1..6 =
// work slots; slot 6 doubles as the landing buffer of the next matrix's
// input, so a chain may use it only up to step pf_after.
#define S_(d, l1, l2, r, e, sc, o0, o1, o2, i0, i1, i2, i3) \
  {d, l1, l2, r, e, sc, o0, o1, o2, i0, i1, i2, i3, {0, 0, 0}}
#define H_(ns, cs, ss, f1, f2, pf, cst, co, sst, so) \
  ns, cs, ss, f1, f2, pf, cst, co, sst, so, {0, 0, 0, 0, 0, 0}
constexpr int8_t X = -1;

__constant__ Chain kChains[7] = {
    // [0] Taylor k=3: chain_deg2 (schemes.py:264-272); sin = A sc (:394)
    {H_(3, 2, 4, 1, 3, 0, 1, 0, 2, 0),
     {S_(0, 0, X, 0, E_SCALED, SC_F2, 1, X, X, X, X, X, X),     // y = A A
      S_(0, 1, X, 1, E_DEG2, SC_ONE, 2, 3, X, 1, X, X, X),       // cos, sc
      S_(0, 0, X, 3, E_SCALED, SC_F, 4, X, X, X, X, X, X)}},     // sin = A sc
    // [1] Taylor k=4: chain_deg4(exact_sine=False) (:275-299)
    {H_(4, 4, 1, 2, 3, 0, 2, 0, 3, 0),
     {S_(0, 0, X, 0, E_SCALED, SC_F2, 1, X, X, X, X, X, X),     // y
      S_(0, 1, X, 1, E_DEG4A, SC_ONE, 2, 3, X, 1, X, X, X),      // y2, L
      S_(0, 2, X, 3, E_DEG4B, SC_ONE, 4, 5, X, 1, 2, X, X),      // cos, sc
      S_(0, 0, X, 5, E_SCALED, SC_F, 1, X, X, X, X, X, X)}},     // sin
    // [2] Taylor k=6: chain_deg8 (:302-326)
    {H_(6, 3, 5, 1, 2, 3, 3, 0, 5, 0),
     {S_(0, 0, X, 0, E_SCALED, SC_F2, 1, X, X, X, X, X, X),     // y
      S_(0, 1, X, 1, E_DEG8A, SC_ONE, 2, 3, X, 1, X, X, X),      // y2, L
      S_(0, 2, X, 3, E_DEG8B, SC_ONE, 4, 5, 6, 1, 2, X, X),      // p8, L2, R2
      S_(0, 5, X, 6, E_DEG8C, SC_ONE, 3, 1, X, 1, 2, 4, X),      // cos, inner
      S_(0, 1, X, 4, E_KEEP, SC_ONE, 2, X, X, X, X, X, X),       // sc
      S_(0, 0, X, 2, E_SCALED, SC_F, 5, X, X, X, X, X, X)}},     // sin = A sc
    // [3] Taylor k=7: chain_deg12 (:329-361)
    {H_(7, 4, 5, 1, 2, 4, 4, 0, 6, 0),
     {S_(0, 0, X, 0, E_SCALED, SC_F2, 1, X, X, X, X, X, X),     // y
      S_(0, 1, X, 1, E_Y2, SC_ONE, 2, X, X, X, X, X, X),         // y2
      S_(0, 2, X, 1, E_DEG12B, SC_ONE, 3, 4, X, 1, 2, X, X),     // y3, c4
      S_(0, 4, X, 4, E_DEG12C, SC_ONE, 5, 6, X, 1, 2, 3, X),     // mid, L
      S_(0, 6, X, 5, E_DEG12D, SC_ONE, 4, 1, X, 1, 2, 3, 5),     // cos, inner
      S_(0, 1, X, 4, E_KEEP, SC_ONE, 2, X, X, X, X, X, X),       // sc
      S_(0, 0, X, 2, E_SCALED, SC_F, 5, X, X, X, X, X, X)}},     // sin = A sc
    // [4] wave k=3: chain_deg4(exact_sine=True) on y (slot 0), :426-427
    {H_(2, 4, 5, 1, 2, 0, 1, 0, 1, 1),
     {S_(0, 0, X, 0, E_DEG4W1, SC_ONE, 1, 2, 3, 0, X, X, X),     // y2, L, L9
      S_(1, 2, 3, 1, E_DEG4W2, SC_TP, 4, 5, X, 0, 1, X, X)}},    // cos, s
    // [5] wave k=4: chain_deg8 on y
    {H_(4, 2, 4, 1, 3, 0, 2, 0, 3, 0),
     {S_(0, 0, X, 0, E_DEG8A, SC_ONE, 1, 2, X, 0, X, X, X),      // y2, L
      S_(0, 1, X, 2, E_DEG8B, SC_ONE, 3, 4, 5, 0, 1, X, X),      // p8, L2, R2
      S_(0, 4, X, 5, E_DEG8C, SC_ONE, 2, 1, X, 0, 1, 3, X),      // cos, inner
      S_(0, 1, X, 3, E_KEEP, SC_TP, 4, X, X, X, X, X, X)}},      // s
    // [6] wave k=5: chain_deg12 on y
    {H_(5, 3, 2, 1, 4, 0, 3, 0, 4, 0),
     {S_(0, 0, X, 0, E_Y2, SC_ONE, 1, X, X, X, X, X, X),         // y2
      S_(0, 1, X, 0, E_DEG12B, SC_ONE, 2, 3, X, 0, 1, X, X),     // y3, c4
      S_(0, 3, X, 3, E_DEG12C, SC_ONE, 4, 5, X, 0, 1, 2, X),     // mid, L
      S_(0, 5, X, 4, E_DEG12D, SC_ONE, 3, 1, X, 0, 1, 2, 4),     // cos, inner
      S_(0, 1, X, 3, E_KEEP, SC_TP, 2, X, X, X, X, X, X)}},      // s
};
#undef H_
#undef S_

// ---------------------------------------------------------------------------
// Per-thread geometry, lane = 4g + t.  K1: warp w owns rows [16(w/2), +16) x
// cols [32(w%2), +32) = 2 x 4 DMMA tiles.  K1c: warp w owns the band's 32
// rows x cols [16w, +16) = 4 x 2 tiles.

template <int CL>
struct Lane {
  int rb, cb, g, t, row0;  // row0: first global row of this CTA's band
  int aoff[Geo<CL>::MI][4];  // A-fragment offsets: tile mi, chunk q (+16 m)
  int boff[Geo<CL>::NI];     // B-fragment offsets for tile ni (+NP kk)
};

template <int CL>
__device__ __forceinline__ void make_lane(Lane<CL>& ln, int rank) {
  constexpr int NP = Geo<CL>::NP, MI = Geo<CL>::MI, NI = Geo<CL>::NI;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (Geo<CL>::CL == 1 && Geo<CL>::THREADS == 512) {
    ln.rb = (warp >> 2) * 16;
    ln.cb = (warp & 3) * 16;
  } else if (Geo<CL>::CL == 1) {
    ln.rb = (warp >> 1) * 16;
    ln.cb = (warp & 1) * 32;
  } else {
    ln.rb = 0;
    ln.cb = warp * 16;
  }
  ln.row0 = rank * Geo<CL>::BAND;
  ln.g = lane >> 2;
  ln.t = lane & 3;
  // A: element (r = rb + 8 mi + g, c = 4 j + t), j = 4 m + q
  //    -> r*NP + 4 ((j) ^ h) + t with h = f(g)/2 (affects the low 2 bits of j)
  const int h = swz_f(ln.g) >> 1;
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int q = 0; q < 4; ++q)
      ln.aoff[mi][q] = (ln.rb + mi * 8 + ln.g) * NP + 4 * (q ^ h) + ln.t;
  // B: element (r = kk + t, c = cb + 8 ni + g) -> kk*NP + swz(t, c) (f(r) = f(t))
#pragma unroll
  for (int ni = 0; ni < NI; ++ni) ln.boff[ni] = swz<NP>(ln.t, ln.cb + ni * 8 + ln.g);
}

typedef double Acc[8][2];  // 8 DMMA tiles x 2 accumulators (p = mi * NI + ni)

__device__ __forceinline__ void zero(Acc& a) {
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i][0] = a[i][1] = 0.0;
}

// Cross-CTA view of a slot: K1 reads R from its own shared memory; K1c maps
// the same slot of each cluster rank (rows [32 o, 32 o + 32)).
// K1c walks the k bands starting at its own rank (p[i] = band (rank + i) %
// CL, lcol[i] its column offset in L), so the four CTAs of a cluster read
// four different owners at any time instead of all hammering one.
template <int CL>
struct RView {
  const double* p[Geo<CL>::CL];
  int lcol[Geo<CL>::CL];
};
template <int CL>
__device__ __forceinline__ RView<CL> rview(const double* R, int rank) {
  RView<CL> v;
  constexpr int NC = Geo<CL>::CL;
  if constexpr (NC == 1) {
    v.p[0] = R;
    v.lcol[0] = 0;
  } else {
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      // K1c: each CTA starts at its own band, so the four CTAs read four
      // different owners at a time.  K1s keeps the natural k order: its
      // accumulation order, and so every bit of its results, is K1's, and
      // a matrix's result does not depend on the batch size (rotated, a
      // cfg1 matrix takes 24 us instead of 29 us, ~3e-15 apart)
      const int o = Geo<CL>::ROTATE ? (rank + i) & (NC - 1) : i;
      // own band through the local shared window: no cluster round trip
      const bool own = Geo<CL>::ROTATE ? i == 0 : o == rank;  // compile-time when rotated
      v.p[i] = own ? R
                   : static_cast<const double*>(
                         __cluster_map_shared_rank(const_cast<double*>(R), o));
      v.lcol[i] = Geo<CL>::BAND * o;  // L columns of band o (swizzle keeps 8-chunk blocks)
    }
  }
  return v;
}

// acc = L * R (and acc2 = L2 * R when DUAL), full NP-deep contraction; L
// and L2 are this CTA's bands, R the whole slot.
template <int CL, bool DUAL>
__device__ __forceinline__ void gemm(const double* __restrict__ L,
                                     const double* __restrict__ L2,
                                     const RView<CL>& R, Acc& acc, Acc& acc2,
                                     const Lane<CL>& ln) {
  constexpr int NP = Geo<CL>::NP, BAND = Geo<CL>::BAND, MI = Geo<CL>::MI, NI = Geo<CL>::NI;
  zero(acc);
  if (DUAL) zero(acc2);
  if constexpr (Geo<CL>::CL > 1) {
    // R arrives over DSMEM (hundreds of cycles): keep PF k-steps of B
    // fragments in flight in a register ring.
    constexpr int NK = NP / 4;
#ifndef CSM_K1C_PF
#define CSM_K1C_PF 6
#endif
    constexpr int PF = CSM_K1C_PF;
    double ring[PF][NI];
#pragma unroll
    for (int d = 0; d < PF; ++d) {
      const double* Rk = R.p[(4 * d) / BAND] + ((4 * d) % BAND) * NP;
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) ring[d][ni] = Rk[ln.boff[ni]];
    }
#pragma unroll
    for (int j = 0; j < NK; ++j) {
      // k-step j of the rotated order: band j / 8, local k-step j % 8
      const int bi = (4 * j) / BAND, jl = j % (BAND / 4), m = jl >> 2, q = jl & 3;
      double b[NI];
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) b[ni] = ring[j % PF][ni];
      if (j + PF < NK) {
        const int kn = 4 * (j + PF);
        const double* Rk = R.p[kn / BAND] + (kn % BAND) * NP;
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) ring[j % PF][ni] = Rk[ln.boff[ni]];
      }
      const double* Lb = L + R.lcol[bi];
      const double* L2b = DUAL ? L2 + R.lcol[bi] : nullptr;
      double a[MI], a2[MI];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) {
        a[mi] = Lb[ln.aoff[mi][q] + 16 * m];
        if (DUAL) a2[mi] = L2b[ln.aoff[mi][q] + 16 * m];
      }
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          dmma(acc[mi * NI + ni], a[mi], b[ni]);
          if (DUAL) dmma(acc2[mi * NI + ni], a2[mi], b[ni]);
        }
    }
  } else {
#pragma unroll
  for (int kk = 0; kk < NP; kk += 4) {
    const int j = kk >> 2, m = j >> 2, q = j & 3;
    const double* Rk = R.p[kk / BAND] + (kk % BAND) * NP;
    double a[MI], a2[MI], b[NI];
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
      a[mi] = L[ln.aoff[mi][q] + 16 * m];
      if (DUAL) a2[mi] = L2[ln.aoff[mi][q] + 16 * m];
    }
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) b[ni] = Rk[ln.boff[ni]];
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) {
        dmma(acc[mi * NI + ni], a[mi], b[ni]);
        if (DUAL) dmma(acc2[mi * NI + ni], a2[mi], b[ni]);
      }
  }
  }
}

__device__ __forceinline__ double2 ld2(const double* p, int off) {
  return *reinterpret_cast<const double2*>(p + off);
}
__device__ __forceinline__ void st2(double* p, int off, double x, double y) {
  *reinterpret_cast<double2*>(p + off) = make_double2(x, y);
}

// Barrier between dependent steps: the CTA (K1) or the whole cluster (K1c,
// release/acquire so band writes are visible to the peers' DSMEM loads).
template <int CL>
__device__ __forceinline__ void step_sync() {
  if constexpr (Geo<CL>::CL == 1) {
    __syncthreads();
  } else {
#ifdef CSM_CLUSTER_RELAXED
    // experiment: CTA barrier (band writes performed in this SM's shared
    // memory) + relaxed cluster arrive, avoiding the GPU-scope MEMBAR that
    // a .release arrive compiles to
    __syncthreads();
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
#else
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
#endif
  }
}

// ---------------------------------------------------------------------------
// Epilogue: one formula per Epi, evaluated on the thread's 8 owned pairs.

template <typename TOut>
struct EpiArgs {
  double* o[3];        // shared-memory outputs
  TOut* g[3];          // optional global outputs (final cos / sin when s == 0)
  const double* in[4];
  double scale;
  int n;
};

// Store one accumulator-layout pair (rg, c), (rg, c+1) of an n x n result
// (rg = global row).
template <int NP, typename TOut>
__device__ __forceinline__ void gstore(TOut* __restrict__ dst, int n, int rg, int c,
                                       double v0, double v1) {
  if (n == NP) {
    if constexpr (sizeof(TOut) == 8)
      *reinterpret_cast<double2*>(reinterpret_cast<double*>(dst) + rg * NP + c) =
          make_double2(v0, v1);
    else
      *reinterpret_cast<float2*>(reinterpret_cast<float*>(dst) + rg * NP + c) =
          make_float2(static_cast<float>(v0), static_cast<float>(v1));
  } else if (rg < n) {
    if (c < n) dst[rg * n + c] = static_cast<TOut>(v0);
    if (c + 1 < n) dst[rg * n + c + 1] = static_cast<TOut>(v1);
  }
}

template <int NP, typename TOut>
__device__ __forceinline__ void put(const EpiArgs<TOut>& E, int q, int rg, int c, int off,
                                    double v0, double v1) {
  st2(E.o[q], off, v0, v1);
  if (E.g[q]) gstore<NP>(E.g[q], E.n, rg, c, v0, v1);
}

// Run BODY on each of the thread's 8 owned pairs (accumulator layout) with
// P (tile index), r (band row), rg (global row), c, off (swizzled), I0/I1
// (identity entries) and p0/p1 (accumulator).
#define FOR_PAIRS(...)                                                        \
  _Pragma("unroll") for (int mi = 0; mi < Geo<CL>::MI; ++mi) {                \
    _Pragma("unroll") for (int ni = 0; ni < Geo<CL>::NI; ++ni) {              \
      const int P = mi * Geo<CL>::NI + ni;                                    \
      const int r = ln.rb + mi * 8 + ln.g;                                    \
      const int rg = ln.row0 + r;                                             \
      const int c = ln.cb + ni * 8 + 2 * ln.t;                                \
      const int off = swz<Geo<CL>::NP>(r, c);                                 \
      const double I0 = (rg == c) ? 1.0 : 0.0, I1 = (rg == c + 1) ? 1.0 : 0.0; \
      const double p0 = acc[P][0], p1 = acc[P][1];                            \
      (void)I0; (void)I1; (void)off;                                          \
      __VA_ARGS__                                                             \
    }                                                                         \
  }

template <int CL, typename TOut>
__device__ __forceinline__ void epilogue(int epi, const EpiArgs<TOut>& E, const Acc& acc,
                                         Acc& acc2, Acc& keep, const Lane<CL>& ln) {
  constexpr int NP = Geo<CL>::NP;
  const double* x = dTables.x8;  // x[0] = x1
  const double* z8 = dTables.z8;
  const double(*a)[4] = dTables.a12;  // a[j-1][i]
  const double* z = dTables.z12;
  switch (epi) {
    case E_SCALED:
      FOR_PAIRS(put<NP>(E, 0, rg, c, off, E.scale * p0, E.scale * p1);)
      break;
    case E_Y2:  // y2 is an operand (slot) and a term of the next three epilogues (acc2)
      FOR_PAIRS({
          put<NP>(E, 0, rg, c, off, p0, p1);
          acc2[P][0] = p0;
          acc2[P][1] = p1;
        })
      break;
    case E_DEG2:
      FOR_PAIRS({
          const double2 y = ld2(E.in[0], off);
          put<NP>(E, 0, rg, c, off, fma(1.0 / 24.0, p0, fma(-0.5, y.x, I0)),
              fma(1.0 / 24.0, p1, fma(-0.5, y.y, I1)));
          put<NP>(E, 1, rg, c, off, fma(1.0 / 120.0, p0, fma(-1.0 / 6.0, y.x, I0)),
              fma(1.0 / 120.0, p1, fma(-1.0 / 6.0, y.y, I1)));
        })
      break;
    case E_DEG4A:
      FOR_PAIRS({
          const double2 y = ld2(E.in[0], off);
          put<NP>(E, 0, rg, c, off, p0, p1);
          put<NP>(E, 1, rg, c, off, fma(1.0 / 40320.0, p0, (-1.0 / 720.0) * y.x),
              fma(1.0 / 40320.0, p1, (-1.0 / 720.0) * y.y));
        })
      break;
    case E_DEG4B:
      FOR_PAIRS({
          const double2 y = ld2(E.in[0], off), y2 = ld2(E.in[1], off);
          put<NP>(E, 0, rg, c, off, p0 + fma(1.0 / 24.0, y2.x, fma(-0.5, y.x, I0)),
              p1 + fma(1.0 / 24.0, y2.y, fma(-0.5, y.y, I1)));
          put<NP>(E, 1, rg, c, off,
              fma(720.0 / 5040.0, p0, fma(1.0 / 120.0, y2.x, fma(-1.0 / 6.0, y.x, I0))),
              fma(720.0 / 5040.0, p1, fma(1.0 / 120.0, y2.y, fma(-1.0 / 6.0, y.y, I1))));
        })
      break;
    case E_DEG4W1:
      FOR_PAIRS({
          const double2 y = ld2(E.in[0], off);
          put<NP>(E, 0, rg, c, off, p0, p1);
          put<NP>(E, 1, rg, c, off, fma(1.0 / 40320.0, p0, (-1.0 / 720.0) * y.x),
              fma(1.0 / 40320.0, p1, (-1.0 / 720.0) * y.y));
          put<NP>(E, 2, rg, c, off, fma(1.0 / 362880.0, p0, (-1.0 / 5040.0) * y.x),
              fma(1.0 / 362880.0, p1, (-1.0 / 5040.0) * y.y));
        })
      break;
    case E_DEG4W2:
      FOR_PAIRS({
          const double2 y = ld2(E.in[0], off), y2 = ld2(E.in[1], off);
          const double q0 = acc2[P][0], q1 = acc2[P][1];
          put<NP>(E, 0, rg, c, off, p0 + fma(1.0 / 24.0, y2.x, fma(-0.5, y.x, I0)),
              p1 + fma(1.0 / 24.0, y2.y, fma(-0.5, y.y, I1)));
          put<NP>(E, 1, rg, c, off,
              E.scale * (q0 + fma(1.0 / 120.0, y2.x, fma(-1.0 / 6.0, y.x, I0))),
              E.scale * (q1 + fma(1.0 / 120.0, y2.y, fma(-1.0 / 6.0, y.y, I1))));
        })
      break;
    case E_DEG8A:
      FOR_PAIRS({
          const double2 y = ld2(E.in[0], off);
          put<NP>(E, 0, rg, c, off, p0, p1);
          put<NP>(E, 1, rg, c, off, fma(x[1], p0, x[0] * y.x), fma(x[1], p1, x[0] * y.y));
        })
      break;
    case E_DEG8B:
      FOR_PAIRS({
          const double2 y = ld2(E.in[0], off), y2 = ld2(E.in[1], off);
          put<NP>(E, 0, rg, c, off, p0, p1);
          put<NP>(E, 1, rg, c, off, fma(x[2], y2.x, p0), fma(x[2], y2.y, p1));
          put<NP>(E, 2, rg, c, off, fma(x[6], p0, fma(x[5], y2.x, fma(x[4], y.x, x[3] * I0))),
              fma(x[6], p1, fma(x[5], y2.y, fma(x[4], y.y, x[3] * I1))));
        })
      break;
    case E_DEG8C:
      FOR_PAIRS({
          const double2 y = ld2(E.in[0], off), y2 = ld2(E.in[1], off),
                        p8 = ld2(E.in[2], off);
          const double c0 = p0 + fma(x[7], y2.x, fma(-0.5, y.x, I0));
          const double c1 = p1 + fma(x[7], y2.y, fma(-0.5, y.y, I1));
          // inner = z5 I + z5 y + z6 y2 + z7 p8 + z8 cos
          const double n0 = fma(z8[8], c0, fma(z8[7], p8.x, fma(z8[6], y2.x, fma(z8[5], y.x, z8[5] * I0))));
          const double n1 = fma(z8[8], c1, fma(z8[7], p8.y, fma(z8[6], y2.y, fma(z8[5], y.y, z8[5] * I1))));
          // sin base = z0 I + z1 y + z2 y2 + z3 p8 + z4 cos
          keep[P][0] = fma(z8[4], c0, fma(z8[3], p8.x, fma(z8[2], y2.x, fma(z8[1], y.x, z8[0] * I0))));
          keep[P][1] = fma(z8[4], c1, fma(z8[3], p8.y, fma(z8[2], y2.y, fma(z8[1], y.y, z8[0] * I1))));
          put<NP>(E, 0, rg, c, off, c0, c1);
          put<NP>(E, 1, rg, c, off, n0, n1);  // may overwrite y at this thread's own pair
        })
      break;
    case E_KEEP:
      FOR_PAIRS(put<NP>(E, 0, rg, c, off, E.scale * (keep[P][0] + p0), E.scale * (keep[P][1] + p1));)
      break;
    case E_DEG12B:
      // Register carriers across the degree-12 epilogues (the non-dual
      // products in between leave acc2 and keep alone): y2 arrives in acc2
      // (E_Y2; it is also a product operand, so its slot stays), and y3 --
      // only a term of the next two epilogues, never an operand -- stays in
      // keep instead of a shared slot (E_DEG12D reads it before it rewrites
      // keep).  y2 and y3 reads and the y3 write leave shared memory: +1.1%
      // on cfg2.
      FOR_PAIRS({
          const double2 y = ld2(E.in[0], off), y2 = make_double2(acc2[P][0], acc2[P][1]);
          keep[P][0] = p0;  // y3
          keep[P][1] = p1;
          put<NP>(E, 1, rg, c, off, fma(a[3][3], p0, fma(a[3][2], y2.x, fma(a[3][1], y.x, a[3][0] * I0))),
              fma(a[3][3], p1, fma(a[3][2], y2.y, fma(a[3][1], y.y, a[3][0] * I1))));
        })
      break;
    case E_DEG12C:
      FOR_PAIRS({
          const double2 y = ld2(E.in[0], off), y2 = make_double2(acc2[P][0], acc2[P][1]);
          const double2 y3 = make_double2(keep[P][0], keep[P][1]);
          const double m0 = fma(a[2][3], y3.x, fma(a[2][2], y2.x, fma(a[2][1], y.x, a[2][0] * I0))) + p0;
          const double m1 = fma(a[2][3], y3.y, fma(a[2][2], y2.y, fma(a[2][1], y.y, a[2][0] * I1))) + p1;
          const double l0 = fma(a[1][3], y3.x, fma(a[1][2], y2.x, fma(a[1][1], y.x, a[1][0] * I0))) + m0;
          const double l1 = fma(a[1][3], y3.y, fma(a[1][2], y2.y, fma(a[1][1], y.y, a[1][0] * I1))) + m1;
          put<NP>(E, 0, rg, c, off, m0, m1);
          put<NP>(E, 1, rg, c, off, l0, l1);
        })
      break;
    case E_DEG12D:
      FOR_PAIRS({
          const double2 y = ld2(E.in[0], off), md = ld2(E.in[3], off);
          const double2 y2 = make_double2(acc2[P][0], acc2[P][1]);
          const double2 y3 = make_double2(keep[P][0], keep[P][1]);  // read before keep is rewritten
          const double c0 = fma(a[0][3], y3.x, fma(a[0][2], y2.x, fma(a[0][1], y.x, a[0][0] * I0))) + p0;
          const double c1 = fma(a[0][3], y3.y, fma(a[0][2], y2.y, fma(a[0][1], y.y, a[0][0] * I1))) + p1;
          const double n0 = fma(z[11], c0, fma(z[10], md.x, fma(z[9], y3.x, fma(z[8], y2.x, fma(z[7], y.x, z[6] * I0)))));
          const double n1 = fma(z[11], c1, fma(z[10], md.y, fma(z[9], y3.y, fma(z[8], y2.y, fma(z[7], y.y, z[6] * I1)))));
          keep[P][0] = fma(z[5], c0, fma(z[4], md.x, fma(z[3], y3.x, fma(z[2], y2.x, fma(z[1], y.x, z[0] * I0)))));
          keep[P][1] = fma(z[5], c1, fma(z[4], md.y, fma(z[3], y3.y, fma(z[2], y2.y, fma(z[1], y.y, z[0] * I1)))));
          put<NP>(E, 0, rg, c, off, c0, c1);
          put<NP>(E, 1, rg, c, off, n0, n1);  // may overwrite y at this thread's own pair
        })
      break;
    default:
      break;
  }
}

// s doubling steps (driver.py:91-98): S <- 2 S C (old C), C <- 2 C C - I as
// one dual product [S; C] * C into the two free slots, then swap; the last
// step writes the results straight from registers to global memory.

// s doubling steps (driver.py:91-98): S <- 2 S C (old C), C <- 2 C C - I as
// one dual product [S; C] * C into the two free slots, then swap; the last
// step writes the results straight from registers to global memory.
template <int CL, typename TOut>
__device__ __forceinline__ void doubling(double*& C, double*& S, double*& F1,
                                         double*& F2, int steps, const Lane<CL>& ln,
                                         TOut* cdst, TOut* sdst, int n) {
  constexpr int NP = Geo<CL>::NP;
  Acc sc, cc;
  for (int it = 0; it < steps; ++it) {
    TRACE_T(6);
    gemm<CL, true>(S, C, rview<CL>(C, ln.row0 / Geo<CL>::BAND), sc, cc, ln);
    const bool last = it == steps - 1;
#pragma unroll
    for (int mi = 0; mi < Geo<CL>::MI; ++mi)
#pragma unroll
      for (int ni = 0; ni < Geo<CL>::NI; ++ni) {
        const int P = mi * Geo<CL>::NI + ni;
        const int r = ln.rb + mi * 8 + ln.g;
        const int rg = ln.row0 + r;
        const int c = ln.cb + ni * 8 + 2 * ln.t;
        const double s0 = 2.0 * sc[P][0], s1 = 2.0 * sc[P][1];
        const double c0 = fma(2.0, cc[P][0], (rg == c) ? -1.0 : 0.0);
        const double c1 = fma(2.0, cc[P][1], (rg == c + 1) ? -1.0 : 0.0);
        if (last) {
          gstore<NP>(sdst, n, rg, c, s0, s1);
          gstore<NP>(cdst, n, rg, c, c0, c1);
        } else {
          const int off = swz<NP>(r, c);
          st2(F1, off, s0, s1);
          st2(F2, off, c0, c1);
        }
      }
    TRACE_T(7);
    if (!last) {
      step_sync<CL>();
      double* t = S; S = F1; F1 = t;
      t = C; C = F2; F2 = t;
    }
  }
}

// ---------------------------------------------------------------------------
// Global <-> shared movement.


__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
  unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src));
}
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(src));
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(src));
}
__device__ __forceinline__ void cp_async8v(void* dst, const void* src) {
  unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::);
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;\n" ::);
}

// Load matrix (n x n, row-major) into slot dst: async for fp64 input.  For
// n < 64 the padding is rewritten with zeros (the slot may hold a previous
// chain's intermediate).
// NaN-fill this CTA's rows [r0, r0 + rows) of an n x n output.
template <int NT, typename TOut>
__device__ __forceinline__ void store_nan(TOut* __restrict__ dst, int n, int r0, int rows) {
  const int lo = r0 * n, hi = min(n, r0 + rows) * n;
  for (int p = lo + threadIdx.x; p < hi; p += NT)
    dst[p] = static_cast<TOut>(__longlong_as_double(0x7ff8000000000000ll));
}

// ---------------------------------------------------------------------------
// Input staging: the next matrix lands, in its natural row-major layout, in
// slot 6 through ONE TMA bulk copy (cp.async.bulk + mbarrier complete_tx)
// issued by thread 0 -- no LSU traffic -- and is converted to the swizzled
// layout (with the wave family's y = (t')^2 A scaling folded in) at the top
// of its turn.  Odd n (not 16-byte aligned rows) falls back to a
// cooperative synchronous copy.

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes,
                                            uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;\n" ::);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// The selection of one matrix from its column sums (thread 0 of a
// self-selecting CTA; out of line so it does not weigh on the chain's
// register allocation): max over columns, then select_one as select_kernel.
__device__ __noinline__ void self_select(const double* colsum, int n, int fin, const double* t,
                                         int family, int precision, int32_t* K, int32_t* S,
                                         int32_t* ST, unsigned long long* normbits, int* meta,
                                         bool write_out) {
  double norm = 0.0;
  for (int j = 0; j < n; ++j) norm = fmax(norm, colsum[j]);
  int st = fin ? kOk : kNonfiniteInput, kk = 0, ss = 0;
  if (write_out) *normbits = static_cast<unsigned long long>(__double_as_longlong(norm));
  if (st == kOk) {
    const double sel = t ? (t[0] * t[0]) * norm : norm;  // driver.py:136
    st = select_one(sel, dTables.theta[family][precision], dTables.kk[family][precision],
                    dTables.nent[family], dTables.log2fix, &kk, &ss);
  }
  if (st != kOk) kk = ss = 0;
  if (write_out) {
    *K = kk;
    *S = ss;
    *ST = st;
  }
  meta[0] = kk;
  meta[1] = ss;
  meta[2] = st;
}

// SELF (K1 only, batch <= grid): no K0 launches before this one -- CTA b
// takes matrix b, computes its 1-norm (column sums in row order, in the
// input dtype, exactly as norm1_kernel), finiteness and (k, s) itself
// (select_one), and writes K / Sx / ST / normbits for the caller.  The
// latency-bound small-batch path (configs[0]) becomes a single launch.
template <int CL, typename TIn, typename TOut, bool WAVE, bool SELF>
__global__ void __launch_bounds__(Geo<CL>::THREADS, 1)
fused64_kernel(const TIn* __restrict__ Ain, TOut* __restrict__ Cout,
             TOut* __restrict__ Sout, const double* __restrict__ T,
             const int32_t* __restrict__ K, const int32_t* __restrict__ Sx,
             const int32_t* __restrict__ ST, const int32_t* __restrict__ order,
             int64_t batch, int n, int tma, int precision,
             unsigned long long* __restrict__ normbits) {
  static_assert(!SELF || CL == 1 || CL == 5, "self-selection: the small-batch variants");
  constexpr int NC = Geo<CL>::CL;  // CTAs per matrix (a cluster when > 1)
  constexpr int NP = Geo<CL>::NP, BAND = Geo<CL>::BAND, THREADS = Geo<CL>::THREADS;
  extern __shared__ __align__(128) double smem[];
  // Static schedule: cluster c takes order[] positions c, 2G-1-c, 2G+c, ...
  // (a snake over the cost-sorted list).  Thread 0 stages the matrix ids two
  // turns ahead and the next matrix's (k, s, status, t) by 4/8-byte
  // cp.async into small rings, so no global latency is ever exposed.
  __shared__ int sh_b[4];
  __shared__ int sh_meta[2][4];
  __shared__ double sh_t[2];
  __shared__ __align__(8) uint64_t sh_bar;
  __shared__ __align__(8) uint64_t sh_bar2;  // K1s self-selection: the whole matrix
  __shared__ Chain sh_chain[7];
  const int tid = threadIdx.x;
  const int G = gridDim.x / NC, cta = blockIdx.x / NC, rank = blockIdx.x % NC;
  Lane<CL> ln;
  make_lane(ln, rank);
  const size_t nn = static_cast<size_t>(n) * n;
  double* const land = smem + 6 * SLOT;
  // this CTA's input band: rows [row0, row0 + rows_here) of each matrix
  const int row0 = ln.row0;
  const int rows_here = max(0, min(BAND, n - row0));
  const size_t band_off = static_cast<size_t>(row0) * n;
  const unsigned in_bytes = static_cast<unsigned>(rows_here * n * sizeof(TIn));
  const bool tma_here = tma && rows_here > 0 && (in_bytes % 16) == 0;
  auto posof = [&](int i) -> long long {
    return static_cast<long long>(i) * G + ((i & 1) ? (G - 1 - cta) : cta);
  };
  auto prefetch = [&](int b) {  // thread 0 only: next input band -> slot 6
    if (tma_here && b >= 0)
      tma_load_1d(land, Ain + static_cast<size_t>(b) * nn + band_off, in_bytes, &sh_bar);
  };

#ifdef CSM_TRACE
  if (tid == CSM_TRACE_TID) trace_count() = 0;
#endif
  for (int i = tid; i < static_cast<int>(sizeof(kChains) / 4); i += THREADS)
    reinterpret_cast<int*>(sh_chain)[i] = reinterpret_cast<const int*>(kChains)[i];
  if (tid == 0) {
    mbar_init(&sh_bar, 1);
    if (SELF && NC > 1) mbar_init(&sh_bar2, 1);
    const long long p0 = posof(0), p1 = posof(1);
    const int b0 = p0 < batch ? (SELF ? static_cast<int>(p0) : order[p0]) : -1;
    sh_b[0] = b0;
    sh_b[1] = (SELF || p1 >= batch) ? -1 : order[p1];
    if (b0 >= 0) {
      if (!SELF) {
        sh_meta[0][0] = K[b0]; sh_meta[0][1] = Sx[b0]; sh_meta[0][2] = ST[b0];
      }
      sh_t[0] = WAVE ? T[b0] : 0.0;
      prefetch(b0);
      if (SELF && NC > 1 && tma)
        tma_load_1d(smem + 5 * SLOT, Ain + static_cast<size_t>(b0) * nn,
                    static_cast<unsigned>(nn * sizeof(TIn)), &sh_bar2);
    }
  }
  __syncthreads();

  Acc acc, acc2, keep;
  for (int it = 0;; ++it) {
    if (tid == 0) cp_async_wait_all();
    __syncthreads();
    const int b = sh_b[it & 3], bn = sh_b[(it + 1) & 3];
    if (b < 0) break;
    if (tma_here) mbar_wait(&sh_bar, it & 1);  // this matrix's band has landed
    if constexpr (SELF) {  // K0 in the CTA: norm1_kernel + select_kernel for matrix b
      // the whole matrix: K1's band is the matrix; each K1s CTA holds a
      // full copy in slot 5's region (free until the chain starts) and
      // selects redundantly, so the cluster agrees without communication
      const TIn* src0 = Ain + static_cast<size_t>(b) * nn;
      TIn* whole = NC == 1 ? reinterpret_cast<TIn*>(land) : reinterpret_cast<TIn*>(smem + 5 * SLOT);
      if (NC > 1 && tma) mbar_wait(&sh_bar2, it & 1);
      if (NC == 1 ? !tma_here : !tma) {  // unaligned: stage the matrix
        for (int p = tid; p < n * n; p += THREADS) whole[p] = src0[p];
        __syncthreads();
      }
      __shared__ double sh_col[64];
      __shared__ int sh_fin;
      if (tid == 0) sh_fin = 1;
      __syncthreads();
      if (tid < n) {
        const TIn* nat = whole;
        TIn sum = TIn(0);
        bool fin = true;
        for (int i = 0; i < n; ++i) {
          const TIn x = nat[i * n + tid];
          fin &= (x - x == TIn(0));
          sum = sum + fabs(x);  // sequential in row order, as norm1_kernel
        }
        sh_col[tid] = static_cast<double>(sum);
        if (!fin) sh_fin = 0;
      }
      __syncthreads();
      if (tid == 0)
        self_select(sh_col, n, sh_fin, WAVE ? T + b : nullptr, WAVE ? 1 : 0, precision,
                    const_cast<int32_t*>(K) + b, const_cast<int32_t*>(Sx) + b,
                    const_cast<int32_t*>(ST) + b, normbits + b, sh_meta[it & 1], rank == 0);
      __syncthreads();
    }
    const int k = sh_meta[it & 1][0], s = sh_meta[it & 1][1], status = sh_meta[it & 1][2];
    const double tcur = sh_t[it & 1];
    TRACE_T(1);
    CSM_TRACE_EV(9, static_cast<unsigned long long>(k * 16 + s));
    if (!SELF && tid == 0) {  // stage ids and metadata for the coming turns
      const long long p2 = posof(it + 2);
      if (p2 < batch) cp_async4(&sh_b[(it + 2) & 3], order + p2);
      else sh_b[(it + 2) & 3] = -1;
      if (bn >= 0) {
        cp_async4(&sh_meta[(it + 1) & 1][0], K + bn);
        cp_async4(&sh_meta[(it + 1) & 1][1], Sx + bn);
        cp_async4(&sh_meta[(it + 1) & 1][2], ST + bn);
        if (WAVE) cp_async8v(&sh_t[(it + 1) & 1], T + bn);
      }
      cp_async_commit();
    }
    const TIn* src = Ain + static_cast<size_t>(b) * nn + band_off;
    if ((!SELF || NC > 1) && !tma_here && rows_here > 0) {  // unaligned band: synchronous copy
      for (int p = tid; p < rows_here * n; p += THREADS)
        reinterpret_cast<TIn*>(land)[p] = src[p];
      __syncthreads();
    }
    TOut* cdst = Cout + static_cast<size_t>(b) * nn;
    TOut* sdst = Sout + static_cast<size_t>(b) * nn;
    if (status != 0) {  // uniform across the cluster (same matrix)
      store_nan<THREADS>(cdst, n, row0, BAND);
      store_nan<THREADS>(sdst, n, row0, BAND);
      __syncthreads();
      if (tid == 0) prefetch(bn);
      continue;
    }
    double f, tp = 0.0;
    if (WAVE) {
      tp = tcur / ldexp(1.0, s);  // driver.py:139, t / 2**s
      f = tp * tp;                // schemes.py:424, y = (t*t) a
    } else {
      f = ldexp(1.0, -s);  // driver.py:115, a * 2**-s (folded into P1/Pk)
    }
    {  // slot 6 (natural band) -> slot 0 (swizzled, zero padded)
      const double g = WAVE ? f : 1.0;
      const TIn* nat = reinterpret_cast<const TIn*>(land);
#pragma unroll 2
      for (int p = tid; p < BAND * NP / 2; p += THREADS) {
        const int r = p / (NP / 2), c = (p % (NP / 2)) * 2;
        double v0 = 0.0, v1 = 0.0;
        if (n == NP) {
          v0 = static_cast<double>(nat[r * NP + c]);
          v1 = static_cast<double>(nat[r * NP + c + 1]);
        } else if (r < rows_here) {
          if (c < n) v0 = static_cast<double>(nat[r * n + c]);
          if (c + 1 < n) v1 = static_cast<double>(nat[r * n + c + 1]);
        }
        st2(smem, swz<NP>(r, c), g * v0, g * v1);
      }
    }
    step_sync<CL>();  // the first product reads slot 0 of every band
    auto slotp = [&](int i) -> double* { return smem + i * SLOT; };
    const int ci = WAVE ? (k == 3 ? 4 : (k == 4 ? 5 : 6))
                        : (k == 3 ? 0 : (k == 4 ? 1 : (k == 6 ? 2 : 3)));
    const Chain& ch = sh_chain[ci];
    const int nsteps = ch.nsteps, pf_after = ch.pf_after;
    CSM_DCHECK(nsteps >= 1 && nsteps <= 7 && ch.cos_slot >= 0 && ch.cos_slot < NSLOTS);
    CSM_DCHECK(ch.cos_slot != 6 && ch.sin_slot != 6 && ch.free1 != 6 && ch.free2 != 6);
    for (int i = 0; i < nsteps; ++i) {
      const Step st = ch.step[i];
      CSM_DCHECK(st.l1 >= 0 && st.l1 < NSLOTS && st.r >= 0 && st.r < NSLOTS &&
                 st.o0 >= 0 && st.o0 < NSLOTS && (!st.dual || (st.l2 >= 0 && st.l2 < NSLOTS)));
      // slot 6 is the next matrix's landing buffer after step pf_after
      CSM_DCHECK(i <= pf_after || (st.o0 != 6 && st.o1 != 6 && st.o2 != 6 && st.l1 != 6 &&
                                   st.r != 6 && st.i0 != 6 && st.i1 != 6 && st.i2 != 6 &&
                                   st.i3 != 6));
      TRACE_T(2);
      if (st.dual)
        gemm<CL, true>(slotp(st.l1), slotp(st.l2), rview<CL>(slotp(st.r), rank), acc, acc2, ln);
      else
        gemm<CL, false>(slotp(st.l1), nullptr, rview<CL>(slotp(st.r), rank), acc, acc2, ln);
      TRACE_T(3);
      EpiArgs<TOut> E;
      E.o[0] = slotp(st.o0);
      E.o[1] = slotp(st.o1);
      E.o[2] = slotp(st.o2);
#pragma unroll
      for (int q = 0; q < 3; ++q)
        E.g[q] = (s != 0) ? nullptr
               : (i == ch.cos_step && q == ch.cos_out) ? cdst
               : (i == ch.sin_step && q == ch.sin_out) ? sdst : nullptr;
      E.in[0] = slotp(st.i0);
      E.in[1] = slotp(st.i1);
      E.in[2] = slotp(st.i2);
      E.in[3] = slotp(st.i3);
      E.scale = st.scale == SC_F ? f : st.scale == SC_F2 ? f * f
              : st.scale == SC_TP ? tp : 1.0;
      E.n = n;
      epilogue<CL>(st.epi, E, acc, acc2, keep, ln);
      TRACE_T(4);
      step_sync<CL>();
      TRACE_T(5);
      if (i == pf_after && tid == 0) prefetch(bn);
    }
    double* C = slotp(ch.cos_slot);
    double* S = slotp(ch.sin_slot);
    double* F1 = slotp(ch.free1);
    double* F2 = slotp(ch.free2);
    doubling<CL>(C, S, F1, F2, s, ln, cdst, sdst, n);
  }
  // no CTA may leave while a peer can still read its bands
  if (NC > 1) step_sync<CL>();
}

}  // namespace f64k

size_t fused64_smem_bytes() {
  return static_cast<size_t>(f64k::NSLOTS) * f64k::SLOT * sizeof(double);
}

// Launch arguments shared by every instantiation.
struct FusedArgs {
  const void* a;
  void *c, *s;
  const double* t;
  const int32_t *k, *sx, *st, *order;
  int64_t batch;
  int n, sms, precision;
  unsigned long long* normbits;  // self-selection only
  cudaStream_t stream;
};

template <int CL, typename TIn, typename TOut, bool WAVE, bool SELF>
static cudaError_t launch_one(const FusedArgs& F) {
  auto kern = f64k::fused64_kernel<CL, TIn, TOut, WAVE, SELF>;
  const size_t smem = fused64_smem_bytes();
  const size_t mat_bytes = static_cast<size_t>(F.n) * F.n * sizeof(TIn);
  // TMA needs 16-byte aligned matrix starts; K1c checks each band's size
  const int tma = (mat_bytes % 16 == 0 && reinterpret_cast<uintptr_t>(F.a) % 16 == 0) ? 1 : 0;
  cudaError_t e = cudaFuncSetAttribute(
      kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  cfg.blockDim = dim3(f64k::Geo<CL>::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = F.stream;
  int clusters = F.sms;
  constexpr int NC = f64k::Geo<CL>::CL;
  if (NC > 1) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = NC;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(NC * (F.sms / NC));
    int active = 0;
    e = cudaOccupancyMaxActiveClusters(&active, kern, &cfg);
    if (e != cudaSuccess) return e;
    clusters = active > 0 ? active : F.sms / NC;  // persistent: every cluster resident
  }
  if (clusters > F.batch) clusters = static_cast<int>(F.batch);
  if (clusters < 1) return cudaSuccess;
  if (SELF && clusters < F.batch) return cudaErrorInvalidValue;  // one matrix per CTA
  cfg.gridDim = dim3(NC * clusters);
  return cudaLaunchKernelEx(&cfg, kern, static_cast<const TIn*>(F.a), static_cast<TOut*>(F.c),
                            static_cast<TOut*>(F.s), F.t, F.k, F.sx, F.st, F.order, F.batch, F.n,
                            tma, F.precision, F.normbits);
}

template <int CL, bool SELF>
static cudaError_t launch_fused(int dtype, bool wave, const FusedArgs& F) {
  if (dtype == 0)
    return wave ? launch_one<CL, double, double, true, SELF>(F)
                : launch_one<CL, double, double, false, SELF>(F);
  if (dtype == 2)
    return wave ? launch_one<CL, float, double, true, SELF>(F)
                : launch_one<CL, float, double, false, SELF>(F);
  return wave ? launch_one<CL, float, float, true, SELF>(F)
              : launch_one<CL, float, float, false, SELF>(F);
}

static int device_sms() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

// SMs the K1c grid occupies (4 x co-resident clusters; the rest of the GPU
// is free for concurrent work).
int k1c_resident_sms() {
  static int cached[32] = {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1,
                           -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1};
  int dev = 0;
  cudaGetDevice(&dev);
  dev = dev < 32 ? dev : 31;
  if (cached[dev] >= 0) return cached[dev];
  auto kern = f64k::fused64_kernel<4, double, double, false, false>;
  const size_t smem = fused64_smem_bytes();
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem)) != cudaSuccess)
    return 0;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 4;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.blockDim = dim3(f64k::Geo<4>::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.gridDim = dim3(4 * 32);
  int active = 0;
  if (cudaOccupancyMaxActiveClusters(&active, kern, &cfg) != cudaSuccess) return 0;
  cached[dev] = 4 * active;
  return cached[dev];
}

// Launch K1 (n <= 64) or K1c (64 < n <= 128) for a batch whose (k, s,
// status) and cost-sorted order[] are already on the device.
cudaError_t launch_fused64(int dtype, bool wave, const void* a, void* c,
                           void* s, const double* t, const int32_t* k,
                           const int32_t* sx, const int32_t* st, const int32_t* order,
                           int64_t batch, int n, cudaStream_t stream) {
  const FusedArgs F{a, c, s, t, k, sx, st, order, batch, n, device_sms(), 0, nullptr, stream};
  if (n <= 64) return launch_fused<1, false>(dtype, wave, F);
  return launch_fused<4, false>(dtype, wave, F);
}

// Co-resident 4-CTA clusters of K1s (0 when CSM_K1S=0 disables it).
static int k1s_clusters() {
  static const bool on = [] {
    const char* e = std::getenv("CSM_K1S");
    return !(e && e[0] == '0');
  }();
  if (!on) return 0;
  static int cached[32] = {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1,
                           -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1};
  int dev = 0;
  cudaGetDevice(&dev);
  dev = dev < 32 ? dev : 31;
  if (cached[dev] >= 0) return cached[dev];
  auto kern = f64k::fused64_kernel<5, double, double, false, true>;
  const size_t smem = fused64_smem_bytes();
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem)) != cudaSuccess)
    return 0;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 4;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.blockDim = dim3(f64k::Geo<5>::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.gridDim = dim3(4 * 32);
  int active = 0;
  if (cudaOccupancyMaxActiveClusters(&active, kern, &cfg) != cudaSuccess) return 0;
  cached[dev] = active;
  return active;
}

// Largest batch K1 runs self-selecting (one CTA per matrix, no K0 launches).
int64_t fused64_self_max(int n) { return n <= 64 ? device_sms() : 0; }

// K1 with the norm, finiteness and (k, s) selection done by each CTA for
// its own matrix: writes k / sx / st / normbits; batch <= fused64_self_max.
cudaError_t launch_fused64_self(int dtype, int precision, bool wave, const void* a, void* c,
                                void* s, const double* t, int32_t* k, int32_t* sx, int32_t* st,
                                unsigned long long* normbits, int64_t batch, int n,
                                cudaStream_t stream) {
  if (n > 64 || n < 1 || batch > fused64_self_max(n)) return cudaErrorInvalidValue;
  const FusedArgs F{a, c, s, t, k, sx, st, nullptr, batch, n, device_sms(), precision,
                    normbits, stream};
  // a batch that fits the co-resident 4-CTA clusters runs on K1s: each
  // matrix over four SMs, a quarter of every product per SM
  if (batch <= k1s_clusters()) return launch_fused<5, true>(dtype, wave, F);
  return launch_fused<1, true>(dtype, wave, F);
}

}  // namespace csm
