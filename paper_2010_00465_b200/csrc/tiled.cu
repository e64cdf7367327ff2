// tiled.cu -- K2: the chain for n > 64 as a sequence of batched, tiled FP64
// DMMA GEMMs whose epilogues carry every linear combination of the scheme
// (and the doubling update), so no elementwise pass ever runs on its own.
//
// Layout in HBM: each matrix owns NSLOT slots of NP x NP float64, NP = n
// rounded up to 64, row-major, zero-padded (block-diagonal padding is exact,
// see fused64.cu).  Slot 0 is the scaled input: for the Taylor family with
// float64 input and n % 64 == 0 it ALIASES the caller's input (2^-s folded
// into the first and last products' epilogues, exact), otherwise
// prepare_kernel writes 2^-s A / (t')^2 A there.  The chain program for
// scheme k is a short list of Ops (host side, build_program).  The outputs
// that are final for a matrix (cos / sin of the chain when s == 0, of the
// last doubling step otherwise) are written straight into the caller's
// buffers in its dtype by the producing epilogue.
//
// GEMM: CTA tile 64x64, 4 warps of 32x32 (4x4 DMMA m8n8k4 tiles), K step 16
// through a 3-stage cp.async pipeline, 4 CTAs per SM; padded smem rows
// (20 / 68 doubles) make both fragment loads bank-conflict free.  One launch
// runs the same step index for every k-group (a work list of segments), and
// each doubling step runs for all groups at once.  (A persistent dataflow
// variant with per-matrix completion counters measured slower; see
// tools/experiments/tiled_dataflow.cu.txt.)
//
// Reference mapping: schemes.py:264-361 (chains), :376-395 / :411-430
// (trig / wave use), driver.py:91-98 (doubling), driver.py:115/:139
// (scaling), matcore.py:107-121 (linear combinations, fused here).
#include <cuda.h>  // CUtensorMap (types only; the encoder is fetched at run time)

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace csm {

namespace tk {

constexpr int BM = 64, BN = 64, BK = 16, STAGES = 3, THREADS = 128;
constexpr int LDA = BK + 4, LDB = BN + 4, LDE = BN + 8;
constexpr int A_STAGE = BM * LDA, B_STAGE = BK * LDB;
constexpr size_t SMEM = static_cast<size_t>(STAGES) * (A_STAGE + B_STAGE) * sizeof(double);
static_assert(BM * LDE <= STAGES * (A_STAGE + B_STAGE), "epilogue tile fits the pipeline buffers");
constexpr int NSLOT = 9;
constexpr int MAXT = 8;
constexpr int MAXSEG = 8;

#ifndef CSM_TILED_PB
#define CSM_TILED_PB 4  // epilogue pairs in flight per thread
#endif

// Term sources
constexpr int SRC_ACC = -1, SRC_I = -2, SRC_OUT0 = -3;  // OUTj = -3 - j
// Output scale modes
enum { SC_NONE = 0, SC_TP = 1, SC_F = 2, SC_F2 = 3 };
// Final-output marks
enum { FIN_NONE = 0, FIN_COS = 1, FIN_SIN = 2 };

struct Term {
  int32_t src;
  int32_t pad;
  double c;
};
struct OutSpec {
  int32_t slot, nterms, scale, final;
  Term t[MAXT];
};
struct Op {
  int32_t lhs, rhs, nout, pad;
  OutSpec out[3];
};

__device__ __forceinline__ void cp16(double* dst, const double* src) {
  unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void wait_group() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

struct Seg {
  int32_t op;       // op index into the op table
  int32_t idx_off;  // offset of this segment's matrices in the index list
  int32_t start;    // first work item (CTA row) of this segment
};

struct LaunchArgs {
  double* ws;
  const double* in0;    // slot-0 alias (float64 input, n == NP) or null
  const int32_t* idx;   // index lists
  const Op* ops;        // op table
  const double* tsc;    // per-matrix t' (wave) or null
  const int32_t* S;     // per-matrix s
  void* cout;           // caller's outputs
  void* sout;
  size_t mat_stride;
  int NP, n, out_f32, dbl_step;  // dbl_step: -1 for chain ops, else i
  int nseg, total, item_base, pad;
  Seg seg[MAXSEG];
  // Block-row (slab) mode for the distributed chain: every slot holds M
  // rows of the NP x NP matrix starting at global row row0, and the right
  // operand is the all-gathered full matrix rhs_full.  Batch mode: M = NP,
  // row0 = 0, rhs_full = null.
  const double* rhs_full;
  int M, row0;
  // Peer mode (fused all-gather): the right operand's row block j lives in
  // rank j's slab, rhs_parts[j] = that slab's base (a peer pointer over
  // NVLink); the product streams its rows straight from the owner, tile by
  // tile, instead of reading an all-gathered copy.  Null otherwise.
  const double* const* rhs_parts;
  // Ozaki accuracy fallback: when set, only items whose flag is nonzero run
  // (flag index = item - only_base); the others leave at once.
  const unsigned* only;
  int only_base;
  // K-split of a slab product, so the all-gather of its right operand
  // overlaps compute (csm_dist_cos_sin): ksplit 1 contracts only k in this
  // rank's own rows [row0, row0 + M), reading them from its own slab slot
  // op.rhs, and stores the raw product to part; ksplit 2 contracts the
  // complementary k range from rhs_full and adds part before the epilogue;
  // 0 is the whole contraction.  part: M x NP doubles per launch item y.
  int ksplit;
  double* part;
  // TMA staging (tma = 1): 2-D tensor maps over the slots (rows of every
  // slot of every matrix stacked: row (b mat_stride + sl M NP) / NP + r),
  // the slot-0 alias in0 and the gathered rhs_full.  *L: 64 x 16 boxes with
  // the 128-byte swizzle (left-operand tile); *R: 16 x 8 boxes with the
  // 64-byte swizzle (8 per right-operand tile), both conflict-free for the
  // DMMA fragment loads.  tma = 0 keeps the cp.async staging (peer mode).
  int tma;
  CUtensorMap tm_wsL, tm_wsR, tm_in0L, tm_in0R, tm_rhsR;
};

// Slot sl of matrix b (slot 0 may alias the caller's input).
__device__ __forceinline__ double* slot_ptr(const LaunchArgs& args, int b, int sl) {
  const size_t slotsz = static_cast<size_t>(args.M) * args.NP;
  if (sl == 0 && args.in0)
    return const_cast<double*>(args.in0) + static_cast<size_t>(b) * slotsz;
  return args.ws + static_cast<size_t>(b) * args.mat_stride + sl * slotsz;
}

// The op's linear combinations for output tile (tm, tn) of matrix b, from
// the product tile E ([BM][LDE] in shared memory): row-contiguous
// (coalesced) global reads of the slot terms and writes of the outputs.
// CSM_TILED_DEDUP=1 builds the variant below that loads each distinct slot
// term once per pair group; measured 3-7% SLOWER than the per-term loads
// (cfg3 0.780 vs 0.834 of the DMMA peak, n = 512 0.876 vs 0.907; profiles/r2/s4/):
// the register-resident copies cost occupancy of the loads in flight.  Off.
#ifndef CSM_TILED_DEDUP
#define CSM_TILED_DEDUP 0
#endif

// One final (cos / sin) pair at flat index o of the caller's n x n output.
__device__ __forceinline__ void store_final(void* dst, int out_f32, size_t o, int c, int n,
                                            double v0, double v1) {
  if (out_f32) {
    float* d = static_cast<float*>(dst);
    if (c < n) d[o] = static_cast<float>(v0);
    if (c + 1 < n) d[o + 1] = static_cast<float>(v1);
  } else {
    double* d = static_cast<double*>(dst);
    if (c + 1 < n && ((o & 1) == 0)) {
      *reinterpret_cast<double2*>(d + o) = make_double2(v0, v1);
    } else {
      if (c < n) d[o] = v0;
      if (c + 1 < n) d[o + 1] = v1;
    }
  }
}

template <int NT>
__device__ __forceinline__ void epilogue_tile(const LaunchArgs& args, const Op& op, int b,
                                              int tm, int tn, const double* E) {
  const int tid = threadIdx.x;
  const int NP = args.NP;
  const int n = args.n;
  const size_t nn = static_cast<size_t>(n) * n;
  const size_t slotsz = static_cast<size_t>(args.M) * NP;
  double* base = args.ws + static_cast<size_t>(b) * args.mat_stride;
  auto slot = [&](int sl) -> double* { return slot_ptr(args, b, sl); };
  const int s_b = args.S[b];
  const double sc_tp = args.tsc ? args.tsc[b] : 1.0;
  const double sc_f = ldexp(1.0, -s_b), sc_f2 = ldexp(1.0, -2 * s_b);
  const bool final_now = args.dbl_step < 0 ? (s_b == 0) : (s_b == args.dbl_step + 1);
  const int nout = op.nout;
  const int r0 = tm * BM, c0 = tn * BN;
  // PB pairs per thread at a time: every slot-sourced term issues PB
  // independent loads before its FMAs, so the workspace reads (HBM for
  // large batches) overlap instead of exposing one latency per term.
  // Distinct slot sources of the op (the heaviest epilogues read y, y2, y3
  // and mid in up to three outputs each): loaded ONCE per pair group, all
  // up front, then every output sums its terms in its listed order from
  // registers -- the same FMA sequence as per-term loads, so bitwise the
  // same results, with all the group's workspace reads in flight at once.
  constexpr int MAXD = 6, PD = 2;  // distinct slots, pairs per thread per group
  int dsrc[MAXD], nd = 0;
#pragma unroll
  for (int d = 0; d < MAXD; ++d) dsrc[d] = -1;
  for (int q = 0; q < nout; ++q)
    for (int tt = 0; tt < op.out[q].nterms; ++tt) {
      const int src = op.out[q].t[tt].src;
      if (src < 0) continue;
      bool seen = false;
#pragma unroll
      for (int d = 0; d < MAXD; ++d) seen |= dsrc[d] == src;
      if (!seen && nd < MAXD) {
#pragma unroll
        for (int d = 0; d < MAXD; ++d)
          if (d == nd) dsrc[d] = src;
      }
      nd += seen ? 0 : 1;
    }
  if (CSM_TILED_DEDUP && nd <= MAXD) {
    static_assert((BM * BN / 2) % (PD * NT) == 0, "pair groups tile the output");
    for (int p0 = tid; p0 < BM * BN / 2; p0 += PD * NT) {
      size_t off[PD];
      double2 xs[MAXD][PD];
#pragma unroll
      for (int m = 0; m < PD; ++m) {
        const int p = p0 + m * NT;
        off[m] = static_cast<size_t>(r0 + (p >> 5)) * NP + c0 + (p & 31) * 2;
      }
#pragma unroll
      for (int d = 0; d < MAXD; ++d)
        if (d < nd) {
          const double* sp = slot(dsrc[d]);
#pragma unroll
          for (int m = 0; m < PD; ++m) xs[d][m] = *reinterpret_cast<const double2*>(sp + off[m]);
        }
      double o0[PD][2], o1[PD][2];
      for (int q = 0; q < nout; ++q) {
        const OutSpec& os = op.out[q];
        double v[PD][2];
#pragma unroll
        for (int m = 0; m < PD; ++m) v[m][0] = v[m][1] = 0.0;
        for (int tt = 0; tt < os.nterms; ++tt) {
          const int src = os.t[tt].src;
          const double cf = os.t[tt].c;
#pragma unroll
          for (int m = 0; m < PD; ++m) {
            const int p = p0 + m * NT;
            double x0 = 0.0, x1 = 0.0;
            if (src >= 0) {
#pragma unroll
              for (int d = 0; d < MAXD; ++d)
                if (dsrc[d] == src) { x0 = xs[d][m].x; x1 = xs[d][m].y; }
            } else if (src == SRC_ACC) {
              const double2 av = *reinterpret_cast<const double2*>(
                  E + (p >> 5) * LDE + (p & 31) * 2);
              x0 = av.x; x1 = av.y;
            } else if (src == SRC_I) {
              const int rg = r0 + (p >> 5) + args.row0, c = c0 + (p & 31) * 2;
              x0 = (rg == c) ? 1.0 : 0.0;
              x1 = (rg == c + 1) ? 1.0 : 0.0;
            } else if (src == SRC_OUT0) {
              x0 = o0[m][0]; x1 = o0[m][1];
            } else {
              x0 = o1[m][0]; x1 = o1[m][1];
            }
            v[m][0] = fma(cf, x0, v[m][0]);
            v[m][1] = fma(cf, x1, v[m][1]);
          }
        }
        if (os.scale != SC_NONE) {
          const double sc = os.scale == SC_TP ? sc_tp : (os.scale == SC_F ? sc_f : sc_f2);
#pragma unroll
          for (int m = 0; m < PD; ++m) { v[m][0] *= sc; v[m][1] *= sc; }
        }
#pragma unroll
        for (int m = 0; m < PD; ++m) {
          if (q == 0) { o0[m][0] = v[m][0]; o0[m][1] = v[m][1]; }
          if (q == 1) { o1[m][0] = v[m][0]; o1[m][1] = v[m][1]; }
          *reinterpret_cast<double2*>(base + os.slot * slotsz + off[m]) =
              make_double2(v[m][0], v[m][1]);
        }
        if (os.final != FIN_NONE && final_now) {
          void* dst = os.final == FIN_COS ? args.cout : args.sout;
#pragma unroll
          for (int m = 0; m < PD; ++m) {
            const int p = p0 + m * NT;
            const int r = r0 + (p >> 5), c = c0 + (p & 31) * 2;
            if (r >= n) continue;
            store_final(dst, args.out_f32, static_cast<size_t>(b) * nn +
                        static_cast<size_t>(r) * n + c, c, n, v[m][0], v[m][1]);
          }
        }
      }
    }
    return;
  }
  constexpr int PB = CSM_TILED_PB;
  static_assert((BM * BN / 2) % (PB * NT) == 0, "pair groups tile the output");
  for (int p0 = tid; p0 < BM * BN / 2; p0 += PB * NT) {
    size_t off[PB];
    int ecol[PB];
    double o0[PB][2], o1[PB][2];  // outputs 0 and 1 (OUTj terms of later outputs)
#pragma unroll
    for (int m = 0; m < PB; ++m) {
      const int p = p0 + m * NT;
      const int rr = p >> 5, cc = (p & 31) * 2;  // 32 pairs per tile row
      off[m] = static_cast<size_t>(r0 + rr) * NP + c0 + cc;
      ecol[m] = rr * LDE + cc;
      o0[m][0] = o0[m][1] = o1[m][0] = o1[m][1] = 0.0;
    }
    for (int q = 0; q < nout; ++q) {
      const OutSpec& os = op.out[q];
      CSM_DCHECK(os.slot >= 1 && os.slot < NSLOT && os.nterms >= 0 && os.nterms <= MAXT);
      double v[PB][2];
#pragma unroll
      for (int m = 0; m < PB; ++m) v[m][0] = v[m][1] = 0.0;
      for (int tt = 0; tt < os.nterms; ++tt) {
        const int src = os.t[tt].src;
        const double cf = os.t[tt].c;
        CSM_DCHECK(src < NSLOT && src >= SRC_OUT0 - 1 && (src > SRC_OUT0 - q || src >= SRC_I));
        if (src >= 0) {
          const double* sp = slot(src);
          double2 x[PB];
#pragma unroll
          for (int m = 0; m < PB; ++m) x[m] = *reinterpret_cast<const double2*>(sp + off[m]);
#pragma unroll
          for (int m = 0; m < PB; ++m) {
            v[m][0] = fma(cf, x[m].x, v[m][0]);
            v[m][1] = fma(cf, x[m].y, v[m][1]);
          }
        } else {
#pragma unroll
          for (int m = 0; m < PB; ++m) {
            double x0, x1;
            if (src == SRC_ACC) {
              const double2 av = *reinterpret_cast<const double2*>(E + ecol[m]);
              x0 = av.x; x1 = av.y;
            } else if (src == SRC_I) {
              const int p = p0 + m * NT;
              const int rg = r0 + (p >> 5) + args.row0, c = c0 + (p & 31) * 2;
              x0 = (rg == c) ? 1.0 : 0.0;
              x1 = (rg == c + 1) ? 1.0 : 0.0;
            } else if (src == SRC_OUT0) {
              x0 = o0[m][0]; x1 = o0[m][1];
            } else {
              x0 = o1[m][0]; x1 = o1[m][1];
            }
            v[m][0] = fma(cf, x0, v[m][0]);
            v[m][1] = fma(cf, x1, v[m][1]);
          }
        }
      }
      if (os.scale != SC_NONE) {
        const double sc = os.scale == SC_TP ? sc_tp : (os.scale == SC_F ? sc_f : sc_f2);
#pragma unroll
        for (int m = 0; m < PB; ++m) { v[m][0] *= sc; v[m][1] *= sc; }
      }
#pragma unroll
      for (int m = 0; m < PB; ++m) {
        if (q == 0) { o0[m][0] = v[m][0]; o0[m][1] = v[m][1]; }
        if (q == 1) { o1[m][0] = v[m][0]; o1[m][1] = v[m][1]; }
        *reinterpret_cast<double2*>(base + os.slot * slotsz + off[m]) =
            make_double2(v[m][0], v[m][1]);
      }
      if (os.final != FIN_NONE && final_now) {
        void* dst = os.final == FIN_COS ? args.cout : args.sout;
#pragma unroll
        for (int m = 0; m < PB; ++m) {
          const int p = p0 + m * NT;
          const int r = r0 + (p >> 5), c = c0 + (p & 31) * 2;
          if (r >= n) continue;
          const double v0 = v[m][0], v1 = v[m][1];
          const size_t o = static_cast<size_t>(b) * nn + static_cast<size_t>(r) * n + c;
          if (args.out_f32) {
            float* d = static_cast<float*>(dst);
            if (c < n) d[o] = static_cast<float>(v0);
            if (c + 1 < n) d[o + 1] = static_cast<float>(v1);
          } else {
            double* d = static_cast<double*>(dst);
            if (c + 1 < n && ((o & 1) == 0)) {
              *reinterpret_cast<double2*>(d + o) = make_double2(v0, v1);
            } else {
              if (c < n) d[o] = v0;
              if (c + 1 < n) d[o + 1] = v1;
            }
          }
        }
      }
    }
  }
}

// After the product: a K-split partial tile goes out raw (ksplit 1) or is
// added in (ksplit 2) before the epilogue.
template <int NT>
__device__ __forceinline__ void finish_tile(const LaunchArgs& args, const Op& op, int b, int tm,
                                            int tn, double* E, size_t slotsz) {
  const int tid = threadIdx.x;
  if (args.ksplit != 0) {  // partial product: raw tile out, or added in
    const int NP = args.NP;
    double* pt = args.part + static_cast<size_t>(blockIdx.y) * slotsz +
                 static_cast<size_t>(tm) * BM * NP + static_cast<size_t>(tn) * BN;
    for (int p = tid; p < BM * BN / 2; p += NT) {
      const int rr = p >> 5, cc = (p & 31) * 2;
      double2* e = reinterpret_cast<double2*>(E + rr * LDE + cc);
      double2* g = reinterpret_cast<double2*>(pt + static_cast<size_t>(rr) * NP + cc);
      if (args.ksplit == 1) {
        *g = *e;
      } else {
        const double2 x = *g;
        *e = make_double2(e->x + x.x, e->y + x.y);
      }
    }
    if (args.ksplit == 1) return;
    __syncthreads();
  }
  epilogue_tile<NT>(args, op, b, tm, tn, E);
}

// One 64x64 output tile of one matrix: acc = L R over the full NP-deep
// contraction, then the op's linear combinations from the staged
// accumulator tile with row-contiguous (coalesced) global reads and writes.
#ifndef CSM_TILED_MINB
#define CSM_TILED_MINB 4  // resident CTAs per SM the register budget targets
#endif
__device__ __forceinline__ unsigned tk_smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void tk_mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(tk_smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 2-D tiled TMA load of one box into shared memory, completing on `bar`.
__device__ __forceinline__ void tk_tma2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(tk_smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(tk_smem_u32(bar))
      : "memory");
}

// CTA of the GEMM over the 64 x 64 tile: W = 4 warps of 32 x 32 (4 CTAs
// per SM; the product of each 256-deep contraction chunk is summed in one
// FMA chain) or W = 8 warps of 32 x 16 (2 CTAs per SM; 16 accumulator
// doubles per thread leave room for the blocked summation below).  TMA:
// operands staged by tensor-map TMA (true) or cp.async (false, peer mode).
//
// Blocked summation (W = 8): the contraction is accumulated in chunks of
// KFLUSH stages (KFLUSH x 16 = 256 terms) that are then added into an outer
// accumulator.  A single sequential FMA chain over K = 8192 carries ~5x the
// rounding error of a blocked BLAS GEMM (tests/test_gpu_fullsize.py: cfg5
// measured 5x the reference's own noise); chunks of 256 match it.  W = 8
// serves NP > kWideNP (launch_gemm), where the epilogue is a small share of
// the tile and 2 CTAs per SM suffice.
#ifndef CSM_TILED_KFLUSH
#define CSM_TILED_KFLUSH 16
#endif
constexpr int kWideNP = 1024;

template <bool TMA, int W, bool BLK>
__global__ void __launch_bounds__(32 * W, W == 8 ? 2 : (BLK ? 3 : CSM_TILED_MINB))
    gemm_epi_kernel(const __grid_constant__ LaunchArgs args) {
  static_assert(W == 4 || W == 8, "4 or 8 warps");
  constexpr int GTHREADS = 32 * W, WNI = W == 8 ? 2 : 4;
  extern __shared__ __align__(16) double sm[];
  __shared__ Op op;
  __shared__ int sh_b;
  __shared__ __align__(8) uint64_t full[STAGES];  // TMA stage barriers
  double* As = sm;
  double* Bs = sm + STAGES * A_STAGE;
  // TMA stages: the swizzle patterns need 1024-byte aligned boxes; the TMA
  // layout (48 KB) leaves room for the shift inside SMEM (56.8 KB)
  double* const tb = sm + (((1024u - (tk_smem_u32(sm) & 1023u)) & 1023u) >> 3);
  static_assert(STAGES * (BM * BK + BK * BN) * sizeof(double) + 1024 <= SMEM, "TMA stages fit");
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int item = static_cast<int>(blockIdx.y) + args.item_base;
  if (args.only && args.only[item - args.only_base] == 0u) return;  // not a fallback item
  Seg sg = args.seg[0];
#pragma unroll
  for (int i = 1; i < MAXSEG; ++i)
    if (i < args.nseg && item >= args.seg[i].start) sg = args.seg[i];
  for (int i = tid; i < static_cast<int>(sizeof(Op) / 4); i += GTHREADS)
    reinterpret_cast<int*>(&op)[i] = reinterpret_cast<const int*>(args.ops + sg.op)[i];
  if (tid == 0) {
    sh_b = args.idx[sg.idx_off + item - sg.start];
    if (TMA) {
#pragma unroll
      for (int s = 0; s < STAGES; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(tk_smem_u32(&full[s])));
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    }
  }
  __syncthreads();
  const int b = sh_b;
  const int NP = args.NP;
  const int M = args.M;
  const int tiles_n = NP / BN;
  const int tm = blockIdx.x / tiles_n, tn = blockIdx.x - tm * tiles_n;
  CSM_DCHECK(b >= 0 && op.lhs >= 0 && op.lhs < NSLOT && op.rhs >= 0 && op.rhs < NSLOT);
  CSM_DCHECK(op.nout >= 1 && op.nout <= 3 && tm * BM < M && tn * BN < NP);
  CSM_DCHECK(args.ksplit == 0 || (args.part && args.row0 % BK == 0 && args.row0 + M <= NP));
  CSM_DCHECK(!args.rhs_parts || args.ksplit == 0);
  const int g = lane >> 2, t = lane & 3;
  const int wm = W == 8 ? (warp >> 2) * 32 : (warp >> 1) * 32;
  const int wn = W == 8 ? (warp & 3) * 16 : (warp & 1) * 32;
  const size_t slotsz = static_cast<size_t>(M) * NP;
  double* base = args.ws + static_cast<size_t>(b) * args.mat_stride;
  auto slot = [&](int sl) -> double* {
    if (sl == 0 && args.in0)
      return const_cast<double*>(args.in0) + static_cast<size_t>(b) * slotsz;
    return base + sl * slotsz;
  };
  // k-stage j -> contraction index (K-split: own rows, or all but them)
  const int nk = (args.ksplit == 0 ? NP : (args.ksplit == 1 ? M : NP - M)) / BK;
  auto kof = [&](int j) -> int {
    const int k = j * BK;
    if (args.ksplit == 1) return args.row0 + k;
    if (args.ksplit == 2 && k >= args.row0) return k + M;
    return k;
  };

  // -- staging: TMA (tensor maps, swizzled boxes) or cp.async (padded rows)
  const double* L = slot(op.lhs) + static_cast<size_t>(tm) * BM * NP;
  const double* R = (args.rhs_full ? args.rhs_full : slot(op.rhs)) + static_cast<size_t>(tn) * BN;
  // row k0 of the right operand (a BK-row stage never crosses a part: M % 64 == 0)
  auto rhs_rows = [&](int k0) -> const double* {
    if (args.ksplit == 1)  // own rows of the (not yet gathered) right operand
      return slot(op.rhs) + static_cast<size_t>(k0 - args.row0) * NP + static_cast<size_t>(tn) * BN;
    if (args.rhs_parts) {
      const int part = k0 / M;
      return args.rhs_parts[part] + static_cast<size_t>(op.rhs) * slotsz +
             static_cast<size_t>(k0 - part * M) * NP + static_cast<size_t>(tn) * BN;
    }
    return R + static_cast<size_t>(k0) * NP;
  };
  auto ws_row = [&](int sl) -> int {
    return static_cast<int>((static_cast<size_t>(b) * args.mat_stride + sl * slotsz) / NP);
  };
  const CUtensorMap* mapL = nullptr;
  const CUtensorMap* mapR = nullptr;
  int rowL = 0, rowR = 0;  // rowR: map row holding contraction index 0
  if constexpr (TMA) {
    const bool l_in0 = op.lhs == 0 && args.in0;
    mapL = l_in0 ? &args.tm_in0L : &args.tm_wsL;
    rowL = (l_in0 ? b * M : ws_row(op.lhs)) + tm * BM;
    if (args.ksplit == 1) {
      mapR = &args.tm_wsR;
      rowR = ws_row(op.rhs) - args.row0;
    } else if (args.rhs_full) {
      mapR = &args.tm_rhsR;
    } else if (op.rhs == 0 && args.in0) {
      mapR = &args.tm_in0R;
      rowR = b * M;
    } else {
      mapR = &args.tm_wsR;
      rowR = ws_row(op.rhs);
    }
  }
  auto load_stage = [&](int stage, int k0) {
    if constexpr (TMA) {  // thread 0: one 64 x 16 box of L, eight 16 x 8 boxes of R
      if (tid != 0) return;
      asm volatile("fence.proxy.async.shared::cta;\n" ::);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                       tk_smem_u32(&full[stage])),
                   "r"(static_cast<unsigned>((BM * BK + BK * BN) * sizeof(double))));
      tk_tma2d(tb + stage * BM * BK, mapL, k0, rowL, &full[stage]);
#pragma unroll
      for (int j = 0; j < BN / 8; ++j)
        tk_tma2d(tb + STAGES * BM * BK + stage * BK * BN + j * BK * 8, mapR, tn * BN + 8 * j,
                 rowR + k0, &full[stage]);
    } else {
    double* as = As + stage * A_STAGE;
    double* bs = Bs + stage * B_STAGE;
#pragma unroll
    for (int i = 0; i < (BM * BK / 2) / GTHREADS; ++i) {
      const int p = tid + i * GTHREADS;
      const int r = p / (BK / 2), c = (p - r * (BK / 2)) * 2;
      cp16(as + r * LDA + c, L + static_cast<size_t>(r) * NP + k0 + c);
    }
    const double* Rk = rhs_rows(k0);
#pragma unroll
    for (int i = 0; i < (BK * BN / 2) / GTHREADS; ++i) {
      const int p = tid + i * GTHREADS;
      const int r = p / (BN / 2), c = (p - r * (BN / 2)) * 2;
      cp16(bs + r * LDB + c, Rk + static_cast<size_t>(r) * NP + c);
    }
    }
  };
  // fragments of k-step kk of stage st
  auto frags = [&](int st, int kk, double (&a)[4], double (&bf)[WNI]) {
    const int k = kk + t;
    if constexpr (TMA) {
      const double* as = tb + st * BM * BK;
      const double* bs = tb + STAGES * BM * BK + st * BK * BN;
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)  // (r, k) -> 16 r + 2 ((k / 2) ^ (r % 8)) + k % 2, r % 8 = g
        a[mi] = as[(wm + mi * 8 + g) * BK + (((k >> 1) ^ g) << 1) + (k & 1)];
#pragma unroll
      for (int ni = 0; ni < WNI; ++ni)  // box j, (k, c) -> 8 k + 2 ((c / 2) ^ (k / 2 % 4)) + c % 2
        bf[ni] = bs[((wn >> 3) + ni) * (BK * 8) + k * 8 + (((g >> 1) ^ ((k >> 1) & 3)) << 1) +
                    (g & 1)];
    } else {
      const double* as = As + st * A_STAGE;
      const double* bs = Bs + st * B_STAGE;
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = as[(wm + mi * 8 + g) * LDA + k];
#pragma unroll
      for (int ni = 0; ni < WNI; ++ni) bf[ni] = bs[k * LDB + wn + ni * 8 + g];
    }
  };

  double acc[4][WNI][2], outer[4][WNI][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < WNI; ++j) acc[i][j][0] = acc[i][j][1] = outer[i][j][0] = outer[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, kof(s));
    if constexpr (!TMA) commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    const int st = kt % STAGES;
    if constexpr (TMA)
      tk_mbar_wait(&full[st], static_cast<unsigned>((kt / STAGES) & 1));
    else
      wait_group<STAGES - 2>();
    __syncthreads();  // every warp is done with the stage refilled next
    {
      const int nxt = kt + STAGES - 1;
      if (nxt < nk) load_stage(nxt % STAGES, kof(nxt));
      if constexpr (!TMA) commit();
    }
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[4], bf[WNI];
      frags(st, kk, a, bf);
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < WNI; ++ni) dmma(acc[mi][ni], a[mi], bf[ni]);
    }
    if (BLK && CSM_TILED_KFLUSH > 0 && (kt + 1) % CSM_TILED_KFLUSH == 0 && kt + 1 < nk) {
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < WNI; ++ni) {
          outer[mi][ni][0] += acc[mi][ni][0];
          outer[mi][ni][1] += acc[mi][ni][1];
          acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
        }
    }
  }
  if constexpr (!TMA) wait_group<0>();
  __syncthreads();  // pipeline buffers are free: stage the accumulator tile

  double* E = sm;  // [BM][LDE]
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < WNI; ++ni)
      *reinterpret_cast<double2*>(E + (wm + mi * 8 + g) * LDE + wn + ni * 8 + 2 * t) =
          BLK ? make_double2(outer[mi][ni][0] + acc[mi][ni][0], outer[mi][ni][1] + acc[mi][ni][1])
                 : make_double2(acc[mi][ni][0], acc[mi][ni][1]);
  __syncthreads();
  finish_tile<GTHREADS>(args, op, b, tm, tn, E, slotsz);
}

// Launch the GEMM variant for A: TMA staging when A.tma; for NP > kWideNP
// the blocked-summation CTA (4 warps at 3 CTAs per SM; CSM_TILED_W=8 picks
// the 8-warp one, CSM_TILED_W=4 the unblocked 4-warp CTA at every size).
inline int gemm_variant(int NP) {
  static const int forced = [] {
    const char* e = std::getenv("CSM_TILED_W");
    return e ? std::atoi(e) : 0;
  }();
  if (forced == 4) return 0;      // 4 warps, one FMA chain
  if (forced == 8) return 2;      // 8 warps, blocked
  return NP > kWideNP ? 1 : 0;    // 1: 4 warps, blocked
}
template <bool TMA>
inline void launch_gemm_t(dim3 grid, const LaunchArgs& A, cudaStream_t st) {
  switch (gemm_variant(A.NP)) {
    case 0: gemm_epi_kernel<TMA, 4, false><<<grid, 128, SMEM, st>>>(A); break;
    case 1: gemm_epi_kernel<TMA, 4, true><<<grid, 128, SMEM, st>>>(A); break;
    default: gemm_epi_kernel<TMA, 8, true><<<grid, 256, SMEM, st>>>(A); break;
  }
}
inline void launch_gemm(dim3 grid, const LaunchArgs& A, cudaStream_t st) {
  if (A.tma) launch_gemm_t<true>(grid, A, st);
  else launch_gemm_t<false>(grid, A, st);
}

#include "ozaki.cuh"

// slot0 <- f * A (zero padded).  Taylor: f = 2^-s; wave: t' = t/2^s,
// f = t' * t', and tsc[b] = t'.  Only when slot 0 cannot alias the input.
template <typename TIn>
__global__ void prepare_kernel(const TIn* __restrict__ A, double* __restrict__ ws,
                               int n, int NP, size_t mat_stride, const int32_t* __restrict__ S,
                               const int32_t* __restrict__ status, const double* __restrict__ T,
                               double* __restrict__ tsc, int copy) {
  const int b = blockIdx.y;
  if (status[b] != 0) return;
  const int s = S[b];
  double f;
  if (T) {
    const double tp = T[b] / ldexp(1.0, s);
    f = tp * tp;
    if (blockIdx.x == 0 && threadIdx.x == 0) tsc[b] = tp;
  } else {
    f = ldexp(1.0, -s);
  }
  if (!copy) return;
  double* dst = ws + static_cast<size_t>(b) * mat_stride;
  const TIn* src = A + static_cast<size_t>(b) * n * n;
  const size_t total = static_cast<size_t>(NP) * NP;
  for (size_t p = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < total;
       p += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(p / NP), c = static_cast<int>(p - static_cast<size_t>(r) * NP);
    double v = 0.0;
    if (r < n && c < n) v = static_cast<double>(src[static_cast<size_t>(r) * n + c]) * f;
    dst[p] = v;
  }
}

// NaN outputs for matrices whose status is non-zero.
template <typename TOut>
__global__ void nan_fill_kernel(TOut* __restrict__ Cout, TOut* __restrict__ Sout, int n,
                                const int32_t* __restrict__ status) {
  const int b = blockIdx.y;
  if (status[b] == 0) return;
  const size_t nn = static_cast<size_t>(n) * n;
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  for (size_t p = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < nn;
       p += static_cast<size_t>(gridDim.x) * blockDim.x) {
    Cout[b * nn + p] = static_cast<TOut>(qnan);
    Sout[b * nn + p] = static_cast<TOut>(qnan);
  }
}

// ---- TMA tensor maps of the GEMM operands --------------------------------
// cuTensorMapEncodeTiled is fetched from the driver at run time (no -lcuda).
typedef CUresult (*PfnEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
inline PfnEncodeTiled encode_tiled() {
  static PfnEncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<PfnEncodeTiled>(nullptr);
    return reinterpret_cast<PfnEncodeTiled>(p);
  }();
  return fn;
}
// float64 rows x NP (row stride NP), boxes of box_r rows x box_c columns.
inline bool encode2d(CUtensorMap* m, const double* base, int NP, size_t rows, int box_c,
                     int box_r, CUtensorMapSwizzle sw) {
  PfnEncodeTiled fn = encode_tiled();
  if (!fn || !base || rows == 0 || rows > 0x7fffffffull ||
      (reinterpret_cast<uintptr_t>(base) & 15))
    return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(NP), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(NP) * sizeof(double)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_c), static_cast<cuuint32_t>(box_r)};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// TMA staging for A when every operand can be described (tma = 0 keeps the
// cp.async staging: peer mode, or CSM_TILED_TMA=0 for A/B measurements).
// ws_rows / in0_rows: rows of the slot stack and of the slot-0 alias.
inline void set_tma(LaunchArgs& A, size_t ws_rows, size_t in0_rows) {
  static const bool enabled = [] {
    const char* e = std::getenv("CSM_TILED_TMA");
    return !(e && e[0] == '0');
  }();
  A.tma = 0;
  if (!enabled || A.rhs_parts) return;
  const CUtensorMapSwizzle L128 = CU_TENSOR_MAP_SWIZZLE_128B, R64 = CU_TENSOR_MAP_SWIZZLE_64B;
  bool ok = encode2d(&A.tm_wsL, A.ws, A.NP, ws_rows, BK, BM, L128) &&
            encode2d(&A.tm_wsR, A.ws, A.NP, ws_rows, 8, BK, R64);
  if (ok && A.in0)
    ok = encode2d(&A.tm_in0L, A.in0, A.NP, in0_rows, BK, BM, L128) &&
         encode2d(&A.tm_in0R, A.in0, A.NP, in0_rows, 8, BK, R64);
  if (ok && A.rhs_full)
    ok = encode2d(&A.tm_rhsR, A.rhs_full, A.NP, static_cast<size_t>(A.NP), 8, BK, R64);
  A.tma = ok ? 1 : 0;
}

// Opt the tiled kernel into its dynamic shared memory, once per device.
inline cudaError_t ensure_smem_attr() {
  static unsigned done_mask = 0;  // bit per device ordinal (< 32)
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 32 && ((done_mask >> dev) & 1u)) return cudaSuccess;
  e = cudaSuccess;
  for (auto k : {gemm_epi_kernel<false, 4, false>, gemm_epi_kernel<false, 4, true>,
                 gemm_epi_kernel<false, 8, true>, gemm_epi_kernel<true, 4, false>,
                 gemm_epi_kernel<true, 4, true>, gemm_epi_kernel<true, 8, true>})
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(SMEM));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(oz_crt_epi<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(SMEM));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(oz_crt_epi<9>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(SMEM));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(oz_gemm<OZ_NSTAGE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(OZ_SMEM));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(oz_gemm_p<OZ_NSTAGE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(OZ_SMEM));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(oz_gemm<OZ_NSTAGE_SMALL>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(OZ_NSTAGE_SMALL * OZ_STAGE));
  if (e == cudaSuccess && dev < 32) done_mask |= 1u << dev;
  return e;
}

// Order-8 Pade: LU with partial pivoting of the shared denominator (slot 5)
// and the two solves for the numerators (slots 6 and 7, in place), one CTA
// per matrix on its n x n block (the padding of den / num_cos is I and of
// num_sin is 0, so the padded solution is block-diagonal too).  Mirrors
// lu_solve_pair (matcore.py:124-151): LAPACK getrf pivoting (first largest
// |a_ik|), singular when min |u_kk| <= 1e3 eps ||den||_1, then getrs.
// Matrices with s == 0 write their final cos / sin here.
__global__ void __launch_bounds__(256) pade_lu_solve_kernel(
    double* __restrict__ ws, size_t mat_stride, int NP, int n, const int32_t* __restrict__ idx,
    const int32_t* __restrict__ S, int32_t* __restrict__ status, void* cout, void* sout,
    int out_f32) {
  const int b = idx[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t slotsz = static_cast<size_t>(NP) * NP;
  double* const Dg = ws + static_cast<size_t>(b) * mat_stride + 5 * slotsz;
  double* D = Dg;
  double* X[2] = {Dg + slotsz, Dg + 2 * slotsz};
  // NP = 64: den and both right-hand sides (3 x 32 KiB) are staged in
  // shared memory for the whole factorisation and solve
  extern __shared__ __align__(16) double lu_sm[];
  const bool staged = NP == 64;
  if (staged) {
    for (int e = tid; e < static_cast<int>(3 * slotsz / 2); e += 256)
      reinterpret_cast<double2*>(lu_sm)[e] = reinterpret_cast<const double2*>(Dg)[e];
    D = lu_sm;
    X[0] = lu_sm + slotsz;
    X[1] = lu_sm + 2 * slotsz;
    __syncthreads();
  }
  __shared__ double red_v[8];
  __shared__ int red_i[8];
  __shared__ int sh_p;
  __shared__ double sh_norm, sh_umin;

  // ||den||_1 (threshold of the singularity test)
  double cmax = 0.0;
  for (int j = tid; j < n; j += 256) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc += fabs(D[static_cast<size_t>(i) * NP + j]);
    cmax = fmax(cmax, acc);
  }
  for (int o = 16; o; o >>= 1) cmax = fmax(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
  if (lane == 0) red_v[warp] = cmax;
  __syncthreads();
  if (tid == 0) {
    double m = red_v[0];
    for (int w = 1; w < 8; ++w) m = fmax(m, red_v[w]);
    sh_norm = m;
    sh_umin = __longlong_as_double(0x7ff0000000000000ll);
  }
  __syncthreads();

  // dot product in 4 independent partial sums (breaks the serial FMA chain)
  auto dot = [&](const double* row, const double* col, int q0, int q1) {
    double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
    int q = q0;
    for (; q + 3 < q1; q += 4) {
      p0 = fma(row[q], col[static_cast<size_t>(q) * NP], p0);
      p1 = fma(row[q + 1], col[static_cast<size_t>(q + 1) * NP], p1);
      p2 = fma(row[q + 2], col[static_cast<size_t>(q + 2) * NP], p2);
      p3 = fma(row[q + 3], col[static_cast<size_t>(q + 3) * NP], p3);
    }
    for (; q < q1; ++q) p0 = fma(row[q], col[static_cast<size_t>(q) * NP], p0);
    return (p0 + p1) + (p2 + p3);
  };
  // M[u0:u1, v0:v1] -= A[u0:u1, q0:q1] * B[q0:q1, v0:v1], register-tiled
  // 4 x 4 per thread (every loaded element feeds 4 FMAs)
  auto rank_update = [&](auto&& Mat, auto&& Aat, auto&& Bat, int u0, int u1, int v0, int v1,
                         int q0, int q1) {
    const int rt = (u1 - u0 + 3) / 4, ct = (v1 - v0 + 3) / 4;
    for (int tile = tid; tile < rt * ct; tile += 256) {
      const int r = u0 + 4 * (tile / ct), c = v0 + 4 * (tile % ct);
      double acc[4][4] = {};
      for (int q = q0; q < q1; ++q) {
        double a[4], x[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = r + i < u1 ? Aat(r + i, q) : 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = c + j < v1 ? Bat(q, c + j) : 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], x[j], acc[i][j]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (r + i < u1 && c + j < v1) Mat(r + i, c + j) -= acc[i][j];
    }
  };
  auto dref = [&](int r, int c) -> double& { return D[static_cast<size_t>(r) * NP + c]; };
  auto dval = [&](int r, int c) -> double { return D[static_cast<size_t>(r) * NP + c]; };
  constexpr int PW = 64;  // panel width of the blocked getrf

  // getrf, right-looking and blocked by 64-column panels: unblocked LU with
  // partial pivoting inside the panel (whole-row swaps, as LAPACK's laswp
  // on both sides), then U12 = L11^-1 A12 and the trailing update
  // A22 -= L21 U12 -- one pass over the trailing matrix per panel instead
  // of one per pivot.
  for (int c0 = 0; c0 < n; c0 += PW) {
    const int c1 = min(n, c0 + PW);
    for (int k = c0; k < c1; ++k) {
      // pivot: first row of max |a_ik|, i >= k (idamax)
      double bv = -1.0;
      int bi = n;
      for (int i = k + tid; i < n; i += 256) {
        const double v = fabs(D[static_cast<size_t>(i) * NP + k]);
        if (v > bv) { bv = v; bi = i; }
      }
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if (lane == 0) { red_v[warp] = bv; red_i[warp] = bi; }
      __syncthreads();
      if (tid == 0) {
        double v = red_v[0];
        int p = red_i[0];
        for (int w = 1; w < 8; ++w)
          if (red_v[w] > v || (red_v[w] == v && red_i[w] < p)) { v = red_v[w]; p = red_i[w]; }
        sh_p = p < n ? p : k;
      }
      __syncthreads();
      const int p = sh_p;
      if (p != k) {  // swap rows k, p of den (whole row) and of both right-hand sides
        for (int j = tid; j < 3 * n; j += 256) {
          double* M = j < n ? D : X[j / n - 1];
          const int c = j % n;
          const double t = M[static_cast<size_t>(k) * NP + c];
          M[static_cast<size_t>(k) * NP + c] = M[static_cast<size_t>(p) * NP + c];
          M[static_cast<size_t>(p) * NP + c] = t;
        }
        __syncthreads();
      }
      const double piv = D[static_cast<size_t>(k) * NP + k];
      if (tid == 0) sh_umin = fmin(sh_umin, fabs(piv));
      const double rcp = 1.0 / piv;
      for (int i = k + 1 + tid; i < n; i += 256) D[static_cast<size_t>(i) * NP + k] *= rcp;
      __syncthreads();
      for (int i = k + 1 + warp; i < n; i += 8) {  // rank-1 update inside the panel
        const double l = D[static_cast<size_t>(i) * NP + k];
        double* row = D + static_cast<size_t>(i) * NP;
        const double* urow = D + static_cast<size_t>(k) * NP;
        for (int j = k + 1 + lane; j < c1; j += 32) row[j] = fma(-l, urow[j], row[j]);
      }
      __syncthreads();
    }
    if (c1 < n) {
      for (int j = c1 + tid; j < n; j += 256) {  // U12 = L11^-1 A12 (unit lower)
        double* col = D + j;
        for (int i = c0 + 1; i < c1; ++i)
          col[static_cast<size_t>(i) * NP] -= dot(D + static_cast<size_t>(i) * NP, col, c0, i);
      }
      __syncthreads();
      rank_update(dref, dval, dval, c1, n, c1, n, c0, c1);  // A22 -= L21 U12
      __syncthreads();
    }
  }
  if (sh_umin <= 1e3 * 0x1p-52 * sh_norm || !(sh_umin == sh_umin)) {
    if (tid == 0) status[b] = kSingular;
    return;
  }
  // getrs, blocked by 64 rows: per block a short triangular solve down each
  // right-hand-side column (one thread per column), then the rank-64
  // update of the remaining rows as a register-tiled (4 x 4 per thread)
  // product, so every loaded L / U / X element feeds 4 FMAs instead of 1.
  constexpr int BSZ = 64;
  auto xat = [&](int r, int c) -> double& {  // column c of [X1 | X2]
    return c < n ? X[0][static_cast<size_t>(r) * NP + c] : X[1][static_cast<size_t>(r) * NP + c - n];
  };
  auto dat = [&](int r, int c) -> double { return D[static_cast<size_t>(r) * NP + c]; };
  // rows [u0, u1) of [X1 | X2] -= F[u0:u1, q0:q1] * X[q0:q1, :], F = L or U of D
  auto update = [&](int u0, int u1, int q0, int q1) {
    rank_update(xat, dval, xat, u0, u1, 0, 2 * n, q0, q1);
  };
  const int nb = (n + BSZ - 1) / BSZ;
  for (int bi = 0; bi < nb; ++bi) {  // forward: unit-lower L
    const int r0 = bi * BSZ, r1 = min(n, r0 + BSZ);
    for (int c = tid; c < 2 * n; c += 256) {
      double* col = &xat(0, c);
      for (int i = r0 + 1; i < r1; ++i)
        col[static_cast<size_t>(i) * NP] -= dot(D + static_cast<size_t>(i) * NP, col, r0, i);
    }
    __syncthreads();
    if (r1 < n) update(r1, n, r0, r1);
    __syncthreads();
  }
  for (int bi = nb - 1; bi >= 0; --bi) {  // backward: upper U
    const int r0 = bi * BSZ, r1 = min(n, r0 + BSZ);
    for (int c = tid; c < 2 * n; c += 256) {
      double* col = &xat(0, c);
      for (int i = r1 - 1; i >= r0; --i) {
        const double* urow = D + static_cast<size_t>(i) * NP;
        col[static_cast<size_t>(i) * NP] =
            (col[static_cast<size_t>(i) * NP] - dot(urow, col, i + 1, r1)) / urow[i];
      }
    }
    __syncthreads();
    if (r0 > 0) update(0, r0, r0, r1);
    __syncthreads();
  }
  __syncthreads();
  if (staged && S[b] != 0)  // the doubling launches read the solutions from the workspace
    for (int e = tid; e < static_cast<int>(slotsz); e += 256) {
      reinterpret_cast<double2*>(Dg + slotsz)[e] = reinterpret_cast<const double2*>(X[0])[e];
    }
  if (S[b] != 0) return;
  const size_t nn = static_cast<size_t>(n) * n;
  for (size_t e = tid; e < 2 * nn; e += 256) {
    const int w = static_cast<int>(e / nn);
    const size_t r = (e % nn) / n, c = (e % nn) % n;
    const double v = X[w][r * NP + c];
    void* dst = w == 0 ? cout : sout;
    if (out_f32) static_cast<float*>(dst)[b * nn + r * n + c] = static_cast<float>(v);
    else static_cast<double*>(dst)[b * nn + r * n + c] = v;
  }
}

}  // namespace tk

// ---------------------------------------------------------------------------
// Host side: chain programs (one per family and k) and the scheduler.

namespace {

using tk::Op;
using tk::OutSpec;
using tk::Term;
constexpr int ACC = tk::SRC_ACC, EYE = tk::SRC_I, OUT0 = tk::SRC_OUT0;

struct OutArg {
  int slot;
  std::vector<std::pair<int, double>> terms;
  int scale = tk::SC_NONE;
  int final = tk::FIN_NONE;
};

Op make_op(int lhs, int rhs, std::initializer_list<OutArg> outs) {
  Op o{};
  o.lhs = lhs;
  o.rhs = rhs;
  for (const OutArg& a : outs) {
    OutSpec& os = o.out[o.nout++];
    os.slot = a.slot;
    os.scale = a.scale;
    os.final = a.final;
    os.nterms = 0;
    for (auto& p : a.terms) {
      os.t[os.nterms].src = p.first;
      os.t[os.nterms].c = p.second;
      ++os.nterms;
    }
  }
  return o;
}

struct Program {
  std::vector<std::vector<Op>> steps;  // each step = 1 or 2 ops in one launch
  int cos_slot, sin_slot;
};

// Taylor family: slot 0 = A (fold: raw A, 2^-s folded into P1 / the sin
// product) or 2^-s A.  Wave family: slot 0 = y = (t')^2 A.
Program build_program(bool wave, int k, bool fold) {
  const Tables& T = host_tables();
  const double* x = T.x8;  // x[0] = x1
  const double* z8 = T.z8;
  const double(*a)[4] = T.a12;
  const double* z = T.z12;
  const int FC = tk::FIN_COS, FS = tk::FIN_SIN;
  const int sy = fold ? tk::SC_F2 : tk::SC_NONE;   // y = A A (scaled)
  const int ss = fold ? tk::SC_F : tk::SC_NONE;    // sin = A sc (scaled)
  Program P;
  auto step = [&](std::initializer_list<Op> ops) { P.steps.emplace_back(ops); };
  if (!wave) {
    const Op p1 = make_op(0, 0, {{1, {{ACC, 1.0}}, sy}});  // y
    if (k == 3) {
      step({p1});
      step({make_op(1, 1, {{2, {{EYE, 1.0}, {1, -0.5}, {ACC, 1.0 / 24.0}}, 0, FC},
                           {3, {{EYE, 1.0}, {1, -1.0 / 6.0}, {ACC, 1.0 / 120.0}}}})});
      step({make_op(0, 3, {{4, {{ACC, 1.0}}, ss, FS}})});
      P.cos_slot = 2; P.sin_slot = 4;
    } else if (k == 4) {
      step({p1});
      step({make_op(1, 1, {{2, {{ACC, 1.0}}}, {3, {{1, -1.0 / 720.0}, {ACC, 1.0 / 40320.0}}}})});
      step({make_op(2, 3, {{4, {{EYE, 1.0}, {1, -0.5}, {2, 1.0 / 24.0}, {ACC, 1.0}}, 0, FC},
                           {5, {{EYE, 1.0}, {1, -1.0 / 6.0}, {2, 1.0 / 120.0},
                                {ACC, 720.0 / 5040.0}}}})});
      step({make_op(0, 5, {{6, {{ACC, 1.0}}, ss, FS}})});
      P.cos_slot = 4; P.sin_slot = 6;
    } else if (k == 6) {
      step({p1});
      step({make_op(1, 1, {{2, {{ACC, 1.0}}}, {3, {{1, x[0]}, {ACC, x[1]}}}})});
      step({make_op(2, 3, {{4, {{ACC, 1.0}}},
                           {5, {{2, x[2]}, {ACC, 1.0}}},
                           {6, {{EYE, x[3]}, {1, x[4]}, {2, x[5]}, {ACC, x[6]}}}})});
      step({make_op(5, 6, {{7, {{EYE, 1.0}, {1, -0.5}, {2, x[7]}, {ACC, 1.0}}, 0, FC},
                           {3, {{EYE, z8[5]}, {1, z8[5]}, {2, z8[6]}, {4, z8[7]}, {OUT0, z8[8]}}},
                           {8, {{EYE, z8[0]}, {1, z8[1]}, {2, z8[2]}, {4, z8[3]}, {OUT0, z8[4]}}}})});
      step({make_op(3, 4, {{1, {{8, 1.0}, {ACC, 1.0}}}})});
      step({make_op(0, 1, {{2, {{ACC, 1.0}}, ss, FS}})});
      P.cos_slot = 7; P.sin_slot = 2;
    } else {  // k == 7
      step({p1});
      step({make_op(1, 1, {{2, {{ACC, 1.0}}}})});
      step({make_op(2, 1, {{3, {{ACC, 1.0}}},
                           {4, {{EYE, a[3][0]}, {1, a[3][1]}, {2, a[3][2]}, {ACC, a[3][3]}}}})});
      step({make_op(4, 4, {{5, {{EYE, a[2][0]}, {1, a[2][1]}, {2, a[2][2]}, {3, a[2][3]}, {ACC, 1.0}}},
                           {6, {{EYE, a[1][0]}, {1, a[1][1]}, {2, a[1][2]}, {3, a[1][3]}, {OUT0, 1.0}}}})});
      step({make_op(6, 5, {{4, {{EYE, a[0][0]}, {1, a[0][1]}, {2, a[0][2]}, {3, a[0][3]}, {ACC, 1.0}}, 0, FC},
                           {7, {{EYE, z[6]}, {1, z[7]}, {2, z[8]}, {3, z[9]}, {5, z[10]}, {OUT0, z[11]}}},
                           {8, {{EYE, z[0]}, {1, z[1]}, {2, z[2]}, {3, z[3]}, {5, z[4]}, {OUT0, z[5]}}}})});
      step({make_op(7, 4, {{1, {{8, 1.0}, {ACC, 1.0}}}})});
      step({make_op(0, 1, {{2, {{ACC, 1.0}}, ss, FS}})});
      P.cos_slot = 4; P.sin_slot = 2;
    }
  } else {
    const int TP = tk::SC_TP;
    if (k == 3) {
      step({make_op(0, 0, {{1, {{ACC, 1.0}}},
                           {2, {{0, -1.0 / 720.0}, {ACC, 1.0 / 40320.0}}},
                           {3, {{0, -1.0 / 5040.0}, {ACC, 1.0 / 362880.0}}}})});
      // q = L y2, q9 = L9 y2 (polynomials in y commute): one dual launch
      step({make_op(2, 1, {{4, {{EYE, 1.0}, {0, -0.5}, {1, 1.0 / 24.0}, {ACC, 1.0}}, 0, FC}}),
            make_op(3, 1, {{5, {{EYE, 1.0}, {0, -1.0 / 6.0}, {1, 1.0 / 120.0}, {ACC, 1.0}}, TP, FS}})});
      P.cos_slot = 4; P.sin_slot = 5;
    } else if (k == 4) {
      step({make_op(0, 0, {{1, {{ACC, 1.0}}}, {2, {{0, x[0]}, {ACC, x[1]}}}})});
      step({make_op(1, 2, {{3, {{ACC, 1.0}}},
                           {4, {{1, x[2]}, {ACC, 1.0}}},
                           {5, {{EYE, x[3]}, {0, x[4]}, {1, x[5]}, {ACC, x[6]}}}})});
      step({make_op(4, 5, {{6, {{EYE, 1.0}, {0, -0.5}, {1, x[7]}, {ACC, 1.0}}, 0, FC},
                           {2, {{EYE, z8[5]}, {0, z8[5]}, {1, z8[6]}, {3, z8[7]}, {OUT0, z8[8]}}},
                           {7, {{EYE, z8[0]}, {0, z8[1]}, {1, z8[2]}, {3, z8[3]}, {OUT0, z8[4]}}}})});
      step({make_op(2, 3, {{1, {{7, 1.0}, {ACC, 1.0}}, TP, FS}})});
      P.cos_slot = 6; P.sin_slot = 1;
    } else {  // k == 5
      step({make_op(0, 0, {{1, {{ACC, 1.0}}}})});
      step({make_op(1, 0, {{2, {{ACC, 1.0}}},
                           {3, {{EYE, a[3][0]}, {0, a[3][1]}, {1, a[3][2]}, {ACC, a[3][3]}}}})});
      step({make_op(3, 3, {{4, {{EYE, a[2][0]}, {0, a[2][1]}, {1, a[2][2]}, {2, a[2][3]}, {ACC, 1.0}}},
                           {5, {{EYE, a[1][0]}, {0, a[1][1]}, {1, a[1][2]}, {2, a[1][3]}, {OUT0, 1.0}}}})});
      step({make_op(5, 4, {{3, {{EYE, a[0][0]}, {0, a[0][1]}, {1, a[0][2]}, {2, a[0][3]}, {ACC, 1.0}}, 0, FC},
                           {6, {{EYE, z[6]}, {0, z[7]}, {1, z[8]}, {2, z[9]}, {4, z[10]}, {OUT0, z[11]}}},
                           {7, {{EYE, z[0]}, {0, z[1]}, {1, z[2]}, {2, z[3]}, {4, z[4]}, {OUT0, z[5]}}}})});
      step({make_op(6, 3, {{1, {{7, 1.0}, {ACC, 1.0}}, TP, FS}})});
      P.cos_slot = 3; P.sin_slot = 1;
    }
  }
  return P;
}

// Standalone sines (schemes.py:398-408, :433-443): special == 1 taylor_sin9
// (the exact-sine degree-4 core, sin = A sc), special == 2 wave_sin34 (the
// inexact-sine degree-4 core on y, s = t sc).  No doubling (s = 0).
Program build_special(int special, bool fold) {
  const int sy = fold ? tk::SC_F2 : tk::SC_NONE;
  const int ss = fold ? tk::SC_F : tk::SC_NONE;
  Program P;
  auto step = [&](std::initializer_list<Op> ops) { P.steps.emplace_back(ops); };
  if (special == 1) {
    step({make_op(0, 0, {{1, {{ACC, 1.0}}, sy}})});
    step({make_op(1, 1, {{2, {{ACC, 1.0}}}, {3, {{1, -1.0 / 5040.0}, {ACC, 1.0 / 362880.0}}}})});
    step({make_op(2, 3, {{4, {{EYE, 1.0}, {1, -1.0 / 6.0}, {2, 1.0 / 120.0}, {ACC, 1.0}}}})});
    step({make_op(0, 4, {{5, {{ACC, 1.0}}, ss, tk::FIN_SIN}})});
    P.cos_slot = 6; P.sin_slot = 5;
  } else if (special == 3) {
    // pade8_cos_sin (schemes.py:446-464): y..y4 with den / num_cos fused
    // into the y4 epilogue and the odd numerator's polynomial into y3's;
    // the LU solve (slots 5 | 6, 7 -> 6, 7) runs between chain and doubling
    const double* D = kPadeDen;
    const double* C = kPadeNumCos;
    const double* N = kPadeNumSin;
    step({make_op(0, 0, {{1, {{ACC, 1.0}}, sy}})});
    step({make_op(1, 1, {{2, {{ACC, 1.0}}}})});
    step({make_op(1, 2, {{3, {{ACC, 1.0}}},
                         {4, {{EYE, N[0]}, {1, N[1]}, {2, N[2]}, {ACC, N[3]}}}})});
    step({make_op(1, 3, {{5, {{EYE, D[0]}, {1, D[1]}, {2, D[2]}, {3, D[3]}, {ACC, D[4]}}},
                         {6, {{EYE, C[0]}, {1, C[1]}, {2, C[2]}, {3, C[3]}, {ACC, C[4]}}}})});
    step({make_op(0, 4, {{7, {{ACC, 1.0}}, ss}})});
    P.cos_slot = 6; P.sin_slot = 7;
  } else {
    step({make_op(0, 0, {{1, {{ACC, 1.0}}}, {2, {{0, -1.0 / 720.0}, {ACC, 1.0 / 40320.0}}}})});
    step({make_op(1, 2, {{3, {{EYE, 1.0}, {0, -1.0 / 6.0}, {1, 1.0 / 120.0},
                              {ACC, 720.0 / 5040.0}}, tk::SC_TP, tk::FIN_SIN}})});
    P.cos_slot = 4; P.sin_slot = 3;
  }
  return P;
}

// Doubling op pair: S' = 2 S C, C' = 2 C C - I, into (c1, s1); final when
// the matrix's s equals this step + 1.
std::vector<Op> doubling_ops(int c0, int s0, int c1, int s1) {
  return {make_op(s0, c0, {{s1, {{ACC, 2.0}}, tk::SC_NONE, tk::FIN_SIN}}),
          make_op(c0, c0, {{c1, {{ACC, 2.0}, {EYE, -1.0}}, tk::SC_NONE, tk::FIN_COS}})};
}

void free_pair(int c0, int s0, int* c1, int* s1) {
  int got[2], m = 0;
  for (int i = 1; i < tk::NSLOT && m < 2; ++i)  // slot 0 may alias the input
    if (i != c0 && i != s0) got[m++] = i;
  *c1 = got[0];
  *s1 = got[1];
}

}  // namespace

size_t tiled_np(int n) { return static_cast<size_t>((n + 63) / 64) * 64; }

// Product engine: 0 = FP64 DMMA (default), 1 = Ozaki-II on the int8 tensor
// cores (ozaki.cuh) for the tiled chain when NP % 256 == 0, 2 = auto: Ozaki
// from NP = 768 up, where its O(n^2 nm) passes are small enough next to the
// GEMM (batched n = 768: 1.06x the DMMA chain, n = 1024: 1.3x, n = 2048:
// 2.1x, cfg5 8192^2: 3.8x; n <= 512 is faster on DMMA, K7), 3 =
// Ozaki without the accuracy guard (experiments).  DMMA is the default
// because its error is componentwise, like the reference's fp64 GEMM
// (matcore.py:97): the Ozaki rounding is relative to row / column maxima,
// and oz_guard bounds it only norm-wise per product -- enough for
// well-scaled operands, not for graded ones whose small entries a long
// doubling recursion amplifies (K7, tests/test_gpu_guard.py).  The process default (csm_set_engine) is atomic; a thread may
// override it (csm_set_thread_engine).  Every entry point reads the engine
// ONCE (engine()) and passes that snapshot down, so a call never mixes
// engines and its workspace check matches what it runs.
static std::atomic<int> g_engine{0};
static thread_local int t_engine = -1;
void set_engine(int e) { g_engine.store(e, std::memory_order_relaxed); }
void set_thread_engine(int e) { t_engine = e; }
int engine() { return t_engine >= 0 ? t_engine : g_engine.load(std::memory_order_relaxed); }
static bool oz_applies(int NP, int eng) {
  if (NP % tk::OZ_TN != 0) return false;
  return eng == 1 || eng == 3 || (eng == 2 && NP >= 768);
}
// moduli: pairwise coprime, <= 256, largest first
static constexpr int kOzMods[tk::OZ_MAXM] = {256, 255, 253, 251, 247, 241, 239, 233,
                                            229, 227, 223, 217, 211, 199, 197, 193};
// oz_store_residues takes modulus 0's residue as the low byte of its group's
// residue: valid only while m_0 = 256 and m_0 opens group 0
static_assert(kOzMods[0] == 256, "the mod-256 shortcut of oz_store_residues needs m_0 = 256");
int oz_moduli(int out_f32) { return out_f32 ? 9 : 16; }

// CRT constants for the first nm moduli and contraction depth K.
tk::OzConst oz_const(int nm, int K) {
  typedef unsigned __int128 u128;
  tk::OzConst C{};
  C.nm = nm;
  u128 M = 1;
  double log2M = 0.0;
  for (int t = 0; t < nm; ++t) {
    M *= static_cast<u128>(kOzMods[t]);
    log2M += std::log2(static_cast<double>(kOzMods[t]));
  }
  // K 2^(2P) <= M / 4: the integer product is exact and |L'R'| < M / 4
  C.P = static_cast<int>(std::floor((log2M - 2.0 - std::log2(static_cast<double>(K))) / 2.0));
  const u128 mask = (static_cast<u128>(1) << tk::OZ_LVB) - 1;
  for (int t = 0; t < nm; ++t) {
    const int m = kOzMods[t];
    C.mod[t] = m;
    C.cdiv[t] = static_cast<uint32_t>((static_cast<uint64_t>(1) << 32) / static_cast<uint64_t>(m));
    const u128 Mt = M / static_cast<u128>(m);
    const int a = static_cast<int>(Mt % static_cast<u128>(m));
    int inv = 0;
    for (int x = 1; x < m; ++x)
      if ((a * x) % m == 1) { inv = x; break; }
    const u128 W = (Mt * static_cast<u128>(inv)) % M;
    for (int l = 0; l < tk::OZ_LV; ++l)
      C.w[t][l] = static_cast<double>(
          static_cast<uint64_t>((W >> (tk::OZ_LVB * (tk::OZ_LV - 1 - l))) & mask));
  }
  // residues go through groups of three consecutive moduli (the last one
  // shorter), each product below 2^24 (oz_store_residues; checked in
  // tests/test_ozaki_math.py)
  for (int g = 0; 3 * g < nm; ++g) {
    double G = 1.0;
    for (int t = 3 * g; t < 3 * g + 3 && t < nm; ++t) G *= kOzMods[t];
    C.gmod[g] = G;
    C.ginv[g] = 1.0 / G;
  }
  for (int l = 0; l < tk::OZ_LV; ++l)
    C.M[l] = static_cast<double>(
        static_cast<uint64_t>((M >> (tk::OZ_LVB * (tk::OZ_LV - 1 - l))) & mask));
  C.invM = 1.0 / (static_cast<double>(static_cast<uint64_t>(M >> 64)) * 18446744073709551616.0 +
                  static_cast<double>(static_cast<uint64_t>(M)));
  return C;
}

// Ozaki scratch, carved from `base` (nullptr: only measure).  nL items own
// an M-row left operand and product, nR items a right operand's maxima and
// column sums, nRp items the right operand's residue planes (a doubling
// pair shares one).  Returns the bytes used; the one function sizes and
// carves, so the two cannot disagree.
static size_t oz_carve(char* base, int64_t nL, int64_t nR, int64_t nRp, size_t M, size_t NP,
                       tk::OzArgs* out) {
  size_t off = 0;
  auto take = [&](size_t bytes) -> char* {
    off = (off + 255) & ~size_t(255);
    char* p = base ? base + off : nullptr;
    off += bytes;
    return p;
  };
  const size_t l = static_cast<size_t>(nL), r = static_cast<size_t>(nR);
  tk::OzArgs O{};
  O.mxL = reinterpret_cast<unsigned long long*>(take(l * M * 8));
  O.rsumL = reinterpret_cast<double*>(take(l * M * 8));
  O.mxR = reinterpret_cast<unsigned long long*>(take(r * NP * 8));
  O.csumR = reinterpret_cast<double*>(take(r * (NP / 64) * NP * 8));
  O.csumC = reinterpret_cast<double*>(take(l * (M / 64) * NP * 8));
  O.bad = reinterpret_cast<unsigned*>(take(std::max(l, r) * 4));
  O.flag = reinterpret_cast<unsigned*>(take(l * 4));
  O.pL = reinterpret_cast<int8_t*>(take(l * tk::OZ_MAXM * M * NP));
  O.pR = reinterpret_cast<int8_t*>(take(static_cast<size_t>(nRp) * tk::OZ_MAXM * NP * NP));
  O.res = reinterpret_cast<int8_t*>(take(l * tk::OZ_MAXM * M * NP));
  if (out) *out = O;
  return off + 256;
}
static size_t oz_item_bytes(size_t NP) { return oz_carve(nullptr, 1, 1, 1, NP, NP, nullptr); }
static int64_t oz_cap_items(int64_t batch, size_t NP) {
  const size_t budget = static_cast<size_t>(4) << 30;
  int64_t cap = static_cast<int64_t>(budget / oz_item_bytes(NP));
  cap = std::max<int64_t>(1, std::min<int64_t>(cap, 2 * batch));
  return std::min<int64_t>(cap, 65535 / tk::OZ_MAXM);
}

size_t tiled_workspace_bytes(int64_t batch, int n, int eng) {
  const size_t NP = tiled_np(n);
  size_t bytes = 0;
  bytes += static_cast<size_t>(batch) * tk::NSLOT * NP * NP * sizeof(double);  // slots
  bytes += static_cast<size_t>(batch) * sizeof(double);                        // tsc
  bytes += static_cast<size_t>(batch) * 2 * sizeof(int32_t) + 256;             // idx
  bytes += 128 * sizeof(Op) + 256;                                             // op table
  if (oz_applies(static_cast<int>(NP), eng)) {
    const int64_t cap = oz_cap_items(batch, NP);
    bytes += oz_carve(nullptr, cap, cap, cap, NP, NP, nullptr) + 256;
  }
  return bytes;
}

struct TiledWs {
  double* slots;
  double* tsc;
  int32_t* idx;
  Op* ops;
  tk::OzArgs oz;  // Ozaki scratch (when the engine runs it)
  int64_t oz_cap;
};

static TiledWs carve(void* ws, int64_t batch, int n, int eng) {
  const size_t NP = tiled_np(n);
  char* p = static_cast<char*>(ws);
  TiledWs w{};
  w.slots = reinterpret_cast<double*>(p);
  p += static_cast<size_t>(batch) * tk::NSLOT * NP * NP * sizeof(double);
  w.tsc = reinterpret_cast<double*>(p);
  p += static_cast<size_t>(batch) * sizeof(double);
  p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255));
  w.idx = reinterpret_cast<int32_t*>(p);
  p += static_cast<size_t>(batch) * 2 * sizeof(int32_t);
  p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255));
  w.ops = reinterpret_cast<Op*>(p);
  p += 128 * sizeof(Op) + 256;
  if (oz_applies(static_cast<int>(NP), eng)) {
    const int64_t cap = oz_cap_items(batch, NP);
    p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255));
    w.oz_cap = cap;
    oz_carve(p, cap, cap, cap, NP, NP, &w.oz);
  }
  return w;
}

// The persistent int8 GEMM (default) or, with CSM_OZ_GEMM=tile, the one-CTA-
// per-tile form (experiments); read once per process.
static bool persistent_layout() {
  static const bool p = [] {
    const char* e = std::getenv("CSM_OZ_GEMM");
    return !(e && std::strcmp(e, "tile") == 0);
  }();
  return p;
}

// Co-resident 2-CTA clusters of the persistent int8 GEMM (one CTA per SM
// by its shared memory), once per device.
static int oz_resident_clusters() {
  static int cached[32] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  dev = dev < 32 ? dev : 31;
  if (cached[dev] > 0) return cached[dev];
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.blockDim = dim3(tk::OZ_PTHREADS);
  cfg.dynamicSmemBytes = tk::OZ_SMEM;
  cfg.gridDim = dim3(2 * 64);
  int active = 0;
  if (cudaOccupancyMaxActiveClusters(&active, tk::oz_gemm_p<tk::OZ_NSTAGE>, &cfg) != cudaSuccess ||
      active <= 0)
    active = 64;
  cached[dev] = active;
  return active;
}

// Column tiles per raster group of the persistent int8 GEMM (oz_gemm_p's
// decode): 8 from NP = 8192 up (nx >= 32), where the 74 co-resident cluster
// pairs then cover about 9 x 8 tiles -- 18 MiB of left and 16 MiB of right
// panels live instead of the whole 64 MiB right plane -- else the whole row.
// Measured on cfg5 (profiles/r2/s12/): GEMM 160.9 ms (row walk), 164.7 (16),
// 154.4 (8), 167.2 (4) per step.  CSM_OZ_GX overrides it (a divisor of nx).
static int oz_group_x(int nx) {
  static const int env = [] {
    const char* e = std::getenv("CSM_OZ_GX");
    return e ? std::atoi(e) : 0;
  }();
  if (env > 0 && env <= nx && nx % env == 0) return env;
  return (nx >= 32 && nx % 8 == 0) ? 8 : nx;
}

// One tiled launch (all items of plan A) through the Ozaki engine, in
// chunks of at most cap items: maxima, residues, nm int8 GEMMs, CRT +
// epilogue, then the accuracy guard (oz_guard) and the DMMA rerun of the
// items it flags (the CTAs of unflagged items leave at once).  An op's
// outputs never alias its operands or epilogue sources (build_program; the
// tile-parallel kernels rely on that too), so the rerun rewrites exactly
// what the CRT epilogue wrote.  Eight launches per chunk.
static cudaError_t run_oz_launch(const tk::LaunchArgs& A, const tk::OzArgs& scratch, int64_t cap,
                                 const tk::OzConst& C, cudaStream_t stream, int64_t* launches,
                                 bool guard) {
  const int NP = A.NP, M = A.M;
  const unsigned tiles = static_cast<unsigned>((M / tk::BM) * (NP / tk::BN));
  for (int done = 0; done < A.total; done += static_cast<int>(cap)) {
    const int cnt = static_cast<int>(std::min<int64_t>(cap, A.total - done));
    tk::OzArgs O = scratch;
    O.item0 = done;
    O.nitems = cnt;
    cudaError_t e = cudaMemsetAsync(O.mxR, 0, static_cast<size_t>(cnt) * NP * 8, stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(O.bad, 0, static_cast<size_t>(cnt) * 4, stream);
    if (e != cudaSuccess) return e;
    tk::oz_rowmax<<<dim3(M / 8, cnt), 256, 0, stream>>>(A, O);
    tk::oz_colmax<<<dim3(NP / 256, NP / 64, cnt), 256, 0, stream>>>(A, O);
    const dim3 gconv_r(M / 128, NP / 16, cnt), gconv_c(NP / 128, NP / 16, cnt);
    const dim3 ggemm(NP / tk::OZ_TN, M / tk::OZ_TM, cnt * C.nm), gcrt(tiles, cnt);
    static const int force_st = [] {  // CSM_OZ_STAGES=2|4 overrides (experiments)
      const char* e = std::getenv("CSM_OZ_STAGES");
      return e ? std::atoi(e) : 0;
    }();
    // NP <= 1024: two 2-stage CTAs per SM, one's epilogue overlapping the
    // other's MMAs (n = 1024: -25% GEMM time); larger: one 4-stage CTA per SM
    const bool small = force_st ? force_st == 2 : NP <= 1024;
    const size_t gsm = (small ? tk::OZ_NSTAGE_SMALL : tk::OZ_NSTAGE) * tk::OZ_STAGE;
    if (C.nm == 16) {
      tk::oz_conv_rows<16><<<gconv_r, 128, 0, stream>>>(A, O, C);
      tk::oz_conv_cols<16><<<gconv_c, 128, 0, stream>>>(A, O, C);
    } else {
      tk::oz_conv_rows<9><<<gconv_r, 128, 0, stream>>>(A, O, C);
      tk::oz_conv_cols<9><<<gconv_c, 128, 0, stream>>>(A, O, C);
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;  // pairs of M tiles share B
    attr[0].val.clusterDim.x = persistent_layout() ? 2 : 1;
    attr[0].val.clusterDim.y = persistent_layout() ? 1 : 2;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = ggemm;
    cfg.blockDim = dim3(tk::OZ_THREADS);
    cfg.dynamicSmemBytes = gsm;
    cfg.stream = stream;
    prof_begin(stream, 2);  // csm_profile_enable(2): the int8 GEMM alone
    if (persistent_layout()) {
      const int pair_tiles = (NP / tk::OZ_TN) * (M / (2 * tk::OZ_TM)) * cnt * C.nm;
      int clusters = oz_resident_clusters();
      if (clusters > pair_tiles) clusters = pair_tiles;
      cfg.gridDim = dim3(2 * clusters);
      cfg.blockDim = dim3(tk::OZ_PTHREADS);
      cfg.dynamicSmemBytes = tk::OZ_SMEM;
      e = cudaLaunchKernelEx(&cfg, tk::oz_gemm_p<tk::OZ_NSTAGE>, A, O, C, pair_tiles,
                             oz_group_x(NP / tk::OZ_TN));
    } else {
      e = small ? cudaLaunchKernelEx(&cfg, tk::oz_gemm<tk::OZ_NSTAGE_SMALL>, A, O, C)
                : cudaLaunchKernelEx(&cfg, tk::oz_gemm<tk::OZ_NSTAGE>, A, O, C);
    }
    prof_end(stream, 2);
    if (e != cudaSuccess) return e;
    if (C.nm == 16)
      tk::oz_crt_epi<16><<<gcrt, tk::THREADS, tk::OZ_CRT_SMEM, stream>>>(A, O, C);
    else
      tk::oz_crt_epi<9><<<gcrt, tk::THREADS, tk::OZ_CRT_SMEM, stream>>>(A, O, C);
    if (guard) {
      tk::oz_guard<<<cnt, 256, 0, stream>>>(A, O, C);
      tk::LaunchArgs R = A;  // DMMA rerun of the flagged items only
      R.item_base = done;
      R.only = O.flag;
      R.only_base = done;
      tk::launch_gemm(dim3(tiles, static_cast<unsigned>(cnt), 1), R, stream);
      *launches += 2;
    }
    *launches += 6;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// Run the tiled pipeline for a batch whose (k, s, status) are on the device.
// Synchronises the stream once to read (k, s, status) back for scheduling.
cudaError_t run_tiled(int dtype, bool wave, const void* a, const double* t, void* c_out,
                      void* s_out, int64_t batch, int n, const int32_t* dK,
                      const int32_t* dS, const int32_t* dStatus, void* ws,
                      cudaStream_t stream, int64_t* launches, int special, int eng) {
  cudaError_t e;
  const int NP = static_cast<int>(tiled_np(n));
  const size_t mat_stride = static_cast<size_t>(tk::NSLOT) * NP * NP;
  TiledWs w = carve(ws, batch, n, eng);
  std::vector<int32_t> hk(batch), hs(batch), hst(batch);
  e = cudaMemcpyAsync(hk.data(), dK, batch * 4, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hs.data(), dS, batch * 4, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hst.data(), dStatus, batch * 4, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return e;

  // slot 0 aliases the caller's input when it already is float64 NP x NP
  const bool fold = !wave && dtype == 0 && n == NP &&
                    reinterpret_cast<uintptr_t>(a) % 16 == 0;
  const int out_f32 = dtype == 1 ? 1 : 0;
  bool any_bad = false;
  for (int64_t b = 0; b < batch; ++b) any_bad |= hst[b] != 0;

  // prepare: wave t' (always), scaled input copy (unless aliased)
  if (wave || !fold) {
    const size_t per = static_cast<size_t>(NP) * NP;
    dim3 grid(static_cast<unsigned>(std::min<size_t>((per + 255) / 256, 64)),
              static_cast<unsigned>(batch));
    if (dtype == 0)
      tk::prepare_kernel<double><<<grid, 256, 0, stream>>>(
          static_cast<const double*>(a), w.slots, n, NP, mat_stride, dS, dStatus,
          wave ? t : nullptr, w.tsc, 1);
    else
      tk::prepare_kernel<float><<<grid, 256, 0, stream>>>(
          static_cast<const float*>(a), w.slots, n, NP, mat_stride, dS, dStatus,
          wave ? t : nullptr, w.tsc, 1);
    ++*launches;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }

  // group by k, each group sorted by s descending (doubling = prefixes)
  const int ks_taylor[4] = {3, 4, 6, 7}, ks_wave[3] = {3, 4, 5}, ks_pade[1] = {5};
  const bool pade = special == 3;
  const int* ks = pade ? ks_pade : (wave ? ks_wave : ks_taylor);
  const int nks = pade ? 1 : (wave ? 3 : 4);
  std::vector<int32_t> order;
  order.reserve(batch);
  struct Group {
    int k;
    size_t off, cnt;
    int max_s;
    Program prog;
    int c1, s1;
    size_t dbl_op[2];
  };
  std::vector<Group> groups;
  for (int gi = 0; gi < nks; ++gi) {
    std::vector<std::pair<int, int32_t>> mem;
    for (int64_t b = 0; b < batch; ++b)
      if (hst[b] == 0 && hk[b] == ks[gi]) mem.emplace_back(hs[b], static_cast<int32_t>(b));
    if (mem.empty()) continue;
    std::stable_sort(mem.begin(), mem.end(),
                     [](const std::pair<int, int32_t>& x, const std::pair<int, int32_t>& y) {
                       return x.first > y.first;
                     });
    Group G;
    G.k = ks[gi];
    G.off = order.size();
    G.cnt = mem.size();
    G.max_s = mem.front().first;
    for (auto& m : mem) order.push_back(m.second);
    G.prog = special ? build_special(special, fold) : build_program(wave, G.k, fold);
    free_pair(G.prog.cos_slot, G.prog.sin_slot, &G.c1, &G.s1);
    groups.push_back(std::move(G));
  }

  if (!order.empty()) {
    // op table: per group, its program ops then its two doubling op pairs
    struct LaunchPlan {
      std::vector<tk::Seg> seg;
      int total;
      int dbl_step;
    };
    std::vector<Op> table;
    std::vector<LaunchPlan> plans;
    std::vector<std::vector<size_t>> prog_off(groups.size());
    for (size_t gi = 0; gi < groups.size(); ++gi) {
      Group& G = groups[gi];
      for (auto& stp : G.prog.steps) {
        prog_off[gi].push_back(table.size());
        for (auto& op : stp) table.push_back(op);
      }
      G.dbl_op[0] = table.size();
      for (auto& op : doubling_ops(G.prog.cos_slot, G.prog.sin_slot, G.c1, G.s1)) table.push_back(op);
      G.dbl_op[1] = table.size();
      for (auto& op : doubling_ops(G.c1, G.s1, G.prog.cos_slot, G.prog.sin_slot)) table.push_back(op);
    }
    if (table.size() > 128) return cudaErrorInvalidValue;
    // chain step j of every group in one launch
    size_t max_steps = 0;
    for (auto& G : groups) max_steps = std::max(max_steps, G.prog.steps.size());
    for (size_t j = 0; j < max_steps; ++j) {
      LaunchPlan L{{}, 0, -1};
      for (size_t gi = 0; gi < groups.size(); ++gi) {
        const Group& G = groups[gi];
        if (j >= G.prog.steps.size()) continue;
        for (size_t o = 0; o < G.prog.steps[j].size(); ++o) {
          L.seg.push_back({static_cast<int32_t>(prog_off[gi][j] + o),
                           static_cast<int32_t>(G.off), L.total});
          L.total += static_cast<int>(G.cnt);
        }
      }
      plans.push_back(L);
    }
    // doubling step i of every group in one launch
    int max_s = 0;
    for (auto& G : groups) max_s = std::max(max_s, G.max_s);
    for (int i = 0; i < max_s; ++i) {
      LaunchPlan L{{}, 0, i};
      for (const Group& G : groups) {
        int cnt = 0;
        for (size_t j = 0; j < G.cnt; ++j)
          if (hs[order[G.off + j]] > i) ++cnt;
        if (!cnt) continue;
        for (int o = 0; o < 2; ++o) {
          L.seg.push_back({static_cast<int32_t>(G.dbl_op[i & 1] + o),
                           static_cast<int32_t>(G.off), L.total});
          L.total += cnt;
        }
      }
      plans.push_back(L);
    }
    for (auto& L : plans)
      if (L.seg.size() > static_cast<size_t>(tk::MAXSEG)) return cudaErrorInvalidValue;

    e = cudaMemcpyAsync(w.idx, order.data(), order.size() * 4, cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(w.ops, table.data(), table.size() * sizeof(Op), cudaMemcpyHostToDevice,
                          stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);  // host vectors die here
    if (e != cudaSuccess) return e;

    if ((e = tk::ensure_smem_attr()) != cudaSuccess) return e;
    const unsigned tiles = static_cast<unsigned>((NP / tk::BM) * (NP / tk::BN));
    tk::LaunchArgs A{};
    A.ws = w.slots;
    A.in0 = fold ? static_cast<const double*>(a) : nullptr;
    A.idx = w.idx;
    A.ops = w.ops;
    A.tsc = wave ? w.tsc : nullptr;
    A.S = dS;
    A.cout = c_out;
    A.sout = s_out;
    A.mat_stride = mat_stride;
    A.NP = NP;
    A.n = n;
    A.out_f32 = out_f32;
    A.M = NP;
    A.row0 = 0;
    A.rhs_full = nullptr;
    A.rhs_parts = nullptr;
    tk::set_tma(A, static_cast<size_t>(batch) * (mat_stride / NP),
                fold ? static_cast<size_t>(batch) * NP : 0);
    const bool use_oz = oz_applies(NP, eng);
    const tk::OzConst ozc = use_oz ? oz_const(oz_moduli(out_f32), NP) : tk::OzConst{};
    size_t lu_smem = 0;
    if (pade && NP == 64) {  // den + both right-hand sides staged in shared memory
      lu_smem = 3 * static_cast<size_t>(NP) * NP * sizeof(double);
      e = cudaFuncSetAttribute(tk::pade_lu_solve_kernel,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(lu_smem));
      if (e != cudaSuccess) return e;
    }
    prof_begin(stream);
    for (size_t pi = 0; pi < plans.size(); ++pi) {
      const LaunchPlan& L = plans[pi];
      if (pade && pi == max_steps) {  // chain done: factor and solve before doubling
        for (const Group& G : groups) {
          tk::pade_lu_solve_kernel<<<static_cast<unsigned>(G.cnt), 256, lu_smem, stream>>>(
              w.slots, mat_stride, NP, n, w.idx + G.off, dS, const_cast<int32_t*>(dStatus),
              c_out, s_out, out_f32);
          ++*launches;
          if ((e = cudaGetLastError()) != cudaSuccess) return e;
        }
      }
      A.dbl_step = L.dbl_step;
      A.nseg = static_cast<int>(L.seg.size());
      for (size_t i = 0; i < L.seg.size(); ++i) A.seg[i] = L.seg[i];
      A.total = L.total;
      if (use_oz) {
        if ((e = run_oz_launch(A, w.oz, w.oz_cap, ozc, stream, launches, eng != 3)) != cudaSuccess)
          return e;
        continue;
      }
      for (int done = 0; done < L.total; done += 65535) {
        A.item_base = done;
        const int cnt = std::min(65535, L.total - done);
        dim3 grid(tiles, static_cast<unsigned>(cnt), 1);
        tk::launch_gemm(grid, A, stream);
        ++*launches;
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
      }
    }
    if (pade && plans.size() == max_steps) {  // no doubling at all
      for (const Group& G : groups) {
        tk::pade_lu_solve_kernel<<<static_cast<unsigned>(G.cnt), 256, lu_smem, stream>>>(
            w.slots, mat_stride, NP, n, w.idx + G.off, dS, const_cast<int32_t*>(dStatus), c_out,
            s_out, out_f32);
        ++*launches;
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
      }
    }
    prof_end(stream);
  }

  if (any_bad || pade) {  // Pade: the LU may have flagged singular denominators
    const size_t nn = static_cast<size_t>(n) * n;
    dim3 grid(static_cast<unsigned>(std::min<size_t>((nn + 255) / 256, 64)),
              static_cast<unsigned>(batch));
    if (dtype == 1)
      tk::nan_fill_kernel<float><<<grid, 256, 0, stream>>>(
          static_cast<float*>(c_out), static_cast<float*>(s_out), n, dStatus);
    else
      tk::nan_fill_kernel<double><<<grid, 256, 0, stream>>>(
          static_cast<double*>(c_out), static_cast<double*>(s_out), n, dStatus);
    ++*launches;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// ---------------------------------------------------------------------------
// Block-row (slab) primitives for the distributed chain (python driver
// paper_2010_00465_b200/distchain.py does the all-gathers).

size_t op_bytes() { return sizeof(Op); }

// Chain program of (family, k) as a flat op list; returns the step count.
int chain_program(bool wave, int k, bool fold, void* ops_out, int max_ops, int32_t* step_nops,
                  int max_steps, int32_t* cos_slot, int32_t* sin_slot) {
  Program P = build_program(wave, k, fold);
  if (static_cast<int>(P.steps.size()) > max_steps) return -1;
  int nops = 0;
  for (auto& st : P.steps) nops += static_cast<int>(st.size());
  if (nops > max_ops) return -1;
  Op* out = static_cast<Op*>(ops_out);
  int o = 0;
  for (size_t i = 0; i < P.steps.size(); ++i) {
    step_nops[i] = static_cast<int32_t>(P.steps[i].size());
    for (auto& op : P.steps[i]) out[o++] = op;
  }
  *cos_slot = P.cos_slot;
  *sin_slot = P.sin_slot;
  return static_cast<int>(P.steps.size());
}

void doubling_program(int c0, int s0, int c1, int s1, void* ops_out) {
  auto v = doubling_ops(c0, s0, c1, s1);
  Op* out = static_cast<Op*>(ops_out);
  out[0] = v[0];
  out[1] = v[1];
}

constexpr int kMaxParts = 64;
size_t slab_scratch_bytes() { return 2 * sizeof(Op) + 64 + kMaxParts * sizeof(double*); }

// Extra slab scratch the Ozaki engine needs for an M x NP slab (0 when the
// DMMA engine runs it).
static bool oz_slab_applies(int M, int NP, int eng) {
  return oz_applies(NP, eng) && M % (2 * tk::OZ_TM) == 0;
}
// Sized for csm_slab_op_pair: two left operands and products, one right
// operand's residue planes (the pair shares it).
size_t slab_engine_bytes(int M, int NP, int eng) {
  if (!oz_slab_applies(M, NP, eng)) return 0;
  return oz_carve(nullptr, 2, 2, 1, static_cast<size_t>(M), static_cast<size_t>(NP), nullptr) + 256;
}

// Run one Op on a block-row slab: out rows = L_rows * rhs_full (+ epilogue).
// scratch: device buffer of slab_scratch_bytes() (op descriptor, s, t').
// Run one op (nops = 1), or the doubling step's two ops sharing the
// right operand (nops = 2: one launch; the Ozaki engine converts it once),
// on a block-row slab.
cudaError_t slab_op(const void* const* op_host, int nops, double* slab, int M, int NP, int row0,
                    const double* rhs_full, const double* in0, int s, double tp, int dbl_step,
                    void* cout, void* sout, int out_f32, void* scratch, cudaStream_t stream,
                    int64_t* launches, const double* const* parts_host, int nparts, int eng) {
  if (M % tk::BM != 0 || NP % tk::BN != 0) return cudaErrorInvalidValue;
  if (nparts < 0 || nparts > kMaxParts || (nparts > 0 && nparts * M != NP))
    return cudaErrorInvalidValue;
  if (nops < 1 || nops > 2 || (nops == 2 && dbl_step < 0)) return cudaErrorInvalidValue;
  struct alignas(16) Staged {
    Op op[2];
    int32_t idx, s, pad0, pad1;
    double tp;
    const double* parts[kMaxParts];
  };
  static_assert(sizeof(Staged) <= 2 * sizeof(Op) + 64 + kMaxParts * sizeof(double*),
                "scratch layout");
  Staged h{};
  for (int i = 0; i < nops; ++i) std::memcpy(&h.op[i], op_host[i], sizeof(Op));
  h.idx = 0;
  h.s = s;
  h.tp = tp;
  for (int i = 0; i < nparts; ++i) h.parts[i] = parts_host[i];
  cudaError_t e = cudaMemcpyAsync(scratch, &h, sizeof(Staged), cudaMemcpyHostToDevice, stream);
  if (e != cudaSuccess) return e;
  e = cudaStreamSynchronize(stream);  // h lives on this stack frame
  if (e != cudaSuccess) return e;
  if ((e = tk::ensure_smem_attr()) != cudaSuccess) return e;
  Staged* d = static_cast<Staged*>(scratch);
  tk::LaunchArgs A{};
  A.ws = slab;
  A.in0 = in0;
  A.idx = &d->idx;
  A.ops = d->op;
  A.tsc = &d->tp;
  A.S = &d->s;
  A.cout = cout;
  A.sout = sout;
  A.mat_stride = 0;
  A.NP = NP;
  A.n = NP;
  A.out_f32 = out_f32;
  A.dbl_step = dbl_step;
  A.nseg = nops;
  A.total = nops;
  A.item_base = 0;
  for (int i = 0; i < nops; ++i) A.seg[i] = {i, 0, i};  // op i on matrix idx[0] = 0
  A.rhs_full = nparts > 0 ? nullptr : rhs_full;
  A.rhs_parts = nparts > 0 ? d->parts : nullptr;
  A.M = M;
  A.row0 = row0;
  tk::set_tma(A, static_cast<size_t>(tk::NSLOT) * M, static_cast<size_t>(M));
  if (nparts == 0 && oz_slab_applies(M, NP, eng)) {  // Ozaki engine (gathered right operand)
    char* p = reinterpret_cast<char*>(
        (reinterpret_cast<uintptr_t>(scratch) + slab_scratch_bytes() + 255) & ~uintptr_t(255));
    tk::OzArgs O{};  // two items' L-side scratch; the pair's right operand once
    oz_carve(p, 2, 2, 1, static_cast<size_t>(M), static_cast<size_t>(NP), &O);
    return run_oz_launch(A, O, nops, oz_const(oz_moduli(out_f32), NP), stream, launches, eng != 3);
  }
  dim3 grid(static_cast<unsigned>((M / tk::BM) * (NP / tk::BN)), static_cast<unsigned>(nops), 1);
  tk::launch_gemm(grid, A, stream);
  ++*launches;
  return cudaGetLastError();
}

}  // namespace csm
