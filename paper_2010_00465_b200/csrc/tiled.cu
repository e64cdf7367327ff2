// tiled.cu -- K2/K3/K4: the chain for n > 64 as a sequence of batched,
// tiled FP64 DMMA GEMMs whose epilogues carry every linear combination of
// the scheme (and the doubling update), so no elementwise pass ever runs
// on its own.
//
// Layout in HBM: each matrix owns NSLOT slots of NP x NP float64, NP = n
// rounded up to 64, row-major, zero-padded (block-diagonal padding is exact,
// see fused64.cu).  Slot 0 receives the scaled input (2^-s A, or (t')^2 A for
// the wave family) from prepare_kernel; the chain program for scheme k is a
// short list of Ops (host side, build_program); finalize_kernel copies the
// final cos/sin slots out in the caller's dtype.
//
// GEMM: CTA tile 64x64, 4 warps of 32x32 (4x4 DMMA m8n8k4 tiles), K step
// 32 through a 3-stage cp.async pipeline; padded smem rows (36 / 68
// doubles) make both fragment loads bank-conflict free.  Grid = tiles x
// matrices-of-this-op (an index list) x ops-in-this-launch (1 or 2: the
// doubling step and the wave k=3 sine are dual launches).
//
// Reference mapping: schemes.py:264-361 (chains), :376-395 / :411-430
// (trig / wave use), driver.py:91-98 (doubling), matcore.py:107-121
// (linear combinations, here fused into epilogues).
#include <algorithm>
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

// Term sources
constexpr int SRC_ACC = -1, SRC_I = -2, SRC_OUT0 = -3;  // OUTj = -3 - j

struct Term {
  int32_t src;
  int32_t pad;
  double c;
};
struct OutSpec {
  int32_t slot, nterms, tscale, pad;
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

// One 64x64 output tile of one matrix: acc = L R over the full n-deep
// contraction (3-stage cp.async pipeline, 4 warps of 32x32 = 4x4 DMMA
// tiles), then the scheme's linear combinations: the accumulator tile is
// staged in shared memory and every output element is formed by a compact
// term loop with row-contiguous (coalesced) global reads and writes.
__global__ void __launch_bounds__(THREADS, 4)
gemm_epi_kernel(double* __restrict__ ws, int NP, size_t mat_stride,
                const int32_t* __restrict__ idx, const Op* __restrict__ ops,
                const double* __restrict__ tsc) {
  extern __shared__ __align__(16) double sm[];
  __shared__ Op op;
  double* As = sm;
  double* Bs = sm + STAGES * A_STAGE;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < static_cast<int>(sizeof(Op) / 4); i += THREADS)
    reinterpret_cast<int*>(&op)[i] = reinterpret_cast<const int*>(ops + blockIdx.z)[i];
  const int b = idx[blockIdx.y];
  const int tiles_n = NP / BN;
  const int tm = blockIdx.x / tiles_n, tn = blockIdx.x - tm * tiles_n;
  double* base = ws + static_cast<size_t>(b) * mat_stride;
  const size_t slotsz = static_cast<size_t>(NP) * NP;
  __syncthreads();
  const double* L = base + op.lhs * slotsz + static_cast<size_t>(tm) * BM * NP;
  const double* R = base + op.rhs * slotsz + static_cast<size_t>(tn) * BN;

  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;

  auto load_stage = [&](int stage, int k0) {
    double* as = As + stage * A_STAGE;
    double* bs = Bs + stage * B_STAGE;
#pragma unroll
    for (int i = 0; i < (BM * BK / 2) / THREADS; ++i) {
      const int p = tid + i * THREADS;
      const int r = p / (BK / 2), c = (p - r * (BK / 2)) * 2;
      cp16(as + r * LDA + c, L + static_cast<size_t>(r) * NP + k0 + c);
    }
#pragma unroll
    for (int i = 0; i < (BK * BN / 2) / THREADS; ++i) {
      const int p = tid + i * THREADS;
      const int r = p / (BN / 2), c = (p - r * (BN / 2)) * 2;
      cp16(bs + r * LDB + c, R + static_cast<size_t>(k0 + r) * NP + c);
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = NP / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, s * BK);
    commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    wait_group<STAGES - 2>();
    __syncthreads();
    {
      const int nxt = kt + STAGES - 1;
      if (nxt < nk) load_stage(nxt % STAGES, nxt * BK);
      commit();
    }
    const double* as = As + (kt % STAGES) * A_STAGE;
    const double* bs = Bs + (kt % STAGES) * B_STAGE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[4], bf[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = as[(wm + mi * 8 + g) * LDA + kk + t];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) bf[ni] = bs[(kk + t) * LDB + wn + ni * 8 + g];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi], bf[ni]);
    }
  }
  wait_group<0>();
  __syncthreads();  // pipeline buffers are free: stage the accumulator tile

  double* E = sm;  // [BM][LDE]
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
      *reinterpret_cast<double2*>(E + (wm + mi * 8 + g) * LDE + wn + ni * 8 + 2 * t) =
          make_double2(acc[mi][ni][0], acc[mi][ni][1]);
  __syncthreads();

  const double ts = tsc ? tsc[b] : 1.0;
  const int nout = op.nout;
  const int r0 = tm * BM, c0 = tn * BN;
#pragma unroll 2
  for (int p = tid; p < BM * BN / 2; p += THREADS) {
    const int rr = p >> 5, cc = (p & 31) * 2;  // 32 pairs per tile row
    const int r = r0 + rr, c = c0 + cc;
    const size_t off = static_cast<size_t>(r) * NP + c;
    const double2 av = *reinterpret_cast<const double2*>(E + rr * LDE + cc);
    const double i0 = (r == c) ? 1.0 : 0.0, i1 = (r == c + 1) ? 1.0 : 0.0;
    double o0[2] = {0.0, 0.0}, o1[2] = {0.0, 0.0};  // outputs 0 and 1 of this pair
    for (int q = 0; q < nout; ++q) {
      const OutSpec& os = op.out[q];
      double v0 = 0.0, v1 = 0.0;
      for (int tt = 0; tt < os.nterms; ++tt) {
        const int src = os.t[tt].src;
        const double cf = os.t[tt].c;
        double x0, x1;
        if (src >= 0) {
          const double2 v = *reinterpret_cast<const double2*>(base + src * slotsz + off);
          x0 = v.x; x1 = v.y;
        } else if (src == SRC_ACC) {
          x0 = av.x; x1 = av.y;
        } else if (src == SRC_I) {
          x0 = i0; x1 = i1;
        } else if (src == SRC_OUT0) {
          x0 = o0[0]; x1 = o0[1];
        } else {
          x0 = o1[0]; x1 = o1[1];
        }
        v0 = fma(cf, x0, v0);
        v1 = fma(cf, x1, v1);
      }
      if (os.tscale) { v0 *= ts; v1 *= ts; }
      if (q == 0) { o0[0] = v0; o0[1] = v1; }
      if (q == 1) { o1[0] = v0; o1[1] = v1; }
      *reinterpret_cast<double2*>(base + os.slot * slotsz + off) = make_double2(v0, v1);
    }
  }
}

// slot0 <- f * A (zero padded).  Taylor: f = 2^-s; wave: t' = t/2^s,
// f = t' * t', and tsc[b] = t'.
template <typename TIn>
__global__ void prepare_kernel(const TIn* __restrict__ A, double* __restrict__ ws,
                               int n, int NP, size_t mat_stride, const int32_t* __restrict__ S,
                               const int32_t* __restrict__ status, const double* __restrict__ T,
                               double* __restrict__ tsc) {
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

// out[b] <- slot (cos/sin) chosen by (k, s parity); NaN for failed matrices.
struct FinalSlots {
  int8_t cos_slot[8][2];  // [k][s & 1]
  int8_t sin_slot[8][2];
};

template <typename TOut>
__global__ void finalize_kernel(const double* __restrict__ ws, TOut* __restrict__ Cout,
                                TOut* __restrict__ Sout, int n, int NP, size_t mat_stride,
                                const int32_t* __restrict__ K, const int32_t* __restrict__ S,
                                const int32_t* __restrict__ status, FinalSlots fs) {
  const int b = blockIdx.y;
  const size_t nn = static_cast<size_t>(n) * n;
  TOut* cd = Cout + b * nn;
  TOut* sd = Sout + b * nn;
  const bool ok = status[b] == 0;
  const double* cs = nullptr;
  const double* ss = nullptr;
  if (ok) {
    const int k = K[b], par = S[b] & 1;
    const double* base = ws + static_cast<size_t>(b) * mat_stride;
    cs = base + static_cast<size_t>(fs.cos_slot[k][par]) * NP * NP;
    ss = base + static_cast<size_t>(fs.sin_slot[k][par]) * NP * NP;
  }
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  for (size_t p = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < nn;
       p += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(p / n), c = static_cast<int>(p - static_cast<size_t>(r) * n);
    const size_t q = static_cast<size_t>(r) * NP + c;
    cd[p] = static_cast<TOut>(ok ? cs[q] : qnan);
    sd[p] = static_cast<TOut>(ok ? ss[q] : qnan);
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

struct ProgBuilder {
  std::vector<Op> ops;
  Op& add(int lhs, int rhs) {
    Op o{};
    o.lhs = lhs;
    o.rhs = rhs;
    ops.push_back(o);
    return ops.back();
  }
  static void out(Op& op, int slot, std::initializer_list<std::pair<int, double>> terms,
                  bool tscale = false) {
    OutSpec& os = op.out[op.nout++];
    os.slot = slot;
    os.tscale = tscale ? 1 : 0;
    os.nterms = 0;
    for (auto& p : terms) {
      os.t[os.nterms].src = p.first;
      os.t[os.nterms].c = p.second;
      ++os.nterms;
    }
  }
};

struct Program {
  std::vector<std::vector<Op>> steps;  // each step = 1 or 2 ops in one launch
  int cos_slot, sin_slot;
};

// Taylor family: slot 0 = 2^-s A.  Wave family: slot 0 = y = (t')^2 A.
Program build_program(bool wave, int k) {
  const Tables& T = host_tables();
  const double* x = T.x8;  // x[0] = x1
  const double* z8 = T.z8;
  const double(*a)[4] = T.a12;
  const double* z = T.z12;
  Program P;
  ProgBuilder B;
  auto step = [&](std::initializer_list<Op> ops) { P.steps.emplace_back(ops); };
  auto mk = [](int l, int r) { Op o{}; o.lhs = l; o.rhs = r; return o; };
  auto O = [](Op& op, int slot, std::initializer_list<std::pair<int, double>> terms,
              bool tscale = false) { ProgBuilder::out(op, slot, terms, tscale); };
  (void)B;
  if (!wave) {
    Op p1 = mk(0, 0);
    O(p1, 1, {{ACC, 1.0}});  // y
    if (k == 3) {
      Op p2 = mk(1, 1);
      O(p2, 2, {{EYE, 1.0}, {1, -0.5}, {ACC, 1.0 / 24.0}});
      O(p2, 3, {{EYE, 1.0}, {1, -1.0 / 6.0}, {ACC, 1.0 / 120.0}});
      Op p3 = mk(0, 3);
      O(p3, 4, {{ACC, 1.0}});
      step({p1}); step({p2}); step({p3});
      P.cos_slot = 2; P.sin_slot = 4;
    } else if (k == 4) {
      Op p2 = mk(1, 1);
      O(p2, 2, {{ACC, 1.0}});
      O(p2, 3, {{1, -1.0 / 720.0}, {ACC, 1.0 / 40320.0}});
      Op p3 = mk(2, 3);
      O(p3, 4, {{EYE, 1.0}, {1, -0.5}, {2, 1.0 / 24.0}, {ACC, 1.0}});
      O(p3, 5, {{EYE, 1.0}, {1, -1.0 / 6.0}, {2, 1.0 / 120.0}, {ACC, 720.0 / 5040.0}});
      Op p4 = mk(0, 5);
      O(p4, 6, {{ACC, 1.0}});
      step({p1}); step({p2}); step({p3}); step({p4});
      P.cos_slot = 4; P.sin_slot = 6;
    } else if (k == 6) {
      Op p2 = mk(1, 1);
      O(p2, 2, {{ACC, 1.0}});
      O(p2, 3, {{1, x[0]}, {ACC, x[1]}});
      Op p3 = mk(2, 3);
      O(p3, 4, {{ACC, 1.0}});
      O(p3, 5, {{2, x[2]}, {ACC, 1.0}});
      O(p3, 6, {{EYE, x[3]}, {1, x[4]}, {2, x[5]}, {ACC, x[6]}});
      Op p4 = mk(5, 6);
      O(p4, 7, {{EYE, 1.0}, {1, -0.5}, {2, x[7]}, {ACC, 1.0}});
      O(p4, 3, {{EYE, z8[5]}, {1, z8[5]}, {2, z8[6]}, {4, z8[7]}, {OUT0, z8[8]}});
      O(p4, 8, {{EYE, z8[0]}, {1, z8[1]}, {2, z8[2]}, {4, z8[3]}, {OUT0, z8[4]}});
      Op p5 = mk(3, 4);
      O(p5, 1, {{8, 1.0}, {ACC, 1.0}});
      Op p6 = mk(0, 1);
      O(p6, 2, {{ACC, 1.0}});
      step({p1}); step({p2}); step({p3}); step({p4}); step({p5}); step({p6});
      P.cos_slot = 7; P.sin_slot = 2;
    } else {  // k == 7
      Op p2 = mk(1, 1);
      O(p2, 2, {{ACC, 1.0}});
      Op p3 = mk(2, 1);
      O(p3, 3, {{ACC, 1.0}});
      O(p3, 4, {{EYE, a[3][0]}, {1, a[3][1]}, {2, a[3][2]}, {ACC, a[3][3]}});
      Op p4 = mk(4, 4);
      O(p4, 5, {{EYE, a[2][0]}, {1, a[2][1]}, {2, a[2][2]}, {3, a[2][3]}, {ACC, 1.0}});
      O(p4, 6, {{EYE, a[1][0]}, {1, a[1][1]}, {2, a[1][2]}, {3, a[1][3]}, {OUT0, 1.0}});
      Op p5 = mk(6, 5);
      O(p5, 4, {{EYE, a[0][0]}, {1, a[0][1]}, {2, a[0][2]}, {3, a[0][3]}, {ACC, 1.0}});
      O(p5, 7, {{EYE, z[6]}, {1, z[7]}, {2, z[8]}, {3, z[9]}, {5, z[10]}, {OUT0, z[11]}});
      O(p5, 8, {{EYE, z[0]}, {1, z[1]}, {2, z[2]}, {3, z[3]}, {5, z[4]}, {OUT0, z[5]}});
      Op p6 = mk(7, 4);
      O(p6, 1, {{8, 1.0}, {ACC, 1.0}});
      Op p7 = mk(0, 1);
      O(p7, 2, {{ACC, 1.0}});
      step({p1}); step({p2}); step({p3}); step({p4}); step({p5}); step({p6}); step({p7});
      P.cos_slot = 4; P.sin_slot = 2;
    }
  } else {
    if (k == 3) {
      Op p1 = mk(0, 0);
      O(p1, 1, {{ACC, 1.0}});
      O(p1, 2, {{0, -1.0 / 720.0}, {ACC, 1.0 / 40320.0}});
      O(p1, 3, {{0, -1.0 / 5040.0}, {ACC, 1.0 / 362880.0}});
      Op q = mk(2, 1), q9 = mk(3, 1);  // L y2, L9 y2 (polynomials in y commute)
      O(q, 4, {{EYE, 1.0}, {0, -0.5}, {1, 1.0 / 24.0}, {ACC, 1.0}});
      O(q9, 5, {{EYE, 1.0}, {0, -1.0 / 6.0}, {1, 1.0 / 120.0}, {ACC, 1.0}}, true);
      step({p1}); step({q, q9});
      P.cos_slot = 4; P.sin_slot = 5;
    } else if (k == 4) {
      Op p1 = mk(0, 0);
      O(p1, 1, {{ACC, 1.0}});
      O(p1, 2, {{0, x[0]}, {ACC, x[1]}});
      Op p2 = mk(1, 2);
      O(p2, 3, {{ACC, 1.0}});
      O(p2, 4, {{1, x[2]}, {ACC, 1.0}});
      O(p2, 5, {{EYE, x[3]}, {0, x[4]}, {1, x[5]}, {ACC, x[6]}});
      Op p3 = mk(4, 5);
      O(p3, 6, {{EYE, 1.0}, {0, -0.5}, {1, x[7]}, {ACC, 1.0}});
      O(p3, 2, {{EYE, z8[5]}, {0, z8[5]}, {1, z8[6]}, {3, z8[7]}, {OUT0, z8[8]}});
      O(p3, 7, {{EYE, z8[0]}, {0, z8[1]}, {1, z8[2]}, {3, z8[3]}, {OUT0, z8[4]}});
      Op p4 = mk(2, 3);
      O(p4, 1, {{7, 1.0}, {ACC, 1.0}}, true);
      step({p1}); step({p2}); step({p3}); step({p4});
      P.cos_slot = 6; P.sin_slot = 1;
    } else {  // k == 5
      Op p1 = mk(0, 0);
      O(p1, 1, {{ACC, 1.0}});
      Op p2 = mk(1, 0);
      O(p2, 2, {{ACC, 1.0}});
      O(p2, 3, {{EYE, a[3][0]}, {0, a[3][1]}, {1, a[3][2]}, {ACC, a[3][3]}});
      Op p3 = mk(3, 3);
      O(p3, 4, {{EYE, a[2][0]}, {0, a[2][1]}, {1, a[2][2]}, {2, a[2][3]}, {ACC, 1.0}});
      O(p3, 5, {{EYE, a[1][0]}, {0, a[1][1]}, {1, a[1][2]}, {2, a[1][3]}, {OUT0, 1.0}});
      Op p4 = mk(5, 4);
      O(p4, 3, {{EYE, a[0][0]}, {0, a[0][1]}, {1, a[0][2]}, {2, a[0][3]}, {ACC, 1.0}});
      O(p4, 6, {{EYE, z[6]}, {0, z[7]}, {1, z[8]}, {2, z[9]}, {4, z[10]}, {OUT0, z[11]}});
      O(p4, 7, {{EYE, z[0]}, {0, z[1]}, {1, z[2]}, {2, z[3]}, {4, z[4]}, {OUT0, z[5]}});
      Op p5 = mk(6, 3);
      O(p5, 1, {{7, 1.0}, {ACC, 1.0}}, true);
      step({p1}); step({p2}); step({p3}); step({p4}); step({p5});
      P.cos_slot = 3; P.sin_slot = 1;
    }
  }
  return P;
}

// Doubling op pair: S' = 2 S C, C' = 2 C C - I, into (c1, s1).
std::vector<Op> doubling_ops(int c0, int s0, int c1, int s1) {
  Op a{}, b{};
  a.lhs = s0; a.rhs = c0;
  ProgBuilder::out(a, s1, {{ACC, 2.0}});
  b.lhs = c0; b.rhs = c0;
  ProgBuilder::out(b, c1, {{ACC, 2.0}, {EYE, -1.0}});
  return {a, b};
}

void free_pair(int c0, int s0, int* c1, int* s1) {
  int got[2], m = 0;
  for (int i = 0; i < tk::NSLOT && m < 2; ++i)
    if (i != c0 && i != s0) got[m++] = i;
  *c1 = got[0];
  *s1 = got[1];
}

}  // namespace

size_t tiled_np(int n) { return static_cast<size_t>((n + 63) / 64) * 64; }

size_t tiled_workspace_bytes(int64_t batch, int n) {
  const size_t NP = tiled_np(n);
  size_t bytes = 0;
  bytes += static_cast<size_t>(batch) * tk::NSLOT * NP * NP * sizeof(double);  // slots
  bytes += static_cast<size_t>(batch) * sizeof(double);                        // tsc
  bytes += static_cast<size_t>(batch) * 2 * sizeof(int32_t) + 256;             // idx
  bytes += 64 * sizeof(Op) + 256;                                              // op table
  return bytes;
}

struct TiledWs {
  double* slots;
  double* tsc;
  int32_t* idx;
  Op* ops;
};

static TiledWs carve(void* ws, int64_t batch, int n) {
  const size_t NP = tiled_np(n);
  char* p = static_cast<char*>(ws);
  TiledWs w;
  w.slots = reinterpret_cast<double*>(p);
  p += static_cast<size_t>(batch) * tk::NSLOT * NP * NP * sizeof(double);
  w.tsc = reinterpret_cast<double*>(p);
  p += static_cast<size_t>(batch) * sizeof(double);
  p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255));
  w.idx = reinterpret_cast<int32_t*>(p);
  p += static_cast<size_t>(batch) * 2 * sizeof(int32_t);
  p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255));
  w.ops = reinterpret_cast<Op*>(p);
  return w;
}

static int64_t g_launches_tiled = 0;

// Run the tiled pipeline for a batch whose (k, s, status) are on the device.
// Synchronises the stream once to read (k, s, status) back for scheduling.
cudaError_t run_tiled(int dtype, bool wave, const void* a, const double* t, void* c_out,
                      void* s_out, int64_t batch, int n, const int32_t* dK,
                      const int32_t* dS, const int32_t* dStatus, void* ws,
                      cudaStream_t stream, int64_t* launches) {
  cudaError_t e;
  const int NP = static_cast<int>(tiled_np(n));
  const size_t mat_stride = static_cast<size_t>(tk::NSLOT) * NP * NP;
  TiledWs w = carve(ws, batch, n);
  std::vector<int32_t> hk(batch), hs(batch), hst(batch);
  e = cudaMemcpyAsync(hk.data(), dK, batch * 4, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hs.data(), dS, batch * 4, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hst.data(), dStatus, batch * 4, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return e;

  // prepare: scaled input into slot 0 (all matrices; failed ones skip)
  {
    dim3 grid(static_cast<unsigned>((static_cast<size_t>(NP) * NP + 255) / 256 < 64
                                        ? (static_cast<size_t>(NP) * NP + 255) / 256 : 64),
              static_cast<unsigned>(batch));
    if (dtype == 0)
      tk::prepare_kernel<double><<<grid, 256, 0, stream>>>(
          static_cast<const double*>(a), w.slots, n, NP, mat_stride, dS, dStatus, wave ? t : nullptr, w.tsc);
    else
      tk::prepare_kernel<float><<<grid, 256, 0, stream>>>(
          static_cast<const float*>(a), w.slots, n, NP, mat_stride, dS, dStatus, wave ? t : nullptr, w.tsc);
    ++*launches;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }

  // group by k, each group sorted by s descending (doubling = prefixes)
  const int ks_taylor[4] = {3, 4, 6, 7}, ks_wave[3] = {3, 4, 5};
  const int* ks = wave ? ks_wave : ks_taylor;
  const int nks = wave ? 3 : 4;
  std::vector<int32_t> order;
  order.reserve(batch);
  struct Group { int k; size_t off, cnt; int max_s; };
  std::vector<Group> groups;
  for (int gi = 0; gi < nks; ++gi) {
    Group G{ks[gi], order.size(), 0, 0};
    std::vector<std::pair<int, int32_t>> mem;
    for (int64_t b = 0; b < batch; ++b)
      if (hst[b] == 0 && hk[b] == ks[gi]) mem.emplace_back(hs[b], static_cast<int32_t>(b));
    std::stable_sort(mem.begin(), mem.end(),
                     [](const std::pair<int, int32_t>& x, const std::pair<int, int32_t>& y) {
                       return x.first > y.first;
                     });
    for (auto& m : mem) order.push_back(m.second);
    G.cnt = mem.size();
    G.max_s = mem.empty() ? 0 : mem.front().first;
    if (G.cnt) groups.push_back(G);
  }

  // op table: programs then doubling pairs, one upload
  std::vector<Op> table;
  struct Launch { size_t op_off; int nops; size_t idx_off; size_t cnt; };
  std::vector<Launch> launches_v;
  tk::FinalSlots fs{};
  for (const Group& G : groups) {
    Program P = build_program(wave, G.k);
    for (auto& stp : P.steps) {
      launches_v.push_back({table.size(), static_cast<int>(stp.size()), G.off, G.cnt});
      for (auto& op : stp) table.push_back(op);
    }
    int c1, s1;
    free_pair(P.cos_slot, P.sin_slot, &c1, &s1);
    fs.cos_slot[G.k][0] = static_cast<int8_t>(P.cos_slot);
    fs.sin_slot[G.k][0] = static_cast<int8_t>(P.sin_slot);
    fs.cos_slot[G.k][1] = static_cast<int8_t>(c1);
    fs.sin_slot[G.k][1] = static_cast<int8_t>(s1);
    const size_t even_off = table.size();
    for (auto& op : doubling_ops(P.cos_slot, P.sin_slot, c1, s1)) table.push_back(op);
    const size_t odd_off = table.size();
    for (auto& op : doubling_ops(c1, s1, P.cos_slot, P.sin_slot)) table.push_back(op);
    for (int i = 0; i < G.max_s; ++i) {
      size_t cnt = 0;
      for (size_t j = 0; j < G.cnt; ++j)
        if (hs[order[G.off + j]] > i) ++cnt;
      launches_v.push_back({(i & 1) ? odd_off : even_off, 2, G.off, cnt});
    }
  }
  if (table.size() > 64) return cudaErrorInvalidValue;
  if (!order.empty()) {
    e = cudaMemcpyAsync(w.idx, order.data(), order.size() * 4, cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(w.ops, table.data(), table.size() * sizeof(Op), cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);  // host vectors die here
    if (e != cudaSuccess) return e;
  }

  static bool attr_done = false;
  if (!attr_done) {
    e = cudaFuncSetAttribute(tk::gemm_epi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(tk::SMEM));
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  const unsigned tiles = static_cast<unsigned>((NP / tk::BM) * (NP / tk::BN));
  prof_begin(stream);
  for (const Launch& L : launches_v) {
    for (size_t done = 0; done < L.cnt; done += 65535) {
      const size_t cnt = std::min<size_t>(65535, L.cnt - done);
      dim3 grid(tiles, static_cast<unsigned>(cnt), static_cast<unsigned>(L.nops));
      tk::gemm_epi_kernel<<<grid, tk::THREADS, tk::SMEM, stream>>>(
          w.slots, NP, mat_stride, w.idx + L.idx_off + done, w.ops + L.op_off,
          wave ? w.tsc : nullptr);
      ++*launches;
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
  }
  prof_end(stream);

  {
    const size_t nn = static_cast<size_t>(n) * n;
    dim3 grid(static_cast<unsigned>((nn + 255) / 256 < 64 ? (nn + 255) / 256 : 64),
              static_cast<unsigned>(batch));
    if (dtype != 1)
      tk::finalize_kernel<double><<<grid, 256, 0, stream>>>(
          w.slots, static_cast<double*>(c_out), static_cast<double*>(s_out), n, NP, mat_stride,
          dK, dS, dStatus, fs);
    else
      tk::finalize_kernel<float><<<grid, 256, 0, stream>>>(
          w.slots, static_cast<float*>(c_out), static_cast<float*>(s_out), n, NP, mat_stride,
          dK, dS, dStatus, fs);
    ++*launches;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace csm
