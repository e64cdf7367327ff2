// ddref.cu -- double-double reference cos/sin on the GPU.
//
// The reference validates its schemes against reference_cos_sin
// (verify.py:480-521): scale by 2^-s until ||A||_1 <= 2^-20, a degree-12
// Taylor pair in compensated double-double arithmetic, then s doubling
// steps, every product being _dd_matmul (verify.py:449-459) -- a k-ordered
// sequence of error-free transformations (_two_sum :417-421, _two_prod
// :423-431, Dekker splitting with 2^27 + 1).  In numpy that is O(n) passes
// of O(n^2) vector ops per product: hours at the 8192^2 config.
//
// Here every output element runs exactly the reference's operation
// sequence -- same k order, same association, every add/mul an explicit
// round-to-nearest intrinsic so nvcc cannot contract anything into an FMA
// -- so the results are bit-identical to the reference (NaN payloads
// aside).  The work is FP64 CUDA-core bound (no tensor core can reproduce
// the error-free transformations): per k step and output element, 9 DMUL /
// DADD for the split product, 4 for the cross terms and 20 for the two
// renormalising additions (the row/column Dekker splits are hoisted into
// the shared-memory stage, where they are computed once per operand).
//
// Kernels
//   dd_gemm_kernel   64x64 output tile per CTA, 256 threads, 4x4 elements
//                    per thread, BK = 8 k-slab in shared memory holding
//                    (hi, split-hi, split-lo, lo) per operand entry.  The
//                    epilogue implements the reference's uses of each
//                    product: plain, series accumulation (_dd_series
//                    :467-477 fused into the power product), the doubling
//                    sine (x2) and cosine (x2 then - I), and per-matrix
//                    pass-through once a matrix's own s steps are done.
//   dd_prologue      bh = a * 2^-s and the identity term of both series.
//   dd_combine       hi + lo -> float64 output.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <utility>

#include "common.cuh"

namespace csm {
namespace dd {

constexpr double kSplit = 134217729.0;  // 2^27 + 1 (verify.py:414)
constexpr int BM = 64, BK = 8, LD = BM + 1, NT = 256;

// 1/j! with their double-double (hi, lo) splits, as _dd_const
// (verify.py:462-464) produces them from the Fractions of
// _REF_COS_CORE / _REF_SIN_CORE (:405-412).  Pinned by the golden test.
struct SeriesConsts {
  double cos_h[7], cos_l[7], sin_h[7], sin_l[7];
};
__constant__ SeriesConsts dSeries;

__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = add(a, b);
  const double bb = sub(s, a);
  e = add(sub(a, sub(s, bb)), sub(b, bb));
}

__device__ __forceinline__ void split(double a, double& hi, double& lo) {
  const double ac = mul(kSplit, a);
  hi = sub(ac, sub(ac, a));
  lo = sub(a, hi);
}

// _dd_mul(xh, xl, yh, yl) with the operands' Dekker splits precomputed.
__device__ __forceinline__ void dd_mul(double xh, double xa, double xb, double xl, double yh,
                                       double ya, double yb, double yl, double& h, double& l) {
  const double p = mul(xh, yh);
  double e = add(sub(mul(xa, ya), p), mul(xa, yb));
  e = add(e, mul(xb, ya));
  e = add(e, mul(xb, yb));
  const double t = add(add(e, mul(xh, yl)), mul(xl, yh));
  two_sum(p, t, h, l);
}

// _dd_add(xh, xl, yh, yl)
__device__ __forceinline__ void dd_add(double xh, double xl, double yh, double yl, double& h,
                                       double& l) {
  double s, e;
  two_sum(xh, yh, s, e);
  two_sum(s, add(add(e, xl), yl), h, l);
}

// acc += power * c, as one step of _dd_series.
__device__ __forceinline__ void series_step(double ph, double pl, double ch, double cl,
                                            double& acc_h, double& acc_l) {
  double pa, pb, ca, cb, th, tl;
  split(ph, pa, pb);
  split(ch, ca, cb);
  dd_mul(ph, pa, pb, pl, ch, ca, cb, cl, th, tl);
  dd_add(acc_h, acc_l, th, tl, acc_h, acc_l);
}

enum Mode { M_PLAIN = 0, M_SERIES = 1, M_DSIN = 2, M_DCOS = 3 };

struct GemmArgs {
  const double *xh, *xl, *yh, *yl;  // xl / yl may be null (the zero matrix)
  double *oh, *ol;
  double *cos_h, *cos_l, *sin_h, *sin_l;  // M_SERIES accumulators
  const int32_t* S;                       // M_DSIN / M_DCOS: per-matrix s
  int n, mode, coef, step;
  int64_t mat;      // n * n
  int64_t b0;       // first matrix of this launch
};

__global__ void __launch_bounds__(NT, 2) dd_gemm_kernel(const GemmArgs g) {
  __shared__ double xs[4][BK][LD];  // x tile, k-major: hi, split-hi, split-lo, lo
  __shared__ double ys[4][BK][LD];  // y tile, k-major
  const int n = g.n;
  const int64_t b = g.b0 + blockIdx.z;
  const int64_t base = b * g.mat;
  const int row0 = blockIdx.y * BM, col0 = blockIdx.x * BM;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;

  if (g.mode >= M_DSIN && g.S[b] <= g.step) {
    // this matrix finished its own doubling: carry x through unchanged
    for (int i = tid; i < BM * BM; i += NT) {
      const int r = row0 + (i >> 6), c = col0 + (i & 63);
      if (r < n && c < n) {
        const int64_t o = base + int64_t(r) * n + c;
        g.oh[o] = g.xh[o];
        g.ol[o] = g.xl[o];
      }
    }
    return;
  }

  double ah[4][4], al[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) ah[i][j] = al[i][j] = 0.0;

  // staging: 64 rows x BK k per operand, (64 BK / NT) entries per thread
  constexpr int RPT = BM * BK / NT, RSTEP = NT / BK;
  const int lk = tid % BK, lr = tid / BK;
  for (int k0 = 0; k0 < n; k0 += BK) {
    const int kc = min(BK, n - k0);
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int r = lr + RSTEP * q;
      // x: row (row0 + r), column (k0 + lk)
      double h = 0.0, l = 0.0;
      if (row0 + r < n && lk < kc) {
        const int64_t o = base + int64_t(row0 + r) * n + k0 + lk;
        h = g.xh[o];
        l = g.xl ? g.xl[o] : 0.0;
      }
      double sa, sb;
      split(h, sa, sb);
      xs[0][lk][r] = h; xs[1][lk][r] = sa; xs[2][lk][r] = sb; xs[3][lk][r] = l;
      // y: k-row (k0 + yk), coalesced along the 64 tile columns
      const int yk = (tid >> 6) + (NT / BM) * q, yc = tid & 63;
      h = 0.0; l = 0.0;
      if (yk < kc && col0 + yc < n) {
        const int64_t o = base + int64_t(k0 + yk) * n + col0 + yc;
        h = g.yh[o];
        l = g.yl ? g.yl[o] : 0.0;
      }
      split(h, sa, sb);
      ys[0][yk][yc] = h; ys[1][yk][yc] = sa; ys[2][yk][yc] = sb; ys[3][yk][yc] = l;
    }
    __syncthreads();
    for (int kk = 0; kk < kc; ++kk) {
      double y[4][4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int c = 0; c < 4; ++c) y[j][c] = ys[c][kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = ty * 4 + i;
        const double x0 = xs[0][kk][r], x1 = xs[1][kk][r], x2 = xs[2][kk][r], x3 = xs[3][kk][r];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          double ph, pl;
          dd_mul(x0, x1, x2, x3, y[j][0], y[j][1], y[j][2], y[j][3], ph, pl);
          dd_add(ah[i][j], al[i][j], ph, pl, ah[i][j], al[i][j]);
        }
      }
    }
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = row0 + ty * 4 + i;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = col0 + tx + 16 * j;
      if (r >= n || c >= n) continue;
      const int64_t o = base + int64_t(r) * n + c;
      double h = ah[i][j], l = al[i][j];
      if (g.mode == M_DSIN) {
        h = mul(2.0, h);
        l = mul(2.0, l);
      } else if (g.mode == M_DCOS) {
        // _dd_add(2 ch, 2 cl, -eye, zero)   (verify.py:517)
        dd_add(mul(2.0, h), mul(2.0, l), r == c ? -1.0 : -0.0, 0.0, h, l);
      }
      g.oh[o] = h;
      g.ol[o] = l;
      if (g.mode == M_SERIES) {
        double a_h = g.cos_h[o], a_l = g.cos_l[o];
        series_step(h, l, dSeries.cos_h[g.coef], dSeries.cos_l[g.coef], a_h, a_l);
        g.cos_h[o] = a_h;
        g.cos_l[o] = a_l;
        a_h = g.sin_h[o];
        a_l = g.sin_l[o];
        series_step(h, l, dSeries.sin_h[g.coef], dSeries.sin_l[g.coef], a_h, a_l);
        g.sin_h[o] = a_h;
        g.sin_l[o] = a_l;
      }
    }
  }
}

// bh = a * 2^-s (verify.py:499) and the identity (power 0) term of both
// series, accumulated onto a zero double-double exactly as _dd_series does.
__global__ void dd_prologue(const double* a, const int32_t* S, double* bh, double* ch, double* cl,
                            double* sh, double* sl, int n, int64_t total) {
  const int64_t mat = int64_t(n) * n;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = i / mat, e = i - b * mat;
    const int r = int(e / n), c = int(e - int64_t(r) * n);
    bh[i] = mul(a[i], ldexp(1.0, -S[b]));
    const double p = (r == c) ? 1.0 : 0.0;
    double h = 0.0, l = 0.0;
    series_step(p, 0.0, dSeries.cos_h[0], dSeries.cos_l[0], h, l);
    ch[i] = h;
    cl[i] = l;
    h = 0.0;
    l = 0.0;
    series_step(p, 0.0, dSeries.sin_h[0], dSeries.sin_l[0], h, l);
    sh[i] = h;
    sl[i] = l;
  }
}

__global__ void dd_combine(const double* h, const double* l, double* out, int64_t total) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = add(h[i], l[i]);
}

}  // namespace dd

// ---------------------------------------------------------------------------
// Host side.

// _dd_const(+-1/j!) (verify.py:462-464): hi = RN(1/N); the residual
// 1 - hi N is an integer multiple of ulp(hi) no larger than N / 2, so the
// fma below is exact and lo = RN((1 - hi N) / N) = RN(1/N - hi) exactly as
// float(value - Fraction(hi)) computes it (signs included).
void ddref_series_consts(double* out28) {
  dd::SeriesConsts c{};
  double fact = 1.0;
  for (int i = 0; i < 7; ++i) {
    if (i > 0) fact *= double(2 * i - 1) * double(2 * i);  // (2i)!
    const double sgn = (i & 1) ? -1.0 : 1.0;
    double hi = sgn / fact;
    c.cos_h[i] = hi;
    c.cos_l[i] = std::fma(-hi, fact, sgn) / fact;
    const double f1 = fact * double(2 * i + 1);  // (2i+1)!
    hi = sgn / f1;
    c.sin_h[i] = hi;
    c.sin_l[i] = std::fma(-hi, f1, sgn) / f1;
  }
  std::memcpy(out28, &c, sizeof(c));
}

static cudaError_t ensure_series() {
  static int done_mask = 0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 32 && (done_mask >> dev) & 1) return cudaSuccess;
  double consts[28];
  ddref_series_consts(consts);
  e = cudaMemcpyToSymbol(dd::dSeries, consts, sizeof(dd::SeriesConsts));
  if (e == cudaSuccess && dev < 32) done_mask |= 1 << dev;
  return e;
}

static unsigned elt_blocks(int64_t total) {
  int64_t b = (total + 255) / 256;
  return unsigned(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}

// C = X Y for a batch, any epilogue mode; launches chunked over grid.z.
static cudaError_t dd_gemm(dd::GemmArgs g, int64_t batch, cudaStream_t stream,
                           int64_t* launches) {
  const int tiles = (g.n + dd::BM - 1) / dd::BM;
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    const int64_t nb = batch - b0 < 65535 ? batch - b0 : 65535;
    g.b0 = b0;
    dd::dd_gemm_kernel<<<dim3(tiles, tiles, unsigned(nb)), dd::NT, 0, stream>>>(g);
    if (launches) ++*launches;
  }
  return cudaGetLastError();
}

size_t ddref_workspace_doubles(int64_t batch, int n) {
  // bh, Y(2), PA(2), PB(2), CS(2), SS(2), SN(2)
  return size_t(batch) * size_t(n) * size_t(n) * 13;
}

cudaError_t dd_matmul(const double* xh, const double* xl, const double* yh, const double* yl,
                      double* oh, double* ol, int64_t batch, int n, cudaStream_t stream,
                      int64_t* launches) {
  dd::GemmArgs g{};
  g.xh = xh; g.xl = xl; g.yh = yh; g.yl = yl; g.oh = oh; g.ol = ol;
  g.n = n; g.mode = dd::M_PLAIN; g.mat = int64_t(n) * n;
  return dd_gemm(g, batch, stream, launches);
}

// The chain of reference_cos_sin (verify.py:495-521) for a batch whose
// per-matrix s is already on the device (dS) and whose maximum is smax.
cudaError_t ddref_chain(const double* a, const int32_t* dS, int smax, double* cos_out,
                        double* sin_out, int64_t batch, int n, double* ws, cudaStream_t stream,
                        int64_t* launches) {
  cudaError_t e = ensure_series();
  if (e != cudaSuccess) return e;
  const int64_t mat = int64_t(n) * n, total = mat * batch;
  double* p = ws;
  auto take = [&]() { double* q = p; p += total; return q; };
  double* bh = take();
  double *yh = take(), *yl = take();
  double *pah = take(), *pal = take(), *pbh = take(), *pbl = take();
  double *csh = take(), *csl = take(), *ssh = take(), *ssl = take();
  double *snh = take(), *snl = take();

  dd::dd_prologue<<<elt_blocks(total), 256, 0, stream>>>(a, dS, bh, csh, csl, ssh, ssl, n, total);
  if (launches) ++*launches;

  dd::GemmArgs g{};
  g.n = n; g.mat = mat;
  g.cos_h = csh; g.cos_l = csl; g.sin_h = ssh; g.sin_l = ssl;
  // y = bh bh, then powers y^2 .. y^6, each folded into both series
  g.mode = dd::M_SERIES;
  g.xh = bh; g.xl = nullptr; g.yh = bh; g.yl = nullptr; g.oh = yh; g.ol = yl; g.coef = 1;
  if ((e = dd_gemm(g, batch, stream, launches)) != cudaSuccess) return e;
  const double *ph = yh, *pl = yl;
  double* bufs[2][2] = {{pah, pal}, {pbh, pbl}};
  for (int j = 2; j <= 6; ++j) {
    double* oh = bufs[j & 1][0];
    double* ol = bufs[j & 1][1];
    g.xh = ph; g.xl = pl; g.yh = yh; g.yl = yl; g.oh = oh; g.ol = ol; g.coef = j;
    if ((e = dd_gemm(g, batch, stream, launches)) != cudaSuccess) return e;
    ph = oh;
    pl = ol;
  }
  // sin = bh * sin_series
  g = dd::GemmArgs{};
  g.n = n; g.mat = mat; g.mode = dd::M_PLAIN;
  g.xh = bh; g.xl = nullptr; g.yh = ssh; g.yl = ssl; g.oh = snh; g.ol = snl;
  if ((e = dd_gemm(g, batch, stream, launches)) != cudaSuccess) return e;
  // doubling: (S, C) -> (2 S C, 2 C C - I), per-matrix step count
  double *S_h = snh, *S_l = snl, *C_h = csh, *C_l = csl;
  double *S2h = pah, *S2l = pal, *C2h = pbh, *C2l = pbl;
  g.S = dS;
  for (int step = 0; step < smax; ++step) {
    g.step = step;
    g.mode = dd::M_DSIN;
    g.xh = S_h; g.xl = S_l; g.yh = C_h; g.yl = C_l; g.oh = S2h; g.ol = S2l;
    if ((e = dd_gemm(g, batch, stream, launches)) != cudaSuccess) return e;
    g.mode = dd::M_DCOS;
    g.xh = C_h; g.xl = C_l; g.yh = C_h; g.yl = C_l; g.oh = C2h; g.ol = C2l;
    if ((e = dd_gemm(g, batch, stream, launches)) != cudaSuccess) return e;
    std::swap(S_h, S2h); std::swap(S_l, S2l); std::swap(C_h, C2h); std::swap(C_l, C2l);
  }
  dd::dd_combine<<<elt_blocks(total), 256, 0, stream>>>(C_h, C_l, cos_out, total);
  dd::dd_combine<<<elt_blocks(total), 256, 0, stream>>>(S_h, S_l, sin_out, total);
  if (launches) *launches += 2;
  return cudaGetLastError();
}

}  // namespace csm
