// fused64.cu -- K1: the whole cos/sin (or wave) pipeline for n <= 64 with
// every intermediate resident in shared memory.
//
// One persistent CTA per SM (256 threads, 8 warps) pulls matrices from an
// atomic work counter.  A matrix is zero-padded to 64x64 (block-diagonal
// padding is exact: the padded block evolves as p(0) I and never touches
// the real block).  Seven 32 KiB slots: six hold the chain's live set
// (peak six for the degree-12 chain) and the
// seventh receives the NEXT matrix by cp.async while this one computes.
//
// Every product is a 64x64x64 FP64 GEMM on the DMMA pipe (mma.sync
// m8n8k4): warp w owns rows [16(w/2), +16) x cols [32(w%2), +32) = 2x4
// DMMA tiles; doubling steps and the wave k=3 sine are DUAL products that
// share the right operand and reuse its fragments.  Linear combinations
// run in the GEMM epilogue on the accumulator registers (never a separate
// pass).  Slots use an XOR swizzle on 32-byte chunks so both DMMA fragment
// loads are bank-conflict free.
//
// Reference mapping: chains schemes.py:264-361, trig use :376-395, wave use
// :411-430, scaling driver.py:115/:139, doubling driver.py:91-98.
#include "common.cuh"

namespace csm {

namespace f64k {

constexpr int NP = 64;
constexpr int SLOT = NP * NP;  // doubles per slot
constexpr int NSLOTS = 7;
constexpr int THREADS = 256;

__device__ __forceinline__ int swz(int r, int c) {
  return r * NP + ((((c >> 2) ^ (r & 7))) << 2) + (c & 3);
}

struct Lane {
  int rb, cb, g, t;
};

typedef double Acc[2][4][2];

__device__ __forceinline__ void zero(Acc& a) {
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) a[i][j][0] = a[i][j][1] = 0.0;
}

// acc = L * R over the full 64-deep contraction.
__device__ __forceinline__ void gemm1(const double* __restrict__ L,
                                      const double* __restrict__ R, Acc& acc,
                                      const Lane& ln) {
  zero(acc);
#pragma unroll
  for (int kk = 0; kk < NP; kk += 4) {
    double a[2], b[4];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) a[mi] = L[swz(ln.rb + mi * 8 + ln.g, kk + ln.t)];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[ni] = R[swz(kk + ln.t, ln.cb + ni * 8 + ln.g)];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
  }
}

// acc1 = L1 * R, acc2 = L2 * R (shared right-operand fragments).
__device__ __forceinline__ void gemm2(const double* __restrict__ L1,
                                      const double* __restrict__ L2,
                                      const double* __restrict__ R, Acc& acc1,
                                      Acc& acc2, const Lane& ln) {
  zero(acc1);
  zero(acc2);
#pragma unroll
  for (int kk = 0; kk < NP; kk += 4) {
    double a1[2], a2[2], b[4];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      a1[mi] = L1[swz(ln.rb + mi * 8 + ln.g, kk + ln.t)];
      a2[mi] = L2[swz(ln.rb + mi * 8 + ln.g, kk + ln.t)];
    }
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[ni] = R[swz(kk + ln.t, ln.cb + ni * 8 + ln.g)];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        dmma(acc1[mi][ni], a1[mi], b[ni]);
        dmma(acc2[mi][ni], a2[mi], b[ni]);
      }
  }
}

// Visit the 8 element pairs this thread owns (its accumulator positions).
// f(mi, ni, off, i0, i1): off = swizzled offset of the pair, i0/i1 = 1.0
// where the pair's first/second element lies on the diagonal, else 0.0.
template <class F>
__device__ __forceinline__ void owned(const Lane& ln, F&& f) {
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int r = ln.rb + mi * 8 + ln.g;
      const int c = ln.cb + ni * 8 + 2 * ln.t;
      f(mi, ni, swz(r, c), r == c ? 1.0 : 0.0, r == c + 1 ? 1.0 : 0.0);
    }
}

__device__ __forceinline__ double2 ld2(const double* p, int off) {
  return *reinterpret_cast<const double2*>(p + off);
}
__device__ __forceinline__ void st2(double* p, int off, double x, double y) {
  *reinterpret_cast<double2*>(p + off) = make_double2(x, y);
}

// Store one result pair: acc values in, slot out.
__device__ __forceinline__ void store_acc(double* dst, const Acc& acc,
                                          const Lane& ln) {
  owned(ln, [&](int mi, int ni, int off, double, double) {
    st2(dst, off, acc[mi][ni][0], acc[mi][ni][1]);
  });
}

// ---------------------------------------------------------------------------
// Chains.  Each leaves cos / sin slot pointers in *pc / *ps.  `Y` is the even
// variable's slot for the wave family (y = t^2 A) and A for Taylor.
// Between a product and its epilogue there is a barrier, so an epilogue may
// overwrite the product's own operands; elementwise reads and writes happen
// only at the thread's own positions.

// Taylor k=3 -- chain_deg2 (schemes.py:264-272) + sin = A sc (:394).
__device__ void taylor3(double* A, double* const* W, const Lane& ln,
                        double** pc, double** ps) {
  Acc acc;
  gemm1(A, A, acc, ln);
  store_acc(W[0], acc, ln);  // y
  __syncthreads();
  gemm1(W[0], W[0], acc, ln);  // y2
  owned(ln, [&](int mi, int ni, int off, double i0, double i1) {
    double2 y = ld2(W[0], off);
    const double* a = acc[mi][ni];
    double c0 = fma(1.0 / 24.0, a[0], fma(-0.5, y.x, i0));
    double c1 = fma(1.0 / 24.0, a[1], fma(-0.5, y.y, i1));
    double s0 = fma(1.0 / 120.0, a[0], fma(-1.0 / 6.0, y.x, i0));
    double s1 = fma(1.0 / 120.0, a[1], fma(-1.0 / 6.0, y.y, i1));
    st2(W[1], off, c0, c1);
    st2(W[2], off, s0, s1);
  });
  __syncthreads();
  gemm1(A, W[2], acc, ln);
  store_acc(W[3], acc, ln);
  __syncthreads();
  *pc = W[1];
  *ps = W[3];
}

// Taylor k=4 -- chain_deg4(exact_sine=False) (schemes.py:275-299).
__device__ void taylor4(double* A, double* const* W, const Lane& ln,
                        double** pc, double** ps) {
  Acc acc;
  gemm1(A, A, acc, ln);
  store_acc(W[0], acc, ln);  // y
  __syncthreads();
  gemm1(W[0], W[0], acc, ln);  // y2
  owned(ln, [&](int mi, int ni, int off, double, double) {
    double2 y = ld2(W[0], off);
    const double* a = acc[mi][ni];
    st2(W[1], off, a[0], a[1]);
    st2(W[2], off, fma(1.0 / 40320.0, a[0], (-1.0 / 720.0) * y.x),
        fma(1.0 / 40320.0, a[1], (-1.0 / 720.0) * y.y));
  });
  __syncthreads();
  gemm1(W[1], W[2], acc, ln);  // q = y2 (-y/720 + y2/40320)
  owned(ln, [&](int mi, int ni, int off, double i0, double i1) {
    double2 y = ld2(W[0], off), y2 = ld2(W[1], off);
    const double* q = acc[mi][ni];
    double c0 = q[0] + fma(1.0 / 24.0, y2.x, fma(-0.5, y.x, i0));
    double c1 = q[1] + fma(1.0 / 24.0, y2.y, fma(-0.5, y.y, i1));
    double s0 = fma(720.0 / 5040.0, q[0], fma(1.0 / 120.0, y2.x, fma(-1.0 / 6.0, y.x, i0)));
    double s1 = fma(720.0 / 5040.0, q[1], fma(1.0 / 120.0, y2.y, fma(-1.0 / 6.0, y.y, i1)));
    st2(W[3], off, c0, c1);
    st2(W[4], off, s0, s1);
  });
  __syncthreads();
  gemm1(A, W[4], acc, ln);
  store_acc(W[0], acc, ln);  // sin (y is dead)
  __syncthreads();
  *pc = W[3];
  *ps = W[0];
}

// Degree-8 core (schemes.py:302-326) on even variable in slot Y; y2 is
// computed first.  Taylor k=6 (sin = A sc) and wave k=4 (s = tp sc).
template <bool WAVE>
__device__ void deg8(double* A, double* Y, double* const* W, double tp,
                     const Lane& ln, double** pc, double** ps) {
  const double* x = dTables.x8;  // x[0] = x1
  const double* z = dTables.z8;
  Acc acc;
  // W slots (4): y2/sc, L/R2/inner/sin, p8, L2/cos
  double *sY2 = W[0], *sL = W[1], *sP8 = W[2], *sL2 = W[3], *sR2 = W[1];
  gemm1(Y, Y, acc, ln);  // y2
  owned(ln, [&](int mi, int ni, int off, double, double) {
    double2 y = ld2(Y, off);
    const double* a = acc[mi][ni];
    st2(sY2, off, a[0], a[1]);
    st2(sL, off, fma(x[1], a[0], x[0] * y.x), fma(x[1], a[1], x[0] * y.y));
  });
  __syncthreads();
  gemm1(sY2, sL, acc, ln);  // p8 = y2 (x1 y + x2 y2)
  __syncthreads();           // sR2 overwrites sL
  owned(ln, [&](int mi, int ni, int off, double i0, double i1) {
    double2 y = ld2(Y, off), y2 = ld2(sY2, off);
    const double* p = acc[mi][ni];
    st2(sP8, off, p[0], p[1]);
    st2(sL2, off, fma(x[2], y2.x, p[0]), fma(x[2], y2.y, p[1]));
    st2(sR2, off, fma(x[6], p[0], fma(x[5], y2.x, fma(x[4], y.x, x[3] * i0))),
        fma(x[6], p[1], fma(x[5], y2.y, fma(x[4], y.y, x[3] * i1))));
  });
  __syncthreads();
  gemm1(sL2, sR2, acc, ln);  // p16
  __syncthreads();            // cos overwrites L2, inner overwrites R2
  double sb[2][4][2];
  double *sCos = sL2, *sInner = sR2;
  owned(ln, [&](int mi, int ni, int off, double i0, double i1) {
    double2 y = ld2(Y, off), y2 = ld2(sY2, off), p8 = ld2(sP8, off);
    const double* p = acc[mi][ni];
    double c0 = p[0] + fma(x[7], y2.x, fma(-0.5, y.x, i0));
    double c1 = p[1] + fma(x[7], y2.y, fma(-0.5, y.y, i1));
    // inner = z5 I + z5 y + z6 y2 + z7 p8 + z8 cos
    double n0 = fma(z[8], c0, fma(z[7], p8.x, fma(z[6], y2.x, fma(z[5], y.x, z[5] * i0))));
    double n1 = fma(z[8], c1, fma(z[7], p8.y, fma(z[6], y2.y, fma(z[5], y.y, z[5] * i1))));
    // sin base = z0 I + z1 y + z2 y2 + z3 p8 + z4 cos
    sb[mi][ni][0] = fma(z[4], c0, fma(z[3], p8.x, fma(z[2], y2.x, fma(z[1], y.x, z[0] * i0))));
    sb[mi][ni][1] = fma(z[4], c1, fma(z[3], p8.y, fma(z[2], y2.y, fma(z[1], y.y, z[0] * i1))));
    st2(sCos, off, c0, c1);
    st2(sInner, off, n0, n1);
  });
  __syncthreads();
  gemm1(sInner, sP8, acc, ln);  // tail
  double* sSc = sY2;             // y2 dead after the p16 epilogue
  owned(ln, [&](int mi, int ni, int off, double, double) {
    double v0 = sb[mi][ni][0] + acc[mi][ni][0];
    double v1 = sb[mi][ni][1] + acc[mi][ni][1];
    if (WAVE) { v0 *= tp; v1 *= tp; }
    st2(sSc, off, v0, v1);
  });
  __syncthreads();
  *pc = sCos;
  if (WAVE) {
    *ps = sSc;
  } else {
    gemm1(A, sSc, acc, ln);
    store_acc(sInner, acc, ln);  // sin (inner dead)
    __syncthreads();
    *ps = sInner;
  }
}

// Degree-12 core (schemes.py:329-361) on even variable in slot Y.
// Taylor k=7 (sin = A sc) and wave k=5 (s = tp sc).
template <bool WAVE>
__device__ void deg12(double* A, double* Y, double* const* W, double tp,
                      const Lane& ln, double** pc, double** ps) {
  const double(*a)[4] = dTables.a12;  // a[j-1][i]
  const double* z = dTables.z12;
  Acc acc;
  double *sY2 = W[0], *sY3 = W[1], *sC4 = W[2], *sMid = W[3];
  gemm1(Y, Y, acc, ln);  // y2
  store_acc(sY2, acc, ln);
  __syncthreads();
  gemm1(sY2, Y, acc, ln);  // y3
  owned(ln, [&](int mi, int ni, int off, double i0, double i1) {
    double2 y = ld2(Y, off), y2 = ld2(sY2, off);
    const double* p = acc[mi][ni];
    st2(sY3, off, p[0], p[1]);
    st2(sC4, off, fma(a[3][3], p[0], fma(a[3][2], y2.x, fma(a[3][1], y.x, a[3][0] * i0))),
        fma(a[3][3], p[1], fma(a[3][2], y2.y, fma(a[3][1], y.y, a[3][0] * i1))));
  });
  __syncthreads();
  gemm1(sC4, sC4, acc, ln);  // c4^2
  __syncthreads();            // L overwrites c4
  double* sL = sC4;
  owned(ln, [&](int mi, int ni, int off, double i0, double i1) {
    double2 y = ld2(Y, off), y2 = ld2(sY2, off), y3 = ld2(sY3, off);
    const double* p = acc[mi][ni];
    double m0 = fma(a[2][3], y3.x, fma(a[2][2], y2.x, fma(a[2][1], y.x, a[2][0] * i0))) + p[0];
    double m1 = fma(a[2][3], y3.y, fma(a[2][2], y2.y, fma(a[2][1], y.y, a[2][0] * i1))) + p[1];
    double l0 = fma(a[1][3], y3.x, fma(a[1][2], y2.x, fma(a[1][1], y.x, a[1][0] * i0))) + m0;
    double l1 = fma(a[1][3], y3.y, fma(a[1][2], y2.y, fma(a[1][1], y.y, a[1][0] * i1))) + m1;
    st2(sMid, off, m0, m1);
    st2(sL, off, l0, l1);
  });
  __syncthreads();
  gemm1(sL, sMid, acc, ln);  // (c2 + mid) mid
  __syncthreads();            // cos overwrites L, inner overwrites mid
  double sb[2][4][2];
  double *sCos = sL, *sInner = sMid;
  owned(ln, [&](int mi, int ni, int off, double i0, double i1) {
    double2 y = ld2(Y, off), y2 = ld2(sY2, off), y3 = ld2(sY3, off),
            md = ld2(sMid, off);
    const double* p = acc[mi][ni];
    double c0 = fma(a[0][3], y3.x, fma(a[0][2], y2.x, fma(a[0][1], y.x, a[0][0] * i0))) + p[0];
    double c1 = fma(a[0][3], y3.y, fma(a[0][2], y2.y, fma(a[0][1], y.y, a[0][0] * i1))) + p[1];
    double n0 = fma(z[11], c0, fma(z[10], md.x, fma(z[9], y3.x, fma(z[8], y2.x, fma(z[7], y.x, z[6] * i0)))));
    double n1 = fma(z[11], c1, fma(z[10], md.y, fma(z[9], y3.y, fma(z[8], y2.y, fma(z[7], y.y, z[6] * i1)))));
    sb[mi][ni][0] = fma(z[5], c0, fma(z[4], md.x, fma(z[3], y3.x, fma(z[2], y2.x, fma(z[1], y.x, z[0] * i0)))));
    sb[mi][ni][1] = fma(z[5], c1, fma(z[4], md.y, fma(z[3], y3.y, fma(z[2], y2.y, fma(z[1], y.y, z[0] * i1)))));
    st2(sCos, off, c0, c1);
    st2(sInner, off, n0, n1);
  });
  __syncthreads();
  gemm1(sInner, sCos, acc, ln);  // tail
  double* sSc = sY2;             // y2 dead
  owned(ln, [&](int mi, int ni, int off, double, double) {
    double v0 = sb[mi][ni][0] + acc[mi][ni][0];
    double v1 = sb[mi][ni][1] + acc[mi][ni][1];
    if (WAVE) { v0 *= tp; v1 *= tp; }
    st2(sSc, off, v0, v1);
  });
  __syncthreads();
  *pc = sCos;
  if (WAVE) {
    *ps = sSc;
  } else {
    gemm1(A, sSc, acc, ln);
    store_acc(sY3, acc, ln);  // sin (y3 dead)
    __syncthreads();
    *ps = sY3;
  }
}

// Wave k=3 -- chain_deg4(exact_sine=True) on y (schemes.py:275-299, :426-427).
// q and q9 share their y2 factor: one dual product L*y2, L9*y2.
__device__ void wave3(double* Y, double* const* W, double tp, const Lane& ln,
                      double** pc, double** ps) {
  Acc acc, acc2;
  gemm1(Y, Y, acc, ln);  // y2
  owned(ln, [&](int mi, int ni, int off, double, double) {
    double2 y = ld2(Y, off);
    const double* p = acc[mi][ni];
    st2(W[0], off, p[0], p[1]);
    st2(W[1], off, fma(1.0 / 40320.0, p[0], (-1.0 / 720.0) * y.x),
        fma(1.0 / 40320.0, p[1], (-1.0 / 720.0) * y.y));
    st2(W[2], off, fma(1.0 / 362880.0, p[0], (-1.0 / 5040.0) * y.x),
        fma(1.0 / 362880.0, p[1], (-1.0 / 5040.0) * y.y));
  });
  __syncthreads();
  gemm2(W[1], W[2], W[0], acc, acc2, ln);  // q, q9
  owned(ln, [&](int mi, int ni, int off, double i0, double i1) {
    double2 y = ld2(Y, off), y2 = ld2(W[0], off);
    const double* q = acc[mi][ni];
    const double* q9 = acc2[mi][ni];
    double c0 = q[0] + fma(1.0 / 24.0, y2.x, fma(-0.5, y.x, i0));
    double c1 = q[1] + fma(1.0 / 24.0, y2.y, fma(-0.5, y.y, i1));
    double s0 = tp * (q9[0] + fma(1.0 / 120.0, y2.x, fma(-1.0 / 6.0, y.x, i0)));
    double s1 = tp * (q9[1] + fma(1.0 / 120.0, y2.y, fma(-1.0 / 6.0, y.y, i1)));
    st2(W[3], off, c0, c1);
    st2(W[4], off, s0, s1);
  });
  __syncthreads();
  *pc = W[3];
  *ps = W[4];
}

// s doubling steps (driver.py:91-98): S <- 2 S C (old C), C <- 2 C C - I,
// as one dual product [S; C] * C, written back in place after a barrier.
__device__ void doubling(double* C, double* S, int steps, const Lane& ln) {
  Acc sc, cc;
  for (int it = 0; it < steps; ++it) {
    gemm2(S, C, C, sc, cc, ln);
    __syncthreads();
    owned(ln, [&](int mi, int ni, int off, double i0, double i1) {
      st2(S, off, 2.0 * sc[mi][ni][0], 2.0 * sc[mi][ni][1]);
      st2(C, off, fma(2.0, cc[mi][ni][0], -i0), fma(2.0, cc[mi][ni][1], -i1));
    });
    __syncthreads();
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
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::);
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;\n" ::);
}

// Issue the load of matrix b into slot dst (async for fp64 input).
template <typename TIn>
__device__ __forceinline__ void load_matrix(double* dst, const TIn* __restrict__ src,
                                            int n) {
  const int tid = threadIdx.x;
  if constexpr (sizeof(TIn) == 8) {
    const double* s = reinterpret_cast<const double*>(src);
    if ((n & 1) == 0) {
      const int half = n >> 1;
      for (int p = tid; p < n * half; p += THREADS) {
        int r = p / half, c = (p - r * half) * 2;
        cp_async16(dst + swz(r, c), s + static_cast<size_t>(r) * n + c);
      }
    } else {
      for (int p = tid; p < n * n; p += THREADS) {
        int r = p / n, c = p - r * n;
        cp_async8(dst + swz(r, c), s + p);
      }
    }
    cp_async_commit();
  } else {
    for (int p = tid; p < n * n; p += THREADS) {
      int r = p / n, c = p - r * n;
      dst[swz(r, c)] = static_cast<double>(src[p]);
    }
  }
}

template <typename TOut>
__device__ __forceinline__ void store_matrix(TOut* __restrict__ dst,
                                             const double* src, int n) {
  const int tid = threadIdx.x;
  if (sizeof(TOut) == 8 && (n & 1) == 0) {
    const int half = n >> 1;
    for (int p = tid; p < n * half; p += THREADS) {
      int r = p / half, c = (p - r * half) * 2;
      double2 v = *reinterpret_cast<const double2*>(src + swz(r, c));
      *reinterpret_cast<double2*>(reinterpret_cast<double*>(dst) +
                                  static_cast<size_t>(r) * n + c) = v;
    }
  } else {
    for (int p = tid; p < n * n; p += THREADS) {
      int r = p / n, c = p - r * n;
      dst[p] = static_cast<TOut>(src[swz(r, c)]);
    }
  }
}

template <typename TOut>
__device__ __forceinline__ void store_nan(TOut* __restrict__ dst, int n) {
  for (int p = threadIdx.x; p < n * n; p += THREADS)
    dst[p] = static_cast<TOut>(__longlong_as_double(0x7ff8000000000000ll));
}

// ---------------------------------------------------------------------------

template <typename TIn, typename TOut, bool WAVE>
__global__ void __launch_bounds__(THREADS, 1)
fused64_kernel(const TIn* __restrict__ Ain, TOut* __restrict__ Cout,
               TOut* __restrict__ Sout, const double* __restrict__ T,
               const int32_t* __restrict__ K, const int32_t* __restrict__ Sx,
               const int32_t* __restrict__ ST, int64_t batch, int n,
               int* __restrict__ counter) {
  extern __shared__ __align__(16) double smem[];
  __shared__ long long sh_next;
  double* slot[NSLOTS];
#pragma unroll
  for (int i = 0; i < NSLOTS; ++i) slot[i] = smem + i * SLOT;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  Lane ln;
  ln.rb = (warp >> 1) * 16;
  ln.cb = (warp & 1) * 32;
  ln.g = lane >> 2;
  ln.t = lane & 3;
  const size_t nn = static_cast<size_t>(n) * n;

  // Both A slots start zero so the padding outside n x n stays exact zero.
  if (n < NP) {
    for (int p = tid; p < SLOT; p += THREADS) slot[0][p] = slot[6][p] = 0.0;
  }
  if (tid == 0) sh_next = atomicAdd(counter, 1);
  __syncthreads();
  long long cur = sh_next;
  double* Acur = slot[0];
  double* Anext = slot[6];
  constexpr bool kAsync = sizeof(TIn) == 8;
  if (kAsync && cur < batch) load_matrix(Acur, Ain + cur * nn, n);
  __syncthreads();

  while (cur < batch) {
    if (tid == 0) sh_next = atomicAdd(counter, 1);
    if (!kAsync) load_matrix(Acur, Ain + cur * nn, n);
    cp_async_wait_all();
    __syncthreads();
    const long long nxt = sh_next;
    if (kAsync && nxt < batch) load_matrix(Anext, Ain + nxt * nn, n);

    TOut* cdst = Cout + cur * nn;
    TOut* sdst = Sout + cur * nn;
    const int st = ST[cur];
    if (st != 0) {
      store_nan(cdst, n);
      store_nan(sdst, n);
    } else {
      const int k = K[cur], s = Sx[cur];
      double tp = 0.0, f;
      if (WAVE) {
        tp = T[cur] / ldexp(1.0, s);  // driver.py:139, t / 2**s
        f = tp * tp;                  // schemes.py:424, y = (t*t) a
      } else {
        f = ldexp(1.0, -s);  // driver.py:115, a * 2**-s
      }
      for (int p = tid; p < SLOT; p += THREADS) Acur[p] *= f;
      __syncthreads();
      double* W[5] = {slot[1], slot[2], slot[3], slot[4], slot[5]};
      double *pc, *ps;
      if (!WAVE) {
        if (k == 3) {
          taylor3(Acur, W, ln, &pc, &ps);
        } else if (k == 4) {
          taylor4(Acur, W, ln, &pc, &ps);
        } else {
          Acc acc;
          gemm1(Acur, Acur, acc, ln);  // y = A A  (schemes.py:388)
          store_acc(W[0], acc, ln);
          __syncthreads();
          if (k == 6) deg8<false>(Acur, W[0], W + 1, 0.0, ln, &pc, &ps);
          else deg12<false>(Acur, W[0], W + 1, 0.0, ln, &pc, &ps);
        }
      } else {
        if (k == 3) wave3(Acur, W, tp, ln, &pc, &ps);
        else if (k == 4) deg8<true>(nullptr, Acur, W, tp, ln, &pc, &ps);
        else deg12<true>(nullptr, Acur, W, tp, ln, &pc, &ps);
      }
      doubling(pc, ps, s, ln);
      store_matrix(cdst, pc, n);
      store_matrix(sdst, ps, n);
    }
    double* tmp = Acur;
    Acur = Anext;
    Anext = tmp;
    cur = nxt;
    __syncthreads();  // sh_next consumed, slots free for the next matrix
  }
}

}  // namespace f64k

size_t fused64_smem_bytes() {
  return static_cast<size_t>(f64k::NSLOTS) * f64k::SLOT * sizeof(double);
}

template <typename TIn, typename TOut, bool WAVE>
static cudaError_t launch_one(const void* a, void* c, void* s, const double* t,
                              const int32_t* k, const int32_t* sx,
                              const int32_t* st, int64_t batch, int n,
                              int* counter, int grid, cudaStream_t stream) {
  auto kern = f64k::fused64_kernel<TIn, TOut, WAVE>;
  const size_t smem = fused64_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(
      kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  kern<<<grid, f64k::THREADS, smem, stream>>>(
      static_cast<const TIn*>(a), static_cast<TOut*>(c), static_cast<TOut*>(s),
      t, k, sx, st, batch, n, counter);
  return cudaGetLastError();
}

// Launch K1 for a batch of n <= 64 matrices whose (k, s, status) are already
// on the device.  `counter` must be a zeroed device int.
cudaError_t launch_fused64(int dtype, bool wave, const void* a, void* c,
                           void* s, const double* t, const int32_t* k,
                           const int32_t* sx, const int32_t* st, int64_t batch,
                           int n, int* counter, cudaStream_t stream) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int grid = static_cast<int>(batch < sms ? batch : sms);
  if (grid < 1) return cudaSuccess;
  if (dtype == 0) {
    return wave ? launch_one<double, double, true>(a, c, s, t, k, sx, st, batch, n, counter, grid, stream)
                : launch_one<double, double, false>(a, c, s, t, k, sx, st, batch, n, counter, grid, stream);
  }
  if (dtype == 2) {
    return wave ? launch_one<float, double, true>(a, c, s, t, k, sx, st, batch, n, counter, grid, stream)
                : launch_one<float, double, false>(a, c, s, t, k, sx, st, batch, n, counter, grid, stream);
  }
  return wave ? launch_one<float, float, true>(a, c, s, t, k, sx, st, batch, n, counter, grid, stream)
              : launch_one<float, float, false>(a, c, s, t, k, sx, st, batch, n, counter, grid, stream);
}

}  // namespace csm
