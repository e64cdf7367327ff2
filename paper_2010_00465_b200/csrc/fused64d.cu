// fused64d.cu -- K1d: the Taylor cos/sin pipeline for n <= 64 with TWO
// persistent CTAs per SM, so that one matrix's epilogue, barrier and input
// staging run under the other matrix's products.
//
// K1 (fused64.cu) keeps one matrix per SM in seven 32 KiB shared-memory
// slots.  Every product of a chain depends on the previous one, so the FP64
// tensor pipe idles through each step's drain, epilogue and barrier: K1
// measures 0.70 of the DMMA peak, 0.90 in the doubling phase and ~0.66 in
// the Taylor phase.  Only a second, independent matrix
// can fill those bubbles, and two K1 contexts do not fit one SM.  K1d shrinks
// a context to fit twice:
//
//  * THREE shared-memory slots (96 KiB) hold only what a coming product
//    reads as an operand.  A step whose outputs replace its own operands is
//    two-phase: product, barrier (every warp has read the operands),
//    epilogue writes, barrier.  The doubling runs S' = 2 S C and
//    C' = 2 C C - I as two products rotating through the three slots.
//  * Values that later epilogues only read ELEMENTWISE (y, y^2, y^3 / p8,
//    mid, the sine base) live in TENSOR MEMORY: each thread parks its own
//    accumulator-layout elements in its TMEM lane (tcgen05.st) and reads them
//    back in 8-column chunks (tcgen05.ld), four carriers x 64 columns = the
//    256 columns a CTA allocates (two CTAs = the SM's 512).
//  * 256 threads (8 warps of 16 x 32), <= 128 registers, so two CTAs share
//    the register file; no dual product (its second accumulator set would
//    not fit), no register carriers.
//  * The degree-8 chain needs A, p8 and two more operands at once; it drops
//    A after the first product and re-reads it (an L2 hit) before the last.
//  * The next matrix's input arrives by per-thread 16-byte cp.async straight
//    into the swizzled layout of whichever slot the chain frees first (no
//    landing slot, no conversion pass); n < 64, float input or unaligned
//    batches load synchronously at the top of the matrix's turn.
//
// The arithmetic is K1's, operation for operation: the same k order in the
// products and the same fma nesting in the epilogues (copied from
// fused64.cu), so K1d's results are bitwise K1's (tests/test_gpu_k1d.py).
//
// Reference mapping: chains schemes.py:264-361, trig use :376-395, scaling
// driver.py:115, doubling driver.py:91-98.  The wave family stays on K1.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace csm {

namespace f64k {

template <> struct Geo<7> {
  static constexpr bool ROTATE = false;
  static constexpr int CL = 1, NP = 64, BAND = 64, THREADS = 256, MI = 2, NI = 4;
};

enum DEpi : int8_t {
  D_Y,       // o0 = y = scale * acc ; T0 = y
  D_DEG2,    // o0 = cos = I - y/2 + acc/24 ; o1 = sc = I - y/6 + acc/120
  D_DEG4A,   // o0 = y2 = acc (T1) ; o1 = -y/720 + acc/40320
  D_DEG4B,   // o0 = cos ; o1 = sc                                  (y, y2)
  D_DEG8A,   // o0 = y2 = acc (T1) ; o1 = x1 y + x2 acc
  D_DEG8B,   // o0 = p8 = acc (T2) ; o1 = x3 y2 + acc ; o2 = x4 I + x5 y + x6 y2 + x7 acc
  D_DEG8C,   // o0 = cos ; o1 = inner ; T3 = sine base              (y, y2, p8)
  D_KEEP8,   // o0 = T3 + acc
  D_Y2,      // o0 = y2 = acc (T1)
  D_DEG12B,  // T2 = y3 = acc ; o0 = c4                             (y, y2)
  D_DEG12C,  // o0 = mid (T3) ; o1 = c2 + mid                       (y, y2, y3)
  D_DEG12D,  // o0 = cos ; o1 = inner ; T0 = sine base              (y, y2, y3, mid)
  D_KEEP12,  // o0 = T0 + acc
  D_SIN,     // o0 = sin = scale * acc
  // wave family (y is the scaled input itself, read from its slot once)
  D_W1,      // o0 = y2 = acc (T1) ; o1 = -y/720 + acc/40320 ; o2 = -y/5040 + acc/9! ; T0 = y
  D_W2C,     // o0 = cos = I - y/2 + y2/24 + acc
  D_W2S,     // o0 = s = scale * (I - y/6 + y2/120 + acc)
  D_W8A,     // D_DEG8A with y from its slot ; T0 = y
  D_WY2,     // D_Y2 with T0 = y copied from its slot
  D_KEEPW8,  // o0 = scale * (T3 + acc)
  D_KEEPW12, // o0 = scale * (T0 + acc)
};

struct __align__(8) DStep {
  int8_t l, r;        // operand slots (logical 0..2)
  int8_t epi;
  int8_t o0, o1, o2;  // output slots (-1 unused)
  int8_t two_phase;   // outputs replace this step's operands: barrier before the writes
  int8_t reload;      // re-read A into this slot once the operands have been read (-1: no)
};
static_assert(sizeof(DStep) == 8, "one 64-bit load per step");

struct __align__(8) DChain {
  int8_t nsteps;
  int8_t pf_step;    // s == 0: logical slot 2 is free once this step's operands have been read
  int8_t wait_step;  // the product of this step reads the reloaded A (-1: none)
  int8_t pad[5];
  DStep step[7];
};
static_assert(sizeof(DChain) == 64, "chain table layout");

// Every chain ends with cos in slot 2, sin in slot 1 and slot 0 free.
#define DS_(l, r, e, o0, o1, o2, tp, rl) {l, r, e, o0, o1, o2, tp, rl}
__constant__ DChain kDChains[7] = {
    // [0] Taylor k=3: chain_deg2 (schemes.py:264-272)
    {3, 1, -1, {0, 0, 0, 0, 0},
     {DS_(0, 0, D_Y, 1, X, X, 0, X),        // y = A A
      DS_(1, 1, D_DEG2, 2, 1, X, 1, X),     // cos, sc (over y)
      DS_(0, 1, D_SIN, 1, X, X, 1, X)}},    // sin = A sc (over sc)
    // [1] Taylor k=4: chain_deg4(exact_sine=False) (:275-299)
    {4, 2, -1, {0, 0, 0, 0, 0},
     {DS_(0, 0, D_Y, 1, X, X, 0, X),
      DS_(1, 1, D_DEG4A, 2, 1, X, 1, X),    // y2, L (over y)
      DS_(2, 1, D_DEG4B, 2, 1, X, 1, X),    // cos (over y2), sc (over L)
      DS_(0, 1, D_SIN, 1, X, X, 1, X)}},
    // [2] Taylor k=6: chain_deg8 (:302-326); A is dropped and re-read
    {6, 3, 5, {0, 0, 0, 0, 0},
     {DS_(0, 0, D_Y, 1, X, X, 0, X),
      DS_(1, 1, D_DEG8A, 2, 0, X, 0, X),    // y2, L (over A)
      DS_(2, 0, D_DEG8B, 1, 2, 0, 1, X),    // p8 (over y), L2 (over y2), R2 (over L)
      DS_(2, 0, D_DEG8C, 2, 0, X, 1, X),    // cos (over L2), inner (over R2)
      DS_(0, 1, D_KEEP8, 1, X, X, 1, 0),    // sc (over p8); A comes back over inner
      DS_(0, 1, D_SIN, 1, X, X, 1, X)}},
    // [3] Taylor k=7: chain_deg12 (:329-361)
    {7, 5, -1, {0, 0, 0, 0, 0},
     {DS_(0, 0, D_Y, 1, X, X, 0, X),
      DS_(1, 1, D_Y2, 2, X, X, 0, X),
      DS_(2, 1, D_DEG12B, 2, X, X, 1, X),   // c4 (over y2); y3 stays in TMEM
      DS_(2, 2, D_DEG12C, 1, 2, X, 1, X),   // mid (over y), L (over c4)
      DS_(2, 1, D_DEG12D, 2, 1, X, 1, X),   // cos (over L), inner (over mid)
      DS_(1, 2, D_KEEP12, 1, X, X, 1, X),   // sc (over inner)
      DS_(0, 1, D_SIN, 1, X, X, 1, X)}},
    // [4] wave k=3: chain_deg4(exact_sine=True) on y = (t')^2 A (schemes.py:426-427);
    // K1's dual product [L; L9] y2 runs as two products
    {3, 1, -1, {0, 0, 0, 0, 0},
     {DS_(0, 0, D_W1, 1, 2, 0, 1, X),       // y2, L, L9 (over y)
      DS_(2, 1, D_W2C, 2, X, X, 1, X),      // cos = ... + L y2 (over L)
      DS_(0, 1, D_W2S, 1, X, X, 1, X)}},    // s = t' (... + L9 y2) (over y2)
    // [5] wave k=4: chain_deg8 on y
    {4, 2, -1, {0, 0, 0, 0, 0},
     {DS_(0, 0, D_W8A, 1, 2, X, 0, X),      // y2, L
      DS_(1, 2, D_DEG8B, 0, 1, 2, 1, X),    // p8 (over y), L2 (over y2), R2 (over L)
      DS_(1, 2, D_DEG8C, 2, 1, X, 1, X),    // cos (over R2), inner (over L2)
      DS_(1, 0, D_KEEPW8, 1, X, X, 1, X)}}, // s (over inner)
    // [6] wave k=5: chain_deg12 on y
    {5, 4, -1, {0, 0, 0, 0, 0},
     {DS_(0, 0, D_WY2, 1, X, X, 0, X),      // y2
      DS_(1, 0, D_DEG12B, 2, X, X, 0, X),   // c4; y3 stays in TMEM
      DS_(2, 2, D_DEG12C, 0, 1, X, 0, X),   // mid (over y), L (over y2)
      DS_(1, 0, D_DEG12D, 2, 1, X, 1, X),   // cos (over c4), inner (over L)
      DS_(1, 2, D_KEEPW12, 1, X, X, 1, X)}},// s (over inner)
};
#undef DS_

// ---------------------------------------------------------------------------
// Tensor memory as a per-thread store.  A carrier is the thread's 16
// accumulator-layout doubles (tile P, element e at columns 4 P + 2 e, +1) in
// its own lane; a chunk is the 8 columns of tiles 2h, 2h + 1.

struct Car { uint32_t w[8]; };

__device__ __forceinline__ void tm_ld8(uint32_t addr, Car& c) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(c.w[0]), "=r"(c.w[1]), "=r"(c.w[2]), "=r"(c.w[3]), "=r"(c.w[4]),
                 "=r"(c.w[5]), "=r"(c.w[6]), "=r"(c.w[7])
               : "r"(addr)
               : "memory");
}
__device__ __forceinline__ void tm_st8(uint32_t addr, const Car& c) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::
                   "r"(addr),
               "r"(c.w[0]), "r"(c.w[1]), "r"(c.w[2]), "r"(c.w[3]), "r"(c.w[4]), "r"(c.w[5]),
               "r"(c.w[6]), "r"(c.w[7])
               : "memory");
}
// The loaded registers pass through the wait so that no use is scheduled
// before it.
__device__ __forceinline__ void tm_wait_ld(Car& a) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(a.w[0]), "+r"(a.w[1]), "+r"(a.w[2]), "+r"(a.w[3]), "+r"(a.w[4]),
                 "+r"(a.w[5]), "+r"(a.w[6]), "+r"(a.w[7])
               :
               : "memory");
}
__device__ __forceinline__ void tm_wait_ld(Car& a, Car& b) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(a.w[0]), "+r"(a.w[1]), "+r"(a.w[2]), "+r"(a.w[3]), "+r"(a.w[4]),
                 "+r"(a.w[5]), "+r"(a.w[6]), "+r"(a.w[7]), "+r"(b.w[0]), "+r"(b.w[1]),
                 "+r"(b.w[2]), "+r"(b.w[3]), "+r"(b.w[4]), "+r"(b.w[5]), "+r"(b.w[6]),
                 "+r"(b.w[7])
               :
               : "memory");
}
__device__ __forceinline__ void tm_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}
// element e of tile j (0 or 1) of the chunk
__device__ __forceinline__ double car_get(const Car& c, int j, int e) {
  return __hiloint2double(static_cast<int>(c.w[4 * j + 2 * e + 1]),
                          static_cast<int>(c.w[4 * j + 2 * e]));
}
__device__ __forceinline__ void car_set(Car& c, int j, int e, double v) {
  c.w[4 * j + 2 * e] = static_cast<uint32_t>(__double2loint(v));
  c.w[4 * j + 2 * e + 1] = static_cast<uint32_t>(__double2hiint(v));
}

// Power-of-two scalings without the FP64 pipe.  The two CTAs of an SM share
// it: while one runs a product, every DMUL / DFMA of the other's epilogue
// queues behind DMMAs (measured: a 16-DMUL epilogue took 3.5 k cycles under
// the other CTA's product).  x * 2^-m and 2 x are exponent arithmetic
// whenever x and the result are normal numbers -- bit for bit the product's
// value; zeros, subnormals, infinities and NaNs take the multiply.
// The caller tests the whole accumulator set once (exp_range_ok) and
// branches between an all-integer and an all-multiply epilogue, so the fast
// path really contains no FP64 instruction (a per-element select would be
// if-converted into multiply + select).
__device__ __forceinline__ bool exp_range_ok(const Acc& acc, int m) {
  // every element: m < biased exponent < 0x7fe (normal, and normal after the
  // shift by -m or +1)
  bool ok = true;
#pragma unroll
  for (int P = 0; P < 8; ++P)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int ex = (__double2hiint(acc[P][e]) >> 20) & 0x7ff;
      ok = ok && ex > m && ex < 0x7fe;
    }
  // warp-uniform: the TMEM stores inside the branches are .sync.aligned
  return __all_sync(0xffffffffu, ok);
}
__device__ __forceinline__ double exp_add(double x, int d) {  // x * 2^d by exponent arithmetic
  return __hiloint2double(__double2hiint(x) + d * (1 << 20), __double2loint(x));
}

template <typename TOut>
struct DArgs {
  double* sm;     // the CTA's slots
  int o[3];       // shared-memory outputs as slot offsets in doubles (-1: not written)
  TOut* g;        // global destination of this step's final output (s == 0), or nullptr
  double scale;   // 2^-shift (Taylor), t' (wave)
  int shift;
  int yin;        // wave: slot offset of y for the epilogues that read it from shared memory
  int n;
  uint32_t tm;    // this thread's TMEM base (lane quarter, warp column half)
};

constexpr uint32_t kCarCols = 64;  // columns per carrier (8 warps: 2 per lane quarter x 32)

// One epilogue over the thread's four chunks.  BODY sees, per tile j of the
// chunk: r, c, off (swizzled), I0/I1 (identity), p0/p1 (accumulator).
#define D_TILES(...)                                                         \
  _Pragma("unroll") for (int j = 0; j < 2; ++j) {                            \
    const int P = 2 * h + j;                                                 \
    const int r = ln.rb + (h >> 1) * 8 + ln.g;                               \
    const int c = ln.cb + (2 * (h & 1) + j) * 8 + 2 * ln.t;                  \
    const int off = swz<64>(r, c);                                           \
    const double I0 = (r == c) ? 1.0 : 0.0, I1 = (r == c + 1) ? 1.0 : 0.0;   \
    const double p0 = acc[P][0], p1 = acc[P][1];                             \
    (void)I0; (void)I1; (void)off;                                           \
    __VA_ARGS__                                                              \
  }
#define D_CHUNKS(...) _Pragma("unroll") for (int h = 0; h < 4; ++h) { __VA_ARGS__ }

// coef * I_rc.  SEL: without a multiply per element -- the coefficient on the
// diagonal, coef * 0.0 (a signed zero, computed once per epilogue) elsewhere:
// the product's value exactly, and one FP64 instruction less per term to
// wait out the other CTA's DMMAs.  Used by the wave kernel (1.778 -> 1.767
// ms); in the Taylor kernel, at the register cap, it spills (2.161 -> 2.177).
template <bool SEL>
__device__ __forceinline__ double idt(double coef, bool on) {
  return SEL ? (on ? coef : coef * 0.0) : coef * (on ? 1.0 : 0.0);
}

template <typename TOut>
__device__ __forceinline__ void dput(const DArgs<TOut>& E, int q, int off, double v0, double v1) {
  if (E.o[q] >= 0) st2(E.sm, E.o[q] + off, v0, v1);
}

template <bool WAVE, typename TOut>
__device__ __forceinline__ void depilogue(int epi, const DArgs<TOut>& E, const Acc& acc,
                                          const Lane<7>& ln) {
  // (each family's kernel compiles only its own cases: the Taylor kernel sits
  // at the register cap, and more code in this switch makes it spill)
  if (WAVE ? (epi == D_Y || epi == D_DEG2 || epi == D_DEG4A || epi == D_DEG4B || epi == D_DEG8A ||
              epi == D_Y2 || epi == D_KEEP8 || epi == D_KEEP12 || epi == D_SIN)
           : epi >= D_W1)
    return;
  // this thread's TMEM stores of the previous epilogue (they completed under
  // the product in between; the wait orders them before the reads below)
  tm_wait_st();
  const double* x = dTables.x8;  // x[0] = x1
  const double* z8 = dTables.z8;
  const double(*a)[4] = dTables.a12;  // a[j-1][i]
  const double* z = dTables.z12;
  const uint32_t T0 = E.tm, T1 = E.tm + kCarCols, T2 = E.tm + 2 * kCarCols,
                 T3 = E.tm + 3 * kCarCols;
  switch (epi) {
    case D_Y:
      if constexpr (!WAVE) {
      if (exp_range_ok(acc, E.shift)) {
        D_CHUNKS({
          Car cy;
          D_TILES({
            const double v0 = exp_add(p0, -E.shift), v1 = exp_add(p1, -E.shift);
            dput(E, 0, off, v0, v1);
            car_set(cy, j, 0, v0);
            car_set(cy, j, 1, v1);
          })
          tm_st8(T0 + 8 * h, cy);
        })
      } else {
        D_CHUNKS({
          Car cy;
          D_TILES({
            const double v0 = E.scale * p0, v1 = E.scale * p1;
            dput(E, 0, off, v0, v1);
            car_set(cy, j, 0, v0);
            car_set(cy, j, 1, v1);
          })
          tm_st8(T0 + 8 * h, cy);
        })
      }
      }
      break;
    case D_SIN:
      if constexpr (!WAVE) {
      if (exp_range_ok(acc, E.shift)) {
        D_CHUNKS({
          D_TILES({
            const double v0 = exp_add(p0, -E.shift), v1 = exp_add(p1, -E.shift);
            dput(E, 0, off, v0, v1);
            if (E.g) gstore<64>(E.g, E.n, r, c, v0, v1);
          })
        })
      } else {
        D_CHUNKS({
          D_TILES({
            const double v0 = E.scale * p0, v1 = E.scale * p1;
            dput(E, 0, off, v0, v1);
            if (E.g) gstore<64>(E.g, E.n, r, c, v0, v1);
          })
        })
      }
      }
      break;
    case D_Y2:
      if constexpr (!WAVE) {
      D_CHUNKS({
        Car cy2;
        D_TILES({
          dput(E, 0, off, p0, p1);
          car_set(cy2, j, 0, p0);
          car_set(cy2, j, 1, p1);
        })
        tm_st8(T1 + 8 * h, cy2);
      })
      }
      break;
    case D_DEG2:
      if constexpr (!WAVE) {
      D_CHUNKS({
        Car cy;
        tm_ld8(T0 + 8 * h, cy);
        tm_wait_ld(cy);
        D_TILES({
          const double y0 = car_get(cy, j, 0), y1 = car_get(cy, j, 1);
          const double c0 = fma(1.0 / 24.0, p0, fma(-0.5, y0, I0));
          const double c1 = fma(1.0 / 24.0, p1, fma(-0.5, y1, I1));
          dput(E, 0, off, c0, c1);
          if (E.g) gstore<64>(E.g, E.n, r, c, c0, c1);
          dput(E, 1, off, fma(1.0 / 120.0, p0, fma(-1.0 / 6.0, y0, I0)),
               fma(1.0 / 120.0, p1, fma(-1.0 / 6.0, y1, I1)));
        })
      })
      }
      break;
    case D_DEG4A:
      if constexpr (!WAVE) {
      D_CHUNKS({
        Car cy, cy2;
        tm_ld8(T0 + 8 * h, cy);
        tm_wait_ld(cy);
        D_TILES({
          const double y0 = car_get(cy, j, 0), y1 = car_get(cy, j, 1);
          dput(E, 0, off, p0, p1);
          car_set(cy2, j, 0, p0);
          car_set(cy2, j, 1, p1);
          dput(E, 1, off, fma(1.0 / 40320.0, p0, (-1.0 / 720.0) * y0),
               fma(1.0 / 40320.0, p1, (-1.0 / 720.0) * y1));
        })
        tm_st8(T1 + 8 * h, cy2);
      })
      }
      break;
    case D_DEG4B:
      if constexpr (!WAVE) {
      D_CHUNKS({
        Car cy, cy2;
        tm_ld8(T0 + 8 * h, cy);
        tm_ld8(T1 + 8 * h, cy2);
        tm_wait_ld(cy, cy2);
        D_TILES({
          const double y0 = car_get(cy, j, 0), y1 = car_get(cy, j, 1);
          const double q0 = car_get(cy2, j, 0), q1 = car_get(cy2, j, 1);
          const double c0 = p0 + fma(1.0 / 24.0, q0, fma(-0.5, y0, I0));
          const double c1 = p1 + fma(1.0 / 24.0, q1, fma(-0.5, y1, I1));
          dput(E, 0, off, c0, c1);
          if (E.g) gstore<64>(E.g, E.n, r, c, c0, c1);
          dput(E, 1, off,
               fma(720.0 / 5040.0, p0, fma(1.0 / 120.0, q0, fma(-1.0 / 6.0, y0, I0))),
               fma(720.0 / 5040.0, p1, fma(1.0 / 120.0, q1, fma(-1.0 / 6.0, y1, I1))));
        })
      })
      }
      break;
    case D_DEG8A:
      if constexpr (!WAVE) {
      D_CHUNKS({
        Car cy, cy2;
        tm_ld8(T0 + 8 * h, cy);
        tm_wait_ld(cy);
        D_TILES({
          const double y0 = car_get(cy, j, 0), y1 = car_get(cy, j, 1);
          dput(E, 0, off, p0, p1);
          car_set(cy2, j, 0, p0);
          car_set(cy2, j, 1, p1);
          dput(E, 1, off, fma(x[1], p0, x[0] * y0), fma(x[1], p1, x[0] * y1));
        })
        tm_st8(T1 + 8 * h, cy2);
      })
      }
      break;
    case D_DEG8B:
      D_CHUNKS({
        Car cy, cy2, cp8;
        tm_ld8(T0 + 8 * h, cy);
        tm_ld8(T1 + 8 * h, cy2);
        tm_wait_ld(cy, cy2);
        D_TILES({
          const double y0 = car_get(cy, j, 0), y1 = car_get(cy, j, 1);
          const double q0 = car_get(cy2, j, 0), q1 = car_get(cy2, j, 1);
          dput(E, 0, off, p0, p1);
          car_set(cp8, j, 0, p0);
          car_set(cp8, j, 1, p1);
          dput(E, 1, off, fma(x[2], q0, p0), fma(x[2], q1, p1));
          dput(E, 2, off, fma(x[6], p0, fma(x[5], q0, fma(x[4], y0, idt<WAVE>(x[3], r == c)))),
               fma(x[6], p1, fma(x[5], q1, fma(x[4], y1, idt<WAVE>(x[3], r == c + 1)))));
        })
        tm_st8(T2 + 8 * h, cp8);
      })
      break;
    case D_DEG8C:
      D_CHUNKS({
        Car cy, cy2, cp8, ck;
        tm_ld8(T0 + 8 * h, cy);
        tm_ld8(T1 + 8 * h, cy2);
        tm_ld8(T2 + 8 * h, cp8);
        tm_wait_ld(cy, cy2);
        tm_wait_ld(cp8);
        D_TILES({
          const double y0 = car_get(cy, j, 0), y1 = car_get(cy, j, 1);
          const double q0 = car_get(cy2, j, 0), q1 = car_get(cy2, j, 1);
          const double e0 = car_get(cp8, j, 0), e1 = car_get(cp8, j, 1);
          const double c0 = p0 + fma(x[7], q0, fma(-0.5, y0, I0));
          const double c1 = p1 + fma(x[7], q1, fma(-0.5, y1, I1));
          // inner = z5 I + z5 y + z6 y2 + z7 p8 + z8 cos
          const double n0 = fma(z8[8], c0, fma(z8[7], e0, fma(z8[6], q0, fma(z8[5], y0, idt<WAVE>(z8[5], r == c)))));
          const double n1 = fma(z8[8], c1, fma(z8[7], e1, fma(z8[6], q1, fma(z8[5], y1, idt<WAVE>(z8[5], r == c + 1)))));
          // sin base = z0 I + z1 y + z2 y2 + z3 p8 + z4 cos
          car_set(ck, j, 0, fma(z8[4], c0, fma(z8[3], e0, fma(z8[2], q0, fma(z8[1], y0, idt<WAVE>(z8[0], r == c))))));
          car_set(ck, j, 1, fma(z8[4], c1, fma(z8[3], e1, fma(z8[2], q1, fma(z8[1], y1, idt<WAVE>(z8[0], r == c + 1))))));
          dput(E, 0, off, c0, c1);
          if (E.g) gstore<64>(E.g, E.n, r, c, c0, c1);
          dput(E, 1, off, n0, n1);
        })
        tm_st8(T3 + 8 * h, ck);
      })
      break;
    case D_KEEP8:
    case D_KEEP12: {
      if constexpr (!WAVE) {
      const uint32_t TK = epi == D_KEEP8 ? T3 : T0;
      D_CHUNKS({
        Car ck;
        tm_ld8(TK + 8 * h, ck);
        tm_wait_ld(ck);
        D_TILES({
          dput(E, 0, off, car_get(ck, j, 0) + p0, car_get(ck, j, 1) + p1);
        })
      })
      }
      break;
    }
    case D_DEG12B:
      D_CHUNKS({
        Car cy, cy2, cy3;
        tm_ld8(T0 + 8 * h, cy);
        tm_ld8(T1 + 8 * h, cy2);
        tm_wait_ld(cy, cy2);
        D_TILES({
          const double y0 = car_get(cy, j, 0), y1 = car_get(cy, j, 1);
          const double q0 = car_get(cy2, j, 0), q1 = car_get(cy2, j, 1);
          car_set(cy3, j, 0, p0);
          car_set(cy3, j, 1, p1);
          dput(E, 0, off, fma(a[3][3], p0, fma(a[3][2], q0, fma(a[3][1], y0, idt<WAVE>(a[3][0], r == c)))),
               fma(a[3][3], p1, fma(a[3][2], q1, fma(a[3][1], y1, idt<WAVE>(a[3][0], r == c + 1)))));
        })
        tm_st8(T2 + 8 * h, cy3);
      })
      break;
    case D_DEG12C:
      D_CHUNKS({
        Car cy, cy2, cy3, cm;
        tm_ld8(T0 + 8 * h, cy);
        tm_ld8(T1 + 8 * h, cy2);
        tm_ld8(T2 + 8 * h, cy3);
        tm_wait_ld(cy, cy2);
        tm_wait_ld(cy3);
        D_TILES({
          const double y0 = car_get(cy, j, 0), y1 = car_get(cy, j, 1);
          const double q0 = car_get(cy2, j, 0), q1 = car_get(cy2, j, 1);
          const double u0 = car_get(cy3, j, 0), u1 = car_get(cy3, j, 1);
          const double m0 = fma(a[2][3], u0, fma(a[2][2], q0, fma(a[2][1], y0, idt<WAVE>(a[2][0], r == c)))) + p0;
          const double m1 = fma(a[2][3], u1, fma(a[2][2], q1, fma(a[2][1], y1, idt<WAVE>(a[2][0], r == c + 1)))) + p1;
          const double l0 = fma(a[1][3], u0, fma(a[1][2], q0, fma(a[1][1], y0, idt<WAVE>(a[1][0], r == c)))) + m0;
          const double l1 = fma(a[1][3], u1, fma(a[1][2], q1, fma(a[1][1], y1, idt<WAVE>(a[1][0], r == c + 1)))) + m1;
          dput(E, 0, off, m0, m1);
          car_set(cm, j, 0, m0);
          car_set(cm, j, 1, m1);
          dput(E, 1, off, l0, l1);
        })
        tm_st8(T3 + 8 * h, cm);
      })
      break;
    case D_DEG12D:
      D_CHUNKS({
        Car cy, cy2, cy3, cm;
        tm_ld8(T0 + 8 * h, cy);
        tm_ld8(T1 + 8 * h, cy2);
        tm_ld8(T2 + 8 * h, cy3);
        tm_ld8(T3 + 8 * h, cm);
        tm_wait_ld(cy, cy2);
        tm_wait_ld(cy3, cm);
        Car ck;
        D_TILES({
          const double y0 = car_get(cy, j, 0), y1 = car_get(cy, j, 1);
          const double q0 = car_get(cy2, j, 0), q1 = car_get(cy2, j, 1);
          const double u0 = car_get(cy3, j, 0), u1 = car_get(cy3, j, 1);
          const double d0 = car_get(cm, j, 0), d1 = car_get(cm, j, 1);
          const double c0 = fma(a[0][3], u0, fma(a[0][2], q0, fma(a[0][1], y0, idt<WAVE>(a[0][0], r == c)))) + p0;
          const double c1 = fma(a[0][3], u1, fma(a[0][2], q1, fma(a[0][1], y1, idt<WAVE>(a[0][0], r == c + 1)))) + p1;
          const double n0 = fma(z[11], c0, fma(z[10], d0, fma(z[9], u0, fma(z[8], q0, fma(z[7], y0, idt<WAVE>(z[6], r == c))))));
          const double n1 = fma(z[11], c1, fma(z[10], d1, fma(z[9], u1, fma(z[8], q1, fma(z[7], y1, idt<WAVE>(z[6], r == c + 1))))));
          car_set(ck, j, 0, fma(z[5], c0, fma(z[4], d0, fma(z[3], u0, fma(z[2], q0, fma(z[1], y0, idt<WAVE>(z[0], r == c)))))));
          car_set(ck, j, 1, fma(z[5], c1, fma(z[4], d1, fma(z[3], u1, fma(z[2], q1, fma(z[1], y1, idt<WAVE>(z[0], r == c + 1)))))));
          dput(E, 0, off, c0, c1);
          if (E.g) gstore<64>(E.g, E.n, r, c, c0, c1);
          dput(E, 1, off, n0, n1);
        })
        tm_st8(T0 + 8 * h, ck);  // the sine base takes y's place
      })
      break;
    case D_W1:
      if constexpr (WAVE) {
      D_CHUNKS({
        Car cy, cy2;
        D_TILES({
          const double2 y = ld2(E.sm, E.yin + off);
          car_set(cy, j, 0, y.x);
          car_set(cy, j, 1, y.y);
          car_set(cy2, j, 0, p0);
          car_set(cy2, j, 1, p1);
          const double l0 = fma(1.0 / 40320.0, p0, (-1.0 / 720.0) * y.x);
          const double l1 = fma(1.0 / 40320.0, p1, (-1.0 / 720.0) * y.y);
          const double m0 = fma(1.0 / 362880.0, p0, (-1.0 / 5040.0) * y.x);
          const double m1 = fma(1.0 / 362880.0, p1, (-1.0 / 5040.0) * y.y);
          dput(E, 0, off, p0, p1);
          dput(E, 1, off, l0, l1);
          dput(E, 2, off, m0, m1);  // over y, at this thread's own pair
        })
        tm_st8(T0 + 8 * h, cy);
        tm_st8(T1 + 8 * h, cy2);
      })
      }
      break;
    case D_W2C:
    case D_W2S:
      if constexpr (WAVE) {
      D_CHUNKS({
        Car cy, cy2;
        tm_ld8(T0 + 8 * h, cy);
        tm_ld8(T1 + 8 * h, cy2);
        tm_wait_ld(cy, cy2);
        D_TILES({
          const double y0 = car_get(cy, j, 0), y1 = car_get(cy, j, 1);
          const double q0 = car_get(cy2, j, 0), q1 = car_get(cy2, j, 1);
          double v0, v1;
          if (epi == D_W2C) {
            v0 = p0 + fma(1.0 / 24.0, q0, fma(-0.5, y0, I0));
            v1 = p1 + fma(1.0 / 24.0, q1, fma(-0.5, y1, I1));
          } else {
            v0 = E.scale * (p0 + fma(1.0 / 120.0, q0, fma(-1.0 / 6.0, y0, I0)));
            v1 = E.scale * (p1 + fma(1.0 / 120.0, q1, fma(-1.0 / 6.0, y1, I1)));
          }
          dput(E, 0, off, v0, v1);
          if (E.g) gstore<64>(E.g, E.n, r, c, v0, v1);
        })
      })
      }
      break;
    case D_W8A:
      if constexpr (WAVE) {
      D_CHUNKS({
        Car cy, cy2;
        D_TILES({
          const double2 y = ld2(E.sm, E.yin + off);
          car_set(cy, j, 0, y.x);
          car_set(cy, j, 1, y.y);
          dput(E, 0, off, p0, p1);
          car_set(cy2, j, 0, p0);
          car_set(cy2, j, 1, p1);
          dput(E, 1, off, fma(x[1], p0, x[0] * y.x), fma(x[1], p1, x[0] * y.y));
        })
        tm_st8(T0 + 8 * h, cy);
        tm_st8(T1 + 8 * h, cy2);
      })
      }
      break;
    case D_WY2:
      if constexpr (WAVE) {
      D_CHUNKS({
        Car cy, cy2;
        D_TILES({
          const double2 y = ld2(E.sm, E.yin + off);
          car_set(cy, j, 0, y.x);
          car_set(cy, j, 1, y.y);
          dput(E, 0, off, p0, p1);
          car_set(cy2, j, 0, p0);
          car_set(cy2, j, 1, p1);
        })
        tm_st8(T0 + 8 * h, cy);
        tm_st8(T1 + 8 * h, cy2);
      })
      }
      break;
    case D_KEEPW8:
    case D_KEEPW12: {
      if constexpr (WAVE) {
      const uint32_t TK = epi == D_KEEPW8 ? T3 : T0;
      D_CHUNKS({
        Car ck;
        tm_ld8(TK + 8 * h, ck);
        tm_wait_ld(ck);
        D_TILES({
          const double v0 = E.scale * (car_get(ck, j, 0) + p0);
          const double v1 = E.scale * (car_get(ck, j, 1) + p1);
          dput(E, 0, off, v0, v1);
          if (E.g) gstore<64>(E.g, E.n, r, c, v0, v1);
        })
      })
      }
      break;
    }
    default:
      break;
  }
}

// Doubling epilogues (driver.py:95-97): S' = 2 acc, or C' = 2 acc - I.  Off
// the diagonal fma(2, p, -0.0) = 2 p (signed zeros included), so only the
// diagonal elements need the FP64 pipe.
template <typename TOut>
__device__ __forceinline__ void ddouble_out(const Acc& acc, bool is_cos, double* dst, TOut* gdst,
                                            int n, const Lane<7>& ln) {
  if (exp_range_ok(acc, 0)) {
    D_CHUNKS({
      D_TILES({
        double v0 = exp_add(p0, 1), v1 = exp_add(p1, 1);
        if (is_cos && r == c) v0 = fma(2.0, p0, -1.0);
        if (is_cos && r == c + 1) v1 = fma(2.0, p1, -1.0);
        if (gdst) gstore<64>(gdst, n, r, c, v0, v1);
        else st2(dst, off, v0, v1);
      })
    })
  } else {
    D_CHUNKS({
      D_TILES({
        const double v0 = is_cos ? fma(2.0, p0, -I0) : 2.0 * p0;
        const double v1 = is_cos ? fma(2.0, p1, -I1) : 2.0 * p1;
        if (gdst) gstore<64>(gdst, n, r, c, v0, v1);
        else st2(dst, off, v0, v1);
      })
    })
  }
}
#undef D_TILES
#undef D_CHUNKS

// Matrix (n x n row-major) -> slot, swizzled.  FAST: n == 64 fp64, 16-byte
// chunks by cp.async (asynchronous; the caller commits and waits).
__device__ __forceinline__ void dload_async(double* slot, const double* src) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int q = threadIdx.x + 256 * i, r = q >> 5, pi = q & 31;
    cp_async16(slot + r * 64 + 2 * (pi ^ swz_f(r)), src + 2 * q);
  }
}
template <bool SCALE, typename TIn>
__device__ __forceinline__ void dload_sync(double* slot, const TIn* src, int n,
                                           double g = 1.0) {
#pragma unroll 2
  for (int p = threadIdx.x; p < 2048; p += 256) {
    const int r = p >> 5, c = (p & 31) * 2;
    double v0 = 0.0, v1 = 0.0;
    if (r < n) {
      if (c < n) v0 = static_cast<double>(src[r * n + c]);
      if (c + 1 < n) v1 = static_cast<double>(src[r * n + c + 1]);
    }
    if (SCALE) st2(slot, swz<64>(r, c), g * v0, g * v1);  // wave: y = (t')^2 A, schemes.py:424
    else st2(slot, swz<64>(r, c), v0, v1);
  }
}

#ifdef CSM_TRACE
__device__ unsigned long long g_k1d_cta[1024][4];  // per CTA: smid, start ns, end ns, matrices
#endif

template <typename TIn, typename TOut, bool WAVE>
__global__ void __launch_bounds__(256, 2)
fused64d_kernel(const TIn* __restrict__ Ain, TOut* __restrict__ Cout, TOut* __restrict__ Sout,
                const double* __restrict__ T, const int32_t* __restrict__ K,
                const int32_t* __restrict__ Sx,
                const int32_t* __restrict__ ST, const int32_t* __restrict__ order,
                int64_t batch, int n, int fast, unsigned* __restrict__ ticket) {
  extern __shared__ __align__(128) double smem[];
  __shared__ int sh_b[4];
  __shared__ int sh_meta[2][4];
  __shared__ double sh_t[2];
  __shared__ uint32_t sh_tmem;
  __shared__ DChain sh_chain[7];
  const int tid = threadIdx.x;
#ifdef CSM_TRACE
  unsigned long long cta_t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(cta_t0));
#endif
  Lane<7> ln;
  make_lane(ln, 0);
  const size_t nn = static_cast<size_t>(n) * n;
  // FAST (fp64, n == 64, aligned): asynchronous input, one matrix ahead.  The
  // wave family then scales it in place, y = (t')^2 A, at the top of its turn.
  const bool is_fast = sizeof(TIn) == 8 && fast != 0;
  auto fetch = [&](int b, double* slot) {  // all threads
    if (is_fast && b >= 0)
      dload_async(slot, reinterpret_cast<const double*>(Ain) + static_cast<size_t>(b) * nn);
    cp_async_commit();
  };

  for (int i = tid; i < static_cast<int>(sizeof(kDChains) / 4); i += 256)
    reinterpret_cast<int*>(sh_chain)[i] = reinterpret_cast<const int*>(kDChains)[i];
  if ((tid >> 5) == 0) {  // warp 0 owns this CTA's 256 TMEM columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(
                     smem_u32(&sh_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  // Work distribution: order[] lists the matrices by descending cost; every
  // CTA draws the next position from one global ticket counter (zeroed by
  // the launcher).  The two CTAs of an SM do not get equal shares of the
  // FP64 pipe, so a static split leaves one of them running alone at the
  // end (measured: 15% of the kernel); tickets end them within a few cheap
  // matrices of each other.  Thread 0 draws three turns ahead, so the
  // atomic's latency is never waited for.
  unsigned pend = 0;  // thread 0: the ticket of turn it + 2
  if (tid == 0) {
    const unsigned t0 = atomicAdd(ticket, 1u), t1 = atomicAdd(ticket, 1u);
    pend = atomicAdd(ticket, 1u);
    const int b0 = t0 < batch ? order[t0] : -1;
    sh_b[0] = b0;
    sh_b[1] = t1 < batch ? order[t1] : -1;
    if (b0 >= 0) {
      sh_meta[0][0] = K[b0]; sh_meta[0][1] = Sx[b0]; sh_meta[0][2] = ST[b0];
      if (WAVE) sh_t[0] = T[b0];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tm = sh_tmem + (static_cast<uint32_t>(32 * ((tid >> 5) & 3)) << 16) +
                      static_cast<uint32_t>(32 * (tid >> 7));
  // logical slot -> offset (in doubles) of its physical slot; pointers are
  // formed as smem + offset at each use so that they stay shared-space
  int so[3] = {0, SLOT, 2 * SLOT};
  fetch(sh_b[0], smem + so[0]);

#ifdef CSM_TRACE
  if (tid == CSM_TRACE_TID) trace_count() = 0;
#endif
  Acc acc, unused;
  for (int it = 0;; ++it) {
    TRACE_T(14);
    cp_async_wait_all();
    __syncthreads();
    const int b = sh_b[it & 3], bn = sh_b[(it + 1) & 3];
    if (b < 0) break;
    const int k = sh_meta[it & 1][0], s = sh_meta[it & 1][1], status = sh_meta[it & 1][2];
    if (tid == 0) {  // stage ids and metadata for the coming turns
      const unsigned p2 = pend;
      pend = atomicAdd(ticket, 1u);
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
    // wave: t' = t / 2**s (driver.py:139), y = (t' t') a (schemes.py:424)
    double tp = 0.0;
    if (WAVE) tp = sh_t[it & 1] / ldexp(1.0, s);
    if (!is_fast && status == 0) {
      dload_sync<WAVE>(smem + so[0], Ain + static_cast<size_t>(b) * nn, n, tp * tp);
      __syncthreads();
    } else if (WAVE && status == 0) {  // each thread scales the chunks it fetched
      const double g = tp * tp;
      double* slot = smem + so[0];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int q = tid + 256 * i, r = q >> 5, pi = q & 31;
        const int off = r * 64 + 2 * (pi ^ swz_f(r));
        const double2 v = ld2(slot, off);
        st2(slot, off, g * v.x, g * v.y);
      }
      __syncthreads();
    }
    TOut* cdst = Cout + static_cast<size_t>(b) * nn;
    TOut* sdst = Sout + static_cast<size_t>(b) * nn;
    if (status != 0) {
      store_nan<256>(cdst, n, 0, 64);
      store_nan<256>(sdst, n, 0, 64);
      fetch(bn, smem + so[0]);  // the unused input's slot takes the next one
      continue;
    }
    TRACE_T(1);
    CSM_TRACE_EV(9, static_cast<unsigned long long>(k * 16 + s));
    // driver.py:115, a * 2**-s (folded into the products).  Built from the
    // exponent: an FP64 instruction here would queue behind the other CTA's
    // DMMAs like the epilogues' do
    const double f = s <= 1022 ? __hiloint2double((1023 - s) << 20, 0) : ldexp(1.0, -s);
    const double ff = s <= 511 ? __hiloint2double((1023 - 2 * s) << 20, 0) : f * f;
    const DChain& ch = sh_chain[WAVE ? (k == 3 ? 4 : (k == 4 ? 5 : 6))
                                     : (k == 3 ? 0 : (k == 4 ? 1 : (k == 6 ? 2 : 3)))];
    const int nsteps = ch.nsteps;
    const int pf_step = s == 0 ? ch.pf_step : -1, wait_step = ch.wait_step;
    // cos must reach shared memory when it is a later operand: doubling, or
    // the degree-12 chains' inner * cos
    const bool cos_smem = s != 0 || k == (WAVE ? 5 : 7);
    for (int i = 0; i < nsteps; ++i) {
      const DStep st = ch.step[i];
      if (i == wait_step) {  // the reloaded A
        cp_async_wait_all();
        __syncthreads();
      }
      TRACE_T(2);
      gemm<7, false>(smem + so[st.l], nullptr, rview<7>(smem + so[st.r], 0), acc, unused, ln);
      TRACE_T(3);
      if (st.two_phase) __syncthreads();  // every warp has read the operands
      TRACE_T(8);
      if (st.reload >= 0) {
        if (is_fast) {
          fetch(b, smem + so[st.reload]);
        } else {
          dload_sync<false>(smem + so[st.reload], Ain + static_cast<size_t>(b) * nn, n);
        }
      }
      if (i == pf_step) fetch(bn, smem + so[2]);
      DArgs<TOut> E;
      E.sm = smem;
      E.o[0] = so[st.o0];
      E.o[1] = st.o1 >= 0 ? so[st.o1] : -1;
      E.o[2] = st.o2 >= 0 ? so[st.o2] : -1;
      E.g = nullptr;
      E.scale = 1.0;
      E.shift = 0;
      E.yin = so[0];  // (wave: y is the input itself, logical slot 0)
      E.n = n;
      E.tm = tm;
      const bool makes_cos = st.epi == D_DEG2 || st.epi == D_DEG4B || st.epi == D_DEG8C ||
                             st.epi == D_DEG12D || st.epi == D_W2C;
      if (makes_cos) {
        if (!cos_smem) E.o[0] = -1;
        if (s == 0) E.g = cdst;
      } else if (st.epi == D_SIN) {
        E.scale = f;
        E.shift = s;
        if (s == 0) { E.o[0] = -1; E.g = sdst; }
      } else if (st.epi == D_W2S || st.epi == D_KEEPW8 || st.epi == D_KEEPW12) {
        E.scale = tp;  // s(t', y) = t' (...), schemes.py:429
        if (s == 0) { E.o[0] = -1; E.g = sdst; }
      } else if (st.epi == D_Y) {
        E.scale = ff;
        E.shift = 2 * s;
      }
      depilogue<WAVE>(st.epi, E, acc, ln);
      TRACE_T(4);
      // (the last step of an s = 0 chain writes only global memory, and the
      // barrier at the top of the next turn follows)
      if (!(s == 0 && i == nsteps - 1)) __syncthreads();
      TRACE_T(5);
    }
    // Doubling (driver.py:91-98): C = slot 2, S = slot 1, slot 0 free.
    int C = so[2], S = so[1], F = so[0];
    for (int d = 0; d < s; ++d) {
      const bool last = d == s - 1;
      if (last) fetch(bn, smem + F);  // nothing is written to shared memory any more
      TRACE_T(6);
      gemm<7, false>(smem + S, nullptr, rview<7>(smem + C, 0), acc, unused, ln);
      TRACE_T(10);
#ifdef CSM_TRACE
      {  // the accumulators' arrival (integer consumer: no FP64 instruction)
        int sink = 0;
#pragma unroll
        for (int P = 0; P < 8; ++P) sink ^= __double2hiint(acc[P][0]) ^ __double2hiint(acc[P][1]);
        if (sink == 0x12345678) sh_b[3] = 1;
      }
      TRACE_T(15);
#endif
      ddouble_out<TOut>(acc, false, smem + F, last ? sdst : nullptr, n, ln);
      TRACE_T(11);
      gemm<7, false>(smem + C, nullptr, rview<7>(smem + C, 0), acc, unused, ln);
      TRACE_T(12);
      if (!last) __syncthreads();  // S and C have been read by every warp
      TRACE_T(13);
      ddouble_out<TOut>(acc, true, smem + S, last ? cdst : nullptr, n, ln);
      TRACE_T(7);
      if (!last) {
        __syncthreads();
        const int t = S; S = F; F = C; C = t;  // S' in F, C' in the old S, the old C is free
      }
    }
    // the next input is arriving in: logical slot 2 (s == 0), or F (after doubling)
    const int nxt = s == 0 ? so[2] : F;
    so[0] = nxt;
    so[1] = nxt == 0 ? SLOT : 0;
    so[2] = nxt == 2 * SLOT ? SLOT : 2 * SLOT;
  }
#ifdef CSM_TRACE
  if (tid == 0 && blockIdx.x < 1024) {
    unsigned smid;
    unsigned long long t1;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    g_k1d_cta[blockIdx.x][0] = smid;
    g_k1d_cta[blockIdx.x][1] = cta_t0;
    g_k1d_cta[blockIdx.x][2] = t1;
  }
#endif
  tm_wait_st();
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if ((tid >> 5) == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(sh_tmem));
}

}  // namespace f64k

size_t fused64d_smem_bytes() { return 3 * static_cast<size_t>(f64k::SLOT) * sizeof(double); }

template <typename TIn, typename TOut, bool WAVE>
static cudaError_t launch_k1d(const void* a, void* c, void* s, const double* t, const int32_t* k,
                              const int32_t* sx, const int32_t* st, const int32_t* order,
                              int64_t batch, int n, unsigned* ticket, cudaStream_t stream) {
  auto kern = f64k::fused64d_kernel<TIn, TOut, WAVE>;
  const size_t smem = fused64d_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                           cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return e;
  static const int env_occ = [] {
    const char* v = std::getenv("CSM_K1D_OCC");
    return v ? std::atoi(v) : 2;
  }();
  size_t smem_launch = smem;
  if (env_occ == 1) {  // experiment: one CTA per SM (pad the allocation)
    smem_launch = 200 * 1024;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem_launch));
    if (e != cudaSuccess) return e;
  }
  // Two CTAs per SM by construction: 2 x (96 KiB + static + 1 KiB reserved)
  // of shared memory, 2 x 256 x 128 registers, 2 x 256 TMEM columns.  The
  // occupancy API is no help here: it reports 1 for any kernel that contains
  // a tcgen05.alloc, while the hardware co-schedules two (tools/occ_tmem.cu).
  cudaFuncAttributes fa;
  e = cudaFuncGetAttributes(&fa, kern);
  if (e != cudaSuccess) return e;
  int dev = 0, smem_sm = 0, regs_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
  const bool two = env_occ != 1 &&
                   2 * (smem_launch + fa.sharedSizeBytes + 1024) <= static_cast<size_t>(smem_sm) &&
                   2 * 256 * fa.numRegs <= regs_sm;
  const int per_sm = two ? 2 : 1;
  if (std::getenv("CSM_K1D_DEBUG"))
    std::fprintf(stderr, "K1d: per_sm=%d regs=%d static_smem=%zu dyn=%zu\n", per_sm, fa.numRegs,
                 fa.sharedSizeBytes, smem_launch);
  int64_t grid = static_cast<int64_t>(device_sms()) * per_sm;
  if (grid > batch) grid = batch;
  if (grid < 1) return cudaSuccess;
  const int fast = (sizeof(TIn) == 8 && n == 64 && reinterpret_cast<uintptr_t>(a) % 16 == 0) ? 1 : 0;
  e = cudaMemsetAsync(ticket, 0, sizeof(unsigned), stream);
  if (e != cudaSuccess) return e;
  kern<<<static_cast<unsigned>(grid), 256, smem_launch, stream>>>(
      static_cast<const TIn*>(a), static_cast<TOut*>(c), static_cast<TOut*>(s), t, k, sx, st, order,
      batch, n, fast, ticket);
  return cudaGetLastError();
}

// K1d: n <= 64, (k, s, status) and order[] on the device; t: the wave
// family's times (nullptr: Taylor cos/sin); ticket: one device word of
// scratch (the work counter, zeroed here).
cudaError_t launch_fused64d(int dtype, bool wave, const void* a, void* c, void* s, const double* t,
                            const int32_t* k, const int32_t* sx, const int32_t* st,
                            const int32_t* order, int64_t batch, int n, unsigned* ticket,
                            cudaStream_t stream) {
  if (n < 1 || n > 64 || !ticket || (wave && !t)) return cudaErrorInvalidValue;
#define K1D_GO(TI, TO)                                                                          \
  (wave ? launch_k1d<TI, TO, true>(a, c, s, t, k, sx, st, order, batch, n, ticket, stream)      \
        : launch_k1d<TI, TO, false>(a, c, s, t, k, sx, st, order, batch, n, ticket, stream))
  if (dtype == 0) return K1D_GO(double, double);
  if (dtype == 2) return K1D_GO(float, double);
  return K1D_GO(float, float);
#undef K1D_GO
}

}  // namespace csm
