// common.cuh -- shared device/host pieces of the cos/sin hot path.
//
//  * the reference's constants (generated header, bit-exact float() values)
//  * (k, s) selection, host+device twin of select_scheme (driver.py:64-88)
//  * the FP64 tensor-core primitive: mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4
//    (sm_100a has no tcgen05 f64 kind; DMMA is the FP64 tensor pipe).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#define CSM_CONST static const
#include "cossin_constants.h"
#undef CSM_CONST

// Device-side bounds checks of the debug build (-DCSM_DEBUG_CHECKS; built by
// tools/build_debug.py and run over the GPU suite in place of compute-sanitizer,
// which is closed on this pool): a failed check traps with its location.
#ifdef CSM_DEBUG_CHECKS
#include <cassert>
#define CSM_DCHECK(cond) assert(cond)
#else
#define CSM_DCHECK(cond) do { } while (0)
#endif

namespace csm {

// ---------------------------------------------------------------------------
// Constant tables, mirrored into __constant__ memory for the device.

struct Tables {
  double theta[3][2][4];  // [family][precision][entry] theta_eff
  int kk[3][2][4];        // scheme k of each entry
  int nent[3];            // entries per family (taylor, wave, pade)
  long long log2fix[1024];
  double x8[8];           // x1..x8       (schemes.py:110-119)
  double z8[9];           // z0..z8       (schemes.py:125-135)
  double a12[4][4];       // [j-1][i]     (schemes.py:149-166)
  double z12[12];         // z0..z11      (schemes.py:174-187)
};

// Defined once: the library is a single translation unit (cossin_b200.cu).
__constant__ Tables dTables;
const Tables& host_tables();

enum Status : int32_t { kOk = 0, kNonfiniteInput = 1, kNonfiniteNorm = 2,
                        kSelectOverflow = 3, kSingular = 4 };

// ceil(log2(q)) as driver.py:67 computes it with glibc's correctly rounded
// log2, for q >= 1 finite.  q = 2^e (1 + j 2^-52): log2(q) rounds down to e
// exactly when j <= fix[e] (table generated from math.log2 itself).
__host__ __device__ inline int ceil_log2_ref(double q, const long long* fix) {
  uint64_t bits;
#ifdef __CUDA_ARCH__
  bits = static_cast<uint64_t>(__double_as_longlong(q));
#else
  __builtin_memcpy(&bits, &q, 8);
#endif
  int e = static_cast<int>((bits >> 52) & 0x7ff) - 1023;
  long long j = static_cast<long long>(bits & ((1ull << 52) - 1));
  if (e < 0) return 0;  // q < 1 cannot reach here (norm > theta); guard
  return (j <= fix[e]) ? e : e + 1;
}

__host__ __device__ inline bool finite_d(double x) {
  return x - x == 0.0;  // false for inf and nan
}

// select_scheme(norm, table) (driver.py:70-88) over a built-in table.
// Returns a Status; writes k and s on kOk.
__host__ __device__ inline int select_one(double norm, const double* theta,
                                          const int* kk, int nent,
                                          const long long* fix, int* k_out,
                                          int* s_out) {
  if (!(norm >= 0.0) || !finite_d(norm)) return kNonfiniteNorm;
  for (int i = 0; i < nent; ++i) {
    if (norm <= theta[i]) { *k_out = kk[i]; *s_out = 0; return kOk; }
  }
  int best_total = 0, best_s = 0, best_k = 0;
  for (int i = 0; i < nent; ++i) {
    int s = 0;
    if (!(norm <= theta[i])) {
      double q = norm / theta[i];
      if (!finite_d(q)) return kSelectOverflow;  // math.ceil(inf) raises
      s = ceil_log2_ref(q, fix);
      if (s < 0) s = 0;
    }
    int total = kk[i] + 2 * s;  // cost == k products for Taylor/wave
    if (i == 0 || total < best_total || (total == best_total && s < best_s)) {
      best_total = total; best_s = s; best_k = kk[i];
    }
  }
  *k_out = best_k; *s_out = best_s;
  return kOk;
}

// ---------------------------------------------------------------------------
// FP64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col).
//   lane = 4*g + t:  a = A[g][t],  b = B[t][g],  d = {D[g][2t], D[g][2t+1]}
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, "
      "{%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// Live-timing hooks (abi.cu): no-ops unless csm_profile_enable(1).
void prof_begin(cudaStream_t stream, int kind = 1);
void prof_end(cudaStream_t stream, int kind = 1);

}  // namespace csm
