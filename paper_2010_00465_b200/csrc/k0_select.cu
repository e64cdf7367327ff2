// k0_select.cu -- K0: per-matrix 1-norm, finiteness check and (k, s)
// selection on the device, plus the constant tables.
//
// norm1 (matcore.py:100-104) is np.abs(a).sum(axis=0).max(): numpy reduces
// axis 0 row by row, so each column sum is a SEQUENTIAL accumulation in row
// order, in the input's dtype (float32 sums for float32 input).  One thread
// per (matrix, column) reproduces exactly that order; loads are coalesced
// across the columns of a row.  The max over columns is exact and
// order-free, so an atomicMax on the (non-negative) double's bit pattern
// finishes the norm.  Selection then runs one thread per matrix with the
// bit-exact twin of select_scheme (common.cuh, driver.py:64-88).
#include "common.cuh"

namespace csm {

// (dTables is defined in common.cuh)

static Tables make_tables() {
  Tables t{};
  for (int i = 0; i < 4; ++i) {
    t.theta[0][0][i] = kTheta_taylor_double[i];
    t.theta[0][1][i] = kTheta_taylor_single[i];
    t.kk[0][0][i] = kK_taylor_double[i];
    t.kk[0][1][i] = kK_taylor_single[i];
  }
  for (int i = 0; i < 3; ++i) {
    t.theta[1][0][i] = kTheta_wave_double[i];
    t.theta[1][1][i] = kTheta_wave_single[i];
    t.kk[1][0][i] = kK_wave_double[i];
    t.kk[1][1][i] = kK_wave_single[i];
  }
  t.theta[2][0][0] = kTheta_pade_double[0];
  t.theta[2][1][0] = kTheta_pade_single[0];
  t.kk[2][0][0] = kK_pade_double[0];
  t.kk[2][1][0] = kK_pade_single[0];
  t.nent[0] = 4;
  t.nent[1] = 3;
  t.nent[2] = 1;
  for (int i = 0; i < 1024; ++i) t.log2fix[i] = kLog2Fix[i];
  for (int i = 0; i < 8; ++i) t.x8[i] = kXDeg8[i];
  for (int i = 0; i < 9; ++i) t.z8[i] = kZDeg8[i];
  for (int j = 0; j < 4; ++j)
    for (int i = 0; i < 4; ++i) t.a12[j][i] = kADeg12[j * 4 + i];
  for (int i = 0; i < 12; ++i) t.z12[i] = kZDeg12[i];
  return t;
}

const Tables& host_tables() {
  static const Tables t = make_tables();
  return t;
}

// Upload the tables once per device (idempotent; cheap check afterwards).
cudaError_t ensure_tables() {
  static int done_mask = 0;  // bit per device ordinal (< 32)
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 32 && (done_mask >> dev) & 1) return cudaSuccess;
  e = cudaMemcpyToSymbol(dTables, &host_tables(), sizeof(Tables));
  if (e == cudaSuccess && dev < 32) done_mask |= 1 << dev;
  return e;
}

template <typename T>
__global__ void norm1_kernel(const T* __restrict__ A, int64_t batch, int n,
                             unsigned long long* __restrict__ normbits,
                             int32_t* __restrict__ status) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= batch * n) return;
  const int64_t b = idx / n;
  const int j = static_cast<int>(idx - b * n);
  const T* p = A + b * n * n + j;
  T acc = T(0);
  bool fin = true;
#pragma unroll 8
  for (int i = 0; i < n; ++i) {
    const T x = p[static_cast<int64_t>(i) * n];
    fin &= (x - x == T(0));
    acc = acc + fabs(x);  // sequential in row order: no reassociation
  }
  if (!fin) status[b] = kNonfiniteInput;
  const double d = static_cast<double>(acc);
  atomicMax(normbits + b, static_cast<unsigned long long>(__double_as_longlong(d)));
}

// family 0 taylor / 1 wave; t may be null for taylor.
__global__ void select_kernel(const unsigned long long* __restrict__ normbits,
                              const double* __restrict__ t, int64_t batch,
                              int family, int precision, int32_t* __restrict__ K,
                              int32_t* __restrict__ S, int32_t* __restrict__ status,
                              double* __restrict__ norms_out) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  double norm = __longlong_as_double(static_cast<long long>(normbits[b]));
  if (norms_out) norms_out[b] = norm;
  int st = status[b];
  int k = 0, s = 0;
  if (st == kOk) {
    if (family == 1) {
      const double tb = t[b];
      norm = (tb * tb) * norm;  // driver.py:136, float(t)*float(t)*norm1(a)
    }
    st = select_one(norm, dTables.theta[family][precision],
                    dTables.kk[family][precision], dTables.nent[family],
                    dTables.log2fix, &k, &s);
  }
  K[b] = k;
  S[b] = s;
  status[b] = st;
}

__global__ void select_norms_kernel(const double* __restrict__ norms,
                                    int64_t count, int family, int precision,
                                    int32_t* __restrict__ K, int32_t* __restrict__ S,
                                    int32_t* __restrict__ status) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= count) return;
  int k = 0, s = 0;
  int st = select_one(norms[b], dTables.theta[family][precision],
                      dTables.kk[family][precision], dTables.nent[family],
                      dTables.log2fix, &k, &s);
  K[b] = k;
  S[b] = s;
  status[b] = st;
}

__global__ void fill_ks_kernel(int32_t* __restrict__ K, int32_t* __restrict__ S,
                               int32_t* __restrict__ status, int64_t batch,
                               int k) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  K[b] = k;
  S[b] = 0;
  status[b] = 0;
}

static inline unsigned blocks_for(int64_t work, int threads) {
  return static_cast<unsigned>((work + threads - 1) / threads);
}

// norm + finiteness: status must be zeroed and normbits zeroed beforehand.
cudaError_t launch_norm1(int dtype, const void* a, int64_t batch, int n,
                         unsigned long long* normbits, int32_t* status,
                         cudaStream_t stream) {
  const int64_t work = batch * n;
  if (work == 0) return cudaSuccess;
  const int threads = 256;
  if (dtype == 0)
    norm1_kernel<double><<<blocks_for(work, threads), threads, 0, stream>>>(
        static_cast<const double*>(a), batch, n, normbits, status);
  else
    norm1_kernel<float><<<blocks_for(work, threads), threads, 0, stream>>>(
        static_cast<const float*>(a), batch, n, normbits, status);
  return cudaGetLastError();
}

cudaError_t launch_select(const unsigned long long* normbits, const double* t,
                          int64_t batch, int family, int precision, int32_t* K,
                          int32_t* S, int32_t* status, double* norms_out,
                          cudaStream_t stream) {
  if (batch == 0) return cudaSuccess;
  select_kernel<<<blocks_for(batch, 256), 256, 0, stream>>>(
      normbits, t, batch, family, precision, K, S, status, norms_out);
  return cudaGetLastError();
}

cudaError_t launch_select_norms(const double* norms, int64_t count, int family,
                                int precision, int32_t* K, int32_t* S,
                                int32_t* status, cudaStream_t stream) {
  if (count == 0) return cudaSuccess;
  select_norms_kernel<<<blocks_for(count, 256), 256, 0, stream>>>(
      norms, count, family, precision, K, S, status);
  return cudaGetLastError();
}

cudaError_t launch_fill_ks(int32_t* K, int32_t* S, int32_t* status,
                           int64_t batch, int k, cudaStream_t stream) {
  if (batch == 0) return cudaSuccess;
  fill_ks_kernel<<<blocks_for(batch, 256), 256, 0, stream>>>(K, S, status, batch, k);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Cost-ordered schedule for the persistent fused kernel: order[] lists the
// matrices by descending product count k + 2s (counting sort; failed
// matrices last), so a snake assignment over the CTAs balances their work
// without a shared atomic queue.

constexpr int kCostBins = 2048;

__global__ void cost_hist_kernel(const int32_t* __restrict__ K, const int32_t* __restrict__ S,
                                 const int32_t* __restrict__ status, int64_t batch,
                                 int* __restrict__ bins) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  int cost = status[b] == 0 ? K[b] + 2 * S[b] : 0;
  cost = cost < kCostBins - 1 ? cost : kCostBins - 1;
  atomicAdd(bins + (kCostBins - 1 - cost), 1);  // bin 0 = most expensive
}

// Exclusive scan of the bins in place (one block).
__global__ void cost_scan_kernel(int* __restrict__ bins) {
  __shared__ int part[1024];
  const int t = threadIdx.x;  // 1024 threads, 2 bins each
  const int a0 = bins[2 * t], a1 = bins[2 * t + 1];
  part[t] = a0 + a1;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const int v = t >= off ? part[t - off] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  const int excl = part[t] - (a0 + a1);
  bins[2 * t] = excl;
  bins[2 * t + 1] = excl + a0;
}

__global__ void cost_scatter_kernel(const int32_t* __restrict__ K, const int32_t* __restrict__ S,
                                    const int32_t* __restrict__ status, int64_t batch,
                                    int* __restrict__ bins, int32_t* __restrict__ order) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  int cost = status[b] == 0 ? K[b] + 2 * S[b] : 0;
  cost = cost < kCostBins - 1 ? cost : kCostBins - 1;
  const int pos = atomicAdd(bins + (kCostBins - 1 - cost), 1);
  order[pos] = static_cast<int32_t>(b);
}

size_t schedule_ws_bytes() { return kCostBins * sizeof(int); }

// bins: device scratch of schedule_ws_bytes(); order: device int32[batch].
__global__ void iota_kernel(int32_t* __restrict__ order, int64_t batch) {
  for (int64_t i = threadIdx.x; i < batch; i += blockDim.x) order[i] = static_cast<int32_t>(i);
}

// Largest batch scheduled unsorted (order = identity, one launch instead of a
// memset and three): at most one matrix per CTA of the persistent fused grid
// (K1: 148 CTAs, K1c: >= 33 resident 4-CTA clusters), so no balancing is
// needed -- the latency-bound single-matrix path of configs[0].
constexpr int64_t kUnsortedMax = 32;

// True when launch_schedule sorts a batch of this size (else order = identity).
bool schedule_sorted(int64_t batch) { return batch > kUnsortedMax; }

// Scan + scatter in one block for batches a single block walks in a few
// microseconds: the scanned bins stay in shared memory.
constexpr int64_t kOneBlockScatterMax = 65536;

__global__ void __launch_bounds__(1024)
cost_scan_scatter_kernel(const int32_t* __restrict__ K, const int32_t* __restrict__ S,
                         const int32_t* __restrict__ status, int64_t batch,
                         const int* __restrict__ bins, int32_t* __restrict__ order) {
  __shared__ int part[1024];
  __shared__ int sb[kCostBins];
  const int t = threadIdx.x;  // 1024 threads, 2 bins each
  const int a0 = bins[2 * t], a1 = bins[2 * t + 1];
  part[t] = a0 + a1;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const int v = t >= off ? part[t - off] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  const int excl = part[t] - (a0 + a1);
  sb[2 * t] = excl;
  sb[2 * t + 1] = excl + a0;
  __syncthreads();
#pragma unroll 4
  for (int64_t b = t; b < batch; b += 1024) {
    int cost = status[b] == 0 ? K[b] + 2 * S[b] : 0;
    cost = cost < kCostBins - 1 ? cost : kCostBins - 1;
    const int pos = atomicAdd(sb + (kCostBins - 1 - cost), 1);
    order[pos] = static_cast<int32_t>(b);
  }
}

// K0 fused for n <= 128: one warp per matrix.  Each lane owns VEC adjacent
// columns of every 32 VEC-column pass and accumulates them sequentially in
// row order in the input's dtype -- the same sums, in the same order, as
// norm1_kernel (matcore.py:100-104) -- with whole rows read as one
// coalesced vector load per lane.  The column maximum is a warp shuffle
// (bit patterns of non-negative doubles order like the values, as the
// atomicMax of norm1_kernel does), lane 0 selects (k, s) like select_kernel
// and, when bins is given, counts the matrix's cost for the schedule: no
// memsets of normbits / status, no atomics on them, one launch instead of
// four stream operations.
template <typename T, int VEC>
__global__ void __launch_bounds__(256)
norm_select_kernel(const T* __restrict__ A, const double* __restrict__ t, int64_t batch, int n,
                   int family, int precision, int32_t* __restrict__ K, int32_t* __restrict__ S,
                   int32_t* __restrict__ status, unsigned long long* __restrict__ normbits,
                   int* __restrict__ bins, int64_t hist_count) {
  const int lane = threadIdx.x & 31;
  const int64_t b = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= batch) return;  // warp-uniform
  const T* base = A + b * n * n;
  unsigned long long mx = 0ull;
  bool fin = true;
  for (int j0 = 0; j0 < n; j0 += 32 * VEC) {
    const int col = j0 + lane * VEC;
    if (col < n) {  // n % VEC == 0: the lane's VEC columns are all inside
      const T* p = base + col;
      T acc[VEC];
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[v] = T(0);
#pragma unroll 8
      for (int i = 0; i < n; ++i) {
        T x[VEC];
        if constexpr (VEC == 1) {
          x[0] = __ldg(p + static_cast<int64_t>(i) * n);
        } else if constexpr (sizeof(T) == 8) {
          const double2 v2 = __ldg(reinterpret_cast<const double2*>(p + static_cast<int64_t>(i) * n));
          x[0] = v2.x; x[1] = v2.y;
        } else {
          const float4 v4 = __ldg(reinterpret_cast<const float4*>(p + static_cast<int64_t>(i) * n));
          x[0] = v4.x; x[1] = v4.y; x[2] = v4.z; x[3] = v4.w;
        }
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          fin &= (x[v] - x[v] == T(0));
          acc[v] = acc[v] + fabs(x[v]);  // sequential in row order: no reassociation
        }
      }
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const unsigned long long bits = static_cast<unsigned long long>(
            __double_as_longlong(static_cast<double>(acc[v])));
        mx = bits > mx ? bits : mx;
      }
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, mx, off);
    mx = o > mx ? o : mx;
  }
  fin = __all_sync(0xffffffffu, fin);
  if (lane != 0) return;
  normbits[b] = mx;
  double norm = __longlong_as_double(static_cast<long long>(mx));
  int st = fin ? kOk : kNonfiniteInput;
  int k = 0, s = 0;
  if (st == kOk) {
    if (family == 1) {
      const double tb = t[b];
      norm = (tb * tb) * norm;  // driver.py:136, float(t)*float(t)*norm1(a)
    }
    st = select_one(norm, dTables.theta[family][precision], dTables.kk[family][precision],
                    dTables.nent[family], dTables.log2fix, &k, &s);
  }
  K[b] = k;
  S[b] = s;
  status[b] = st;
  if (bins && b < hist_count) {
    int cost = st == 0 ? k + 2 * s : 0;
    cost = cost < kCostBins - 1 ? cost : kCostBins - 1;
    atomicAdd(bins + (kCostBins - 1 - cost), 1);  // bin 0 = most expensive
  }
}

constexpr int kNormSelectMaxN = 128;
bool norm_select_fits(int n) { return n > 0 && n <= kNormSelectMaxN; }

// bins (zeroed by the caller) may be null: no cost histogram then.
cudaError_t launch_norm_select(int dtype, const void* a, const double* t, int64_t batch, int n,
                               int family, int precision, int32_t* K, int32_t* S,
                               int32_t* status, unsigned long long* normbits, int* bins,
                               int64_t hist_count, cudaStream_t stream) {
  if (batch == 0) return cudaSuccess;
  const unsigned blocks = blocks_for(batch, 8);  // 8 warps = 8 matrices per block
  const bool al16 = (reinterpret_cast<uintptr_t>(a) & 15) == 0;
  if (dtype == 0) {
    const double* A = static_cast<const double*>(a);
    if (al16 && n % 2 == 0)
      norm_select_kernel<double, 2><<<blocks, 256, 0, stream>>>(
          A, t, batch, n, family, precision, K, S, status, normbits, bins, hist_count);
    else
      norm_select_kernel<double, 1><<<blocks, 256, 0, stream>>>(
          A, t, batch, n, family, precision, K, S, status, normbits, bins, hist_count);
  } else {
    const float* A = static_cast<const float*>(a);
    if (al16 && n % 4 == 0)
      norm_select_kernel<float, 4><<<blocks, 256, 0, stream>>>(
          A, t, batch, n, family, precision, K, S, status, normbits, bins, hist_count);
    else
      norm_select_kernel<float, 1><<<blocks, 256, 0, stream>>>(
          A, t, batch, n, family, precision, K, S, status, normbits, bins, hist_count);
  }
  return cudaGetLastError();
}

// prehist: the bins already hold the cost histogram of [0, batch)
// (norm_select_kernel counted it), so the memset and the histogram launch
// are skipped, and a batch one block can walk is scanned and scattered in
// one launch.
cudaError_t launch_schedule(const int32_t* K, const int32_t* S, const int32_t* status,
                            int64_t batch, int* bins, int32_t* order, cudaStream_t stream,
                            int64_t* launches, bool prehist) {
  if (batch == 0) return cudaSuccess;
  if (batch <= kUnsortedMax) {
    iota_kernel<<<1, 32, 0, stream>>>(order, batch);
    *launches += 1;
    return cudaGetLastError();
  }
  if (prehist) {
    if (batch <= kOneBlockScatterMax) {
      cost_scan_scatter_kernel<<<1, 1024, 0, stream>>>(K, S, status, batch, bins, order);
      *launches += 1;
    } else {
      cost_scan_kernel<<<1, 1024, 0, stream>>>(bins);
      cost_scatter_kernel<<<blocks_for(batch, 256), 256, 0, stream>>>(K, S, status, batch, bins,
                                                                      order);
      *launches += 2;
    }
    return cudaGetLastError();
  }
  cudaError_t e = cudaMemsetAsync(bins, 0, schedule_ws_bytes(), stream);
  if (e != cudaSuccess) return e;
  cost_hist_kernel<<<blocks_for(batch, 256), 256, 0, stream>>>(K, S, status, batch, bins);
  cost_scan_kernel<<<1, 1024, 0, stream>>>(bins);
  cost_scatter_kernel<<<blocks_for(batch, 256), 256, 0, stream>>>(K, S, status, batch, bins,
                                                                  order);
  *launches += 3;
  return cudaGetLastError();
}

}  // namespace csm
