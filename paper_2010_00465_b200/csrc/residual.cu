// residual.cu -- the Pythagorean residual ||C^2 + S^2 - I||_1 of computed
// pairs, on the device (csm_pythagorean_residual).
//
// The reference reports this identity as its accuracy witness
// (pkg/README.md:172-176; tests/test_driver.py:149-157 asserts it <= 1e-12
// on a symmetric 8 x 8 at norm 50).  It is a diagnostic, not part of the
// cos/sin path: bench.py evaluates it over the whole batch outside the
// timed region, so the bench line can carry it without any library GEMM.
//
// One CTA per 64 x 64 tile of C C + S S - I: both products accumulate into
// the same DMMA m8n8k4 registers (4 warps x 32 x 32, K step 16 through
// shared memory, bounds-checked loads so any n works), then each tile's
// column sums of |.| go to a per-tile partial; a second kernel adds the
// partials in a fixed order and takes the max over columns (deterministic).
#include "common.cuh"

namespace csm {
namespace rk {

constexpr int T = 64, BK = 16, LDA = BK + 4, LDB = T + 4;

template <typename TIn>
__global__ void __launch_bounds__(128) residual_tile_kernel(const TIn* __restrict__ C,
                                                            const TIn* __restrict__ S, int n,
                                                            double* __restrict__ part) {
  // C, S row panels and column panels; after the K loop the same buffer
  // holds the finished tile E (static shared memory stays below 48 KiB)
  constexpr int PANELS = 2 * T * LDA + 2 * BK * LDB, ETILE = T * (T + 1);
  __shared__ double buf[PANELS > ETILE ? PANELS : ETILE];
  double(*As)[T * LDA] = reinterpret_cast<double(*)[T * LDA]>(buf);
  double(*Bs)[BK * LDB] = reinterpret_cast<double(*)[BK * LDB]>(buf + 2 * T * LDA);
  double(*E)[T + 1] = reinterpret_cast<double(*)[T + 1]>(buf);
  const int tiles = (n + T - 1) / T;
  const int b = blockIdx.y;
  const int tm = blockIdx.x / tiles, tn = blockIdx.x % tiles;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const size_t nn = static_cast<size_t>(n) * n;
  const TIn* M[2] = {C + b * nn, S + b * nn};
  double acc[4][4][2] = {};
  for (int k0 = 0; k0 < n; k0 += BK) {
    for (int q = 0; q < 2; ++q) {
      for (int p = tid; p < T * BK; p += 128) {
        const int r = p / BK, c = p % BK;
        const int gr = tm * T + r, gc = k0 + c;
        As[q][r * LDA + c] =
            (gr < n && gc < n) ? static_cast<double>(M[q][static_cast<size_t>(gr) * n + gc]) : 0.0;
      }
      for (int p = tid; p < BK * T; p += 128) {
        const int r = p / T, c = p % T;
        const int gr = k0 + r, gc = tn * T + c;
        Bs[q][r * LDB + c] =
            (gr < n && gc < n) ? static_cast<double>(M[q][static_cast<size_t>(gr) * n + gc]) : 0.0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        double a[4], bf[4];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) a[mi] = As[q][(wm + mi * 8 + g) * LDA + kk + t];
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) bf[ni] = Bs[q][(kk + t) * LDB + wn + ni * 8 + g];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi], bf[ni]);
      }
    __syncthreads();
  }
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = wm + mi * 8 + g, c = wn + ni * 8 + 2 * t + h;
        const bool diag = tm * T + r == tn * T + c;
        E[r][c] = acc[mi][ni][h] - (diag ? 1.0 : 0.0);
      }
  __syncthreads();
  if (tid < T) {
    const int c = tn * T + tid;
    double s = 0.0;
    for (int r = 0; r < T && tm * T + r < n; ++r) s += fabs(E[r][tid]);
    if (c < n) part[(static_cast<size_t>(b) * tiles + tm) * n + c] = s;
  }
}

// out[b] = max_j sum_tm part[b][tm][j]  (one CTA per matrix)
__global__ void __launch_bounds__(256) residual_reduce_kernel(const double* __restrict__ part,
                                                              int n, double* __restrict__ out) {
  const int b = blockIdx.x, tiles = (n + T - 1) / T;
  __shared__ double red[8];
  double m = 0.0;
  for (int j = threadIdx.x; j < n; j += 256) {
    double s = 0.0;
    for (int tm = 0; tm < tiles; ++tm) s += part[(static_cast<size_t>(b) * tiles + tm) * n + j];
    m = (s > m || s != s) ? s : m;  // a NaN residual stays NaN
  }
  for (int o = 16; o; o >>= 1) {
    const double x = __shfl_xor_sync(0xffffffffu, m, o);
    m = (x > m || x != x) ? x : m;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) m = (red[w] > m || red[w] != red[w]) ? red[w] : m;
    m = (red[0] > m || red[0] != red[0]) ? red[0] : m;
    out[b] = m;
  }
}

}  // namespace rk

size_t residual_workspace_bytes(int64_t batch, int n) {
  const size_t tiles = static_cast<size_t>((n + rk::T - 1) / rk::T);
  return static_cast<size_t>(batch) * tiles * static_cast<size_t>(n) * sizeof(double) + 256;
}

cudaError_t pythagorean_residual(bool f32, const void* c, const void* s, int64_t batch, int n,
                                 double* out, void* ws, cudaStream_t stream, int64_t* launches) {
  const int tiles = (n + rk::T - 1) / rk::T;
  double* part = static_cast<double*>(ws);
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    const int cnt = static_cast<int>(std::min<int64_t>(65535, batch - b0));
    const size_t off = static_cast<size_t>(b0) * n * n;
    dim3 grid(static_cast<unsigned>(tiles * tiles), static_cast<unsigned>(cnt));
    double* p = part + static_cast<size_t>(b0) * tiles * n;
    if (f32)
      rk::residual_tile_kernel<float><<<grid, 128, 0, stream>>>(
          static_cast<const float*>(c) + off, static_cast<const float*>(s) + off, n, p);
    else
      rk::residual_tile_kernel<double><<<grid, 128, 0, stream>>>(
          static_cast<const double*>(c) + off, static_cast<const double*>(s) + off, n, p);
    rk::residual_reduce_kernel<<<cnt, 256, 0, stream>>>(p, n, out + b0);
    *launches += 2;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace csm
