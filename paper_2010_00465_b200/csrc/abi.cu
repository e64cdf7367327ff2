// abi.cu -- the extern "C" boundary (include/cossin_b200.h).
//
// Each entry point validates its arguments the way the reference's Python
// layer does (driver.py:101-105 shape/finiteness, driver.py:77-78 norm,
// schemes.py:78-84 scheme id), then runs K0 (norm + selection) and either
// the fused n <= 64 kernel (K1) or the tiled chain (K2-K4).  There is no
// CPU fallback: without a device every compute call returns
// CSM_ERR_NO_DEVICE.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "../../include/cossin_b200.h"
#include "common.cuh"

namespace csm {
cudaError_t ensure_tables();
cudaError_t launch_norm1(int dtype, const void* a, int64_t batch, int n,
                         unsigned long long* normbits, int32_t* status, cudaStream_t stream);
cudaError_t launch_select(const unsigned long long* normbits, const double* t, int64_t batch,
                          int family, int precision, int32_t* K, int32_t* S, int32_t* status,
                          double* norms_out, cudaStream_t stream);
cudaError_t launch_select_norms(const double* norms, int64_t count, int family, int precision,
                                int32_t* K, int32_t* S, int32_t* status, cudaStream_t stream);
cudaError_t launch_fill_ks(int32_t* K, int32_t* S, int32_t* status, int64_t batch, int k,
                           cudaStream_t stream);
int64_t fused64_self_max(int n);
cudaError_t launch_fused64_self(int dtype, int precision, bool wave, const void* a, void* c,
                                void* s, const double* t, int32_t* k, int32_t* sx, int32_t* st,
                                unsigned long long* normbits, int64_t batch, int n,
                                cudaStream_t stream);
cudaError_t launch_fused64(int dtype, bool wave, const void* a, void* c, void* s,
                           const double* t, const int32_t* k, const int32_t* sx,
                           const int32_t* st, const int32_t* order, int64_t batch, int n,
                           cudaStream_t stream);
size_t schedule_ws_bytes();
cudaError_t launch_schedule(const int32_t* K, const int32_t* S, const int32_t* status,
                            int64_t batch, int* bins, int32_t* order, cudaStream_t stream,
                            int64_t* launches, bool prehist);
bool schedule_sorted(int64_t batch);
bool norm_select_fits(int n);
cudaError_t launch_norm_select(int dtype, const void* a, const double* t, int64_t batch, int n,
                               int family, int precision, int32_t* K, int32_t* S,
                               int32_t* status, unsigned long long* normbits, int* bins,
                               int64_t hist_count, cudaStream_t stream);
size_t tiled_workspace_bytes(int64_t batch, int n, int eng);
void set_engine(int e);
void set_thread_engine(int e);
int engine();
int k1c_resident_sms();
cudaError_t launch_fused64d(int dtype, bool wave, const void* a, void* c, void* s, const double* t,
                            const int32_t* k, const int32_t* sx, const int32_t* st,
                            const int32_t* order, int64_t batch, int n, unsigned* ticket,
                            cudaStream_t stream);
size_t op_bytes();
int chain_program(bool wave, int k, bool fold, void* ops_out, int max_ops, int32_t* step_nops,
                  int max_steps, int32_t* cos_slot, int32_t* sin_slot);
void doubling_program(int c0, int s0, int c1, int s1, void* ops_out);
size_t slab_scratch_bytes();
size_t slab_engine_bytes(int M, int NP, int eng);
cudaError_t slab_op(const void* const* op_host, int nops, double* slab, int M, int NP, int row0,
                    const double* rhs_full, const double* in0, int s, double tp, int dbl_step,
                    void* cout, void* sout, int out_f32, void* scratch, cudaStream_t stream,
                    int64_t* launches, const double* const* parts_host, int nparts, int eng);
cudaError_t run_tiled(int dtype, bool wave, const void* a, const double* t, void* c_out,
                      void* s_out, int64_t batch, int n, const int32_t* dK, const int32_t* dS,
                      const int32_t* dStatus, void* ws, cudaStream_t stream, int64_t* launches,
                      int special, int eng);
size_t residual_workspace_bytes(int64_t batch, int n);
cudaError_t pythagorean_residual(bool f32, const void* c, const void* s, int64_t batch, int n,
                                 double* out, void* ws, cudaStream_t stream, int64_t* launches);
size_t ddref_workspace_doubles(int64_t batch, int n);
void ddref_series_consts(double* out28);
cudaError_t dd_matmul(const double* xh, const double* xl, const double* yh, const double* yl,
                      double* oh, double* ol, int64_t batch, int n, cudaStream_t stream,
                      int64_t* launches);
cudaError_t ddref_chain(const double* a, const int32_t* dS, int smax, double* cos_out,
                        double* sin_out, int64_t batch, int n, double* ws, cudaStream_t stream,
                        int64_t* launches);
}  // namespace csm

namespace {
thread_local int g_prof = 0;  // 0 off, 1 pipeline intervals, 2 int8 GEMM launches, 3 fused K0 launches
thread_local std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_prof_ev;
thread_local cudaEvent_t g_prof_open = nullptr;
thread_local bool g_prof_hold = false;  // an enclosing interval is open
}  // namespace

namespace csm {
void prof_begin(cudaStream_t stream, int kind) {
  if (g_prof != kind || g_prof_hold) return;
  if (cudaEventCreate(&g_prof_open) != cudaSuccess) { g_prof_open = nullptr; return; }
  cudaEventRecord(g_prof_open, stream);
}
void prof_end(cudaStream_t stream, int kind) {
  if (g_prof != kind || g_prof_hold || !g_prof_open) return;
  cudaEvent_t e1;
  if (cudaEventCreate(&e1) != cudaSuccess) return;
  cudaEventRecord(e1, stream);
  g_prof_ev.emplace_back(g_prof_open, e1);
  g_prof_open = nullptr;
}
}  // namespace csm

namespace {

void prof_clear() {
  for (auto& p : g_prof_ev) {
    cudaEventDestroy(p.first);
    cudaEventDestroy(p.second);
  }
  g_prof_ev.clear();
}

thread_local std::string g_err;
thread_local int64_t g_launches = 0;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(CSM_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct CommonWs {
  unsigned long long* normbits;
  int32_t* kbuf;
  int32_t* sbuf;
  int32_t* order;  // cost-sorted schedule of the fused kernel
  int* bins;       // counting-sort scratch
  void* tiled;
};

size_t common_bytes(int64_t batch) {
  return align256(static_cast<size_t>(batch) * 8) + 3 * align256(static_cast<size_t>(batch) * 4) +
         align256(csm::schedule_ws_bytes());
}

CommonWs carve(void* ws, int64_t batch) {
  char* p = static_cast<char*>(ws);
  CommonWs w;
  w.normbits = reinterpret_cast<unsigned long long*>(p);
  p += align256(static_cast<size_t>(batch) * 8);
  w.kbuf = reinterpret_cast<int32_t*>(p);
  p += align256(static_cast<size_t>(batch) * 4);
  w.sbuf = reinterpret_cast<int32_t*>(p);
  p += align256(static_cast<size_t>(batch) * 4);
  w.order = reinterpret_cast<int32_t*>(p);
  p += align256(static_cast<size_t>(batch) * 4);
  w.bins = reinterpret_cast<int*>(p);
  p += align256(csm::schedule_ws_bytes());
  w.tiled = p;
  return w;
}

int check_device() {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) return fail(CSM_ERR_NO_DEVICE, "no CUDA device available");
  int dev = 0, major = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10) return fail(CSM_ERR_NO_DEVICE, "kernels are built for sm_100a (B200) only");
  e = csm::ensure_tables();
  if (e != cudaSuccess) return cuda_fail(e, "constant tables");
  return CSM_SUCCESS;
}

size_t workspace_size(int64_t batch, int n, int eng) {
  if (batch < 0 || n < 0) return 0;
  size_t bytes = common_bytes(batch);
  if (n > 64) bytes += csm::tiled_workspace_bytes(batch, n, eng) + 256;
  return bytes;
}

int check_common(int dtype, int64_t batch, int n, size_t ws_bytes, int eng) {
  if (dtype != CSM_F64 && dtype != CSM_F32 && dtype != CSM_F32_IN_F64_OUT)
    return fail(CSM_ERR_ARG, "dtype must be CSM_F64, CSM_F32 or CSM_F32_IN_F64_OUT");
  if (batch < 0 || n < 0) return fail(CSM_ERR_ARG, "batch and n must be nonnegative");
  if (batch > (int64_t(1) << 31) - 1) return fail(CSM_ERR_ARG, "batch too large");
  if (ws_bytes < workspace_size(batch, n, eng))
    return fail(CSM_ERR_WORKSPACE, "workspace smaller than csm_workspace_size() for this call's engine");
  return CSM_SUCCESS;
}

// Largest n served by the fused kernels (K1: n <= 64, K1c: n <= 128); larger
// n runs the tiled chain.  CSM_FUSED_MAX=64 (environment) keeps 64 < n <=
// 128 on the tiled chain, for A/B measurements.
int fused_max() {
  static const int v = [] {
    const char* e = std::getenv("CSM_FUSED_MAX");
    const int x = e ? std::atoi(e) : 128;
    return x >= 128 ? 128 : (x >= 64 ? 64 : 0);
  }();
  return v;
}

// K1d (two CTAs per SM, fused64d.cu) runs n <= 64 (both families);
// CSM_K1D=0 (environment) keeps those batches on K1, for A/B measurements
// and the bitwise cross-check test.
int k1_variant() {
  static const int v = [] {
    const char* e = std::getenv("CSM_K1D");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return v;
}

// Matrices of a 64 < n <= 128 batch given to the side tiled chain.
int64_t side_count(int64_t batch) {
  static const double share = [] {
    const char* e = std::getenv("CSM_SIDE_SHARE");
    const double x = e ? std::atof(e) : 0.12;
    return x < 0.0 ? 0.0 : (x > 0.5 ? 0.5 : x);
  }();
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int idle = sms - csm::k1c_resident_sms();
  if (share <= 0.0 || idle < 8 || batch < 1024) return 0;
  return static_cast<int64_t>(share * static_cast<double>(batch));
}

// One non-blocking side stream per device (created on first use).
cudaStream_t side_stream() {
  static cudaStream_t streams[32] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 32) dev = 31;
  if (!streams[dev]) cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking);
  return streams[dev];
}

// After K/S/status are on the device: run K1/K1c or the tiled chain.
int run_compute(int dtype, bool wave, const void* a, const double* t, void* c, void* s,
                int64_t batch, int n, const int32_t* K, const int32_t* S, const int32_t* st,
                const CommonWs& w, cudaStream_t stream, int eng, bool prehist = false) {
  if (n == 0 || batch == 0) return CSM_SUCCESS;
  cudaError_t e;
  if (n <= fused_max()) {
    // K1c leaves the SMs outside whole 4-SM clusters idle (GPC boundaries):
    // a share of the batch sized to them runs the tiled chain concurrently
    // on a side stream (CSM_SIDE_SHARE, default 0.12; 0 disables).
    int64_t bf = batch;
    if (n > 64) bf = batch - side_count(batch);
    cudaEvent_t ev_sel = nullptr, ev_done = nullptr;
    if (bf < batch) {
      cudaEventCreateWithFlags(&ev_sel, cudaEventDisableTiming);
      cudaEventRecord(ev_sel, stream);  // (k, s, status) are final here
    }
    struct EventGuard {  // events are released on every exit path
      cudaEvent_t* ev[2];
      ~EventGuard() {
        for (auto* p : ev)
          if (*p) cudaEventDestroy(*p);
      }
    } guard{{&ev_sel, &ev_done}};
    e = csm::launch_schedule(K, S, st, bf, w.bins, w.order, stream, &g_launches, prehist);
    if (e != cudaSuccess) return cuda_fail(e, "schedule kernels");
    csm::prof_begin(stream);
    // (the schedule's histogram scratch is free again: its first word is the work counter)
    if (n <= 64 && k1_variant() == 1)
      e = csm::launch_fused64d(dtype, wave, a, c, s, t, K, S, st, w.order, bf, n,
                               reinterpret_cast<unsigned*>(w.bins), stream);
    else
      e = csm::launch_fused64(dtype, wave, a, c, s, t, K, S, st, w.order, bf, n, stream);
    if (e != cudaSuccess) return cuda_fail(e, "fused64 launch");
    ++g_launches;
    if (bf < batch) {
      cudaStream_t side = side_stream();
      cudaStreamWaitEvent(side, ev_sel, 0);
      const size_t in_elt = dtype == CSM_F64 ? 8 : 4, out_elt = dtype == CSM_F32 ? 4 : 8;
      const size_t nn = static_cast<size_t>(n) * n;
      g_prof_hold = true;
      e = csm::run_tiled(dtype, wave, static_cast<const char*>(a) + bf * nn * in_elt,
                         t ? t + bf : nullptr, static_cast<char*>(c) + bf * nn * out_elt,
                         static_cast<char*>(s) + bf * nn * out_elt, batch - bf, n, K + bf, S + bf,
                         st + bf, w.tiled, side, &g_launches, 0, eng);
      g_prof_hold = false;
      if (e != cudaSuccess) return cuda_fail(e, "side tiled chain");
      cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming);
      cudaEventRecord(ev_done, side);
      cudaStreamWaitEvent(stream, ev_done, 0);
    }
    csm::prof_end(stream);
  } else {
    e = csm::run_tiled(dtype, wave, a, t, c, s, batch, n, K, S, st, w.tiled, stream, &g_launches,
                       0, eng);
    if (e != cudaSuccess) return cuda_fail(e, "tiled chain");
  }
  return CSM_SUCCESS;
}

// CSM_SELF_SELECT=0 keeps the separate K0 launches for small batches too
// (A/B measurements and the cross-check test).
bool self_select_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("CSM_SELF_SELECT");
    return !(e && e[0] == '0');
  }();
  return on;
}

// CSM_K0_FUSED=0 keeps the separate norm1 / select / histogram launches for
// n <= 128 too (A/B measurements and the cross-check test).
bool k0_fused_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("CSM_K0_FUSED");
    return !(e && e[0] == '0');
  }();
  return on;
}

int pipeline(int dtype, int precision, bool wave, const void* a, const double* t, void* c,
             void* s, int64_t batch, int n, int32_t* k, int32_t* sx, int32_t* status, void* ws,
             size_t ws_bytes, void* stream_v) {
  g_launches = 0;
  const int eng = csm::engine();  // one engine for the whole call
  int rc = check_common(dtype, batch, n, ws_bytes, eng);
  if (rc) return rc;
  if (precision != CSM_PREC_DOUBLE && precision != CSM_PREC_SINGLE)
    return fail(CSM_ERR_ARG, "precision must be CSM_PREC_DOUBLE or CSM_PREC_SINGLE");
  if (batch == 0) return CSM_SUCCESS;
  if (!k || !sx || !status || !ws || (n > 0 && (!a || !c || !s)) || (wave && !t))
    return fail(CSM_ERR_ARG, "null pointer argument");
  if ((rc = check_device())) return rc;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  CommonWs w = carve(ws, batch);
  cudaError_t e;
  if (n > 0 && n <= 64 && batch <= csm::fused64_self_max(n) && self_select_enabled()) {
    // small batch: K1 selects per CTA, one launch for the whole call
    csm::prof_begin(stream);
    e = csm::launch_fused64_self(dtype, precision, wave, a, c, s, t, k, sx, status, w.normbits,
                                 batch, n, stream);
    if (e != cudaSuccess) return cuda_fail(e, "fused64 (self-selecting) launch");
    ++g_launches;
    csm::prof_end(stream, 1);
    return CSM_SUCCESS;
  }
  if (csm::norm_select_fits(n) && k0_fused_enabled()) {
    // n <= 128: norm, finiteness, (k, s) and the schedule's cost histogram in one launch
    int64_t hist_n = 0;
    if (n <= fused_max()) {
      const int64_t bf = n > 64 ? batch - side_count(batch) : batch;
      if (csm::schedule_sorted(bf)) hist_n = bf;
    }
    if (hist_n) {
      e = cudaMemsetAsync(w.bins, 0, csm::schedule_ws_bytes(), stream);
      if (e != cudaSuccess) return cuda_fail(e, "memset");
    }
    csm::prof_begin(stream, 3);  // csm_profile_enable(3): the K0 launch alone
    e = csm::launch_norm_select(dtype, a, t, batch, n, wave ? 1 : 0, precision, k, sx, status,
                                w.normbits, hist_n ? w.bins : nullptr, hist_n, stream);
    csm::prof_end(stream, 3);
    if (e != cudaSuccess) return cuda_fail(e, "norm/select kernel");
    ++g_launches;
    return run_compute(dtype, wave, a, t, c, s, batch, n, k, sx, status, w, stream, eng,
                       hist_n > 0);
  }
  e = cudaMemsetAsync(w.normbits, 0, static_cast<size_t>(batch) * 8, stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(status, 0, static_cast<size_t>(batch) * 4, stream);
  if (e != cudaSuccess) return cuda_fail(e, "memset");
  if (n > 0) {
    e = csm::launch_norm1(dtype, a, batch, n, w.normbits, status, stream);
    if (e != cudaSuccess) return cuda_fail(e, "norm1 kernel");
    ++g_launches;
  }
  e = csm::launch_select(w.normbits, t, batch, wave ? 1 : 0, precision, k, sx, status, nullptr,
                         stream);
  if (e != cudaSuccess) return cuda_fail(e, "select kernel");
  ++g_launches;
  return run_compute(dtype, wave, a, t, c, s, batch, n, k, sx, status, w, stream, eng);
}

int core(int dtype, bool wave, int kval, const void* a, const double* t, void* c, void* s,
         int64_t batch, int n, int32_t* status, void* ws, size_t ws_bytes, void* stream_v) {
  g_launches = 0;
  const int eng = csm::engine();
  int rc = check_common(dtype, batch, n, ws_bytes, eng);
  if (rc) return rc;
  const bool ok = wave ? (kval == 3 || kval == 4 || kval == 5)
                       : (kval == 3 || kval == 4 || kval == 6 || kval == 7);
  if (!ok) return fail(CSM_ERR_ARG, "k_products is not valid for this scheme family");
  if (batch == 0) return CSM_SUCCESS;
  if (!status || !ws || (n > 0 && (!a || !c || !s)) || (wave && !t))
    return fail(CSM_ERR_ARG, "null pointer argument");
  if ((rc = check_device())) return rc;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  CommonWs w = carve(ws, batch);
  cudaError_t e = csm::launch_fill_ks(w.kbuf, w.sbuf, status, batch, kval, stream);
  if (e != cudaSuccess) return cuda_fail(e, "fill kernel");
  ++g_launches;
  return run_compute(dtype, wave, a, t, c, s, batch, n, w.kbuf, w.sbuf, status, w, stream, eng);
}

// ---- FP64 DMMA peak probe --------------------------------------------------
__global__ void dmma_peak_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) csm::dmma(c[i], a, b);
  }
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc += c[i][0] + c[i][1];
  if (acc == 1234.5) out[0] = acc;
}

}  // namespace

extern "C" {
#ifdef CSM_TRACE
int csm_trace_k1d_ctas(unsigned long long* out);
#endif

const char* csm_version(void) { return "cossin_b200 0.1.0 (sm_100a, FP64 DMMA)"; }

const char* csm_last_error(void) { return g_err.c_str(); }

int64_t csm_last_launch_count(void) { return g_launches; }

size_t csm_workspace_size(int dtype, int64_t batch, int n) {
  (void)dtype;
  return workspace_size(batch, n, csm::engine());
}

int csm_norm1(int dtype, const void* a, int64_t batch, int n, double* norms, int32_t* status,
              void* stream_v) {
  g_launches = 0;
  if (dtype != CSM_F64 && dtype != CSM_F32 && dtype != CSM_F32_IN_F64_OUT)
    return fail(CSM_ERR_ARG, "bad dtype");
  if (batch < 0 || n < 0) return fail(CSM_ERR_ARG, "batch and n must be nonnegative");
  if (batch == 0) return CSM_SUCCESS;
  if (!norms || !status || (n > 0 && !a)) return fail(CSM_ERR_ARG, "null pointer argument");
  int rc = check_device();
  if (rc) return rc;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  // norms doubles as the bit accumulator (same size, zero bits == 0.0)
  auto* bits = reinterpret_cast<unsigned long long*>(norms);
  cudaError_t e = cudaMemsetAsync(bits, 0, static_cast<size_t>(batch) * 8, stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(status, 0, static_cast<size_t>(batch) * 4, stream);
  if (e != cudaSuccess) return cuda_fail(e, "memset");
  if (n > 0) {
    e = csm::launch_norm1(dtype, a, batch, n, bits, status, stream);
    if (e != cudaSuccess) return cuda_fail(e, "norm1 kernel");
    ++g_launches;
  }
  return CSM_SUCCESS;
}

static bool family_ok(int family) {
  return family == CSM_FAMILY_TAYLOR || family == CSM_FAMILY_WAVE || family == CSM_FAMILY_PADE;
}

int csm_select_host(const double* norms, int64_t count, int family, int precision, int32_t* k,
                    int32_t* s, int32_t* status) {
  if (!family_ok(family)) return fail(CSM_ERR_ARG, "bad family");
  if (precision != CSM_PREC_DOUBLE && precision != CSM_PREC_SINGLE)
    return fail(CSM_ERR_ARG, "bad precision");
  if (count < 0) return fail(CSM_ERR_ARG, "count must be nonnegative");
  if (count > 0 && (!norms || !k || !s || !status)) return fail(CSM_ERR_ARG, "null pointer argument");
  const csm::Tables& T = csm::host_tables();
  for (int64_t i = 0; i < count; ++i) {
    int kk = 0, ss = 0;
    status[i] = csm::select_one(norms[i], T.theta[family][precision], T.kk[family][precision],
                                T.nent[family], T.log2fix, &kk, &ss);
    k[i] = kk;
    s[i] = ss;
  }
  return CSM_SUCCESS;
}

int csm_select_device(const double* norms, int64_t count, int family, int precision, int32_t* k,
                      int32_t* s, int32_t* status, void* stream) {
  g_launches = 0;
  if (!family_ok(family)) return fail(CSM_ERR_ARG, "bad family");
  if (precision != CSM_PREC_DOUBLE && precision != CSM_PREC_SINGLE)
    return fail(CSM_ERR_ARG, "bad precision");
  if (count < 0) return fail(CSM_ERR_ARG, "count must be nonnegative");
  if (count == 0) return CSM_SUCCESS;
  if (!norms || !k || !s || !status) return fail(CSM_ERR_ARG, "null pointer argument");
  int rc = check_device();
  if (rc) return rc;
  cudaError_t e = csm::launch_select_norms(norms, count, family, precision, k, s, status,
                                           static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "select kernel");
  ++g_launches;
  return CSM_SUCCESS;
}

int csm_select_table(const double* norms, int64_t count, const double* theta_eff,
                     const int64_t* cost_num, const int64_t* cost_den, int n_entries,
                     int32_t* entry_index, int32_t* s, int32_t* status) {
  if (count < 0 || n_entries <= 0) return fail(CSM_ERR_ARG, "need count >= 0 and n_entries > 0");
  if (count > 0 && (!norms || !theta_eff || !cost_num || !cost_den || !entry_index || !s || !status))
    return fail(CSM_ERR_ARG, "null pointer argument");
  for (int i = 0; i < n_entries; ++i)
    if (cost_den[i] <= 0) return fail(CSM_ERR_ARG, "cost denominators must be positive");
  const long long* fix = csm::host_tables().log2fix;
  for (int64_t q = 0; q < count; ++q) {
    const double norm = norms[q];
    entry_index[q] = 0;
    s[q] = 0;
    if (!(norm >= 0.0) || !csm::finite_d(norm)) { status[q] = CSM_NONFINITE_NORM; continue; }
    int chosen = -1;
    for (int i = 0; i < n_entries; ++i)
      if (norm <= theta_eff[i]) { chosen = i; break; }
    if (chosen >= 0) { entry_index[q] = chosen; status[q] = CSM_OK; continue; }
    int st = CSM_OK, best_i = -1, best_s = 0;
    __int128 bnum = 0, bden = 1;
    for (int i = 0; i < n_entries; ++i) {
      int si = 0;
      if (!(norm <= theta_eff[i])) {
        const double qv = norm / theta_eff[i];
        if (!csm::finite_d(qv)) { st = CSM_SELECT_OVERFLOW; break; }
        si = std::max(0, csm::ceil_log2_ref(qv, fix));
      }
      const __int128 num = static_cast<__int128>(cost_num[i]) + 2 * static_cast<__int128>(si) * cost_den[i];
      const __int128 den = cost_den[i];
      bool better = best_i < 0;
      if (!better) {
        const __int128 lhs = num * bden, rhs = bnum * den;
        better = lhs < rhs || (lhs == rhs && si < best_s);
      }
      if (better) { best_i = i; best_s = si; bnum = num; bden = den; }
    }
    status[q] = st;
    if (st == CSM_OK) { entry_index[q] = best_i; s[q] = best_s; }
  }
  return CSM_SUCCESS;
}

int csm_cos_sin(int dtype, int precision, const void* a, void* cos_out, void* sin_out,
                int64_t batch, int n, int32_t* k, int32_t* s, int32_t* status, void* workspace,
                size_t ws_bytes, void* stream) {
  return pipeline(dtype, precision, false, a, nullptr, cos_out, sin_out, batch, n, k, s, status,
                  workspace, ws_bytes, stream);
}

int csm_wave(int dtype, int precision, const void* a, const double* t, void* c_out, void* s_out,
             int64_t batch, int n, int32_t* k, int32_t* s, int32_t* status, void* workspace,
             size_t ws_bytes, void* stream) {
  return pipeline(dtype, precision, true, a, t, c_out, s_out, batch, n, k, s, status, workspace,
                  ws_bytes, stream);
}

int csm_taylor_core(int dtype, int k, const void* a, void* cos_out, void* sin_out, int64_t batch,
                    int n, int32_t* status, void* workspace, size_t ws_bytes, void* stream) {
  return core(dtype, false, k, a, nullptr, cos_out, sin_out, batch, n, status, workspace, ws_bytes,
              stream);
}

int csm_wave_core(int dtype, int k, const void* a, const double* t, void* c_out, void* s_out,
                  int64_t batch, int n, int32_t* status, void* workspace, size_t ws_bytes,
                  void* stream) {
  return core(dtype, true, k, a, t, c_out, s_out, batch, n, status, workspace, ws_bytes, stream);
}

int csm_theta_table(int family, int precision, double* theta_cos, double* theta_sin, int32_t* k,
                    int capacity) {
  if (!family_ok(family)) return fail(CSM_ERR_ARG, "bad family");
  if (precision != CSM_PREC_DOUBLE && precision != CSM_PREC_SINGLE)
    return fail(CSM_ERR_ARG, "bad precision");
  const double* tc[3][2] = {{kThetaCos_taylor_double, kThetaCos_taylor_single},
                            {kThetaCos_wave_double, kThetaCos_wave_single},
                            {kThetaCos_pade_double, kThetaCos_pade_single}};
  const double* ts[3][2] = {{kThetaSin_taylor_double, kThetaSin_taylor_single},
                            {kThetaSin_wave_double, kThetaSin_wave_single},
                            {kThetaSin_pade_double, kThetaSin_pade_single}};
  const int* kk[3][2] = {{kK_taylor_double, kK_taylor_single}, {kK_wave_double, kK_wave_single},
                         {kK_pade_double, kK_pade_single}};
  const int count = family == CSM_FAMILY_TAYLOR ? 4 : (family == CSM_FAMILY_WAVE ? 3 : 1);
  if (capacity < count || !theta_cos || !theta_sin || !k) return fail(CSM_ERR_ARG, "capacity too small");
  for (int i = 0; i < count; ++i) {
    theta_cos[i] = tc[family][precision][i];
    theta_sin[i] = ts[family][precision][i];
    k[i] = kk[family][precision][i];
  }
  return count;
}

#ifdef CSM_TRACE
int csm_trace_k1d_ctas(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, csm::f64k::g_k1d_cta, sizeof(unsigned long long) * 1024 * 4);
  return 0;
}
int csm_trace_dump(unsigned long long* out, int cap) {
  int n = 0;
  cudaMemcpyFromSymbol(&n, csm::f64k::g_trace_n, sizeof(int));
  if (n > cap) n = cap;
  if (n > (1 << 16)) n = 1 << 16;
  cudaMemcpyFromSymbol(out, csm::f64k::g_trace, sizeof(unsigned long long) * n);
  int zero = 0;
  cudaMemcpyToSymbol(csm::f64k::g_trace_n, &zero, sizeof(int));
  return n;
}
#endif

size_t csm_op_bytes(void) { return csm::op_bytes(); }

size_t csm_slab_scratch_bytes(void) { return csm::slab_scratch_bytes(); }

int csm_chain_program(int family, int k, int fold, void* ops_out, int max_ops, int32_t* step_nops,
                      int max_steps, int32_t* cos_slot, int32_t* sin_slot) {
  if (family != CSM_FAMILY_TAYLOR && family != CSM_FAMILY_WAVE) return fail(CSM_ERR_ARG, "bad family");
  const bool wave = family == CSM_FAMILY_WAVE;
  const bool ok = wave ? (k == 3 || k == 4 || k == 5) : (k == 3 || k == 4 || k == 6 || k == 7);
  if (!ok) return fail(CSM_ERR_ARG, "k_products is not valid for this scheme family");
  if (!ops_out || !step_nops || !cos_slot || !sin_slot) return fail(CSM_ERR_ARG, "null pointer argument");
  const int r = csm::chain_program(wave, k, fold != 0 && !wave, ops_out, max_ops, step_nops,
                                   max_steps, cos_slot, sin_slot);
  if (r < 0) return fail(CSM_ERR_ARG, "output arrays too small");
  return r;
}

int csm_doubling_program(int c0, int s0, int c1, int s1, void* ops_out) {
  if (!ops_out) return fail(CSM_ERR_ARG, "null pointer argument");
  const int v[4] = {c0, s0, c1, s1};
  for (int i = 0; i < 4; ++i)
    if (v[i] < 1 || v[i] >= CSM_SLAB_SLOTS) return fail(CSM_ERR_ARG, "slot out of range");
  csm::doubling_program(c0, s0, c1, s1, ops_out);
  return CSM_SUCCESS;
}

size_t csm_slab_engine_bytes(int M, int NP) {
  if (M <= 0 || NP <= 0) return 0;
  return csm::slab_engine_bytes(M, NP, csm::engine());
}

// Shared checks of the slab entry points; on success *eng is the call's
// engine snapshot (peer products always run DMMA and need no engine bytes).
static int slab_checks(const double* slab, int M, int NP, int row0, const void* scratch,
                       size_t scratch_bytes, bool peer, int* eng) {
  if (!slab || !scratch) return fail(CSM_ERR_ARG, "null pointer argument");
  if (M <= 0 || NP <= 0 || M % 64 || NP % 64 || row0 < 0 || row0 + M > NP)
    return fail(CSM_ERR_ARG, "slab shape must be M x NP with M, NP multiples of 64");
  *eng = csm::engine();
  const size_t need = csm::slab_scratch_bytes() + (peer ? 0 : csm::slab_engine_bytes(M, NP, *eng));
  if (scratch_bytes < need)
    return fail(CSM_ERR_WORKSPACE,
                "scratch smaller than csm_slab_scratch_bytes() + csm_slab_engine_bytes(M, NP) "
                "for this call's engine");
  return check_device();
}

int csm_slab_op(const void* op, double* slab, int M, int NP, int row0, const double* rhs_full,
                const double* in0, int s, double tp, int dbl_step, void* cos_out, void* sin_out,
                int out_f32, void* scratch, size_t scratch_bytes, void* stream) {
  g_launches = 0;
  if (!op || !rhs_full) return fail(CSM_ERR_ARG, "null pointer argument");
  int eng = 0;
  int rc = slab_checks(slab, M, NP, row0, scratch, scratch_bytes, false, &eng);
  if (rc) return rc;
  const void* ops[1] = {op};
  cudaError_t e = csm::slab_op(ops, 1, slab, M, NP, row0, rhs_full, in0, s, tp, dbl_step,
                               cos_out, sin_out, out_f32, scratch,
                               static_cast<cudaStream_t>(stream), &g_launches, nullptr, 0, eng);
  if (e != cudaSuccess) return cuda_fail(e, "slab op");
  return CSM_SUCCESS;
}

int csm_slab_op_pair(const void* op_a, const void* op_b, double* slab, int M, int NP, int row0,
                     const double* rhs_full, const double* in0, int s, double tp, int dbl_step,
                     void* cos_out, void* sin_out, int out_f32, void* scratch,
                     size_t scratch_bytes, void* stream) {
  g_launches = 0;
  if (!op_a || !op_b || !rhs_full) return fail(CSM_ERR_ARG, "null pointer argument");
  if (dbl_step < 0) return fail(CSM_ERR_ARG, "csm_slab_op_pair runs a doubling step (dbl_step >= 0)");
  int eng = 0;
  int rc = slab_checks(slab, M, NP, row0, scratch, scratch_bytes, false, &eng);
  if (rc) return rc;
  const void* ops[2] = {op_a, op_b};
  cudaError_t e = csm::slab_op(ops, 2, slab, M, NP, row0, rhs_full, in0, s, tp, dbl_step,
                               cos_out, sin_out, out_f32, scratch,
                               static_cast<cudaStream_t>(stream), &g_launches, nullptr, 0, eng);
  if (e != cudaSuccess) return cuda_fail(e, "slab op pair");
  return CSM_SUCCESS;
}

int csm_slab_op_peer(const void* op, double* slab, int M, int NP, int row0,
                     const double* const* rhs_slabs, int nparts, const double* in0, int s,
                     double tp, int dbl_step, void* cos_out, void* sin_out, int out_f32,
                     void* scratch, size_t scratch_bytes, void* stream) {
  g_launches = 0;
  if (!op || !rhs_slabs) return fail(CSM_ERR_ARG, "null pointer argument");
  if (nparts <= 0 || nparts > 64 || nparts * M != NP)
    return fail(CSM_ERR_ARG, "need M, NP multiples of 64 and nparts * M == NP (<= 64 parts)");
  for (int i = 0; i < nparts; ++i)
    if (!rhs_slabs[i]) return fail(CSM_ERR_ARG, "null peer slab");
  int eng = 0;
  int rc = slab_checks(slab, M, NP, row0, scratch, scratch_bytes, true, &eng);
  if (rc) return rc;
  const void* ops[1] = {op};
  cudaError_t e = csm::slab_op(ops, 1, slab, M, NP, row0, nullptr, in0, s, tp, dbl_step, cos_out,
                               sin_out, out_f32, scratch, static_cast<cudaStream_t>(stream),
                               &g_launches, rhs_slabs, nparts, CSM_ENGINE_DMMA);
  if (e != cudaSuccess) return cuda_fail(e, "peer slab op");
  return CSM_SUCCESS;
}

size_t csm_sine_workspace_size(int dtype, int64_t batch, int n) {
  (void)dtype;
  if (batch < 0 || n < 0) return 0;
  return common_bytes(batch) + csm::tiled_workspace_bytes(batch, n, csm::engine()) + 256;
}

static int standalone_sine(int dtype, bool wave, const void* a, const double* t, void* s_out,
                           int64_t batch, int n, int32_t* status, void* ws, size_t ws_bytes,
                           void* stream_v) {
  g_launches = 0;
  if (dtype != CSM_F64 && dtype != CSM_F32 && dtype != CSM_F32_IN_F64_OUT)
    return fail(CSM_ERR_ARG, "bad dtype");
  if (batch < 0 || n < 0) return fail(CSM_ERR_ARG, "batch and n must be nonnegative");
  const int eng = csm::engine();
  if (ws_bytes < common_bytes(batch) + csm::tiled_workspace_bytes(batch, n, eng) + 256)
    return fail(CSM_ERR_WORKSPACE, "workspace smaller than csm_sine_workspace_size()");
  if (batch == 0 || n == 0) return CSM_SUCCESS;
  if (!a || !s_out || !status || !ws || (wave && !t)) return fail(CSM_ERR_ARG, "null pointer argument");
  int rc = check_device();
  if (rc) return rc;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  CommonWs w = carve(ws, batch);
  cudaError_t e = csm::launch_fill_ks(w.kbuf, w.sbuf, status, batch, 3, stream);
  if (e != cudaSuccess) return cuda_fail(e, "fill kernel");
  ++g_launches;
  e = csm::run_tiled(dtype, wave, a, t, nullptr, s_out, batch, n, w.kbuf, w.sbuf, status, w.tiled,
                     stream, &g_launches, wave ? 2 : 1, eng);
  if (e != cudaSuccess) return cuda_fail(e, "standalone sine");
  return CSM_SUCCESS;
}

int csm_taylor_sin9(int dtype, const void* a, void* sin_out, int64_t batch, int n,
                    int32_t* status, void* workspace, size_t ws_bytes, void* stream) {
  return standalone_sine(dtype, false, a, nullptr, sin_out, batch, n, status, workspace, ws_bytes,
                         stream);
}

int csm_wave_sin34(int dtype, const void* a, const double* t, void* s_out, int64_t batch, int n,
                   int32_t* status, void* workspace, size_t ws_bytes, void* stream) {
  return standalone_sine(dtype, true, a, t, s_out, batch, n, status, workspace, ws_bytes, stream);
}

// ---------------------------------------------------------------------------
// Pythagorean residual of computed pairs (diagnostic; pkg/README.md:172-176).

size_t csm_residual_workspace_size(int64_t batch, int n) {
  if (batch < 0 || n < 0) return 0;
  return csm::residual_workspace_bytes(batch, n);
}

int csm_pythagorean_residual(int dtype, const void* cos_in, const void* sin_in, int64_t batch,
                             int n, double* out, void* workspace, size_t ws_bytes, void* stream) {
  g_launches = 0;
  if (dtype != CSM_F64 && dtype != CSM_F32) return fail(CSM_ERR_ARG, "dtype must be CSM_F64 or CSM_F32");
  if (batch < 0 || n < 0) return fail(CSM_ERR_ARG, "batch and n must be nonnegative");
  if (ws_bytes < csm_residual_workspace_size(batch, n))
    return fail(CSM_ERR_WORKSPACE, "workspace smaller than csm_residual_workspace_size()");
  if (batch == 0) return CSM_SUCCESS;
  if (!out || (n > 0 && (!cos_in || !sin_in || !workspace)))
    return fail(CSM_ERR_ARG, "null pointer argument");
  int rc = check_device();
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n == 0) {
    cudaError_t e = cudaMemsetAsync(out, 0, static_cast<size_t>(batch) * 8, st);
    return e == cudaSuccess ? CSM_SUCCESS : cuda_fail(e, "memset");
  }
  cudaError_t e = csm::pythagorean_residual(dtype == CSM_F32, cos_in, sin_in, batch, n, out,
                                            workspace, st, &g_launches);
  if (e != cudaSuccess) return cuda_fail(e, "residual kernels");
  return CSM_SUCCESS;
}

// ---------------------------------------------------------------------------
// Double-double reference cos/sin (verify.py:480-521) and its product.

size_t csm_ddref_workspace_size(int64_t batch, int n) {
  if (batch < 0 || n < 0) return 0;
  return 3 * align256(static_cast<size_t>(batch) * 8) +
         csm::ddref_workspace_doubles(batch, n) * 8 + 256;
}

int csm_ddref_series_consts(double* out28) {
  if (!out28) return fail(CSM_ERR_ARG, "null pointer argument");
  csm::ddref_series_consts(out28);
  return CSM_SUCCESS;
}

int csm_dd_matmul(const double* xh, const double* xl, const double* yh, const double* yl,
                  double* oh, double* ol, int64_t batch, int n, void* stream) {
  g_launches = 0;
  if (batch < 0 || n < 0) return fail(CSM_ERR_ARG, "batch and n must be nonnegative");
  if (batch == 0 || n == 0) return CSM_SUCCESS;
  if (!xh || !yh || !oh || !ol) return fail(CSM_ERR_ARG, "null pointer argument");
  int rc = check_device();
  if (rc) return rc;
  cudaError_t e = csm::dd_matmul(xh, xl, yh, yl, oh, ol, batch, n,
                                 static_cast<cudaStream_t>(stream), &g_launches);
  if (e != cudaSuccess) return cuda_fail(e, "dd_matmul");
  return CSM_SUCCESS;
}

int csm_ddref_cos_sin(const double* a, double* cos_out, double* sin_out, int64_t batch, int n,
                      int32_t* s_host, int32_t* status_host, void* ws, size_t ws_bytes,
                      void* stream_v) {
  g_launches = 0;
  if (batch < 0 || n < 0) return fail(CSM_ERR_ARG, "batch and n must be nonnegative");
  if (ws_bytes < csm_ddref_workspace_size(batch, n))
    return fail(CSM_ERR_WORKSPACE, "workspace smaller than csm_ddref_workspace_size()");
  if (batch == 0 || n == 0) return CSM_SUCCESS;
  if (!a || !cos_out || !sin_out || !s_host || !status_host || !ws)
    return fail(CSM_ERR_ARG, "null pointer argument");
  int rc = check_device();
  if (rc) return rc;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  char* p = static_cast<char*>(ws);
  auto* bits = reinterpret_cast<unsigned long long*>(p);
  p += align256(static_cast<size_t>(batch) * 8);
  auto* dst = reinterpret_cast<int32_t*>(p);
  p += align256(static_cast<size_t>(batch) * 8);
  auto* dS = reinterpret_cast<int32_t*>(p);
  p += align256(static_cast<size_t>(batch) * 8);
  cudaError_t e = cudaMemsetAsync(bits, 0, static_cast<size_t>(batch) * 8, stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(dst, 0, static_cast<size_t>(batch) * 4, stream);
  if (e == cudaSuccess) e = csm::launch_norm1(CSM_F64, a, batch, n, bits, dst, stream);
  if (e != cudaSuccess) return cuda_fail(e, "ddref norm");
  ++g_launches;
  std::vector<unsigned long long> hb(static_cast<size_t>(batch));
  e = cudaMemcpyAsync(hb.data(), bits, hb.size() * 8, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return cuda_fail(e, "ddref norm readback");
  // verify.py:495-498: s = ceil(log2(norm / 2^-20)) when norm > 2^-20;
  // a nan norm compares false (s = 0), an infinite quotient is the
  // reference's OverflowError.
  const double cap = 0x1p-20;
  std::vector<int32_t> hs(hb.size(), 0);
  int smax = 0;
  for (size_t b = 0; b < hb.size(); ++b) {
    double norm;
    std::memcpy(&norm, &hb[b], 8);
    status_host[b] = CSM_OK;
    if (norm > cap) {
      const double q = norm / cap;
      if (!csm::finite_d(q)) {
        status_host[b] = CSM_SELECT_OVERFLOW;
      } else {
        hs[b] = csm::ceil_log2_ref(q, csm::host_tables().log2fix);
      }
    }
    s_host[b] = hs[b];
    smax = std::max(smax, hs[b]);
  }
  e = cudaMemcpyAsync(dS, hs.data(), hs.size() * 4, cudaMemcpyHostToDevice, stream);
  if (e != cudaSuccess) return cuda_fail(e, "ddref s upload");
  e = csm::ddref_chain(a, dS, smax, cos_out, sin_out, batch, n,
                       reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255)),
                       stream, &g_launches);
  if (e != cudaSuccess) return cuda_fail(e, "ddref chain");
  // the host vector hs must outlive the async upload
  e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return cuda_fail(e, "ddref chain");
  return CSM_SUCCESS;
}

// ---------------------------------------------------------------------------
// Order-8 Pade baseline (driver.py:149-164).

size_t csm_pade_workspace_size(int dtype, int64_t batch, int n) {
  (void)dtype;
  if (batch < 0 || n < 0) return 0;
  return common_bytes(batch) + csm::tiled_workspace_bytes(batch, n, csm::engine()) + 256;
}

int csm_pade_cos_sin(int dtype, int precision, const void* a, void* cos_out, void* sin_out,
                     int64_t batch, int n, int32_t* k, int32_t* sx, int32_t* status, void* ws,
                     size_t ws_bytes, void* stream_v) {
  g_launches = 0;
  if (dtype != CSM_F64 && dtype != CSM_F32 && dtype != CSM_F32_IN_F64_OUT)
    return fail(CSM_ERR_ARG, "bad dtype");
  if (precision != CSM_PREC_DOUBLE && precision != CSM_PREC_SINGLE)
    return fail(CSM_ERR_ARG, "bad precision");
  if (batch < 0 || n < 0) return fail(CSM_ERR_ARG, "batch and n must be nonnegative");
  const int eng = csm::engine();
  if (ws_bytes < common_bytes(batch) + csm::tiled_workspace_bytes(batch, n, eng) + 256)
    return fail(CSM_ERR_WORKSPACE, "workspace smaller than csm_pade_workspace_size()");
  if (batch == 0) return CSM_SUCCESS;
  if (!k || !sx || !status || !ws || (n > 0 && (!a || !cos_out || !sin_out)))
    return fail(CSM_ERR_ARG, "null pointer argument");
  int rc = check_device();
  if (rc) return rc;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  CommonWs w = carve(ws, batch);
  cudaError_t e = cudaMemsetAsync(w.normbits, 0, static_cast<size_t>(batch) * 8, stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(status, 0, static_cast<size_t>(batch) * 4, stream);
  if (e != cudaSuccess) return cuda_fail(e, "memset");
  if (n > 0) {
    e = csm::launch_norm1(dtype, a, batch, n, w.normbits, status, stream);
    if (e != cudaSuccess) return cuda_fail(e, "norm1 kernel");
    ++g_launches;
  }
  e = csm::launch_select(w.normbits, nullptr, batch, CSM_FAMILY_PADE, precision, k, sx, status,
                         nullptr, stream);
  if (e != cudaSuccess) return cuda_fail(e, "select kernel");
  ++g_launches;
  if (n == 0) return CSM_SUCCESS;
  e = csm::run_tiled(dtype, false, a, nullptr, cos_out, sin_out, batch, n, k, sx, status, w.tiled,
                     stream, &g_launches, 3, eng);
  if (e != cudaSuccess) return cuda_fail(e, "pade chain");
  return CSM_SUCCESS;
}

// The Pade base pair alone (schemes.py:446-464 pade8_cos_sin): k = 5,
// s = 0 for every matrix, no selection, then the same chain as above.
int csm_pade_core(int dtype, const void* a, void* cos_out, void* sin_out, int64_t batch, int n,
                  int32_t* status, void* ws, size_t ws_bytes, void* stream_v) {
  g_launches = 0;
  if (dtype != CSM_F64 && dtype != CSM_F32 && dtype != CSM_F32_IN_F64_OUT)
    return fail(CSM_ERR_ARG, "bad dtype");
  if (batch < 0 || n < 0) return fail(CSM_ERR_ARG, "batch and n must be nonnegative");
  const int eng = csm::engine();
  if (ws_bytes < common_bytes(batch) + csm::tiled_workspace_bytes(batch, n, eng) + 256)
    return fail(CSM_ERR_WORKSPACE, "workspace smaller than csm_pade_workspace_size()");
  if (batch == 0) return CSM_SUCCESS;
  if (!status || !ws || (n > 0 && (!a || !cos_out || !sin_out)))
    return fail(CSM_ERR_ARG, "null pointer argument");
  int rc = check_device();
  if (rc) return rc;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  CommonWs w = carve(ws, batch);
  cudaError_t e = csm::launch_fill_ks(w.kbuf, w.sbuf, status, batch, 5, stream);
  if (e != cudaSuccess) return cuda_fail(e, "fill kernel");
  ++g_launches;
  if (n == 0) return CSM_SUCCESS;
  e = csm::run_tiled(dtype, false, a, nullptr, cos_out, sin_out, batch, n, w.kbuf, w.sbuf, status,
                     w.tiled, stream, &g_launches, 3, eng);
  if (e != cudaSuccess) return cuda_fail(e, "pade chain");
  return CSM_SUCCESS;
}

// ---- distributed chain (distchain.cu) ------------------------------------
namespace {
thread_local int32_t g_dist_gathers = 0, g_dist_products = 0;

int dist_common(int precision, const double* a, int n, int world, size_t ws_bytes, size_t need) {
  if (precision != CSM_PREC_DOUBLE && precision != CSM_PREC_SINGLE)
    return fail(CSM_ERR_ARG, "bad precision");
  if (world < 1) return fail(CSM_ERR_ARG, "world must be >= 1");
  if (n <= 0 || n % (64 * world)) return fail(CSM_ERR_ARG, "n must be a positive multiple of 64 x world");
  if (!a) return fail(CSM_ERR_ARG, "null pointer argument");
  if (ws_bytes < need) return fail(CSM_ERR_WORKSPACE, "workspace smaller than csm_dist_workspace_size()");
  return check_device();
}
}  // namespace

size_t csm_dist_workspace_size(int n, int world, int flags) {
  if (n <= 0 || world < 1 || n % world) return 0;
  return csm::dc::rank_bytes(n, world, world > 1 || (flags & CSM_DIST_FORCE_GATHER));
}

int csm_dist_cos_sin(int precision, const double* a, double* cos_rows, double* sin_rows, int n,
                     ncclComm_t comm, int flags, int32_t* k, int32_t* s, int32_t* status,
                     void* ws, size_t ws_bytes, void* stream_v) {
  g_launches = 0;
  g_dist_gathers = g_dist_products = 0;
  int world = 1, rank = 0;
  const bool force = (flags & CSM_DIST_FORCE_GATHER) != 0;
  if (comm) {
    if (!csm::dc::nccl().ok) return fail(CSM_ERR_ARG, "NCCL entry points not found in the process or libnccl.so.2");
    if (csm::dc::nccl().comm_count(comm, &world) != 0 ||
        csm::dc::nccl().comm_user_rank(comm, &rank) != 0)
      return fail(CSM_ERR_ARG, "invalid NCCL communicator");
  } else if (force) {
    return fail(CSM_ERR_ARG, "CSM_DIST_FORCE_GATHER needs a communicator");
  }
  int rc = dist_common(precision, a, n, world, ws_bytes, csm_dist_workspace_size(n, world, flags));
  if (rc) return rc;
  if (!cos_rows || !sin_rows || !k || !s || !status || !ws) return fail(CSM_ERR_ARG, "null pointer argument");
  csm::dc::Exchange ex;
  ex.comm = comm;
  ex.world = world;
  csm::dc::Result res;
  std::string why;
  void* wsv[1] = {ws};
  double* cr[1] = {cos_rows};
  double* sr[1] = {sin_rows};
  cudaError_t e = csm::dc::run(precision, a, n, world, rank, 1, wsv, cr, sr, ex, force,
                               static_cast<cudaStream_t>(stream_v), &res, &g_launches, &why);
  *k = res.k;
  *s = res.s;
  *status = res.status;
  g_dist_gathers = res.gathers;
  g_dist_products = res.products;
  if (e != cudaSuccess) return why.empty() ? cuda_fail(e, "distributed chain") : fail(CSM_ERR_CUDA, why);
  return CSM_SUCCESS;
}

int csm_dist_cos_sin_virtual(int precision, const double* a, double* cos_out, double* sin_out,
                             int n, int world, int32_t* k, int32_t* s, int32_t* status, void* ws,
                             size_t ws_bytes, void* stream_v) {
  g_launches = 0;
  g_dist_gathers = g_dist_products = 0;
  const size_t per = csm_dist_workspace_size(n, world, CSM_DIST_FORCE_GATHER);
  int rc = dist_common(precision, a, n, world, ws_bytes, per * static_cast<size_t>(world));
  if (rc) return rc;
  if (!cos_out || !sin_out || !k || !s || !status || !ws) return fail(CSM_ERR_ARG, "null pointer argument");
  std::vector<void*> wsv(world);
  std::vector<double*> cr(world), sr(world);
  const size_t M = static_cast<size_t>(n) / world;
  for (int q = 0; q < world; ++q) {
    wsv[q] = static_cast<char*>(ws) + q * per;
    cr[q] = cos_out + q * M * n;
    sr[q] = sin_out + q * M * n;
  }
  csm::dc::Exchange ex;
  ex.world = world;
  csm::dc::Result res;
  std::string why;
  cudaError_t e = csm::dc::run(precision, a, n, world, 0, world, wsv.data(), cr.data(), sr.data(),
                               ex, world == 1, static_cast<cudaStream_t>(stream_v), &res,
                               &g_launches, &why);
  *k = res.k;
  *s = res.s;
  *status = res.status;
  g_dist_gathers = res.gathers;
  g_dist_products = res.products;
  if (e != cudaSuccess) return why.empty() ? cuda_fail(e, "virtual distributed chain") : fail(CSM_ERR_CUDA, why);
  return CSM_SUCCESS;
}

int csm_dist_last_stats(int32_t* gathers, int32_t* products) {
  if (!gathers || !products) return fail(CSM_ERR_ARG, "null pointer argument");
  *gathers = g_dist_gathers;
  *products = g_dist_products;
  return CSM_SUCCESS;
}

int csm_nccl_get_unique_id(void* id) {
  if (!id) return fail(CSM_ERR_ARG, "null pointer argument");
  if (!csm::dc::nccl().ok) return fail(CSM_ERR_ARG, "NCCL entry points not found");
  const int rc = csm::dc::nccl_unique_id(id);
  return rc ? fail(CSM_ERR_CUDA, "ncclGetUniqueId failed: " + std::to_string(rc)) : CSM_SUCCESS;
}

int csm_nccl_comm_init_rank(ncclComm_t* comm, int nranks, const void* id, int rank) {
  if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks) return fail(CSM_ERR_ARG, "bad argument");
  if (!csm::dc::nccl().ok) return fail(CSM_ERR_ARG, "NCCL entry points not found");
  void* c = nullptr;
  const int rc = csm::dc::nccl_comm_init(&c, nranks, id, rank);
  if (rc) return fail(CSM_ERR_CUDA, "ncclCommInitRank failed: " + std::to_string(rc));
  *comm = static_cast<ncclComm_t>(c);
  return CSM_SUCCESS;
}

int csm_nccl_comm_destroy(ncclComm_t comm) {
  if (!comm) return CSM_SUCCESS;
  if (!csm::dc::nccl().ok) return fail(CSM_ERR_ARG, "NCCL entry points not found");
  const int rc = csm::dc::nccl().comm_destroy(comm);
  return rc ? fail(CSM_ERR_CUDA, "ncclCommDestroy failed: " + std::to_string(rc)) : CSM_SUCCESS;
}

int csm_graph_safe(int dtype, int64_t batch, int n) {
  (void)dtype;
  if (batch < 0 || n < 0) return 0;
  if (n <= 64) return 1;
  return (n <= fused_max() && side_count(batch) == 0) ? 1 : 0;
}

int csm_profile_enable(int on) {
  prof_clear();
  if (on < 0 || on > 3) return fail(CSM_ERR_ARG, "profile mode must be 0, 1, 2 or 3");
  g_prof = on;
  return CSM_SUCCESS;
}

int csm_profile_collect(double* total_ms, int64_t* intervals) {
  if (!total_ms || !intervals) return fail(CSM_ERR_ARG, "null pointer argument");
  double sum = 0.0;
  for (auto& p : g_prof_ev) {
    cudaError_t e = cudaEventSynchronize(p.second);
    if (e != cudaSuccess) return cuda_fail(e, "profile events");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.first, p.second);
    sum += ms;
  }
  *total_ms = sum;
  *intervals = static_cast<int64_t>(g_prof_ev.size());
  prof_clear();
  return CSM_SUCCESS;
}

int csm_set_engine(int engine) {
  if (engine != CSM_ENGINE_DMMA && engine != CSM_ENGINE_OZAKI && engine != CSM_ENGINE_AUTO &&
      engine != CSM_ENGINE_OZAKI_UNGUARDED)
    return fail(CSM_ERR_ARG, "engine must be CSM_ENGINE_DMMA, CSM_ENGINE_OZAKI or CSM_ENGINE_AUTO");
  csm::set_engine(engine);
  return CSM_SUCCESS;
}

int csm_get_engine(void) { return csm::engine(); }

int csm_set_thread_engine(int engine) {
  if (engine != -1 && engine != CSM_ENGINE_DMMA && engine != CSM_ENGINE_OZAKI &&
      engine != CSM_ENGINE_AUTO && engine != CSM_ENGINE_OZAKI_UNGUARDED)
    return fail(CSM_ERR_ARG, "thread engine must be -1 (none) or a CSM_ENGINE_* value");
  csm::set_thread_engine(engine);
  return CSM_SUCCESS;
}

int csm_fp64_peak(int iters, double* tflops, void* stream_v) {
  if (!tflops || iters <= 0) return fail(CSM_ERR_ARG, "bad arguments");
  int rc = check_device();
  if (rc) return rc;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* scratch = nullptr;
  cudaError_t e = cudaMalloc(&scratch, 8);
  if (e != cudaSuccess) return cuda_fail(e, "malloc");
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int warps = 8;
  dmma_peak_kernel<<<sms, 32 * warps, 0, stream>>>(scratch, iters / 8 + 1);  // warm-up
  cudaEventRecord(e0, stream);
  dmma_peak_kernel<<<sms, 32 * warps, 0, stream>>>(scratch, iters);
  cudaEventRecord(e1, stream);
  e = cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(scratch);
  if (e != cudaSuccess) return cuda_fail(e, "peak kernel");
  const double flops = 2.0 * 256.0 * 8.0 * static_cast<double>(iters) * warps * sms;
  *tflops = flops / (static_cast<double>(ms) * 1e-3) / 1e12;
  return CSM_SUCCESS;
}

}  // extern "C"
