// distchain.cu -- block-row distributed cos/sin of ONE large matrix
// (configs[4], 8192^2) driven from C++: the program of the Taylor chain
// (chain_deg{2,4,8,12}, schemes.py:264-361) and the doubling steps
// (driver.py:91-98) over W ranks, every product out_rows = L_rows R_full on
// the tiled DMMA kernel in slab mode, the right operand all-gathered over
// NCCL (csm_dist_cos_sin) -- the C-ABI twin of distchain.py's gather mode.
//
// Gathers overlap compute.  A product whose right operand R is not yet
// gathered is split along k: the all-gather of R runs on a side stream
// while the rank contracts the k range of its OWN rows of R (already in its
// slab; ksplit 1, raw partial product to a scratch slab), then the
// complementary k range from the gathered copy adds the partial product
// before the fused epilogue (ksplit 2).  At W ranks the first part is 1/W
// of the product, so the gather (7/8 x 512 MiB per product at W = 8)
// hides behind ~1/8 of a 137 GFLOP product ("cfg5 time model").
// A gathered copy is cached until its slot is rewritten; products whose
// right operand is the replicated input A (A A, and the final sin = A sc
// evaluated as sc A: polynomials in A commute) need no gather at all.
//
// The same schedule runs W virtual ranks in one process
// (csm_dist_cos_sin_virtual: all slabs on one device, the all-gather as
// device copies) so the split products and the cache are tested on one GPU.
//
// NCCL is not linked: its entry points are resolved at run time from the
// library the process already loaded (torch's) or libnccl.so.2.
#include <dlfcn.h>

#include <map>
#include <string>

namespace csm {

namespace dc {

constexpr size_t kStageBytes = 16384;  // op table + idx + s + tp + selection scratch

// -- NCCL entry points (resolved lazily) -------------------------------------
typedef int (*PfnGetUniqueId)(void*);
typedef int (*PfnCommDestroy)(void*);
typedef int (*PfnAllGather)(const void*, void*, size_t, int, void*, cudaStream_t);
typedef int (*PfnCommCount)(const void*, int*);
typedef int (*PfnCommUserRank)(const void*, int*);
typedef const char* (*PfnGetErrorString)(int);

struct Nccl {
  PfnGetUniqueId get_unique_id = nullptr;
  void* comm_init_rank = nullptr;  // called through a by-value thunk below
  PfnCommDestroy comm_destroy = nullptr;
  PfnAllGather all_gather = nullptr;
  PfnCommCount comm_count = nullptr;
  PfnCommUserRank comm_user_rank = nullptr;
  PfnGetErrorString error_string = nullptr;
  bool ok = false;
};

struct UniqueId {
  char internal[128];
};
typedef int (*PfnCommInitRankV)(void**, int, UniqueId, int);

const Nccl& nccl() {
  static Nccl api = [] {
    Nccl a;
    void* h = RTLD_DEFAULT;
    if (!dlsym(h, "ncclAllGather")) {
      h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) return a;
    }
    a.get_unique_id = reinterpret_cast<PfnGetUniqueId>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = dlsym(h, "ncclCommInitRank");
    a.comm_destroy = reinterpret_cast<PfnCommDestroy>(dlsym(h, "ncclCommDestroy"));
    a.all_gather = reinterpret_cast<PfnAllGather>(dlsym(h, "ncclAllGather"));
    a.comm_count = reinterpret_cast<PfnCommCount>(dlsym(h, "ncclCommCount"));
    a.comm_user_rank = reinterpret_cast<PfnCommUserRank>(dlsym(h, "ncclCommUserRank"));
    a.error_string = reinterpret_cast<PfnGetErrorString>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.all_gather &&
           a.comm_count && a.comm_user_rank;
    return a;
  }();
  return api;
}
constexpr int kNcclFloat64 = 8;  // ncclDataType_t ncclFloat64 / ncclDouble

int nccl_unique_id(void* out) { return nccl().get_unique_id(out); }
int nccl_comm_init(void** comm, int nranks, const void* id, int rank) {
  UniqueId u;
  std::memcpy(u.internal, id, sizeof(u.internal));
  return reinterpret_cast<PfnCommInitRankV>(nccl().comm_init_rank)(comm, nranks, u, rank);
}

// -- schedule -----------------------------------------------------------------
struct Action {
  int op, nops, rhs, dbl_step;
  std::vector<int> writes;  // slots rewritten by this step (invalidate their gathered copies)
};

struct Schedule {
  std::vector<tk::Op> ops;  // chain ops, then doubling pairs (c0,s0->c1,s1), (c1,s1->c0,s0)
  std::vector<Action> acts;
};

Schedule schedule(int k, int s) {
  Schedule S;
  Program P = build_program(false, k, true);
  for (auto& step : P.steps) {
    std::vector<int> written;
    std::vector<int> first;
    for (auto& op0 : step) {
      tk::Op op = op0;
      if (op.lhs == 0 && op.rhs != 0) std::swap(op.lhs, op.rhs);  // A X = X A
      first.push_back(static_cast<int>(S.ops.size()));
      S.ops.push_back(op);
      for (int q = 0; q < op.nout; ++q) written.push_back(op.out[q].slot);
    }
    for (size_t i = 0; i < step.size(); ++i)
      S.acts.push_back({first[i], 1, S.ops[first[i]].rhs, -1,
                        i + 1 == step.size() ? written : std::vector<int>{}});
  }
  int c0 = P.cos_slot, s0 = P.sin_slot, c1, s1;
  free_pair(c0, s0, &c1, &s1);
  const int pairA = static_cast<int>(S.ops.size());
  for (auto& op : doubling_ops(c0, s0, c1, s1)) S.ops.push_back(op);
  const int pairB = static_cast<int>(S.ops.size());
  for (auto& op : doubling_ops(c1, s1, c0, s0)) S.ops.push_back(op);
  for (int i = 0; i < s; ++i) {
    const bool a = (i & 1) == 0;
    S.acts.push_back({a ? pairA : pairB, 2, a ? c0 : c1, i, {a ? c1 : c0, a ? s1 : s0}});
  }
  return S;
}

// Gathered copies alive at once, over every Taylor k (the doubling adds at
// most one): sizes the per-rank gather pool.
int max_live_gathers() {
  static int m = [] {
    int best = 1;
    for (int k : {3, 4, 6, 7}) {
      Schedule S = schedule(k, 4);
      std::map<int, int> live;
      for (auto& a : S.acts) {
        if (a.rhs != 0) live[a.rhs] = 1;
        best = std::max(best, static_cast<int>(live.size()));
        for (int w : a.writes) live.erase(w);
      }
    }
    return best;
  }();
  return m;
}

// Per-rank workspace: staging | slab (NSLOT x M x n) | partial products
// (2 x M x n) | gather pool (G x n x n, only when W > 1 or gathers forced).
struct RankWs {
  char* stage;
  double* slab;
  double* part;
  double* pool;
};

size_t rank_bytes(int n, int world, bool gathers) {
  const size_t M = static_cast<size_t>(n) / world;
  size_t b = kStageBytes + static_cast<size_t>(tk::NSLOT) * M * n * 8 + 2 * M * n * 8;
  if (gathers) b += static_cast<size_t>(max_live_gathers()) * n * n * 8;
  return b + 256;
}

RankWs carve_rank(void* ws, int n, int world) {
  const size_t M = static_cast<size_t>(n) / world;
  char* p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
  RankWs r;
  r.stage = p;
  p += kStageBytes;
  r.slab = reinterpret_cast<double*>(p);
  p += static_cast<size_t>(tk::NSLOT) * M * n * 8;
  r.part = reinterpret_cast<double*>(p);
  p += 2 * M * n * 8;
  r.pool = reinterpret_cast<double*>(p);
  return r;
}

struct Staged {  // device copy, at the start of local rank 0's stage
  int32_t idx, s, k, status;
  double tp;
  unsigned long long normbits;
  int32_t pad[2];
};
constexpr size_t kOpsOffset = 256;

// One launch of the tiled kernel in slab mode for local rank q.
cudaError_t launch(const tk::Op* d_ops, const Staged* d_st, int op, int nops, double* slab,
                   int M, int n, int row0, const double* in0, const double* rhs_full,
                   int ksplit, double* part, int dbl_step, double* cos_rows, double* sin_rows,
                   cudaStream_t st, int64_t* launches) {
  tk::LaunchArgs A{};
  A.ws = slab;
  A.in0 = in0;
  A.idx = &d_st->idx;
  A.ops = d_ops + op;
  A.tsc = &d_st->tp;
  A.S = &d_st->s;
  A.cout = cos_rows;
  A.sout = sin_rows;
  A.mat_stride = 0;
  A.NP = n;
  A.n = n;
  A.out_f32 = 0;
  A.dbl_step = dbl_step;
  A.nseg = nops;
  A.total = nops;
  A.item_base = 0;
  for (int i = 0; i < nops; ++i) A.seg[i] = {i, 0, i};
  A.rhs_full = rhs_full;
  A.M = M;
  A.row0 = row0;
  A.ksplit = ksplit;
  A.part = part;
  tk::set_tma(A, static_cast<size_t>(tk::NSLOT) * M, static_cast<size_t>(M));
  dim3 grid(static_cast<unsigned>((M / tk::BM) * (n / tk::BN)), static_cast<unsigned>(nops), 1);
  tk::launch_gemm(grid, A, st);
  ++*launches;
  return cudaGetLastError();
}

// The all-gather of slot `slot`: NCCL (one local rank) or, for virtual
// ranks, every rank's block copied into every rank's pool buffer.
struct Exchange {
  void* comm = nullptr;  // NCCL communicator (null: virtual or W = 1)
  int world = 1;
};

struct Result {
  int k = 0, s = 0, status = 0, gathers = 0, products = 0;
};

// Run the schedule for `nlocal` ranks held by this process (1 with NCCL,
// W when virtual).  ws[q], cos_rows[q], sin_rows[q]: local rank q's
// buffers; rank ids rank0 + q.
cudaError_t run(int precision, const double* a, int n, int world, int rank0, int nlocal,
                void* const* ws, double* const* cos_rows, double* const* sin_rows,
                const Exchange& ex, bool force_gather, cudaStream_t st, Result* res,
                int64_t* launches, std::string* why) {
  const int M = n / world;
  std::vector<RankWs> R(nlocal);
  for (int q = 0; q < nlocal; ++q) R[q] = carve_rank(ws[q], n, world);
  Staged* d_st = reinterpret_cast<Staged*>(R[0].stage);
  tk::Op* d_ops = reinterpret_cast<tk::Op*>(R[0].stage + kOpsOffset);
  // selection on the replicated input (bit-exact norm, driver.py:64-88)
  cudaError_t e = cudaMemsetAsync(d_st, 0, sizeof(Staged), st);
  if (e == cudaSuccess)
    e = launch_norm1(0, a, 1, n, &d_st->normbits, &d_st->status, st);
  if (e == cudaSuccess)
    e = launch_select(&d_st->normbits, nullptr, 1, 0, precision, &d_st->k, &d_st->s,
                      &d_st->status, nullptr, st);
  *launches += 2;
  Staged h{};
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d_st, sizeof(Staged), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return e;
  res->k = h.k;
  res->s = h.s;
  res->status = h.status;
  if (h.status != 0) return cudaSuccess;  // the caller reports the status
  Schedule S = schedule(h.k, h.s);
  if (kOpsOffset + S.ops.size() * sizeof(tk::Op) > kStageBytes) {
    *why = "op table exceeds the staging area";
    return cudaErrorInvalidValue;
  }
  h.idx = 0;
  h.tp = 1.0;
  std::vector<char> blob(kOpsOffset + S.ops.size() * sizeof(tk::Op));
  std::memcpy(blob.data(), &h, sizeof(Staged));
  std::memcpy(blob.data() + kOpsOffset, S.ops.data(), S.ops.size() * sizeof(tk::Op));
  e = cudaMemcpyAsync(d_st, blob.data(), blob.size(), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // blob lives on this frame
  if (e == cudaSuccess) e = tk::ensure_smem_attr();
  if (e != cudaSuccess) return e;

  const bool gathers = world > 1 || force_gather;
  cudaStream_t cs = nullptr;
  std::vector<cudaEvent_t> events;
  auto new_event = [&](cudaEvent_t* ev) {
    cudaError_t r = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    if (r == cudaSuccess) events.push_back(*ev);
    return r;
  };
  if (gathers) e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  const int G = max_live_gathers();
  std::map<int, int> cache;           // slot -> pool buffer
  std::vector<bool> busy(G, false);
  const size_t nn = static_cast<size_t>(n) * n, Mn = static_cast<size_t>(M) * n;
  for (const Action& act : S.acts) {
    if (e != cudaSuccess) break;
    const int r = act.rhs;
    auto each = [&](auto&& fn) {
      for (int q = 0; q < nlocal && e == cudaSuccess; ++q) e = fn(q, (rank0 + q) * M);
    };
    auto prod = [&](int q, int row0, const double* rhs, int ksplit) {
      if (q == 0 && ksplit != 1) res->products += act.nops;  // per rank
      return launch(d_ops, d_st, act.op, act.nops, R[q].slab, M, n, row0, a + row0 * size_t(n),
                    rhs, ksplit, R[q].part, act.dbl_step, cos_rows[q], sin_rows[q], st,
                    launches);
    };
    if (r == 0) {  // the replicated input
      each([&](int q, int row0) { return prod(q, row0, a, 0); });
    } else if (!gathers) {  // W = 1: the slab is the whole matrix
      each([&](int q, int row0) { return prod(q, row0, R[q].slab + r * Mn, 0); });
    } else if (cache.count(r)) {
      const int g = cache[r];
      each([&](int q, int row0) { return prod(q, row0, R[q].pool + g * nn, 0); });
    } else {
      int g = 0;
      while (g < G && busy[g]) ++g;
      if (g == G) {
        *why = "gather pool exhausted";
        e = cudaErrorInvalidValue;
        break;
      }
      busy[g] = true;
      cache[r] = g;
      cudaEvent_t ready, done;
      if ((e = new_event(&ready)) != cudaSuccess || (e = new_event(&done)) != cudaSuccess) break;
      if ((e = cudaEventRecord(ready, st)) != cudaSuccess) break;
      if ((e = cudaStreamWaitEvent(cs, ready, 0)) != cudaSuccess) break;
      if (ex.comm) {
        const int rc = nccl().all_gather(R[0].slab + r * Mn, R[0].pool + g * nn, Mn,
                                         kNcclFloat64, ex.comm, cs);
        if (rc != 0) {
          *why = std::string("ncclAllGather: ") +
                 (nccl().error_string ? nccl().error_string(rc) : std::to_string(rc));
          e = cudaErrorUnknown;
          break;
        }
      } else {
        for (int q = 0; q < nlocal && e == cudaSuccess; ++q)
          for (int p = 0; p < world && e == cudaSuccess; ++p)
            e = cudaMemcpyAsync(R[q].pool + g * nn + p * Mn, R[p].slab + r * Mn, Mn * 8,
                                cudaMemcpyDeviceToDevice, cs);
      }
      if (e == cudaSuccess) e = cudaEventRecord(done, cs);
      ++res->gathers;
      if (world > 1) {  // own rows first, while the gather is in flight
        each([&](int q, int row0) { return prod(q, row0, nullptr, 1); });
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, done, 0);
        each([&](int q, int row0) { return prod(q, row0, R[q].pool + g * nn, 2); });
      } else {
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, done, 0);
        each([&](int q, int row0) { return prod(q, row0, R[q].pool + g * nn, 0); });
      }
    }
    for (int w : act.writes) {
      auto it = cache.find(w);
      if (it != cache.end()) {
        busy[it->second] = false;
        cache.erase(it);
      }
    }
  }
  for (cudaEvent_t ev : events) cudaEventDestroy(ev);
  if (cs) cudaStreamDestroy(cs);
  return e;
}

}  // namespace dc

}  // namespace csm
