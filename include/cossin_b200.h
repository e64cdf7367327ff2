/*
 * cossin_b200.h -- C-ABI of the B200-native cos/sin hot path.
 *
 * Drop-in boundary for the reference package `cossinm`
 * (/root/reference/pkg/src/cossinm).  The reference has no native layer:
 * its entry points are Python functions, and every product funnels into
 * numpy `@` (matcore.py:90-97).  Each function below replaces one of those
 * entry points (file:line cited per function) for a whole BATCH of
 * matrices in one call; the Python package paper_2010_00465_b200 binds
 * them with ctypes and keeps the reference's names and signatures.
 *
 * Conventions
 *   - All matrix pointers are DEVICE pointers to row-major (C-order),
 *     contiguous [batch][n][n] arrays of the given dtype.
 *   - k / s / status are DEVICE int32 arrays of length batch (outputs).
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Every call
 *     is stream-ordered and reentrant; the only globals are immutable
 *     constant tables.  One workspace per concurrent stream.
 *   - Return value: CSM_SUCCESS or a negative CSM_ERR_* code; the message
 *     of the last failure on the calling thread is csm_last_error().
 *   - Per-matrix status (mirrors the reference's exceptions):
 *       CSM_OK                0
 *       CSM_NONFINITE_INPUT   1  MatrixInputError  (driver.py:101-105)
 *       CSM_NONFINITE_NORM    2  ValueError        (driver.py:77-78)
 *       CSM_SELECT_OVERFLOW   3  OverflowError     (math.ceil(inf), driver.py:67)
 *       CSM_SINGULAR          4  SingularMatrixError (Pade only, matcore.py:141-147)
 *     Matrices with a nonzero status are skipped; their outputs are NaN.
 */
#ifndef COSSIN_B200_H
#define COSSIN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* matrix dtype: input/output element types (compute is always float64) */
enum { CSM_F64 = 0, CSM_F32 = 1, CSM_F32_IN_F64_OUT = 2 };
enum { CSM_PREC_DOUBLE = 0, CSM_PREC_SINGLE = 1 };    /* theta table       */
enum { CSM_FAMILY_TAYLOR = 0, CSM_FAMILY_WAVE = 1,    /* scheme family     */
       CSM_FAMILY_PADE = 2 };                          /* theta_tables.py:108-119 */

enum {
  CSM_OK = 0,
  CSM_NONFINITE_INPUT = 1,
  CSM_NONFINITE_NORM = 2,
  CSM_SELECT_OVERFLOW = 3,
  CSM_SINGULAR = 4         /* Pade denominator singular (matcore.py:141-147) */
};

enum {
  CSM_SUCCESS = 0,
  CSM_ERR_ARG = -1,        /* bad argument (shape, dtype, k, null ptr) */
  CSM_ERR_CUDA = -2,       /* a CUDA runtime call failed               */
  CSM_ERR_WORKSPACE = -3,  /* workspace too small                      */
  CSM_ERR_NO_DEVICE = -4   /* no usable sm_100 device                  */
};

/* Library version string and last error message (thread-local). */
const char* csm_version(void);
const char* csm_last_error(void);

/* Bytes of device workspace csm_cos_sin / csm_wave / the *_core calls need
 * for `batch` matrices of order n (independent of precision). */
size_t csm_workspace_size(int dtype, int64_t batch, int n);

/* ---- K0: norm + selection ------------------------------------------------
 * csm_norm1: norms[b] = max_j sum_i |a_bij|, each column summed
 * sequentially in row order in the input dtype, exactly as numpy's
 * np.abs(a).sum(axis=0).max() (matcore.py:100-104).  status[b] is set to
 * CSM_NONFINITE_INPUT for a non-finite entry (driver.py:101-105), else 0.
 * norms: device double[batch]. */
int csm_norm1(int dtype, const void* a, int64_t batch, int n, double* norms,
              int32_t* status, void* stream);

/* Selection of (k, s) from norms with a built-in theta table
 * (select_scheme, driver.py:64-88; tables theta_tables.py:79-144).
 * Host twin: all pointers are HOST pointers.  Returns per-norm status
 * (0, CSM_NONFINITE_NORM, CSM_SELECT_OVERFLOW). */
int csm_select_host(const double* norms, int64_t count, int family,
                    int precision, int32_t* k, int32_t* s, int32_t* status);

/* Device twin: norms, k, s, status are DEVICE pointers. */
int csm_select_device(const double* norms, int64_t count, int family,
                      int precision, int32_t* k, int32_t* s, int32_t* status,
                      void* stream);

/* Host selection over an arbitrary caller-supplied table (the reference's
 * select_scheme(norm, table) with a user-built ThetaTable, driver.py:70-88):
 * entries in table order, theta_eff[i] = min(theta_cos, theta_sin), cost =
 * cost_num[i] / cost_den[i] (the Fraction ThetaEntry.cost).  Writes the
 * chosen entry INDEX and s.  Host pointers. */
int csm_select_table(const double* norms, int64_t count,
                     const double* theta_eff, const int64_t* cost_num,
                     const int64_t* cost_den, int n_entries,
                     int32_t* entry_index, int32_t* s, int32_t* status);

/* ---- Full pipelines ------------------------------------------------------
 * csm_cos_sin: for every matrix b: validate, norm, select (k, s) with the
 * Taylor table of `precision`, scale by 2^-s, run the k-product factored
 * chain, double s times; cos_out[b] = cos(a_b), sin_out[b] = sin(a_b).
 * Replaces cos_sin(a, precision) (driver.py:108-123) for a batch.
 * dtype CSM_F32 reads/writes float32, CSM_F32_IN_F64_OUT reads float32 and
 * writes float64; both compute in float64 and take the 1-norm in float32
 * like numpy does for a float32 array. */
int csm_cos_sin(int dtype, int precision, const void* a, void* cos_out,
                void* sin_out, int64_t batch, int n, int32_t* k, int32_t* s,
                int32_t* status, void* workspace, size_t ws_bytes,
                void* stream);

/* csm_wave: c_out[b] = c(t_b^2 A_b), s_out[b] = s(t_b, A_b), with selection
 * on (t_b*t_b)*norm1(A_b) and the wave table, the chain at t_b/2^s and s
 * doubling steps.  Replaces wave_cos_sin(a, t, precision)
 * (driver.py:126-146).  t: DEVICE double[batch]. */
int csm_wave(int dtype, int precision, const void* a, const double* t,
             void* c_out, void* s_out, int64_t batch, int n, int32_t* k,
             int32_t* s, int32_t* status, void* workspace, size_t ws_bytes,
             void* stream);

/* ---- Fixed-scheme cores (no selection, no doubling) ----------------------
 * csm_taylor_core: taylor_cos_sin(a, SchemeId(COS_SIN_TAYLOR, k), ledger)
 * (schemes.py:376-395), k in {3,4,6,7}, for every matrix of the batch.
 * csm_wave_core: wave_kernels(a, t, SchemeId(WAVE_KERNEL, k), ledger)
 * (schemes.py:411-430), k in {3,4,5}; t: DEVICE double[batch].
 * status: DEVICE int32[batch] (non-finite input is NOT checked here, as in
 * the reference, whose scheme layer never validates finiteness). */
int csm_taylor_core(int dtype, int k, const void* a, void* cos_out,
                    void* sin_out, int64_t batch, int n, int32_t* status,
                    void* workspace, size_t ws_bytes, void* stream);
int csm_wave_core(int dtype, int k, const void* a, const double* t,
                  void* c_out, void* s_out, int64_t batch, int n,
                  int32_t* status, void* workspace, size_t ws_bytes,
                  void* stream);

/* Standalone sines (off the cos/sin pair path; schemes.py:398-408 and
 * :433-443): csm_taylor_sin9 = taylor_sin9(a) (degree-9 sine, exact-sine
 * degree-4 core; the reference's ledger charges 5 products),
 * csm_wave_sin34 = wave_sin34(a, t) (order-3 wave sine, 2 products).  No
 * scaling, no selection.  Workspace: csm_sine_workspace_size(). */
size_t csm_sine_workspace_size(int dtype, int64_t batch, int n);
int csm_taylor_sin9(int dtype, const void* a, void* sin_out, int64_t batch, int n,
                    int32_t* status, void* workspace, size_t ws_bytes, void* stream);
int csm_wave_sin34(int dtype, const void* a, const double* t, void* s_out,
                   int64_t batch, int n, int32_t* status, void* workspace,
                   size_t ws_bytes, void* stream);

/* Double-double reference values (verify.py:480-521 reference_cos_sin):
 * scale to ||A||_1 <= 2^-20, degree-12 Taylor pair and s doublings, every
 * product the k-ordered compensated _dd_matmul (verify.py:449-459).  Each
 * element follows the reference's exact operation sequence, so the float64
 * outputs (hi + lo) are bit-identical to the reference's.  float64 input
 * only.  s_host / status_host are HOST arrays of `batch` entries (status
 * CSM_SELECT_OVERFLOW where norm / 2^-20 overflows, the reference's
 * OverflowError); the call synchronises `stream` (s is chosen on the host,
 * as the reference does).  csm_dd_matmul is the bare product (xl / yl may
 * be NULL for a zero low part); csm_ddref_series_consts writes the 28
 * _dd_const splits of 1/(2i)! and 1/(2i+1)! (cos hi[7], cos lo[7],
 * sin hi[7], sin lo[7]; verify.py:405-412, :462-464). */
size_t csm_ddref_workspace_size(int64_t batch, int n);
int csm_ddref_cos_sin(const double* a, double* cos_out, double* sin_out,
                      int64_t batch, int n, int32_t* s_host,
                      int32_t* status_host, void* workspace, size_t ws_bytes,
                      void* stream);
int csm_dd_matmul(const double* xh, const double* xl, const double* yh,
                  const double* yl, double* oh, double* ol, int64_t batch,
                  int n, void* stream);
int csm_ddref_series_consts(double* out28);

/* Pythagorean residual of computed pairs: out[b] = ||C_b C_b + S_b S_b -
 * I||_1 (max column sum), the reference's accuracy witness (pkg/README.md:
 * 172-176, tests/test_driver.py:149-157).  A diagnostic beside the path:
 * both products on DMMA, deterministic reduction.  dtype CSM_F64 or CSM_F32
 * (the inputs' type); out: DEVICE double[batch]. */
size_t csm_residual_workspace_size(int64_t batch, int n);
int csm_pythagorean_residual(int dtype, const void* cos_in, const void* sin_in,
                             int64_t batch, int n, double* out, void* workspace,
                             size_t ws_bytes, void* stream);

/* Order-8 Pade baseline (driver.py:149-164, schemes.py:446-464): selection
 * over PADE_TABLE, a * 2^-s, five products (A^2, A^4, A^6, A^8 and A times
 * the odd numerator) with the three polynomials fused into their epilogues,
 * ONE batched LU with partial pivoting of the shared denominator and two
 * solves (matcore.py:124-151, singularity test 1e3 eps ||den||_1), then s
 * doublings.  k[] reports 5 (the PADE8 scheme id); the ledger cost is
 * 22/3 + 2 s.  Every n runs the tiled chain; workspace:
 * csm_pade_workspace_size(). */
size_t csm_pade_workspace_size(int dtype, int64_t batch, int n);
int csm_pade_cos_sin(int dtype, int precision, const void* a, void* cos_out,
                     void* sin_out, int64_t batch, int n, int32_t* k, int32_t* s,
                     int32_t* status, void* workspace, size_t ws_bytes,
                     void* stream);

/* The Pade base pair alone (schemes.py:446-464 pade8_cos_sin): no
 * selection and no scaling (k = 5, s = 0 for every matrix), the same five
 * products, LU and two solves as csm_pade_cos_sin.  status[] reports
 * CSM_SINGULAR per matrix; workspace: csm_pade_workspace_size(). */
int csm_pade_core(int dtype, const void* a, void* cos_out, void* sin_out, int64_t batch, int n,
                  int32_t* status, void* workspace, size_t ws_bytes, void* stream);

/* Copy the built-in theta table of (family, precision) -- the reference's
 * TAYLOR_TABLE / WAVE_TABLE (theta_tables.py:79-144) -- into host arrays of
 * `capacity` entries; returns the entry count (or a negative error). */
int csm_theta_table(int family, int precision, double* theta_cos,
                    double* theta_sin, int32_t* k, int capacity);

/* ---- Block-row (slab) primitives of the distributed chain ----------------
 * One very large matrix (configs[4], 8192^2) is split by rows over the
 * ranks; every product is  out_rows = L_rows * R_full  with R_full the
 * all-gathered right operand (the gather is the caller's: NCCL through
 * torch.distributed in paper_2010_00465_b200/distchain.py).  The chain
 * programs are exported as opaque op descriptors (csm_op_bytes() each) so
 * the driver can interleave gathers and products step by step.
 *   csm_chain_program: ops of scheme (family, k) in step order (fold = 1:
 *     slot 0 is the raw input and 2^-s is folded into the products); returns
 *     the step count, step_nops[i] = ops in step i, and the slots that hold
 *     cos / sin after the chain (schemes.py:264-430).
 *   csm_doubling_program: the two ops of one doubling step from (c0, s0)
 *     into (c1, s1) (driver.py:91-98).
 *   csm_slab_op: run one op on a slab of CSM_SLAB_SLOTS x M x NP float64
 *     (M rows from global row row0, M and NP multiples of 64).  in0 = the
 *     input rows (slot 0 alias), s / tp = the matrix's s and t', dbl_step =
 *     -1 for chain ops or the doubling index; outputs that are final are
 *     also written to cos_out / sin_out (the caller's M x NP rows).
 *     scratch: device buffer of scratch_bytes >= csm_slab_scratch_bytes()
 *     + csm_slab_engine_bytes(M, NP) (the latter is the Ozaki engine's
 *     scratch for the calling thread's engine, 0 under the DMMA engine;
 *     csm_slab_op_peer always runs DMMA and needs only the former).  A
 *     smaller scratch_bytes returns CSM_ERR_WORKSPACE, never overflows. */
#define CSM_SLAB_SLOTS 9
size_t csm_op_bytes(void);
size_t csm_slab_scratch_bytes(void);
size_t csm_slab_engine_bytes(int M, int NP);
int csm_chain_program(int family, int k, int fold, void* ops_out, int max_ops,
                      int32_t* step_nops, int max_steps, int32_t* cos_slot,
                      int32_t* sin_slot);
int csm_doubling_program(int c0, int s0, int c1, int s1, void* ops_out);
int csm_slab_op(const void* op, double* slab, int M, int NP, int row0,
                const double* rhs_full, const double* in0, int s, double tp,
                int dbl_step, void* cos_out, void* sin_out, int out_f32,
                void* scratch, size_t scratch_bytes, void* stream);
/* csm_slab_op_pair: the doubling step's two ops (csm_doubling_program: S C
 * and C C, both with right operand C = rhs_full) in one launch; on the
 * Ozaki engine C is converted once for both (dbl_step >= 0 required). */
int csm_slab_op_pair(const void* op_a, const void* op_b, double* slab, int M, int NP,
                     int row0, const double* rhs_full, const double* in0, int s,
                     double tp, int dbl_step, void* cos_out, void* sin_out,
                     int out_f32, void* scratch, size_t scratch_bytes, void* stream);
/* Fused all-gather + product: like csm_slab_op, but the right operand is
 * NOT gathered -- rhs_slabs (HOST array of nparts pointers) holds each
 * rank's slab base, peer pointers over NVLink (e.g. from torch symmetric
 * memory), row block j of slot op.rhs living in rhs_slabs[j].  The GEMM's
 * cp.async stages stream those rows straight from the owning GPU, so the
 * transfer overlaps the math tile by tile.  Requires nparts * M == NP.
 * The caller orders steps with a cross-rank barrier (all writers of the
 * operand done before any reader starts). */
int csm_slab_op_peer(const void* op, double* slab, int M, int NP, int row0,
                     const double* const* rhs_slabs, int nparts,
                     const double* in0, int s, double tp, int dbl_step,
                     void* cos_out, void* sin_out, int out_f32, void* scratch,
                     size_t scratch_bytes, void* stream);

/* ---- The distributed chain driven from C (cfg5 across GPUs) -------------
 * csm_dist_cos_sin: cos / sin of ONE n x n float64 matrix `a` (device,
 * replicated on every rank) over the ranks of an NCCL communicator, block
 * row: rank r computes rows [r M, r M + M), M = n / W, into cos_rows /
 * sin_rows (device, M x n).  Selection, the Taylor chain and the doubling
 * steps run as in csm_cos_sin (driver.py:108-123); every product is
 * out_rows = L_rows R_full on the FP64 DMMA tiled kernel, with R_full
 * all-gathered by ncclAllGather on a side stream while the rank contracts
 * its own rows of R (K-split), and a gathered operand is reused until its
 * slot is rewritten (distchain.py's schedule).  comm = NULL runs W = 1.
 * n must be a multiple of 64 W.  k / s / status: host outputs (status as
 * in csm_cos_sin; on a non-zero status nothing is computed).  Stream
 * ordered; the call synchronises `stream` twice (selection read-back and
 * op-table staging).  NCCL is resolved at run time from the process (or
 * libnccl.so.2); it is not a link dependency.  All ranks must call with
 * the same a, n and precision.  workspace: csm_dist_workspace_size(n, W,
 * flags) bytes per rank.
 *   flags: CSM_DIST_FORCE_GATHER gathers every non-A right operand even at
 *   W = 1 (exercises the NCCL path on one GPU).
 * csm_dist_cos_sin_virtual: the same schedule for W virtual ranks in this
 * process (every slab on the current device, the all-gather as device
 * copies) -- the K-split products and the gather cache on one GPU.
 * cos / sin: full n x n outputs; workspace: W x csm_dist_workspace_size(n,
 * W, CSM_DIST_FORCE_GATHER).
 * csm_dist_last_stats: gathers and products of the calling thread's last
 * distributed call. */
#if !defined(NCCL_H_)
typedef struct ncclComm* ncclComm_t;
#endif
#define CSM_DIST_FORCE_GATHER 1
size_t csm_dist_workspace_size(int n, int world, int flags);
int csm_dist_cos_sin(int precision, const double* a, double* cos_rows, double* sin_rows, int n,
                     ncclComm_t comm, int flags, int32_t* k, int32_t* s, int32_t* status,
                     void* workspace, size_t ws_bytes, void* stream);
int csm_dist_cos_sin_virtual(int precision, const double* a, double* cos_out, double* sin_out,
                             int n, int world, int32_t* k, int32_t* s, int32_t* status,
                             void* workspace, size_t ws_bytes, void* stream);
int csm_dist_last_stats(int32_t* gathers, int32_t* products);
/* NCCL communicator helpers for callers without their own NCCL setup
 * (id: 128 bytes, made on one rank and shared out of band). */
int csm_nccl_get_unique_id(void* id);
int csm_nccl_comm_init_rank(ncclComm_t* comm, int nranks, const void* id, int rank);
int csm_nccl_comm_destroy(ncclComm_t comm);

/* 1 when csm_cos_sin / csm_wave for (dtype, batch, n) never synchronises
 * the host (K1, or K1c without the side chain), so the call can be
 * captured in a CUDA graph; 0 for the tiled chain (it reads (k, s) back to
 * plan its launches). */
int csm_graph_safe(int dtype, int64_t batch, int n);

/* Product engine of the tiled chain (n > 128; also the Pade and standalone
 * sine calls) and of csm_slab_op.  CSM_ENGINE_DMMA: FP64 DMMA (mma.sync
 * m8n8k4).  CSM_ENGINE_OZAKI: each product exactly on integers by the
 * Ozaki-II scheme -- rows / columns scaled to P-bit integers, one tcgen05
 * int8 GEMM per modulus (16 moduli for float64 results, 9 for float32),
 * Chinese-remainder reconstruction fused with the op's epilogue -- whenever
 * the padded order is a multiple of 256 (DMMA otherwise).  Every Ozaki
 * product is checked by an a-priori error bound: when the rounding of the
 * operands to P bits relative to their row / column maxima could exceed
 * n u ||C||_1 (the fp64 GEMM's norm-wise bound), that product is recomputed
 * on DMMA.  The guarantee is norm-wise per product: on graded operands a
 * long doubling recursion can amplify the Ozaki rounding of small entries
 * beyond the reference's accuracy, which an fp64 GEMM (componentwise
 * error, matcore.py:97) does not do -- hence DMMA is the DEFAULT engine.
 * CSM_ENGINE_AUTO: Ozaki for padded orders >= 768 that are multiples of
 * 256, where it is faster; DMMA below.  The chain, (k, s) and the
 * reference interface are unchanged.
 *   csm_set_engine: the process default (atomic; CSM_ENGINE_DMMA at load).
 *   csm_set_thread_engine: an override for the calling thread (-1 clears).
 * Each call reads the engine once; workspace sizes (csm_workspace_size,
 * csm_slab_engine_bytes, ...) depend on it, and a call whose workspace is
 * too small for its engine returns CSM_ERR_WORKSPACE.  Returns CSM_ERR_ARG
 * for an unknown engine. */
#define CSM_ENGINE_DMMA 0
#define CSM_ENGINE_OZAKI 1
#define CSM_ENGINE_AUTO 2
/* Experiments and tests only: the Ozaki engine WITHOUT the accuracy guard
 * (shows what the guard prevents on badly scaled operands). */
#define CSM_ENGINE_OZAKI_UNGUARDED 3
int csm_set_engine(int engine);
int csm_get_engine(void);
int csm_set_thread_engine(int engine);

/* ---- Measurement helpers (not part of the reference surface) ------------
 * csm_fp64_peak: time a DMMA (mma.sync m8n8k4 f64) throughput loop on the
 * current device for ~`iters` iterations; returns TFLOP/s in *tflops.
 * csm_last_launch_count: number of kernels the last pipeline call on this
 * thread launched. */
int csm_fp64_peak(int iters, double* tflops, void* stream);
int64_t csm_last_launch_count(void);

/* Live timing of the dominant kernel: while enabled, every pipeline call on
 * this thread records a CUDA event pair on its stream around the dominant
 * kernel (the fused n <= 64 kernel, or the tiled GEMM launches).
 * csm_profile_collect synchronises those events, returns the summed
 * milliseconds and the number of intervals, and clears them.
 * csm_profile_enable(0/1) also clears; mode 2 records the Ozaki engine's
 * int8 GEMM launches (one interval per launch) instead, mode 3 the fused
 * K0 launch (norm1 + finiteness + selection, n <= 128) of each call. */
int csm_profile_enable(int on);
int csm_profile_collect(double* total_ms, int64_t* intervals);

#ifdef __cplusplus
}
#endif

#endif /* COSSIN_B200_H */
