/*
 * turbo_ns.h -- C ABI of libturbons.so: AOL-preconditioned Newton-Schulz
 * orthogonalisation ("Turbo-Muon", arxiv 2512.04632) on NVIDIA B200 (sm_100a).
 *
 * What is computed (PAPER.md line numbers, "P:Lnnn"):
 *   Let X be m x n and Xh its short-side orientation (Xh = X if m >= n, else X^T;
 *   reading R2), N = min(m,n), M = max(m,n).  With coefficients
 *   (a_k, b_k, c_k), k = 1..T:
 *     precond = AOL        : A0 = Xh^T Xh (Eq. 7); s_i = (sum_j |A0_ij|)^(-1/2)
 *                            (Eq. 8); X1 = Xh diag(s) (Eq. 9); A1 = diag(s) A0
 *                            diag(s) (Alg. 2 l.4) -- the Gram is reused.
 *     precond = FROBENIUS  : s = 1/||Xh||_F (Eqs. 10-11; Alg. 1).
 *     precond = NONE       : X1 = Xh (caller guarantees ||X||_2 <= 1).
 *     for k = 1..T:  A_k = X_k^T X_k   (Eq. 3; k = 1 reuses A1)
 *                    B_k = b_k A_k + c_k A_k A_k          (Eq. 4)
 *                    X_{k+1} = a_k X_k + X_k B_k          (Eq. 5)
 *   The result X_{T+1} (transposed back for m < n) is written in the caller's layout.
 *
 * Conventions for every entry point:
 *   - Matrices are dense row-major, leading dimension = number of columns, in DEVICE
 *     memory of the current CUDA device, 16-byte aligned.  Element type = `dtype`
 *     (NS_BF16: bfloat16 storage, fp32 accumulation; NS_FP32: fp32 throughout).
 *   - `coeffs` is a HOST array of 3*iters floats (a_1,b_1,c_1,a_2,...); it is read
 *     before the call returns (the caller may free it afterwards).
 *   - Calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy default
 *     stream) and never block the host on the device -- including the first call for
 *     a problem list, whose plan build allocates (cudaMallocAsync), zeroes
 *     (cudaMemsetAsync) and uploads its tables (cudaMemcpyAsync) stream-ordered on
 *     `stream`.  Exceptions, each documented at its entry point: ns_read_flags,
 *     ns_profile_read, nsx_epilogue_counters, ns_shutdown, the nsx_* single-step test
 *     entry points, and the first call of the process on a device (context set-up).
 *     The plan-building call cannot itself be stream-captured (NS_ERR_NOT_SUPPORTED);
 *     later calls can.
 *   - Caller-owned memory is never freed by the library.  Workspace (a ping-pong
 *     buffer of the matrix size plus two N x N buffers and small tables per matrix)
 *     is owned by the library, cached per problem list (keyed by device pointers and
 *     shapes), and released stream-ordered (cudaFreeAsync after an event recorded at
 *     the plan's last launch) when the cache evicts it, or by ns_shutdown.
 *   - All argument checks happen on the host before anything is enqueued; on any
 *     error nothing is enqueued and no memory is touched.  Numerical conditions
 *     (zero row-sum, zero matrix, non-finite values) do NOT fail a call: they set
 *     device flags readable with ns_read_flags (reading R4).
 *   - From the second call with the same problem list on, the call's launches are
 *     replayed as one CUDA graph captured by the library (same kernels, same results;
 *     not while `stream` is itself being captured; TNS_NOGRAPH=1 disables it).
 *   - Thread-safety: calls are serialised by an internal mutex; distinct streams are
 *     fine for distinct problem lists.  Calls with the SAME problem list share its cached
 *     workspace: a call on another stream than the previous call with that list waits
 *     (cudaStreamWaitEvent) for the previous call's last launch; only while `stream` is
 *     being captured must the caller order such calls itself.
 *   - Determinism: results are bitwise reproducible for identical inputs, and
 *     independent of how matrices are grouped into calls: every routing and tiling
 *     decision that changes the arithmetic (cluster kernel vs step engine, split-K Gram
 *     of N <= 256 matrices) depends on the matrix shape alone.
 */
#ifndef TURBO_NS_H_
#define TURBO_NS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NS_ABI_VERSION 2

typedef enum {
  NS_OK = 0,
  NS_ERR_INVALID_VALUE = 1, /* bad shape / iters / coeffs / enum / NULL pointer      */
  NS_ERR_NOT_SUPPORTED = 2, /* e.g. misaligned pointer                               */
  NS_ERR_WORKSPACE = 3,     /* device allocation failed                              */
  NS_ERR_CUDA = 4           /* a CUDA runtime/driver call or launch failed           */
} ns_status;

typedef enum {
  NS_PRECOND_NONE = 0,      /* no scaling; caller guarantees ||X||_2 <= 1             */
  NS_PRECOND_FROBENIUS = 1, /* Alg. 1: X / ||X||_F   (Muon, Muon+)                   */
  NS_PRECOND_AOL = 2        /* Alg. 2: AOL column scaling with Gram reuse (Turbo-Muon) */
} ns_precond;

typedef enum {
  NS_BF16 = 0, /* bf16 storage of X, A, B; fp32 accumulation (tcgen05 tensor cores) */
  NS_FP32 = 1  /* fp32 storage and fp32 FFMA arithmetic ("exact" mode)              */
} ns_dtype;

/* Flag bits reported by ns_read_flags. */
#define NS_FLAG_ZERO_SCALE 0x1u /* a zero AOL row-sum (zero column) or zero matrix (Frobenius) */
#define NS_FLAG_NONFINITE 0x2u  /* a non-finite value was produced                        */

/* The north-star call (Alg. 2 P:L163-176 for AOL, Alg. 1
 * for FROBENIUS / NONE, Eqs. 3-5 P:L116-118 per iteration).  In place: `batch` matrices of
 * m x n at X, X + m*n, ... (contiguous, device) are each overwritten with
 * NS_T(precond(X_i)), T = iters (1..64), coeffs = T triples (host).  Errors:
 * NS_ERR_INVALID_VALUE (m, n, batch < 1; iters outside 1..64; NULL or non-finite coeffs;
 * bad enum), NS_ERR_NOT_SUPPORTED (X not aligned to its element size; stream-captured
 * plan build), NS_ERR_WORKSPACE (allocation), NS_ERR_CUDA; nothing enqueued on error. */
ns_status ns_orthogonalize(void* X, int64_t m, int64_t n, int64_t batch, int iters,
                           const float* coeffs, ns_precond precond, ns_dtype dtype,
                           void* stream);

/* Mixed precision: as ns_orthogonalize_batched with dtype NS_BF16,
 * but X[i] / out[i] are fp32 device matrices (4-byte aligned; out = NULL or out[i] == X[i]
 * for in place).  Each X[i] is cast to bf16 (round to nearest even) into a workspace
 * staging copy in one grouped launch, the NS runs in bf16 on the copies exactly as for a
 * bf16 caller, and the bf16 results are widened into out[i] in one more launch -- so the
 * result is bitwise float(NS_bf16(bf16(X[i]))).  X[i] is read once and not modified unless
 * it is also the output.  The workspace holds 2*m*n bytes per matrix more than
 * ns_workspace_size(..., NS_BF16) reports. */
ns_status ns_orthogonalize_cast(const void* const* X, void* const* out, const int64_t* m,
                                const int64_t* n, int64_t count, int iters, const float* coeffs,
                                ns_precond precond, void* stream);

/* Grouped (the paper batches layer matrices, "batches of 32"):
 * the same computation as ns_orthogonalize for `count` matrices of arbitrary shapes
 * m[i] x n[i] (count < 2^20).  X is a HOST array of
 * device pointers (inputs); out is a HOST array of device pointers receiving the
 * results (out may be NULL, or out[i] == X[i], for in place; out[i] must not
 * otherwise overlap any X[j]).  Every NS step runs as ONE launch over all matrices
 * (3*iters + 1 launches in total), plus ONE cluster launch for all small matrices
 * (see ns_set_path); bf16 matrices whose row pitch TMA cannot address (not a multiple of
 * 16 bytes) run as a second group on the CUDA-core kernels.  Results are bitwise identical
 * to calling ns_orthogonalize on each matrix alone (split-K exception: see above). */
ns_status ns_orthogonalize_batched(void* const* X, void* const* out, const int64_t* m,
                                   const int64_t* n, int64_t count, int iters,
                                   const float* coeffs, ns_precond precond, ns_dtype dtype,
                                   void* stream);

/* Fused collective (the GEMM -> all-gather of the sharded path as ONE
 * kernel): as ns_orthogonalize_batched, and the LAST iteration's epilogue also stores every
 * output tile into npeer more destinations, peer_out[i * npeer + r] = matrix i's slot on
 * peer r (device addresses valid in this process, e.g. other GPUs' gather buffers mapped
 * over NVLink by symmetric memory), so the exchange overlaps the final GEMM tile by tile.
 * out[i] (or X[i]) receives the result as well.  bf16 tcgen05 path only (16-byte aligned
 * pointers, m and n multiples of 8), else NS_ERR_NOT_SUPPORTED; 0 <= npeer <= 64.  The
 * caller orders the peers (e.g. a symmetric-memory barrier before and after the call). */
ns_status ns_orthogonalize_peers(void* const* X, void* const* out, void* const* peer_out, int npeer,
                                 const int64_t* m, const int64_t* n, int64_t count, int iters,
                                 const float* coeffs, ns_precond precond, ns_dtype dtype, void* stream);

/* One Muon / Turbo-Muon optimizer step over `count` weight matrices (
 * PAPER.md P:L16/L97 "momentum -> orthogonalize -> update", reading R13 for the formulas of
 * the cited public Muon):
 *   G' = grad_scale G (e.g. 1/world: the data-parallel mean of summed gradients)
 *   M <- beta M + (1-beta) G' ;  U <- nesterov ? (1-beta) G' + beta M : M   (U rounded to bf16)
 *   U <- NS_iters(precond(U))  (as ns_orthogonalize_batched, in place on U)
 *   W <- W (1 - lr weight_decay) - lr * max(1, m/n)^(1/2) * U
 * W[i] (w_dtype), G[i] (g_dtype), M[i] (fp32, caller-initialised, e.g. zeros) and U[i]
 * (bf16 staging, contents overwritten) are m[i] x n[i] device matrices; 0 <= beta < 1.
 * 3*iters + 3 launches, asynchronous on `stream`. */
ns_status ns_muon_step(void* const* W, const void* const* G, float* const* M, void* const* U,
                       const int64_t* m, const int64_t* n, int64_t count, ns_dtype w_dtype, ns_dtype g_dtype,
                       float lr, float beta, float weight_decay, float grad_scale, int nesterov, int iters,
                       const float* coeffs, ns_precond precond, void* stream);

/* The update half of a Muon step on its own (the distributed optimizer applies updates
 * orthogonalised on other ranks; reading R13):  W <- W (1 - lr weight_decay) - lr *
 * max(1, m/n)^(1/2) * U for `count` matrices, W[i] (w_dtype) and U[i] (bf16, e.g. an
 * ns_orthogonalize result) m[i] x n[i] device matrices.  The same kernel ns_muon_step uses
 * (bitwise the same W).  One launch, asynchronous on `stream`. */
ns_status ns_muon_apply(void* const* W, const void* const* U, const int64_t* m, const int64_t* n,
                        int64_t count, ns_dtype w_dtype, float lr, float weight_decay, void* stream);

/* Workspace of the north-star signature: bytes of device workspace the
 * library holds for the problem list of `count` shapes m[i] x n[i], each repeated `batch`
 * times (ns_orthogonalize with `batch`, or a grouped list) -- per matrix W (m x n), A and B
 * (N x N), s and the AOL partials (Eq. 8 row sums), plus a 1 KiB header per plan
 * (a list mixing TMA-unaligned bf16 shapes runs as two plans).  An upper bound for any
 * device and path: a matrix served by the tcgen05 cluster kernel needs only its Gram-partial
 * scratch and A image (counted with the larger of the two footprints), the FFMA cluster
 * kernel none.  Host only
 * (no device call).  NS_ERR_INVALID_VALUE for NULL pointers, count/batch/m/n < 1, bad
 * dtype. */
ns_status ns_workspace_size(const int64_t* m, const int64_t* n, int64_t count, int64_t batch,
                            ns_dtype dtype, size_t* bytes);

/* Optional caller-owned workspace: `ptr` (device memory of the current
 * device, 256-byte aligned, `bytes` >= 256) from which every plan built afterwards carves
 * its workspace (bump allocation; a problem list needs at most ns_workspace_size bytes)
 * instead of allocating its own.  A call whose new plan does not fit fails with
 * NS_ERR_WORKSPACE and enqueues nothing.  Drops the cached plans that used the previous
 * caller buffer without synchronising: `stream` is made to wait (events) for their last
 * launches, so work enqueued on `stream` afterwards is ordered after them; the caller keeps
 * the previous buffer alive until that work has run, and `ptr` alive until the next
 * ns_set_workspace or ns_shutdown.  ptr = NULL returns to library-owned workspace. */
ns_status ns_set_workspace(void* ptr, size_t bytes, void* stream);

/* Numerical conditions of the path (reading R4: the paper's Eq. 8 has no epsilon, P:L206;
 * SPEC's zero-column / non-finite errors, become flags so that no call has
 * to synchronise).  SYNCHRONISES `stream`, returns the OR of NS_FLAG_* raised since the
 * last read on the current device, and clears them.  NS_ERR_INVALID_VALUE if flags is
 * NULL. */
ns_status ns_read_flags(void* stream, uint32_t* flags);

/* Number of kernels the library launched on this process since load (host counter). */
uint64_t ns_launch_count(void);

/* Execution-path override for testing.  0 = auto: bf16 matrices with short side N <= 128
 * that TMA can address and that fit 16 row slabs (M <= 4096) run the WHOLE NS in ONE launch of
 * a 4- to 16-CTA cluster on the tensor cores (cluster_tc_ns_kernel: X slabs and A / B'
 * resident in shared memory, lower-triangle Gram partials reduced through L2 in a fixed
 * order into an A image every CTA bulk-loads); other
 * matrices with N <= 128 whose fp32 copy
 * fits in shared memory (fp32 always, bf16 while M*N^2 <= 2.2e6) run the whole NS in one
 * launch of a 16- or 8-CTA FFMA cluster (cluster_ns_kernel; row a-10); all other matrices go
 * through the step engine (tcgen05, 256x256 tiles on CTA pairs, for aligned bf16, else SIMT;
 * one PDL-chained launch per step); when several kinds are present the cluster launches run
 * on internal side streams joined back by events; 1 = force the SIMT (CUDA-core) step
 * kernels, 2 = tcgen05 with single-CTA 128x256 tiles, 4 = per-step launches for every matrix
 * (no cluster kernels), 5 = as 0 but every matrix that fits the FFMA cluster kernel takes it,
 * 7 = as 0 but every bf16 matrix with N <= 256 that fits the tcgen05 cluster kernel (M <= 3072
 * for N > 128) takes it.  Results of a matrix never depend on the rest of the call.  Returns
 * the previous value; any other `path` returns -1 and changes nothing. */
int ns_set_path(int path);

/* Per-kernel event timing (measurement support for bench.py; off by default).
 * When enabled, every launch the library enqueues is bracketed by CUDA events recorded
 * on the SAME stream.  ns_profile_read SYNCHRONISES on the last event, writes for each
 * kind k (0 GRAM, 1 PRECOND, 2 POLY, 3 XB, 4 SIMT, 5 COPY, 6 CLUSTER_TC, 7 CLUSTER; nkinds <= 8) the summed
 * device milliseconds ms[k] and the launch count counts[k], then clears the records. */
void ns_profile_enable(int on);
ns_status ns_profile_read(double* ms, uint64_t* counts, int nkinds);
/* Measurement only: epilogue clock counters collected when the environment variable
 * TNS_DBG has bit 8 set (tiles, cycles waiting for the accumulator, TMEM load, aux wait,
 * math, staging wait, store issue, -).  SYNCHRONISES the device; reset != 0 zeroes them. */
ns_status nsx_epilogue_counters(uint64_t* out8, int reset);

const char* ns_status_string(ns_status s);
const char* ns_last_error(void); /* detail of the last non-OK status (thread-local) */
int ns_abi_version(void);
void ns_shutdown(void); /* synchronises the device, frees workspace and plan caches */

/* ---------------------------------------------------------------------------------
 * Single-step entry points (each is one step of the path; used by the step-level
 * parity tests).  X is m x n row-major; N = min(m,n); all outputs are dtype.
 * --------------------------------------------------------------------------------- */

/* A = Xh^T Xh (N x N, both triangles written)        -- Eq. 3 / Eq. 7.  part != NULL
 * (aligned bf16 only, else NS_ERR_NOT_SUPPORTED): also the AOL row-sum partials of |A|
 * that the iteration-1 Gram epilogue emits (Eq. 8), fp32[N * L] with
 * L = ceil(N/64) + ceil(N/32): part[i*L + c] = sum of |A_ij| over the 64 columns of
 * direct slot c, part[i*L + ceil(N/64) + r] = the same over the 32 rows of mirrored slot r
 * (only slots the lower-triangle tiling writes; zero the buffer first). */
ns_status nsx_gram(const void* X, int64_t m, int64_t n, void* A, float* part, ns_dtype dtype,
                   void* stream);

/* In place on A (N x N symmetric): s from A (AOL: Eq. 8; FROBENIUS: 1/sqrt(trace A) =
 * 1/||X||_F, Eq. 10), then A <- diag(s) A diag(s) (Alg. 2 l.4).  s: device fp32[N].
 * part != NULL (AOL, bf16): the row sums come from nsx_gram's partials instead of A --
 * the production branches (one lane per row while L <= 64, i.e. N <= 1344, else a warp
 * tree). */
ns_status nsx_precondition(void* A, int64_t N, ns_precond precond, const float* part, float* s,
                           ns_dtype dtype, void* stream);

/* B = (b A + c A A) diag(s)  (Eq. 4; s == NULL means s = 1). */
ns_status nsx_poly(const void* A, int64_t N, float b, float c, const float* s, void* B,
                   ns_dtype dtype, void* stream);

/* Out = a Xh diag(s) + Xh B^T in the caller's (m x n) layout, B as produced by
 * nsx_poly.  With B = B1 diag(s) this is a X1 + X1 B1 for X1 = Xh diag(s): Eq. 5 with
 * the AOL scaling of iteration 1 folded in (X1 is never materialised).  s == NULL
 * means s = 1 (then B is symmetric and B^T = B).  Out must not overlap X. */
ns_status nsx_update(const void* X, int64_t m, int64_t n, const void* B, float a,
                     const float* s, void* Out, ns_dtype dtype, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TURBO_NS_H_ */
