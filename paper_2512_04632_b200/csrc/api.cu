// C ABI of libturbons.so (include/turbo_ns.h): argument checking, planning (shape
// orientation, ping-pong buffers, workspace, TMA descriptors, grouped job tables) and
// stream-ordered enqueueing of the 3*T + 1 launches of one Newton-Schulz call.
//
// The step order follows PAPER.md Alg. 2 (L163-176) and Eqs. 3-5 (L116-118):
//   k = 1:   GRAM(X0) -> A0 ; PRECOND: s (Eq. 8 / Eq. 10), A1 = diag(s) A0 diag(s)
//            POLY: B1' = (b1 A1 + c1 A1^2) diag(s)
//            XB:   X2 = a1 X0 diag(s) + X0 B1'^T    (= a1 X1 + X1 B1, X1 never stored)
//   k >= 2:  GRAM(Xk) -> Ak ; POLY: Bk = bk Ak + ck Ak^2 ; XB: Xk+1 = ak Xk + Xk Bk
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/turbo_ns.h"
#include "jobs.h"
#include "kernels.h"

namespace tns {

// ---------------------------------------------------------------------------- globals
static std::mutex g_mu;
static uint64_t g_launches = 0;
static int g_path = 0;
static thread_local std::string g_err;

// ---- optional per-launch event timing (ns_profile_*)
struct ProfRec { int kind; cudaEvent_t a, b; };
static bool g_prof = false;
static std::vector<ProfRec> g_prof_recs;
static std::vector<cudaEvent_t> g_ev_pool;
static cudaEvent_t ev_get() {
  if (!g_ev_pool.empty()) { cudaEvent_t e = g_ev_pool.back(); g_ev_pool.pop_back(); return e; }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
struct ProfScope {
  bool on; int kind; cudaStream_t s; cudaEvent_t a = nullptr, b = nullptr;
  ProfScope(int k, cudaStream_t st) : on(g_prof), kind(k), s(st) {
    if (on) { a = ev_get(); cudaEventRecord(a, s); }
  }
  ~ProfScope() {
    if (on) { b = ev_get(); cudaEventRecord(b, s); g_prof_recs.push_back({kind, a, b}); }
  }
};

static ns_status fail(ns_status s, const std::string& msg) {
  g_err = msg;
  return s;
}
#define CU_TRY(expr)                                                                       \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      return fail(NS_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));        \
  } while (0)

struct DevCtx {
  bool init = false;
  int sms = 0;
  int cc_major = 0, cc_minor = 0;
  uint32_t* flags = nullptr;  // device word
  // side stream for the cluster-resident small-matrix launch, joined back by events
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // side streams of the tcgen05 cluster kernel's launches (one per cluster size 2, 4, 8, 16),
  // so they run beside each other and beside the step engine
  cudaStream_t tside[4] = {};
  cudaEvent_t tfork[4] = {}, tjoin[4] = {};
  cudaStream_t cap = nullptr;  // private stream on which plans are captured into CUDA graphs
  // private stream on which evicted plans' device memory is released (cudaFreeAsync), ordered
  // after the plan's last use by an event -- eviction never synchronises the host
  cudaStream_t freer = nullptr;
};
static DevCtx g_dev[64];
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static ns_status dev_ctx(DevCtx** out) {
  int dev = 0;
  CU_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail(NS_ERR_NOT_SUPPORTED, "device index >= 64");
  DevCtx& d = g_dev[dev];
  if (!d.init) {
    CU_TRY(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev));
    CU_TRY(cudaDeviceGetAttribute(&d.cc_major, cudaDevAttrComputeCapabilityMajor, dev));
    CU_TRY(cudaDeviceGetAttribute(&d.cc_minor, cudaDevAttrComputeCapabilityMinor, dev));
    CU_TRY(cudaMalloc(&d.flags, sizeof(uint32_t)));
    CU_TRY(cudaMemset(d.flags, 0, sizeof(uint32_t)));
    CU_TRY(cudaStreamCreateWithFlags(&d.side, cudaStreamNonBlocking));
    CU_TRY(cudaEventCreateWithFlags(&d.ev_fork, cudaEventDisableTiming));
    CU_TRY(cudaEventCreateWithFlags(&d.ev_join, cudaEventDisableTiming));
    for (int i = 0; i < 4; ++i) {
      CU_TRY(cudaStreamCreateWithFlags(&d.tside[i], cudaStreamNonBlocking));
      CU_TRY(cudaEventCreateWithFlags(&d.tfork[i], cudaEventDisableTiming));
      CU_TRY(cudaEventCreateWithFlags(&d.tjoin[i], cudaEventDisableTiming));
    }
    CU_TRY(cudaStreamCreateWithFlags(&d.freer, cudaStreamNonBlocking));
    if (!g_encode) {
      cudaDriverEntryPointQueryResult q;
      void* fn = nullptr;
      CU_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
      if (q != cudaDriverEntryPointSuccess || !fn)
        return fail(NS_ERR_CUDA, "cuTensorMapEncodeTiled entry point not found");
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    d.init = true;
  }
  *out = &d;
  return NS_OK;
}

static inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Stream-ordered release of library-owned device memory (allocated with cudaMallocAsync):
// the private `freer` stream waits for `last` (an event recorded after the memory's last
// use) and frees there -- no host synchronisation.
static void release_async(int dev, void* p, cudaEvent_t last) {
  if (!p) return;
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != dev) cudaSetDevice(dev);
  DevCtx& d = g_dev[dev & 63];
  cudaStream_t s = d.init ? d.freer : nullptr;
  if (last && s) cudaStreamWaitEvent(s, last, 0);
  if (cudaFreeAsync(p, s) != cudaSuccess) cudaGetLastError();
  if (cur != dev) cudaSetDevice(cur);
}

// Row-major R x C bf16 matrix, zero OOB fill.  box = 64: 64 x 64 boxes with 128-byte
// swizzle (GEMM operands); box = 32: 32 x 32 boxes with 64-byte swizzle (epilogue).
static ns_status encode_tmap(CUtensorMap* tm, const void* base, int64_t rows, int64_t cols, int box_dim = 64) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_dim, (cuuint32_t)box_dim};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        box_dim == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(NS_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return NS_OK;
}
// Both maps of one buffer, consecutively: [64-box operand map, 32-box epilogue map].
static ns_status encode_pair(std::vector<CUtensorMap>& v, const void* base, int64_t rows, int64_t cols, int* idx) {
  CUtensorMap tm[2];
  ns_status st;
  if ((st = encode_tmap(&tm[0], base, rows, cols, 64)) != NS_OK) return st;
  if ((st = encode_tmap(&tm[1], base, rows, cols, 32)) != NS_OK) return st;
  *idx = (int)v.size();
  v.push_back(tm[0]);
  v.push_back(tm[1]);
  return NS_OK;
}

// ---------------------------------------------------------------------------- planning
struct Mat {
  void* x;
  void* out;
  int64_t m, n, M, N;
  bool wide;
  bool copy_in;
  // workspace byte offsets
  size_t w_off, a_off, b_off, s_off, part_off, split_off;
  int part_ld;
  int split;  // split-K factor of this matrix's Gram (0: none), see choose_splits
  // mixed-precision call (ns_orthogonalize_cast): the caller's fp32 buffers; x / out then
  // point at a bf16 staging copy in the workspace (stage_off)
  const void* user_x = nullptr;
  void* user_out = nullptr;
  size_t stage_off = 0;
  // tensormap indices (tcgen05 path)
  int tm_x, tm_out, tm_w, tm_a, tm_b;
  size_t tc_part_off = 0;  // cluster tcgen05 kernel: Gram partials + A image (tc_part_floats)
  size_t cl_off = 0;       // FFMA cluster kernel: row-exchange scratch (cl_xchg_floats)
  // fused collective: extra destinations of the final result (peers' buffers)
  std::vector<void*> peer;
  int tm_peer;
};

enum PhaseKind { PH_GEMM = 0, PH_SIMT = 1, PH_PRECOND = 2, PH_COPY = 3, PH_CLUSTER = 5, PH_SPLIT = 6,
                 PH_CAST_IN = 7, PH_CAST_OUT = 8, PH_TC = 9 };
struct Phase {
  PhaseKind kind;
  size_t dev_off;  // offset of the job array in the device table
  int njobs;
  int64_t total;    // tiles (GEMM/SIMT) or items (PRECOND)
  int64_t total_rows;
  bool vec8;
  bool lane_rows = false;  // PH_PRECOND: AOL from the Gram partials for every job
  int row_kinds = 0;       // PH_PRECOND: OR of precond_lane_kind over the jobs
  int gemm_kind;  // profiling kind: 0 GRAM, 2 POLY, 3 XB
  size_t tiles_off = 0;   // offset of the TaskDesc list (PH_GEMM)
  int64_t max_tiles = 0;  // tiles of the GEMM step
  size_t coeff_off = 0;   // PH_CLUSTER: 3*iters floats
  size_t smem = 0;        // PH_CLUSTER: dynamic shared memory per CTA
  int ctas = 8;           // PH_CLUSTER: CTAs per cluster
  bool has_split = false; // PH_GEMM: the task list holds split-K tasks
  int64_t max_numel = 0;  // PH_CAST_*: largest matrix
  // copies (PH_COPY)
  std::vector<std::pair<std::pair<void*, const void*>, size_t>> copies;
};

struct Plan {
  int device = 0;
  ns_dtype dtype = NS_BF16;
  bool simt = false;
  int cg = 2;  // tcgen05 CTA group (2: 256x256 tiles on CTA pairs)
  int bn = 256;  // tile width: 128 for tile-starved plans (see choose_bn)
  bool cast = false;  // fp32 caller buffers, bf16 compute (ns_orthogonalize_cast)
  int iters = 0;
  ns_precond precond = NS_PRECOND_AOL;
  std::vector<Mat> mats;   // tcgen05 / SIMT step engine
  std::vector<Mat> tiny;   // cluster-resident whole-NS kernel (row a-10)
  std::vector<Mat> tc;     // cluster-resident tcgen05 whole-NS kernel (mid-size, §8(f) rank 4)
  void* ws = nullptr;
  size_t ws_bytes = 0;
  void* dtab = nullptr;
  size_t dtab_bytes = 0;
  unsigned* barrier = nullptr;
  std::vector<Phase> phases;
  uint64_t last_use = 0;
  bool ws_borrowed = false;  // carved from the caller's ns_set_workspace buffer
  // the plan's launch sequence captured once into a CUDA graph (see launch_plan)
  cudaGraphExec_t gexec = nullptr;
  uint64_t glaunches = 0;
  uint64_t uses = 0;
  bool graph_failed = false;
  bool pinned = false;             // resolved for a call in progress: never evicted
  cudaEvent_t last = nullptr;      // recorded on the caller's stream after every launch
  cudaStream_t last_stream = nullptr;  // ... on this stream (a call on another stream waits for it)
  ~Plan() {
    // an executable graph still in flight is released on completion (cudaGraphExecDestroy);
    // device memory is freed stream-ordered after the last launch (release_async)
    if (gexec) cudaGraphExecDestroy(gexec);
    if (ws && !ws_borrowed) release_async(device, ws, last);
    if (dtab) release_async(device, dtab, last);
    if (last) cudaEventDestroy(last);
  }
};

static std::map<std::vector<uint64_t>, std::unique_ptr<Plan>> g_plans;
// Caller-owned workspace (ns_set_workspace): plans built while it is set carve their
// workspace from it (bump allocation), instead of cudaMalloc.
struct UserWs { uint8_t* base = nullptr; size_t bytes = 0, used = 0; };
static UserWs g_uws[64];
static uint64_t g_tick = 0;
static const size_t kMaxPlans = 256;  // distinct problem lists (e.g. buckets of a pipeline)

static size_t elem_size(ns_dtype d) { return d == NS_BF16 ? 2 : 4; }

static bool tma_ok(const Mat& mt, ns_dtype dt) {
  if (dt != NS_BF16) return false;
  if ((mt.n % 8) != 0 || (mt.m % 8) != 0) return false;
  if ((reinterpret_cast<uintptr_t>(mt.x) & 15) || (reinterpret_cast<uintptr_t>(mt.out) & 15)) return false;
  if (mt.m > (int64_t)1 << 31 || mt.n > (int64_t)1 << 31) return false;
  return true;
}

// s is padded with zeros to a multiple of the 256-wide tile (+32): the epilogue reads
// s[q .. q+32) and s[p] for whole tiles without bounds checks.
static size_t s_floats(int64_t N) { return (size_t)((N + 255) / 256 * 256 + 32); }
// AOL row-sum partial slots per row (see GemmJob::part).
static int part_ld_for(int64_t N) { return (int)((N + 63) / 64 + (N + 31) / 32); }

// Split-K Gram.  For N <= 256 the Gram is one 256 x 256 block per matrix, walked over the
// whole K = M by a single CTA pair: with a long K (tall matrices, e.g. 256 x 2304 conv
// weights) a handful of pairs would stream K at single-SM bandwidth while the rest of the GPU
// idles.  Such Grams (N <= 256, nk = ceil(M / 64) >= 16 k-blocks) are cut into
// S = min(16, ceil(nk / 8)) k-ranges, computed as independent tiles whose fp32 partials a
// reduction launch sums in a fixed order.  S depends on the matrix shape ALONE -- never on
// the rest of the call -- so a matrix's result is bitwise the same in every call (single,
// batched, or on any rank of the sharded path, §8(e)).  Per-step launches only.
static const int64_t kSplitLd = 256;  // floats per partial row; rows padded to 256 too
static int split_factor(int64_t M, int64_t N) {
  if (N > kSplitMaxN) return 0;
  const int64_t nk = (M + kBK - 1) / kBK;
  if (nk < 16) return 0;
  return (int)std::min<int64_t>(16, (nk + 7) / 8);
}
static void choose_splits(std::vector<Mat>& mats) {
  const char* e = getenv("TNS_NOSPLIT");  // A/B knob, read at plan build
  const bool off = e && atoi(e);
  for (Mat& mt : mats) mt.split = off ? 0 : split_factor(mt.M, mt.N);
}
// Tile width.  A plan whose every GEMM step has at most half as many 256-wide tiles as there
// are CTA-pair workers (small problems: one tile per pair, latency-bound) uses 128-wide
// tiles: twice the tiles, and each epilogue warp drains 2 chunks instead of 4 -- the
// epilogue is the longest stretch of such a launch.  Results are bitwise the same as with
// 256-wide tiles (every output element is the same sequence of K = 16 UMMA steps; the AOL
// partials are per 64 columns either way), so the choice never breaks batch invariance.
// Per-step launches on CTA pairs only; TNS_BN=256 forces the wide tiles (A/B knob).
static int choose_bn(const std::vector<Mat>& mats, int cg, int workers) {
  if (cg != 2) return 256;
  if (const char* e = getenv("TNS_BN")) {  // A/B knob: force either width
    if (atoi(e) == 256) return 256;
    if (atoi(e) == 128) return 128;
  }
  int64_t sym = 0, xb = 0;
  for (const Mat& mt : mats) {
    const int64_t nb = (mt.N + kSymBlock - 1) / kSymBlock;
    sym += nb * (nb + 1) / 2;
    const int64_t P = mt.wide ? mt.N : mt.M, Q = mt.wide ? mt.M : mt.N;
    xb += ((P + 255) / 256) * ((Q + 255) / 256);
  }
  return 2 * std::max(sym, xb) <= workers ? 128 : 256;
}

static size_t split_bytes(const Mat& mt) { return mt.split ? (size_t)mt.split * kSplitLd * kSplitLd * 4 : 0; }

static size_t tc_part_bytes(int64_t M, int64_t N) {
  const int C = tc_cluster(M, N);
  return C ? tc_part_floats(tc_np(N), C) * 4 : 0;
}
// CTAs of the FFMA cluster kernel for a matrix (16 when it fits that layout; TNS_CL_CTAS=8
// forces 8 -- an A/B knob), and its exchange scratch
static int cl_ctas(int64_t M, int64_t N) {
  static const bool only8 = [] { const char* e = getenv("TNS_CL_CTAS"); return e && atoi(e) == 8; }();
  return !only8 && cl_fits(M, N, kClCtasMax) ? kClCtasMax : kClCtas;
}
static size_t cl_xchg_bytes(int64_t M, int64_t N) {
  return cl_fits(M, N) ? cl_xchg_floats((int)M, (int)N, cl_ctas(M, N)) * 4 : 0;
}

// Workspace of a problem list as the step engine lays it out; a bf16 matrix the tcgen05
// cluster kernel could take counts with the larger of its two footprints (an upper bound
// whatever the routing).
static size_t workspace_bytes_for(const std::vector<Mat>& mats, ns_dtype dt) {
  size_t off = 1024;  // [0,1024): grid-barrier words
  const size_t es = elem_size(dt);
  for (const Mat& mt : mats) {
    size_t o = 0;
    o = align_up(o, 256) + (size_t)mt.M * mt.N * es;
    o = align_up(o, 256) + (size_t)mt.N * mt.N * es;
    o = align_up(o, 256) + (size_t)mt.N * mt.N * es;
    o = align_up(o, 256) + s_floats(mt.N) * 4;
    o = align_up(o, 256) + (size_t)mt.N * part_ld_for(mt.N) * 4;
    if (dt == NS_BF16) o = align_up(o, 256) + (size_t)split_factor(mt.M, mt.N) * kSplitLd * kSplitLd * 4;
    if (dt == NS_BF16 && tc_fits(mt.M, mt.N)) o = std::max(o, tc_part_bytes(mt.M, mt.N));
    o = std::max(o, cl_xchg_bytes(mt.M, mt.N));  // or the FFMA cluster kernel's exchange scratch
    off = align_up(off, 256) + align_up(o, 256);
  }
  return align_up(off, 256);
}

// Host tables assembled for one plan before upload.
struct HostTables {
  std::vector<uint8_t> bytes;
  size_t push(const void* p, size_t n, size_t align = 128) {
    size_t off = align_up(bytes.size(), align);
    bytes.resize(off + n);
    std::memcpy(bytes.data() + off, p, n);
    return off;
  }
};

// Measurement knob (A/B of the half-storage symmetric matrices): TNS_NOHALF=1 stores A
// and B' whole (mirrored) and reads them K-major only.
static bool half_storage_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TNS_NOHALF");
    v = (e && atoi(e)) ? 0 : 1;
  }
  return v == 1;
}

// Persistent workers take tasks t = w, w + nw, w + 2 nw, ...  When a step mixes tile
// lengths (e.g. a Gram over K = 1024 and K = 4096 matrices), plain round-robin leaves up to
// ~5 % imbalance; instead assign tiles greedily longest-first to the least-loaded worker
// (cost = k-blocks + 4 for the epilogue) and lay each worker's list out on its stride,
// padding with TK_NONE.  Within a worker the original (rasterised) order is kept.
static void balance_tasks(std::vector<TaskDesc>& tasks, const std::vector<GemmJob>& jobs, int workers) {
  const int64_t n = (int64_t)tasks.size();
  if (workers < 2 || n <= workers) return;
  auto cost = [&](const TaskDesc& td) {
    return (int64_t)(td.nkb ? td.nkb : (jobs[td.tile & 0xFFFFFu].K + kBK - 1) / kBK) + 4;
  };
  int64_t cmin = INT64_MAX, cmax = 0;
  for (const TaskDesc& td : tasks) { cmin = std::min(cmin, cost(td)); cmax = std::max(cmax, cost(td)); }
  if (cmin == cmax) return;  // uniform tiles: round-robin is already balanced
  std::vector<int64_t> order(n);
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return cost(tasks[a]) > cost(tasks[b]); });
  std::vector<int64_t> load(workers, 0);
  std::vector<std::vector<int64_t>> lists(workers);
  for (int64_t i : order) {
    int w = 0;
    for (int k = 1; k < workers; ++k) if (load[k] < load[w]) w = k;
    load[w] += cost(tasks[i]);
    lists[w].push_back(i);
  }
  size_t rounds = 0;
  for (auto& l : lists) { std::sort(l.begin(), l.end()); rounds = std::max(rounds, l.size()); }
  TaskDesc pad;
  std::memset(&pad, 0, sizeof(pad));
  pad.kind = TK_NONE;
  std::vector<TaskDesc> out(rounds * workers, pad);
  for (int w = 0; w < workers; ++w)
    for (size_t r = 0; r < lists[w].size(); ++r) out[r * workers + w] = tasks[lists[w][r]];
  tasks.swap(out);
}

static ns_status build_plan(Plan& P, HostTables& H, DevCtx* dc, const float* coeffs, cudaStream_t stream) {
  const int hs = half_storage_enabled() ? 1 : 0;
  const int T = P.iters;
  const size_t es = elem_size(P.dtype);
  const bool bf16 = P.dtype == NS_BF16;
  if (!P.simt) choose_splits(P.mats);
  else for (Mat& mt : P.mats) mt.split = 0;
  P.bn = P.simt ? 256 : choose_bn(P.mats, P.cg, dc->sms / 2);
  // -- workspace layout
  size_t off = 1024;  // [0,16): preconditioner grid barrier; [64, 1024): phase counters
  for (Mat& mt : P.mats) {
    off = align_up(off, 256); mt.w_off = off; off += (size_t)mt.M * mt.N * es;
    off = align_up(off, 256); mt.a_off = off; off += (size_t)mt.N * mt.N * es;
    off = align_up(off, 256); mt.b_off = off; off += (size_t)mt.N * mt.N * es;
    off = align_up(off, 256); mt.s_off = off; off += s_floats(mt.N) * 4;
    mt.part_ld = part_ld_for(mt.N);
    off = align_up(off, 256); mt.part_off = off;
    if (P.precond == NS_PRECOND_AOL && !P.simt) off += (size_t)mt.N * mt.part_ld * 4;
    off = align_up(off, 256); mt.split_off = off; off += split_bytes(mt);
  }
  for (Mat& mt : P.tc) {  // Gram partials of the tcgen05 cluster kernel
    off = align_up(off, 256); mt.tc_part_off = off; off += tc_part_bytes(mt.M, mt.N);
  }
  for (Mat& mt : P.tiny) {  // row-exchange scratch of the FFMA cluster kernel
    off = align_up(off, 256); mt.cl_off = off; off += cl_xchg_bytes(mt.M, mt.N);
  }
  if (P.cast) {  // bf16 staging copies of the caller's fp32 matrices
    for (Mat& mt : P.mats) { off = align_up(off, 256); mt.stage_off = off; off += (size_t)mt.m * mt.n * 2; }
    for (Mat& mt : P.tiny) { off = align_up(off, 256); mt.stage_off = off; off += (size_t)mt.m * mt.n * 2; }
    for (Mat& mt : P.tc) { off = align_up(off, 256); mt.stage_off = off; off += (size_t)mt.m * mt.n * 2; }
  }
  P.ws_bytes = align_up(off, 256);
  cudaError_t e = cudaSuccess;
  UserWs& uw = g_uws[P.device & 63];
  if (uw.base) {
    const size_t at = align_up(uw.used, 256);
    if (at + P.ws_bytes > uw.bytes)
      return fail(NS_ERR_WORKSPACE, "caller workspace too small: this problem list needs " +
                                        std::to_string(P.ws_bytes) + " more bytes, " +
                                        std::to_string(uw.bytes > at ? uw.bytes - at : 0) + " left");
    P.ws = uw.base + at;
    P.ws_borrowed = true;
    uw.used = at + P.ws_bytes;
  } else {
    e = cudaMallocAsync(&P.ws, P.ws_bytes, stream);  // stream-ordered: no host synchronisation
    if (e != cudaSuccess) {
      cudaGetLastError();
      P.ws = nullptr;
      return fail(NS_ERR_WORKSPACE, "workspace cudaMallocAsync(" + std::to_string(P.ws_bytes) + ") failed");
    }
  }
  uint8_t* ws = reinterpret_cast<uint8_t*>(P.ws);
  P.barrier = reinterpret_cast<unsigned*>(ws);
  CU_TRY(cudaMemsetAsync(P.ws, 0, P.ws_bytes, stream));  // zero padding of s (and everything else) once
  auto W = [&](const Mat& mt) { return (void*)(ws + mt.w_off); };
  auto Am = [&](const Mat& mt) { return (void*)(ws + mt.a_off); };
  auto Bm = [&](const Mat& mt) { return (void*)(ws + mt.b_off); };
  auto Sv = [&](const Mat& mt) { return (float*)(ws + mt.s_off); };
  auto Part = [&](const Mat& mt) { return (float*)(ws + mt.part_off); };
  const bool use_part = (P.precond == NS_PRECOND_AOL) && !P.simt;

  // -- mixed precision: cast the caller's fp32 matrices into bf16 staging (in place from
  //    then on), cast the results back at the end
  std::vector<CastJob> cast_out;
  if (P.cast) {
    std::vector<CastJob> cin;
    int64_t mx = 0;
    for (std::vector<Mat>* v : {&P.mats, &P.tiny, &P.tc})
      for (Mat& mt : *v) {
        mt.user_x = mt.x; mt.user_out = mt.out;
        void* st = ws + mt.stage_off;
        cin.push_back({mt.user_x, st, mt.m * mt.n});
        cast_out.push_back({st, mt.user_out, mt.m * mt.n});
        mt.x = mt.out = st;
        mt.copy_in = (T % 2 == 1);
        mx = std::max<int64_t>(mx, mt.m * mt.n);
      }
    Phase ph{PH_CAST_IN};
    ph.dev_off = H.push(cin.data(), cin.size() * sizeof(CastJob), 64);
    ph.njobs = (int)cin.size();
    ph.max_numel = mx;
    P.phases.push_back(ph);
  }

  // -- tensormaps (tcgen05 path)
  std::vector<CUtensorMap> tmaps;
  if (!P.simt) {
    for (Mat& mt : P.mats) {
      ns_status st;
      if ((st = encode_pair(tmaps, mt.x, mt.m, mt.n, &mt.tm_x)) != NS_OK) return st;
      if (mt.out != mt.x) {
        if ((st = encode_pair(tmaps, mt.out, mt.m, mt.n, &mt.tm_out)) != NS_OK) return st;
      } else {
        mt.tm_out = mt.tm_x;
      }
      if ((st = encode_pair(tmaps, W(mt), mt.m, mt.n, &mt.tm_w)) != NS_OK) return st;
      if ((st = encode_pair(tmaps, Am(mt), mt.N, mt.N, &mt.tm_a)) != NS_OK) return st;
      if ((st = encode_pair(tmaps, Bm(mt), mt.N, mt.N, &mt.tm_b)) != NS_OK) return st;
      mt.tm_peer = (int)tmaps.size();
      for (void* pp : mt.peer) {
        CUtensorMap tm;
        if ((st = encode_tmap(&tm, pp, mt.m, mt.n, 32)) != NS_OK) return st;
        tmaps.push_back(tm);
      }
    }
  }
  for (Mat& mt : P.tc) {  // tcgen05 cluster kernel: 64 x 64-box maps of the input and output
    ns_status st;
    CUtensorMap tm;
    if ((st = encode_tmap(&tm, mt.x, mt.m, mt.n, 64)) != NS_OK) return st;
    mt.tm_x = (int)tmaps.size();
    tmaps.push_back(tm);
    if ((st = encode_tmap(&tm, mt.out, mt.m, mt.n, 64)) != NS_OK) return st;
    mt.tm_out = (int)tmaps.size();
    tmaps.push_back(tm);
  }
  size_t tm_off = tmaps.empty() ? 0 : H.push(tmaps.data(), tmaps.size() * sizeof(CUtensorMap), 128);
  struct TcFix { size_t job_off; int tin, tout; };
  std::vector<TcFix> tc_fixes;

  // Device addresses of tensormaps are known only after allocation: record indices now,
  // patch pointers after cudaMalloc of the table (two-pass).  We first compute the final
  // table size by building jobs with placeholder bases, then fix them up.
  struct Fix { size_t job_off; int ta, tb, tout, taux, tpeer = -1; };
  std::vector<Fix> fixes;
  struct Step {  // one tcgen05-path step before it is laid out as launches
    int kind = PHK_GEMM;
    int gemm_kind = 0;
    std::vector<GemmJob> jobs;
    std::vector<std::array<int, 5>> tmi;
    size_t job_base = 0;
    std::vector<PrecondJob> pj;
    int64_t rows = 0, items = 0;
    bool vec8 = false;
    std::vector<int> jsplit;   // PHK_GEMM: split-K factor per job (0: none)
    std::vector<SplitJob> sj;  // PHK_SPLIT
  };
  std::vector<Step> steps;

  // -- phases
  if (P.mats.size() > 0) {
    Phase cp{PH_COPY};
    for (Mat& mt : P.mats)
      if (mt.copy_in) cp.copies.push_back({{W(mt), mt.x}, (size_t)mt.m * mt.n * es});
    if (!cp.copies.empty()) P.phases.push_back(cp);
  }
  auto cur_ptr = [&](const Mat& mt, int k) -> void* {  // X_k (k = 1..T+1), caller layout
    if (k == 1) return mt.copy_in ? W(mt) : mt.x;
    return ((T - (k - 1)) % 2 == 0) ? mt.out : W(mt);  // dst of iteration k-1
  };
  auto cur_tm = [&](const Mat& mt, int k) -> int {
    if (k == 1) return mt.copy_in ? mt.tm_w : mt.tm_x;
    return ((T - (k - 1)) % 2 == 0) ? mt.tm_out : mt.tm_w;
  };

  // -- small matrices: the whole NS in one cluster launch (enqueued first, on a side stream
  //    when the step engine has work too, so the two overlap)
  if (!P.tiny.empty()) {
    // 16-CTA clusters for the matrices that fit that layout, 8-CTA for the others: the
    // choice depends on the matrix alone, so batched results stay bitwise equal to single
    // calls (one cluster launch per group)
    for (int ctas : {kClCtasMax, kClCtas}) {
      std::vector<ClusterJob> cj;
      size_t smem = 0;
      for (const Mat& mt : P.tiny) {
        if (cl_ctas(mt.M, mt.N) != ctas) continue;
        ClusterJob J;
        std::memset(&J, 0, sizeof(J));
        J.x = mt.x; J.out = mt.out;
        J.xchg = reinterpret_cast<float*>(ws + mt.cl_off);
        J.m = (int)mt.m; J.n = (int)mt.n; J.M = (int)mt.M; J.N = (int)mt.N; J.wide = mt.wide ? 1 : 0;
        cj.push_back(J);
        smem = std::max(smem, cl_layout(J.M, J.N, ctas).floats * 4 + kClHdr);
      }
      if (cj.empty()) continue;
      Phase ph{PH_CLUSTER};
      ph.dev_off = H.push(cj.data(), cj.size() * sizeof(ClusterJob), 64);
      ph.coeff_off = H.push(coeffs, (size_t)3 * T * sizeof(float), 16);
      ph.njobs = (int)cj.size();
      ph.smem = smem;
      ph.ctas = ctas;
      P.phases.push_back(ph);
    }
  }
  // -- mid-size bf16 matrices: the whole NS on the tensor cores in one 16-CTA cluster each,
  //    one launch for all of them (on a second side stream when other work is present)
  if (!P.tc.empty()) {
    // one launch per cluster size (a function of the shape alone, tc_cluster)
    for (int C = 2; C <= kTcCtas; C *= 2) {
      std::vector<TcJob> jobs;
      std::vector<TcFix> fx;
      size_t smem = 0;
      for (const Mat& mt : P.tc) {
        if (tc_cluster(mt.M, mt.N) != C) continue;
        TcJob J;
        std::memset(&J, 0, sizeof(J));
        J.m = (int)mt.m; J.n = (int)mt.n; J.M = (int)mt.M; J.N = (int)mt.N; J.wide = mt.wide ? 1 : 0;
        J.Np = tc_np(mt.N); J.C = C; J.R = tc_rows(mt.M, C);
        J.part = reinterpret_cast<float*>(ws + mt.tc_part_off);
        fx.push_back({jobs.size() * sizeof(TcJob), mt.tm_x, mt.tm_out});
        jobs.push_back(J);
        smem = std::max(smem, tc_smem(J.Np, J.R, C));
      }
      if (jobs.empty()) continue;
      Phase ph{PH_TC};
      ph.dev_off = H.push(jobs.data(), jobs.size() * sizeof(TcJob), 64);
      for (TcFix& f : fx) { f.job_off += ph.dev_off; tc_fixes.push_back(f); }
      ph.coeff_off = H.push(coeffs, (size_t)3 * T * sizeof(float), 16);
      ph.njobs = (int)jobs.size();
      ph.smem = smem;
      ph.ctas = C;
      P.phases.push_back(ph);
    }
  }
  for (int k = 1; k <= T && !P.mats.empty(); ++k) {
    const float a = coeffs[3 * (k - 1)], b = coeffs[3 * (k - 1) + 1], c = coeffs[3 * (k - 1) + 2];
    const bool scaled = (k == 1 && P.precond != NS_PRECOND_NONE);
    for (int step = 0; step < 3; ++step) {
      const int mode = step;  // GRAM, POLY, XB
      if (!P.simt) {
        std::vector<GemmJob> jobs;
        std::vector<std::array<int, 5>> tmi;
        for (Mat& mt : P.mats) {
          GemmJob J;
          std::memset(&J, 0, sizeof(J));
          J.mode = mode;
          int ta = 0, tb = 0, tout = -1, taux = -1;
          if (mode == MODE_GRAM) {
            ta = tb = cur_tm(mt, k);
            tout = mt.tm_a;
            J.a_mn = J.b_mn = mt.wide ? 0 : 1;
            J.sym = 1; J.P = J.Q = (int)mt.N; J.K = (int)mt.M;
            J.out = Am(mt); J.aux = nullptr; J.ld = mt.N;
            J.half = hs;  // A: lower-triangle blocks only (readers take the upper transposed)
            if (k == 1 && use_part) {
              J.part = Part(mt); J.part_ld = mt.part_ld;
              J.part_sm = precond_part_sm(mt.part_ld);  // precond_rows.cuh: per-N summation
            }
            if (mt.split) {  // partials only; the reduction launch writes A (and the AOL sums)
              J.split_ws = reinterpret_cast<float*>(ws + mt.split_off);
              J.split_stride = kSplitLd * kSplitLd;
              J.split_ld = (int)kSplitLd;
              J.part = nullptr; J.part_ld = 0;
            }
          } else if (mode == MODE_POLY) {
            ta = tb = mt.tm_a;
            tout = mt.tm_b; taux = mt.tm_a;
            J.a_mn = J.b_mn = 0;
            J.sym = 1; J.P = J.Q = J.K = (int)mt.N;
            J.out = Bm(mt); J.aux = Am(mt); J.ld = mt.N;
            J.s = scaled ? Sv(mt) : nullptr;
            J.b = b; J.c = c;
            J.diag_add = a;  // B' = bA + cA^2 + aI: Eq. 5 becomes the single product X B'
            J.a_sym = J.b_sym = hs;       // A is half-stored
            J.half = scaled ? 0 : hs;     // B1' = sym * diag(s) is not symmetric: store it whole
          } else {
            if (!mt.wide) {
              ta = cur_tm(mt, k); tb = mt.tm_b; J.a_mn = 0; J.b_mn = 0;
              J.P = (int)mt.M; J.Q = (int)mt.N; J.s_by_row = 0;
              J.b_sym = scaled ? 0 : hs;  // B' half-stored except the scaled iteration 1
            } else {
              ta = mt.tm_b; tb = cur_tm(mt, k); J.a_mn = 0; J.b_mn = 1;
              J.P = (int)mt.N; J.Q = (int)mt.M; J.s_by_row = 1;
              J.a_sym = scaled ? 0 : hs;
            }
            J.sym = 0; J.K = (int)mt.N;
            J.out = cur_ptr(mt, k + 1); J.aux = nullptr; J.ld = mt.n;
            tout = ((T - k) % 2 == 0) ? mt.tm_out : mt.tm_w;
            if (k == T && !mt.peer.empty()) J.npeer = (int)mt.peer.size();
            // a_k and diag(s) are folded into B' by the POLY epilogue: no aux, plain store
            J.s = nullptr;
            J.a = 0.f;
          }
          J.tiles_q = J.sym ? (J.P + kSymBlock - 1) / kSymBlock : (J.Q + kBN - 1) / kBN;
          jobs.push_back(J);
          tmi.push_back({ta, tb, tout, taux, J.npeer ? mt.tm_peer : -1});
        }
        Step stp;
        stp.kind = PHK_GEMM;
        stp.gemm_kind = mode == MODE_GRAM ? 0 : (mode == MODE_POLY ? 2 : 3);
        stp.jobs = std::move(jobs);
        stp.tmi = std::move(tmi);
        for (Mat& mt : P.mats) stp.jsplit.push_back(mode == MODE_GRAM ? mt.split : 0);
        steps.push_back(std::move(stp));
        if (mode == MODE_GRAM) {
          Step red;
          red.kind = PHK_SPLIT;
          for (Mat& mt : P.mats) {
            if (!mt.split) continue;
            SplitJob S;
            std::memset(&S, 0, sizeof(S));
            S.ws = reinterpret_cast<const float*>(ws + mt.split_off);
            S.stride = kSplitLd * kSplitLd; S.ld = (int)kSplitLd;
            S.S = mt.split; S.N = (int)mt.N;
            S.A = Am(mt);
            if (k == 1 && use_part) { S.part = Part(mt); S.part_ld = mt.part_ld; S.part_sm = precond_part_sm(mt.part_ld); }
            S.row_start = red.rows;
            red.rows += mt.N;
            red.sj.push_back(S);
          }
          if (!red.sj.empty()) steps.push_back(std::move(red));
        }
      } else {
        std::vector<SimtJob> jobs;
        int64_t total = 0;
        for (Mat& mt : P.mats) {
          SimtJob J;
          std::memset(&J, 0, sizeof(J));
          J.mode = mode;
          if (mode == MODE_GRAM) {
            void* X = cur_ptr(mt, k);
            J.A = J.B = X;
            if (!mt.wide) { J.sa_p = J.sb_q = 1; J.sa_k = J.sb_k = mt.n; }
            else          { J.sa_p = J.sb_q = mt.n; J.sa_k = J.sb_k = 1; }
            J.P = J.Q = (int)mt.N; J.K = (int)mt.M;
            J.out = Am(mt); J.ld = mt.N;
          } else if (mode == MODE_POLY) {
            J.A = J.B = Am(mt);
            J.sa_p = J.sb_q = mt.N; J.sa_k = J.sb_k = 1;
            J.P = J.Q = J.K = (int)mt.N;
            J.out = Bm(mt); J.aux = Am(mt); J.ld = mt.N;
            J.s = scaled ? Sv(mt) : nullptr;
            J.b = b; J.c = c;
          } else {
            void* X = cur_ptr(mt, k);
            if (!mt.wide) {
              J.A = X; J.sa_p = mt.n; J.sa_k = 1;
              J.B = Bm(mt); J.sb_q = mt.N; J.sb_k = 1;
              J.P = (int)mt.M; J.Q = (int)mt.N; J.s_by_row = 0;
            } else {
              J.A = Bm(mt); J.sa_p = mt.N; J.sa_k = 1;
              J.B = X; J.sb_q = 1; J.sb_k = mt.n;
              J.P = (int)mt.N; J.Q = (int)mt.M; J.s_by_row = 1;
            }
            J.K = (int)mt.N;
            J.out = cur_ptr(mt, k + 1); J.aux = X; J.ld = mt.n;
            J.s = scaled ? Sv(mt) : nullptr;
            J.a = a;
          }
          J.tiles_q = (J.Q + kSimtTile - 1) / kSimtTile;
          J.tiles = ((J.P + kSimtTile - 1) / kSimtTile) * J.tiles_q;
          J.tile_start = total;
          total += J.tiles;
          jobs.push_back(J);
        }
        Phase ph{PH_SIMT};
        ph.dev_off = H.push(jobs.data(), jobs.size() * sizeof(SimtJob), 64);
        ph.njobs = (int)jobs.size();
        ph.total = total;
        P.phases.push_back(ph);
      }
      if (mode == MODE_GRAM && scaled) {
        std::vector<PrecondJob> pj;
        int64_t rows = 0, items = 0;
        bool vec8 = bf16;
        for (Mat& mt : P.mats) vec8 = vec8 && (mt.N % 8 == 0);
        for (Mat& mt : P.mats) {
          PrecondJob J;
          std::memset(&J, 0, sizeof(J));
          J.A = Am(mt); J.s = Sv(mt); J.N = (int)mt.N; J.precond = (int)P.precond;
          if (use_part) { J.part = Part(mt); J.part_ld = mt.part_ld; J.part_sm = precond_part_sm(mt.part_ld); }
          J.half = P.simt ? 0 : hs;
          J.row_start = rows; J.seg_start = items;
          rows += mt.N;
          items += precond_segments(J.N, J.half);  // phase-2 work units (256-column row segments)
          pj.push_back(J);
        }
        if (P.simt) {
          Phase ph{PH_PRECOND};
          ph.dev_off = H.push(pj.data(), pj.size() * sizeof(PrecondJob), 64);
          ph.njobs = (int)pj.size();
          ph.total = items;
          ph.total_rows = rows;
          ph.vec8 = vec8;
          P.phases.push_back(ph);
        } else {
          Step stp;
          stp.kind = PHK_PRE_S;
          stp.pj = std::move(pj);
          stp.rows = rows;
          stp.items = items;
          stp.vec8 = vec8;
          steps.push_back(std::move(stp));
        }
      }
    }
  }

  // -- tcgen05 steps: one launch each (PDL-chained)
  if (!P.simt && !steps.empty()) {
    auto tile_list = [&](const Step& st) {
      // longest-K jobs first (LPT-like): long tiles do not end up in the last wave
      std::vector<size_t> order(st.jobs.size());
      for (size_t j = 0; j < st.jobs.size(); ++j) order[j] = j;
      std::stable_sort(order.begin(), order.end(), [&](size_t x, size_t y) { return st.jobs[x].K > st.jobs[y].K; });
      std::vector<uint64_t> tl;
      for (size_t j : order) umma_tile_list(st.jobs[j], (uint32_t)j, P.cg, P.bn, tl);
      return tl;
    };
    auto mk_task = [](uint64_t w) {
      TaskDesc td;
      std::memset(&td, 0, sizeof(td));
      td.tile = w; td.kind = TK_TILE;
      return td;
    };
    for (Step& st : steps) {
      if (st.kind == PHK_GEMM) {
        std::vector<TaskDesc> tasks;
        std::vector<uint64_t> tl = tile_list(st);
        for (uint64_t w : tl) {
          const size_t j = w & 0xFFFFFu;
          const int S = j < st.jsplit.size() ? st.jsplit[j] : 0;
          if (!S) { tasks.push_back(mk_task(w)); continue; }
          const int nk = (st.jobs[j].K + kBK - 1) / kBK;
          for (int sp = 0; sp < S; ++sp) {  // k-blocks [sp*nk/S, (sp+1)*nk/S)
            TaskDesc td = mk_task(w);
            td.kb0 = (uint32_t)(sp * nk / S);
            td.nkb = (uint32_t)((sp + 1) * nk / S) - td.kb0;
            td.split = (uint32_t)sp + 1;
            tasks.push_back(td);
          }
        }
        balance_tasks(tasks, st.jobs, dc->sms / P.cg);
        Phase ph{PH_GEMM};
        ph.gemm_kind = st.gemm_kind;
        for (const TaskDesc& td : tasks) ph.has_split = ph.has_split || td.split != 0;
        ph.dev_off = H.push(st.jobs.data(), st.jobs.size() * sizeof(GemmJob), 64);
        ph.njobs = (int)st.jobs.size();
        ph.tiles_off = H.push(tasks.data(), tasks.size() * sizeof(TaskDesc), 64);
        ph.total = (int64_t)tasks.size();
        ph.max_tiles = ph.total;
        for (size_t j = 0; j < st.jobs.size(); ++j)
          fixes.push_back({ph.dev_off + j * sizeof(GemmJob), st.tmi[j][0], st.tmi[j][1], st.tmi[j][2], st.tmi[j][3],
                           st.tmi[j][4]});
        P.phases.push_back(ph);
      } else if (st.kind == PHK_SPLIT) {
        Phase ph{PH_SPLIT};
        ph.dev_off = H.push(st.sj.data(), st.sj.size() * sizeof(SplitJob), 64);
        ph.njobs = (int)st.sj.size();
        ph.total_rows = st.rows;
        P.phases.push_back(ph);
      } else {
        Phase ph{PH_PRECOND};
        ph.dev_off = H.push(st.pj.data(), st.pj.size() * sizeof(PrecondJob), 64);
        ph.njobs = (int)st.pj.size();
        ph.total = st.items;
        ph.total_rows = st.rows;
        ph.vec8 = st.vec8;
        ph.lane_rows = true;
        for (const PrecondJob& pj : st.pj) {
          ph.lane_rows = ph.lane_rows && pj.precond == 2 && pj.part != nullptr;
          if (pj.part != nullptr) ph.row_kinds |= precond_lane_kind(pj.part_ld);
        }
        P.phases.push_back(ph);
      }
    }
  }

  if (P.cast) {
    Phase ph{PH_CAST_OUT};
    ph.dev_off = H.push(cast_out.data(), cast_out.size() * sizeof(CastJob), 64);
    ph.njobs = (int)cast_out.size();
    for (const CastJob& c : cast_out) ph.max_numel = std::max<int64_t>(ph.max_numel, c.numel);
    P.phases.push_back(ph);
  }

  // -- upload
  if (!H.bytes.empty()) {
    P.dtab_bytes = align_up(H.bytes.size(), 256);
    e = cudaMallocAsync(&P.dtab, P.dtab_bytes, stream);
    if (e != cudaSuccess) {
      cudaGetLastError();
      P.dtab = nullptr;
      return fail(NS_ERR_WORKSPACE, "job-table cudaMallocAsync failed");
    }
    uint8_t* dbase = reinterpret_cast<uint8_t*>(P.dtab);
    for (const Fix& f : fixes) {
      GemmJob* J = reinterpret_cast<GemmJob*>(H.bytes.data() + f.job_off);
      J->tmA = dbase + tm_off + (size_t)f.ta * sizeof(CUtensorMap);
      J->tmB = dbase + tm_off + (size_t)f.tb * sizeof(CUtensorMap);
      J->tmOut = dbase + tm_off + (size_t)(f.tout + 1) * sizeof(CUtensorMap);
      J->tmAux = f.taux >= 0 ? dbase + tm_off + (size_t)(f.taux + 1) * sizeof(CUtensorMap) : nullptr;
      J->tmPeer = f.tpeer >= 0 ? dbase + tm_off + (size_t)f.tpeer * sizeof(CUtensorMap) : nullptr;
    }
    for (const TcFix& f : tc_fixes) {
      TcJob* J = reinterpret_cast<TcJob*>(H.bytes.data() + f.job_off);
      J->tm_in = dbase + tm_off + (size_t)f.tin * sizeof(CUtensorMap);
      J->tm_out = dbase + tm_off + (size_t)f.tout * sizeof(CUtensorMap);
    }
    // pageable host -> device, stream-ordered: the runtime stages the bytes before returning
    // and does not wait for the stream's earlier work
    CU_TRY(cudaMemcpyAsync(P.dtab, H.bytes.data(), H.bytes.size(), cudaMemcpyHostToDevice, stream));
  }
  (void)dc;
  return NS_OK;
}

static ns_status enqueue_plan(Plan& P, DevCtx* dc, cudaStream_t stream) {
  uint8_t* dbase = reinterpret_cast<uint8_t*>(P.dtab);
  bool joined = true;
  uint32_t tjoined = 0xFu;  // bit i clear: tc side stream i must be joined back
  for (const Phase& ph : P.phases) {
    switch (ph.kind) {
      case PH_CLUSTER: {
        // alone: on the caller's stream; with step-engine work: forked onto the side stream
        const bool fork = !P.mats.empty();
        cudaStream_t s = stream;
        if (fork) {
          CU_TRY(cudaEventRecord(dc->ev_fork, stream));
          CU_TRY(cudaStreamWaitEvent(dc->side, dc->ev_fork, 0));
          s = dc->side;
          joined = false;
        }
        {
          ProfScope ps(7, s);
          CU_TRY(launch_cluster_ns(reinterpret_cast<const ClusterJob*>(dbase + ph.dev_off), ph.njobs,
                                   reinterpret_cast<const float*>(dbase + ph.coeff_off), P.iters, (int)P.precond,
                                   P.dtype == NS_BF16, ph.smem, ph.ctas, dc->flags, s));
        }
        ++g_launches;
        if (fork) CU_TRY(cudaEventRecord(dc->ev_join, dc->side));
        break;
      }
      case PH_TC: {
        // alone: on the caller's stream; beside other work (the step engine, the FFMA cluster
        // kernel, or a tc launch of another cluster size): forked onto its own side stream
        int ntc = 0;
        for (const Phase& q : P.phases) ntc += q.kind == PH_TC;
        const bool fork = !P.mats.empty() || !P.tiny.empty() || ntc > 1;
        const int si = ph.ctas == 2 ? 0 : ph.ctas == 4 ? 1 : ph.ctas == 8 ? 2 : 3;
        cudaStream_t s = stream;
        if (fork) {
          CU_TRY(cudaEventRecord(dc->tfork[si], stream));
          CU_TRY(cudaStreamWaitEvent(dc->tside[si], dc->tfork[si], 0));
          s = dc->tside[si];
          tjoined &= ~(1u << si);
        }
        {
          ProfScope ps(6, s);
          CU_TRY(launch_cluster_tc_ns(reinterpret_cast<const TcJob*>(dbase + ph.dev_off), ph.njobs, ph.ctas,
                                      reinterpret_cast<const float*>(dbase + ph.coeff_off), P.iters, (int)P.precond,
                                      ph.smem, dc->flags, s));
        }
        ++g_launches;
        if (fork) CU_TRY(cudaEventRecord(dc->tjoin[si], dc->tside[si]));
        break;
      }
      case PH_COPY: {
        ProfScope ps(5, stream);
        for (auto& c : ph.copies)
          CU_TRY(cudaMemcpyAsync(c.first.first, c.first.second, c.second, cudaMemcpyDeviceToDevice, stream));
        break;
      }
      case PH_GEMM: {
        ProfScope ps(ph.gemm_kind, stream);
        CU_TRY(launch_umma_gemm(reinterpret_cast<const GemmJob*>(dbase + ph.dev_off),
                                reinterpret_cast<const TaskDesc*>(dbase + ph.tiles_off), ph.total, ph.max_tiles, P.cg,
                                dc->sms, dc->flags, ph.has_split, P.bn, stream));
        ++g_launches;
        break;
      }
      case PH_SIMT: {
        ProfScope ps(4, stream);
        CU_TRY(launch_simt_gemm(reinterpret_cast<const SimtJob*>(dbase + ph.dev_off), ph.njobs, ph.total,
                                dc->sms, P.dtype == NS_BF16, dc->flags, stream));
        ++g_launches;
        break;
      }
      case PH_CAST_IN:
      case PH_CAST_OUT: {
        if (ph.kind == PH_CAST_OUT && !joined) {  // after the side-stream cluster launch too
          CU_TRY(cudaStreamWaitEvent(stream, dc->ev_join, 0));
          joined = true;
        }
        if (ph.kind == PH_CAST_OUT)
          for (int i = 0; i < 4; ++i)
            if (!(tjoined >> i & 1u)) { CU_TRY(cudaStreamWaitEvent(stream, dc->tjoin[i], 0)); tjoined |= 1u << i; }
        ProfScope ps(5, stream);
        CU_TRY(launch_cast(reinterpret_cast<const CastJob*>(dbase + ph.dev_off), ph.njobs, ph.max_numel,
                           ph.kind == PH_CAST_IN, dc->sms, stream));
        ++g_launches;
        break;
      }
      case PH_SPLIT: {
        ProfScope ps(0, stream);  // part of the Gram step
        CU_TRY(launch_split_reduce(reinterpret_cast<const SplitJob*>(dbase + ph.dev_off), ph.njobs, ph.total_rows,
                                   dc->flags, stream));
        ++g_launches;
        break;
      }
      case PH_PRECOND: {
        ProfScope ps(1, stream);
        CU_TRY(launch_precondition(reinterpret_cast<const PrecondJob*>(dbase + ph.dev_off), ph.njobs,
                                   ph.total_rows, ph.total, ph.vec8, P.dtype == NS_BF16, P.barrier,
                                   dc->flags, ph.lane_rows ? 1 | ph.row_kinds : 0, stream));
        ++g_launches;
        break;
      }
    }
  }
  if (!joined) CU_TRY(cudaStreamWaitEvent(stream, dc->ev_join, 0));
  for (int i = 0; i < 4; ++i)
    if (!(tjoined >> i & 1u)) CU_TRY(cudaStreamWaitEvent(stream, dc->tjoin[i], 0));
  return NS_OK;
}

// Replay through a CUDA graph: from a plan's second use on, its launch sequence (all steps,
// PDL edges, the cluster launch's fork/join) is captured once on a private stream and then
// launched into the caller's stream as one graph -- one host call instead of 13-18 launches
// (the host cost of a small call drops from ~40-70 us to a graph launch).  Not used while
// the caller's stream is itself being captured (the launches go into the caller's graph),
// while per-launch profiling is on, or with TNS_NOGRAPH=1 (measurement knob); a capture
// that fails leaves the plan on direct launches.
static bool graphs_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TNS_NOGRAPH");
    v = (e && atoi(e)) ? 0 : 1;
  }
  return v == 1;
}

static void capture_plan(Plan& P, DevCtx* dc) {
  if (!dc->cap && cudaStreamCreateWithFlags(&dc->cap, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    P.graph_failed = true;
    return;
  }
  const uint64_t l0 = g_launches;
  cudaGraph_t g = nullptr;
  ns_status st = NS_OK;
  cudaError_t e = cudaStreamBeginCapture(dc->cap, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    st = enqueue_plan(P, dc, dc->cap);
    e = cudaStreamEndCapture(dc->cap, &g);  // ends the capture even if the enqueue failed
  }
  const uint64_t n = g_launches - l0;
  g_launches = l0;  // nothing ran
  if (e == cudaSuccess && st == NS_OK && g) e = cudaGraphInstantiate(&P.gexec, g, 0);
  if (g) cudaGraphDestroy(g);
  if (e != cudaSuccess || st != NS_OK || !P.gexec) {
    cudaGetLastError();
    if (P.gexec) cudaGraphExecDestroy(P.gexec);
    P.gexec = nullptr;
    P.graph_failed = true;
    return;
  }
  P.glaunches = n;
}

static ns_status launch_plan(Plan& P, DevCtx* dc, cudaStream_t stream) {
  bool graph = graphs_enabled() && !g_prof && !P.graph_failed;
  if (graph) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess) {
      cudaGetLastError();
      graph = false;
    } else if (cs != cudaStreamCaptureStatusNone) {
      graph = false;
    }
  }
  // the plan's workspace is shared by every call with this problem list: a call on another
  // stream than the previous one waits for that call's last launch (not while `stream` is
  // being captured -- the caller's graph then owns the ordering)
  if (P.last && P.last_stream != stream) {
    cudaStreamCaptureStatus cs0 = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cs0) == cudaSuccess && cs0 == cudaStreamCaptureStatusNone)
      CU_TRY(cudaStreamWaitEvent(stream, P.last, 0));
    cudaGetLastError();
  }
  if (graph && !P.gexec && P.uses >= 1) capture_plan(P, dc);
  ++P.uses;
  ns_status st = NS_OK;
  if (graph && P.gexec) {
    CU_TRY(cudaGraphLaunch(P.gexec, stream));
    g_launches += P.glaunches;
  } else {
    st = enqueue_plan(P, dc, stream);
  }
  // last use, for the stream-ordered release of the plan's memory on eviction (not while
  // the caller captures `stream`: its graph then owns the ordering)
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (st == NS_OK && cudaStreamIsCapturing(stream, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone) {
    if (!P.last && cudaEventCreateWithFlags(&P.last, cudaEventDisableTiming) != cudaSuccess) P.last = nullptr;
    if (P.last) {
      CU_TRY(cudaEventRecord(P.last, stream));
      P.last_stream = stream;
    }
  }
  cudaGetLastError();
  return st;
}

// ---------------------------------------------------------------------------- validation
static ns_status validate_common(int64_t count, int iters, const float* coeffs, ns_precond precond,
                                 ns_dtype dtype) {
  if (count < 1) return fail(NS_ERR_INVALID_VALUE, "count/batch must be >= 1");
  if (iters < 1 || iters > 64) return fail(NS_ERR_INVALID_VALUE, "iters must be in [1, 64]");
  if (!coeffs) return fail(NS_ERR_INVALID_VALUE, "coeffs is NULL");
  for (int i = 0; i < 3 * iters; ++i)
    if (!std::isfinite(coeffs[i])) return fail(NS_ERR_INVALID_VALUE, "non-finite coefficient");
  if (precond != NS_PRECOND_NONE && precond != NS_PRECOND_FROBENIUS && precond != NS_PRECOND_AOL)
    return fail(NS_ERR_INVALID_VALUE, "bad precond");
  if (dtype != NS_BF16 && dtype != NS_FP32) return fail(NS_ERR_INVALID_VALUE, "bad dtype");
  return NS_OK;
}

static ns_status validate_mat(const void* x, int64_t m, int64_t n, ns_dtype dtype) {
  if (!x) return fail(NS_ERR_INVALID_VALUE, "NULL matrix pointer");
  if (m < 1 || n < 1) return fail(NS_ERR_INVALID_VALUE, "m and n must be >= 1");
  if (m > ((int64_t)1 << 30) || n > ((int64_t)1 << 30) || m * n > ((int64_t)1 << 40))
    return fail(NS_ERR_INVALID_VALUE, "matrix too large");
  if (reinterpret_cast<uintptr_t>(x) % elem_size(dtype))
    return fail(NS_ERR_NOT_SUPPORTED, "matrix pointer not aligned to its element size");
  return NS_OK;
}

// Tile words pack the job index and p0/128, q0/bn in 20 bits each (jobs.h pack_tile): a
// tcgen05 matrix needs M < 2^27 rows and a call fewer than 2^20 matrices.
static const int64_t kMaxTmaRows = (int64_t)1 << 27;
static const int64_t kMaxJobs = (int64_t)1 << 20;

// Does matrix `mt` take the cluster-resident whole-NS kernel?  Path 0 routes by measured
// cost (tools/cl_sizes.py, profiles/r01_v12_cluster_routing.log): the bf16 step engine of a
// lone small matrix costs ~63 us (13 launches, graph replay), the cluster kernel grows with
// its FMA work M*N^2 (64x216: 43 us, 128^2: 64 us, 64x576: 79 us) -- so bf16 matrices take
// it up to M*N^2 = 2.2e6; fp32 always (the SIMT step kernels are slower).  Path 5 takes it
// whenever the matrix fits.  Shape-only: batching never changes a result.
static bool to_cluster(const Mat& mt, ns_dtype dtype, bool any_peer, int cc_major) {
  const bool use_cluster = (g_path == 0 || g_path == 5) && !any_peer && cc_major == 10;
  if (!use_cluster || !cl_fits(mt.M, mt.N)) return false;
  return g_path == 5 || dtype != NS_BF16 || (double)mt.M * (double)mt.N * (double)mt.N <= 2.2e6;
}

static bool tma_ok_call(const Mat& mt, ns_dtype dtype, bool cast);

// Does matrix `mt` take the cluster-resident tcgen05 whole-NS kernel (cluster_tc.cu)?  Paths 0
// and 5: bf16 matrices with short side N <= 128 (padded to 128) whose slabs fit 16 CTAs (M <=
// 4096) and that TMA can address -- measured faster than both the step engine and the FFMA
// cluster kernel (graph replay, profiles/r02_cluster_tc.log: 1024x128 43 vs 79 us, 64x576 43
// vs 64, 128^2 43 vs 60 / 66; round-2 third pass: 37-39 us).  For 128 < N <= 256 (padded to
// 256) the kernel now beats the step engine on lone matrices (256x2304 82 vs 91 us, 768x256 76
// vs 78, 3072x192 86 vs 88; 256x576 77 vs 76) but holds 16 SMs per matrix for the whole call,
// so a batch of such matrices runs in waves (64 x 256x2304 ~7 waves) where the step engine
// shares tiles across the GPU; routing is per shape (batching never changes a result), so only
// path 7 sends N > 128 here (the CIFAR set: 86 us on path 7, 104 on path 0); path 4 sends none.
// Shape-only (plus TMA alignment, as for the step engine): batching never changes a result.
static bool to_tc(const Mat& mt, ns_dtype dtype, bool any_peer, int cc_major, bool cast) {
  if (dtype != NS_BF16 || any_peer || cc_major != 10) return false;
  if (!(g_path == 0 || g_path == 5 || g_path == 7)) return false;
  if (!tc_fits(mt.M, mt.N) || !tma_ok_call(mt, dtype, cast)) return false;
  return g_path == 7 || mt.N <= 128;
}

static bool tma_ok_call(const Mat& mt, ns_dtype dtype, bool cast) {
  Mat chk = mt;  // mixed precision: the step engine reads the 256-byte aligned staging copy
  if (cast) chk.x = chk.out = reinterpret_cast<void*>(256);
  if (!tma_ok(chk, dtype) || chk.M >= kMaxTmaRows) return false;
  for (void* pp : mt.peer)
    if (reinterpret_cast<uintptr_t>(pp) & 15) return false;
  return true;
}

// A call's matrices as plans.  A bf16 list that mixes TMA-addressable matrices with step-
// engine matrices TMA cannot address (a row pitch that is not a multiple of 16 bytes) runs as
// two plans on the stream: the unaligned ones on the CUDA-core step kernels, the rest on the
// tcgen05 engine (and the cluster kernel) -- so one unaligned matrix neither slows the others
// down nor changes their results (batching stays invisible).  Matrices that take the cluster
// kernel stay with the aligned group, whatever their pitch (the cluster kernel reads any
// layout), so they keep running beside the tcgen05 launches.
static void group_mats(const std::vector<Mat>& mats, ns_dtype dtype, bool cast, int cc_major,
                       std::vector<std::vector<Mat>>& groups) {
  groups.clear();
  if (dtype == NS_BF16 && g_path != 1 && mats.size() > 1) {
    bool any_peer = false;
    for (const Mat& mt : mats) any_peer = any_peer || !mt.peer.empty();
    std::vector<Mat> aligned, unaligned;
    for (const Mat& mt : mats) {
      const bool un = !to_cluster(mt, dtype, any_peer, cc_major) && !tma_ok_call(mt, dtype, cast);
      (un ? unaligned : aligned).push_back(mt);
    }
    if (!aligned.empty() && !unaligned.empty()) {
      groups.push_back(std::move(unaligned));
      groups.push_back(std::move(aligned));
      return;
    }
  }
  groups.push_back(mats);
}

// Find the cached plan of this problem list, or build it (workspace and tables allocated and
// uploaded stream-ordered on `stream`).  The plan comes back pinned: it cannot be evicted
// until unpinned, so a call can resolve all its plans before launching any.
static ns_status resolve_plan(const std::vector<Mat>& mats_in, int iters, const float* coeffs, ns_precond precond,
                              ns_dtype dtype, cudaStream_t stream, bool cast, DevCtx* dc, Plan** out) {
  std::vector<Mat> tiny, tcs, big;
  bool any_peer = false;
  for (const Mat& mt : mats_in) any_peer = any_peer || !mt.peer.empty();
  for (const Mat& mt : mats_in) {
    // path 5 keeps every matrix the FFMA cluster kernel fits there (its tests); otherwise the
    // tcgen05 cluster kernel first, then the FFMA one (fp32, TMA-unaligned small bf16)
    if (g_path == 5 && to_cluster(mt, dtype, any_peer, dc->cc_major)) tiny.push_back(mt);
    else if (to_tc(mt, dtype, any_peer, dc->cc_major, cast)) tcs.push_back(mt);
    else if (to_cluster(mt, dtype, any_peer, dc->cc_major)) tiny.push_back(mt);
    else big.push_back(mt);
  }
  bool simt = (g_path == 1) || dtype != NS_BF16 || dc->cc_major != 10;
  bool peers = false;
  for (const Mat& mt : big) {
    simt = simt || !tma_ok_call(mt, dtype, cast);
    peers = peers || !mt.peer.empty();
  }
  if (peers && simt)
    return fail(NS_ERR_NOT_SUPPORTED, "fused peer stores need the bf16 tcgen05 path (aligned shapes/pointers)");
  int dev = 0;
  CU_TRY(cudaGetDevice(&dev));
  // plan key: device, routing, coefficients, and per matrix the buffers and shape
  std::vector<uint64_t> key;
  key.reserve(mats_in.size() * 5 + 8 + 3 * iters);
  const int cg = (g_path == 2) ? 1 : 2;
  key.push_back((uint64_t)dev); key.push_back((uint64_t)dtype); key.push_back(simt ? 1 : 0);
  key.push_back(cast ? 1 : 0);
  key.push_back((uint64_t)cg);
  key.push_back((uint64_t)g_path);
  key.push_back((uint64_t)iters); key.push_back((uint64_t)precond);
  for (int i = 0; i < 3 * iters; ++i) { uint32_t u; std::memcpy(&u, &coeffs[i], 4); key.push_back(u); }
  key.push_back((uint64_t)tiny.size());
  key.push_back((uint64_t)tcs.size());
  for (const Mat& mt : mats_in) {
    key.push_back(reinterpret_cast<uint64_t>(mt.x)); key.push_back(reinterpret_cast<uint64_t>(mt.out));
    key.push_back((uint64_t)mt.m); key.push_back((uint64_t)mt.n);
    key.push_back((uint64_t)mt.peer.size());
    for (void* pp : mt.peer) key.push_back(reinterpret_cast<uint64_t>(pp));
  }
  auto it = g_plans.find(key);
  Plan* P = nullptr;
  if (it == g_plans.end()) {
    // Evict least-recently-used plans while the cache is full by count or would hold more
    // workspace than max(4 GiB, 2 x this list's): a caller that passes new buffers every step
    // (fresh pointers, fresh plans) must not accumulate workspaces.  Eviction releases the
    // victim's memory stream-ordered after its last launch (Plan::~Plan): no host sync.
    std::vector<Mat> sized(big);
    sized.insert(sized.end(), tcs.begin(), tcs.end());
    const size_t need = workspace_bytes_for(sized, dtype);
    const size_t budget = std::max<size_t>((size_t)4 << 30, 2 * need);
    auto held = [&]() {
      size_t b = 0;
      for (auto& kv : g_plans) if (!kv.second->ws_borrowed) b += kv.second->ws_bytes;
      return b;
    };
    while (g_plans.size() >= kMaxPlans || held() + need > budget) {
      auto victim = g_plans.end();
      for (auto jt = g_plans.begin(); jt != g_plans.end(); ++jt)
        if (!jt->second->pinned && (victim == g_plans.end() || jt->second->last_use < victim->second->last_use))
          victim = jt;
      if (victim == g_plans.end()) break;
      g_plans.erase(victim);
    }
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CU_TRY(cudaStreamIsCapturing(stream, &cs));
    if (cs != cudaStreamCaptureStatusNone)
      return fail(NS_ERR_NOT_SUPPORTED, "the first call of a problem list builds its plan (device allocations, "
                                        "table upload) and cannot be stream-captured: call it once uncaptured");
    std::unique_ptr<Plan> np(new Plan());
    np->device = dev; np->dtype = dtype; np->simt = simt; np->cg = cg; np->iters = iters; np->precond = precond;
    np->cast = cast;
    np->mats = big;
    np->tiny = tiny;
    np->tc = tcs;
    HostTables H;
    ns_status st = build_plan(*np, H, dc, coeffs, stream);
    if (st != NS_OK) {
      // nothing was launched; the partly built plan's memory goes back stream-ordered, after
      // the memset / upload already enqueued on `stream`
      if (np->ws_borrowed && np->ws)
        g_uws[dev & 63].used = (size_t)(reinterpret_cast<uint8_t*>(np->ws) - g_uws[dev & 63].base);
      if (cudaEventCreateWithFlags(&np->last, cudaEventDisableTiming) == cudaSuccess) cudaEventRecord(np->last, stream);
      cudaGetLastError();
      return st;
    }
    P = np.get();
    g_plans[key] = std::move(np);
  } else {
    P = it->second.get();
  }
  P->pinned = true;
  P->last_use = ++g_tick;
  *out = P;
  return NS_OK;
}

// One call: resolve (find or build) every plan of the call first, then launch them in order,
// so a failure while building the second plan leaves nothing enqueued and no caller memory
// touched (the header's error contract).
static ns_status run(const std::vector<Mat>& mats_in, int iters, const float* coeffs, ns_precond precond,
                     ns_dtype dtype, cudaStream_t stream, bool cast = false) {
  if ((int64_t)mats_in.size() >= kMaxJobs)
    return fail(NS_ERR_NOT_SUPPORTED, "more than 2^20 - 1 matrices in one call");
  DevCtx* dc = nullptr;
  ns_status st = dev_ctx(&dc);
  if (st != NS_OK) return st;
  std::vector<std::vector<Mat>> groups;
  group_mats(mats_in, dtype, cast, dc->cc_major, groups);
  std::vector<Plan*> plans;
  for (const auto& g : groups) {
    Plan* P = nullptr;
    st = resolve_plan(g, iters, coeffs, precond, dtype, stream, cast, dc, &P);
    if (st != NS_OK) break;
    plans.push_back(P);
  }
  if (st == NS_OK)
    for (Plan* P : plans)
      if ((st = launch_plan(*P, dc, stream)) != NS_OK) break;
  for (Plan* P : plans) P->pinned = false;
  return st;
}

static Mat make_mat(void* x, void* out, int64_t m, int64_t n, int iters) {
  Mat mt{};
  mt.x = x; mt.out = out ? out : x; mt.m = m; mt.n = n;
  mt.wide = m < n;
  mt.M = mt.wide ? n : m;
  mt.N = mt.wide ? m : n;
  mt.copy_in = (mt.out == mt.x) && (iters % 2 == 1);
  return mt;
}

}  // namespace tns

using namespace tns;

extern "C" {

int ns_abi_version(void) { return NS_ABI_VERSION; }

const char* ns_status_string(ns_status s) {
  switch (s) {
    case NS_OK: return "NS_OK";
    case NS_ERR_INVALID_VALUE: return "NS_ERR_INVALID_VALUE";
    case NS_ERR_NOT_SUPPORTED: return "NS_ERR_NOT_SUPPORTED";
    case NS_ERR_WORKSPACE: return "NS_ERR_WORKSPACE";
    case NS_ERR_CUDA: return "NS_ERR_CUDA";
  }
  return "NS_ERR_UNKNOWN";
}

const char* ns_last_error(void) { return g_err.c_str(); }

uint64_t ns_launch_count(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  return g_launches;
}

void ns_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_prof = on != 0;
}

ns_status ns_profile_read(double* ms, uint64_t* counts, int nkinds) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!ms || !counts || nkinds < 1 || nkinds > 8) return fail(NS_ERR_INVALID_VALUE, "bad arguments");
  for (int k = 0; k < nkinds; ++k) { ms[k] = 0.0; counts[k] = 0; }
  if (!g_prof_recs.empty()) CU_TRY(cudaEventSynchronize(g_prof_recs.back().b));
  for (const ProfRec& r : g_prof_recs) {
    float t = 0.f;
    CU_TRY(cudaEventElapsedTime(&t, r.a, r.b));
    if (r.kind < nkinds) { ms[r.kind] += t; counts[r.kind] += 1; }
    g_ev_pool.push_back(r.a);
    g_ev_pool.push_back(r.b);
  }
  g_prof_recs.clear();
  return NS_OK;
}

ns_status nsx_epilogue_counters(uint64_t* out8, int reset) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!out8) return fail(NS_ERR_INVALID_VALUE, "NULL");
  CU_TRY(cudaDeviceSynchronize());
  const char* dbg = getenv("TNS_DBG");
  if (dbg && (atoi(dbg) & 128)) {  // cluster-kernel timeline: 7 phase marks averaged per launch + count
    unsigned long long t[9];
    CU_TRY(cluster_timeline(t, reset != 0));
    const unsigned long long n = t[8] ? t[8] : 1;
    for (int i = 0; i < 7; ++i) out8[i] = t[i] / n;
    out8[7] = t[8];
    return NS_OK;
  }
  CU_TRY(umma_epi_prof(reinterpret_cast<unsigned long long*>(out8), reset != 0));
  return NS_OK;
}

int ns_set_path(int path) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (path != 0 && path != 1 && path != 2 && path != 4 && path != 5 && path != 7) return -1;
  int old = g_path;
  g_path = path;
  return old;
}

ns_status ns_orthogonalize(void* X, int64_t m, int64_t n, int64_t batch, int iters, const float* coeffs,
                           ns_precond precond, ns_dtype dtype, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  ns_status st = validate_common(batch, iters, coeffs, precond, dtype);
  if (st != NS_OK) return st;
  if ((st = validate_mat(X, m, n, dtype)) != NS_OK) return st;
  std::vector<Mat> mats;
  const size_t stride = (size_t)m * n * elem_size(dtype);
  for (int64_t i = 0; i < batch; ++i) {
    void* xi = reinterpret_cast<uint8_t*>(X) + i * stride;
    mats.push_back(make_mat(xi, xi, m, n, iters));
  }
  return run(mats, iters, coeffs, precond, dtype, reinterpret_cast<cudaStream_t>(stream));
}

ns_status ns_orthogonalize_cast(const void* const* X, void* const* out, const int64_t* m, const int64_t* n,
                                int64_t count, int iters, const float* coeffs, ns_precond precond, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  ns_status st = validate_common(count, iters, coeffs, precond, NS_BF16);
  if (st != NS_OK) return st;
  if (!X || !m || !n) return fail(NS_ERR_INVALID_VALUE, "NULL array argument");
  std::vector<Mat> mats;
  for (int64_t i = 0; i < count; ++i) {
    void* x = const_cast<void*>(X[i]);
    if ((st = validate_mat(x, m[i], n[i], NS_FP32)) != NS_OK) return st;
    void* o = out ? out[i] : nullptr;
    if (o && (st = validate_mat(o, m[i], n[i], NS_FP32)) != NS_OK) return st;
    Mat mt = make_mat(x, o, m[i], n[i], iters);
    mt.copy_in = false;  // decided on the staging copy (build_plan)
    mats.push_back(mt);
  }
  return run(mats, iters, coeffs, precond, NS_BF16, reinterpret_cast<cudaStream_t>(stream), true);
}

ns_status ns_orthogonalize_batched(void* const* X, void* const* out, const int64_t* m, const int64_t* n,
                                   int64_t count, int iters, const float* coeffs, ns_precond precond,
                                   ns_dtype dtype, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  ns_status st = validate_common(count, iters, coeffs, precond, dtype);
  if (st != NS_OK) return st;
  if (!X || !m || !n) return fail(NS_ERR_INVALID_VALUE, "NULL array argument");
  std::vector<Mat> mats;
  for (int64_t i = 0; i < count; ++i) {
    if ((st = validate_mat(X[i], m[i], n[i], dtype)) != NS_OK) return st;
    void* o = out ? out[i] : nullptr;
    if (o && (st = validate_mat(o, m[i], n[i], dtype)) != NS_OK) return st;
    mats.push_back(make_mat(X[i], o, m[i], n[i], iters));
  }
  return run(mats, iters, coeffs, precond, dtype, reinterpret_cast<cudaStream_t>(stream));
}

ns_status ns_orthogonalize_peers(void* const* X, void* const* out, void* const* peer_out, int npeer,
                                 const int64_t* m, const int64_t* n, int64_t count, int iters,
                                 const float* coeffs, ns_precond precond, ns_dtype dtype, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  ns_status st = validate_common(count, iters, coeffs, precond, dtype);
  if (st != NS_OK) return st;
  if (!X || !m || !n) return fail(NS_ERR_INVALID_VALUE, "NULL array argument");
  if (npeer < 0 || npeer > 64 || (npeer > 0 && !peer_out)) return fail(NS_ERR_INVALID_VALUE, "bad npeer/peer_out");
  if (dtype != NS_BF16) return fail(NS_ERR_NOT_SUPPORTED, "fused peer stores are bf16 only");
  std::vector<Mat> mats;
  for (int64_t i = 0; i < count; ++i) {
    if ((st = validate_mat(X[i], m[i], n[i], dtype)) != NS_OK) return st;
    void* o = out ? out[i] : nullptr;
    if (o && (st = validate_mat(o, m[i], n[i], dtype)) != NS_OK) return st;
    Mat mt = make_mat(X[i], o, m[i], n[i], iters);
    for (int r = 0; r < npeer; ++r) {
      void* pp = peer_out[i * npeer + r];
      if ((st = validate_mat(pp, m[i], n[i], dtype)) != NS_OK) return st;
      mt.peer.push_back(pp);
    }
    mats.push_back(mt);
  }
  return run(mats, iters, coeffs, precond, dtype, reinterpret_cast<cudaStream_t>(stream));
}

// Muon step: cached device job tables, keyed by the pointer lists (allocated and uploaded
// stream-ordered; `last` = event after the table's last use).
struct MuonTab {
  int device = 0;
  void* d = nullptr;
  cudaEvent_t last = nullptr;
  ~MuonTab() {
    release_async(device, d, last);
    if (last) cudaEventDestroy(last);
  }
};
static std::map<std::vector<uint64_t>, std::unique_ptr<MuonTab>> g_muon_tabs;

// The Muon job tables are keyed by pointer lists; a caller with fresh buffers every step
// would add one per step: past 1024 tables, drop them all (stream-ordered release).
static void muon_tabs_trim() {
  if (g_muon_tabs.size() < 1024) return;
  g_muon_tabs.clear();
}

static ns_status muon_table(const std::vector<uint64_t>& key, const std::vector<MuonJob>& jobs, cudaStream_t s,
                            MuonTab** out) {
  auto it = g_muon_tabs.find(key);
  if (it != g_muon_tabs.end()) { *out = it->second.get(); return NS_OK; }
  muon_tabs_trim();
  std::unique_ptr<MuonTab> t(new MuonTab());
  CU_TRY(cudaGetDevice(&t->device));
  const size_t bytes = jobs.size() * sizeof(MuonJob);
  if (cudaMallocAsync(&t->d, bytes, s) != cudaSuccess) {
    cudaGetLastError();
    t->d = nullptr;
    return fail(NS_ERR_WORKSPACE, "Muon job-table cudaMallocAsync failed");
  }
  CU_TRY(cudaMemcpyAsync(t->d, jobs.data(), bytes, cudaMemcpyHostToDevice, s));
  CU_TRY(cudaEventCreateWithFlags(&t->last, cudaEventDisableTiming));
  *out = t.get();
  g_muon_tabs[key] = std::move(t);
  return NS_OK;
}
static void muon_table_used(MuonTab* t, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone) cudaEventRecord(t->last, s);
  cudaGetLastError();
}

ns_status ns_muon_step(void* const* W, const void* const* G, float* const* M, void* const* U,
                       const int64_t* m, const int64_t* n, int64_t count, ns_dtype w_dtype, ns_dtype g_dtype,
                       float lr, float beta, float weight_decay, float grad_scale, int nesterov, int iters,
                       const float* coeffs, ns_precond precond, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  ns_status st = validate_common(count, iters, coeffs, precond, NS_BF16);
  if (st != NS_OK) return st;
  if (!W || !G || !M || !U || !m || !n) return fail(NS_ERR_INVALID_VALUE, "NULL array argument");
  if ((w_dtype != NS_BF16 && w_dtype != NS_FP32) || (g_dtype != NS_BF16 && g_dtype != NS_FP32))
    return fail(NS_ERR_INVALID_VALUE, "bad dtype");
  if (!std::isfinite(lr) || !std::isfinite(beta) || !std::isfinite(weight_decay) || !std::isfinite(grad_scale) ||
      beta < 0.f || beta >= 1.f)
    return fail(NS_ERR_INVALID_VALUE, "lr / beta / weight_decay / grad_scale out of range");
  std::vector<Mat> mats;
  std::vector<MuonJob> jobs;
  std::vector<uint64_t> key;
  int64_t max_numel = 0;
  for (int64_t i = 0; i < count; ++i) {
    if ((st = validate_mat(U[i], m[i], n[i], NS_BF16)) != NS_OK) return st;
    if ((st = validate_mat(W[i], m[i], n[i], w_dtype)) != NS_OK) return st;
    if ((st = validate_mat(G[i], m[i], n[i], g_dtype)) != NS_OK) return st;
    if ((st = validate_mat(M[i], m[i], n[i], NS_FP32)) != NS_OK) return st;
    mats.push_back(make_mat(U[i], U[i], m[i], n[i], iters));
    MuonJob J;
    J.M = M[i]; J.G = G[i]; J.U = U[i]; J.W = W[i];
    J.numel = m[i] * n[i];
    J.scale = (float)std::sqrt(std::max(1.0, (double)m[i] / (double)n[i]));
    jobs.push_back(J);
    max_numel = std::max(max_numel, J.numel);
    for (const void* p : {(const void*)W[i], G[i], (const void*)M[i], (const void*)U[i]})
      key.push_back(reinterpret_cast<uint64_t>(p));
    key.push_back((uint64_t)m[i]); key.push_back((uint64_t)n[i]);
  }
  if (count > 65535) return fail(NS_ERR_NOT_SUPPORTED, "more than 65535 matrices in one Muon step");
  DevCtx* dc = nullptr;
  if ((st = dev_ctx(&dc)) != NS_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  MuonTab* tab = nullptr;
  if ((st = muon_table(key, jobs, s, &tab)) != NS_OK) return st;
  const MuonJob* dtab = reinterpret_cast<const MuonJob*>(tab->d);
  CU_TRY(launch_muon_momentum(dtab, (int)count, max_numel, g_dtype == NS_BF16, beta, grad_scale, nesterov, dc->sms, s));
  ++g_launches;
  st = run(mats, iters, coeffs, precond, NS_BF16, s);
  if (st == NS_OK) {
    CU_TRY(launch_muon_apply(dtab, (int)count, max_numel, w_dtype == NS_BF16, lr, weight_decay, dc->sms, s));
    ++g_launches;
  }
  muon_table_used(tab, s);
  return st;
}

ns_status ns_muon_apply(void* const* W, const void* const* U, const int64_t* m, const int64_t* n, int64_t count,
                        ns_dtype w_dtype, float lr, float weight_decay, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (count < 1) return fail(NS_ERR_INVALID_VALUE, "count must be >= 1");
  if (count > 65535) return fail(NS_ERR_NOT_SUPPORTED, "more than 65535 matrices in one call");
  if (!W || !U || !m || !n) return fail(NS_ERR_INVALID_VALUE, "NULL array argument");
  if (w_dtype != NS_BF16 && w_dtype != NS_FP32) return fail(NS_ERR_INVALID_VALUE, "bad dtype");
  if (!std::isfinite(lr) || !std::isfinite(weight_decay)) return fail(NS_ERR_INVALID_VALUE, "lr / weight_decay not finite");
  ns_status st;
  std::vector<MuonJob> jobs;
  std::vector<uint64_t> key{0xA991ull};  // distinct from the ns_muon_step tables
  int64_t max_numel = 0;
  for (int64_t i = 0; i < count; ++i) {
    if ((st = validate_mat(U[i], m[i], n[i], NS_BF16)) != NS_OK) return st;
    if ((st = validate_mat(W[i], m[i], n[i], w_dtype)) != NS_OK) return st;
    MuonJob J;
    std::memset(&J, 0, sizeof(J));
    J.U = const_cast<void*>(U[i]); J.W = W[i];
    J.numel = m[i] * n[i];
    J.scale = (float)std::sqrt(std::max(1.0, (double)m[i] / (double)n[i]));
    jobs.push_back(J);
    max_numel = std::max(max_numel, J.numel);
    key.push_back(reinterpret_cast<uint64_t>(W[i])); key.push_back(reinterpret_cast<uint64_t>(U[i]));
    key.push_back((uint64_t)m[i]); key.push_back((uint64_t)n[i]);
  }
  DevCtx* dc = nullptr;
  if ((st = dev_ctx(&dc)) != NS_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  MuonTab* tab = nullptr;
  if ((st = muon_table(key, jobs, s, &tab)) != NS_OK) return st;
  CU_TRY(launch_muon_apply(reinterpret_cast<const MuonJob*>(tab->d), (int)count, max_numel, w_dtype == NS_BF16, lr,
                           weight_decay, dc->sms, s));
  ++g_launches;
  muon_table_used(tab, s);
  return NS_OK;
}

ns_status ns_workspace_size(const int64_t* m, const int64_t* n, int64_t count, int64_t batch, ns_dtype dtype,
                            size_t* bytes) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!m || !n || !bytes || count < 1 || batch < 1) return fail(NS_ERR_INVALID_VALUE, "bad arguments");
  if (dtype != NS_BF16 && dtype != NS_FP32) return fail(NS_ERR_INVALID_VALUE, "bad dtype");
  std::vector<Mat> mats;
  for (int64_t i = 0; i < count; ++i) {
    if (m[i] < 1 || n[i] < 1) return fail(NS_ERR_INVALID_VALUE, "m and n must be >= 1");
    for (int64_t b = 0; b < batch; ++b) mats.push_back(make_mat((void*)256, nullptr, m[i], n[i], 2));
  }
  // the same plan grouping as a call (group_mats), with every matrix counted as needing
  // workspace (cluster routing depends on the device): an upper bound for any device/path
  std::vector<std::vector<Mat>> groups;
  const int old = g_path;
  g_path = 4;  // no cluster routing: every matrix is counted in its step-engine group
  group_mats(mats, dtype, false, 10, groups);
  g_path = old;
  size_t total = 0;
  for (const auto& g : groups) total += workspace_bytes_for(g, dtype);
  *bytes = total;
  return NS_OK;
}

ns_status ns_set_workspace(void* ptr, size_t bytes, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (ptr && (bytes < 256 || (reinterpret_cast<uintptr_t>(ptr) & 255)))
    return fail(NS_ERR_INVALID_VALUE, "workspace must be >= 256 bytes and 256-byte aligned");
  int dev = 0;
  CU_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail(NS_ERR_NOT_SUPPORTED, "device index >= 64");
  DevCtx* dc = nullptr;
  ns_status st = dev_ctx(&dc);
  if (st != NS_OK) return st;
  // drop the cached plans that live in the previous caller buffer; their job tables are
  // released stream-ordered after their last launch, and work already enqueued keeps its
  // buffers (the caller keeps the old buffer alive until that work is done, or orders the
  // new buffer's first use after it on `stream`)
  for (auto it = g_plans.begin(); it != g_plans.end();) {
    if (it->second->ws_borrowed && it->second->device == dev) {
      if (it->second->last && stream) cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), it->second->last, 0);
      it = g_plans.erase(it);
    } else {
      ++it;
    }
  }
  cudaGetLastError();
  g_uws[dev] = UserWs{reinterpret_cast<uint8_t*>(ptr), ptr ? bytes : 0, 0};
  return NS_OK;
}

ns_status ns_read_flags(void* stream, uint32_t* flags) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!flags) return fail(NS_ERR_INVALID_VALUE, "flags is NULL");
  DevCtx* dc = nullptr;
  ns_status st = dev_ctx(&dc);
  if (st != NS_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  uint32_t h = 0;
  CU_TRY(cudaMemcpyAsync(&h, dc->flags, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  CU_TRY(cudaMemsetAsync(dc->flags, 0, sizeof(uint32_t), s));
  CU_TRY(cudaStreamSynchronize(s));
  *flags = h;
  return NS_OK;
}

void ns_shutdown(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  cudaDeviceSynchronize();
  g_plans.clear();
  g_muon_tabs.clear();
  cudaDeviceSynchronize();
  for (auto& d : g_dev) {
    if (d.init && d.flags) cudaFree(d.flags);
    if (d.init && d.side) cudaStreamDestroy(d.side);
    if (d.init && d.ev_fork) cudaEventDestroy(d.ev_fork);
    if (d.init && d.ev_join) cudaEventDestroy(d.ev_join);
    for (int i = 0; i < 4; ++i) {
      if (d.init && d.tside[i]) cudaStreamDestroy(d.tside[i]);
      if (d.init && d.tfork[i]) cudaEventDestroy(d.tfork[i]);
      if (d.init && d.tjoin[i]) cudaEventDestroy(d.tjoin[i]);
    }
    if (d.init && d.cap) cudaStreamDestroy(d.cap);
    if (d.init && d.freer) cudaStreamDestroy(d.freer);
    d = DevCtx();
  }
}

// ------------------------------------------------------------------------------ single steps
// These build a one-off job table, launch one kernel and synchronise (test entry points).
struct TDesc { const void* ptr; int rows, cols; };
static ns_status one_gemm(GemmJob J, TDesc ta, TDesc tb, TDesc tout, TDesc taux, SimtJob S, bool simt,
                          ns_dtype dtype, cudaStream_t stream, int64_t s_len = 0) {
  DevCtx* dc = nullptr;
  ns_status st = dev_ctx(&dc);
  if (st != NS_OK) return st;
  void* dmem = nullptr;
  if (!simt) {
    float* spad = nullptr;  // the tcgen05 epilogue reads s in whole tiles: pad with zeros
    if (J.s) {
      CU_TRY(cudaMalloc(&spad, s_floats(s_len) * 4));
      CU_TRY(cudaMemsetAsync(spad, 0, s_floats(s_len) * 4, stream));
      CU_TRY(cudaMemcpyAsync(spad, J.s, s_len * 4, cudaMemcpyDeviceToDevice, stream));
      J.s = spad;
    }
    struct FreeS { float* p; ~FreeS() { if (p) { cudaDeviceSynchronize(); cudaFree(p); } } } free_s{spad};
    std::vector<CUtensorMap> tm;
    int ia, ib, io, ix = -1;
    if ((st = encode_pair(tm, ta.ptr, ta.rows, ta.cols, &ia)) != NS_OK) return st;
    if ((st = encode_pair(tm, tb.ptr, tb.rows, tb.cols, &ib)) != NS_OK) return st;
    if ((st = encode_pair(tm, tout.ptr, tout.rows, tout.cols, &io)) != NS_OK) return st;
    if (taux.ptr && (st = encode_pair(tm, taux.ptr, taux.rows, taux.cols, &ix)) != NS_OK) return st;
    const int cg = g_path == 2 ? 1 : 2;
    std::vector<uint64_t> tl;
    umma_tile_list(J, 0, cg, 256, tl);
    std::vector<TaskDesc> tasks(tl.size());
    for (size_t i = 0; i < tl.size(); ++i) {
      std::memset(&tasks[i], 0, sizeof(TaskDesc));
      tasks[i].tile = tl[i]; tasks[i].kind = TK_TILE;
    }
    const size_t jo = tm.size() * sizeof(CUtensorMap), to = jo + align_up(sizeof(GemmJob), 64);
    const size_t bytes = to + tasks.size() * sizeof(TaskDesc);
    CU_TRY(cudaMalloc(&dmem, bytes));
    uint8_t* d = reinterpret_cast<uint8_t*>(dmem);
    J.tmA = d + ia * sizeof(CUtensorMap);
    J.tmB = d + ib * sizeof(CUtensorMap);
    J.tmOut = d + (io + 1) * sizeof(CUtensorMap);
    J.tmAux = ix >= 0 ? d + (ix + 1) * sizeof(CUtensorMap) : nullptr;
    std::vector<uint8_t> h(bytes);
    std::memcpy(h.data(), tm.data(), jo);
    std::memcpy(h.data() + jo, &J, sizeof(J));
    std::memcpy(h.data() + to, tasks.data(), tasks.size() * sizeof(TaskDesc));
    CU_TRY(cudaMemcpy(dmem, h.data(), bytes, cudaMemcpyHostToDevice));
    cudaError_t e = launch_umma_gemm(reinterpret_cast<const GemmJob*>(d + jo), reinterpret_cast<const TaskDesc*>(d + to),
                                     (int64_t)tasks.size(), (int64_t)tasks.size(), cg, dc->sms, dc->flags, false, 256,
                                     stream);
    ++g_launches;
    cudaError_t e2 = cudaStreamSynchronize(stream);
    cudaFree(dmem);
    if (e != cudaSuccess) return fail(NS_ERR_CUDA, std::string("umma launch: ") + cudaGetErrorString(e));
    if (e2 != cudaSuccess) return fail(NS_ERR_CUDA, std::string("umma exec: ") + cudaGetErrorString(e2));
  } else {
    CU_TRY(cudaMalloc(&dmem, sizeof(SimtJob)));
    CU_TRY(cudaMemcpy(dmem, &S, sizeof(S), cudaMemcpyHostToDevice));
    cudaError_t e = launch_simt_gemm(reinterpret_cast<const SimtJob*>(dmem), 1, S.tiles, dc->sms,
                                     dtype == NS_BF16, dc->flags, stream);
    ++g_launches;
    cudaError_t e2 = cudaStreamSynchronize(stream);
    cudaFree(dmem);
    if (e != cudaSuccess) return fail(NS_ERR_CUDA, std::string("simt launch: ") + cudaGetErrorString(e));
    if (e2 != cudaSuccess) return fail(NS_ERR_CUDA, std::string("simt exec: ") + cudaGetErrorString(e2));
  }
  return NS_OK;
}

static bool step_simt(ns_dtype dtype, int64_t m, int64_t n, std::initializer_list<const void*> ptrs) {
  DevCtx* dc = nullptr;
  if (dev_ctx(&dc) != NS_OK) return true;
  if (g_path == 1 || dtype != NS_BF16 || dc->cc_major != 10) return true;
  if (m % 8 || n % 8) return true;
  for (const void* p : ptrs)
    if (reinterpret_cast<uintptr_t>(p) & 15) return true;
  return false;
}

static void finish_tiles(GemmJob& J, SimtJob& S) {
  J.tiles_q = J.sym ? (J.P + kSymBlock - 1) / kSymBlock : (J.Q + kBN - 1) / kBN;
  S.tiles_q = (S.Q + kSimtTile - 1) / kSimtTile;
  S.tiles = ((S.P + kSimtTile - 1) / kSimtTile) * S.tiles_q;
}

ns_status nsx_gram(const void* X, int64_t m, int64_t n, void* A, float* part, ns_dtype dtype, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  ns_status st;
  if ((st = validate_mat(X, m, n, dtype)) != NS_OK) return st;
  if (!A) return fail(NS_ERR_INVALID_VALUE, "A is NULL");
  const bool wide = m < n;
  const int64_t M = wide ? n : m, N = wide ? m : n;
  GemmJob J; SimtJob S;
  std::memset(&J, 0, sizeof(J)); std::memset(&S, 0, sizeof(S));
  J.mode = S.mode = MODE_GRAM;
  J.sym = 1; J.P = J.Q = S.P = S.Q = (int)N; J.K = S.K = (int)M;
  J.a_mn = J.b_mn = wide ? 0 : 1;
  J.out = S.out = A; J.ld = S.ld = N;
  S.A = S.B = X;
  if (!wide) { S.sa_p = S.sb_q = 1; S.sa_k = S.sb_k = n; } else { S.sa_p = S.sb_q = n; S.sa_k = S.sb_k = 1; }
  finish_tiles(J, S);
  const bool simt = step_simt(dtype, m, n, {X, A});
  if (part) {  // AOL row-sum partials of the Gram epilogue (production layout, GemmJob::part)
    if (simt) return fail(NS_ERR_NOT_SUPPORTED, "Gram partials come from the tcgen05 epilogue (aligned bf16 only)");
    J.part = part; J.part_ld = part_ld_for(N);
  }
  return one_gemm(J, {X, (int)m, (int)n}, {X, (int)m, (int)n}, {A, (int)N, (int)N}, {nullptr, 0, 0}, S, simt, dtype,
                  reinterpret_cast<cudaStream_t>(stream));
}

ns_status nsx_poly(const void* A, int64_t N, float b, float c, const float* s, void* B, ns_dtype dtype,
                   void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  ns_status st;
  if ((st = validate_mat(A, N, N, dtype)) != NS_OK) return st;
  if (!B) return fail(NS_ERR_INVALID_VALUE, "B is NULL");
  GemmJob J; SimtJob S;
  std::memset(&J, 0, sizeof(J)); std::memset(&S, 0, sizeof(S));
  J.mode = S.mode = MODE_POLY;
  J.sym = 1; J.P = J.Q = J.K = S.P = S.Q = S.K = (int)N;
  J.out = S.out = B; J.aux = S.aux = A; J.ld = S.ld = N;
  J.s = S.s = s; J.b = S.b = b; J.c = S.c = c;
  S.A = S.B = A; S.sa_p = S.sb_q = N; S.sa_k = S.sb_k = 1;
  finish_tiles(J, S);
  const bool simt = step_simt(dtype, N, N, {A, B});
  return one_gemm(J, {A, (int)N, (int)N}, {A, (int)N, (int)N}, {B, (int)N, (int)N}, {A, (int)N, (int)N}, S, simt,
                  dtype, reinterpret_cast<cudaStream_t>(stream), N);
}

ns_status nsx_update(const void* X, int64_t m, int64_t n, const void* B, float a, const float* s, void* Out,
                     ns_dtype dtype, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  ns_status st;
  if ((st = validate_mat(X, m, n, dtype)) != NS_OK) return st;
  if (!B || !Out) return fail(NS_ERR_INVALID_VALUE, "B/Out is NULL");
  const bool wide = m < n;
  const int64_t M = wide ? n : m, N = wide ? m : n;
  GemmJob J; SimtJob S;
  std::memset(&J, 0, sizeof(J)); std::memset(&S, 0, sizeof(S));
  J.mode = S.mode = MODE_XB;
  J.sym = 0; J.K = S.K = (int)N;
  J.out = S.out = Out; J.aux = S.aux = X; J.ld = S.ld = n;
  J.s = S.s = s; J.a = S.a = a;
  int ta_r, ta_c, tb_r, tb_c; const void *ta, *tb;
  if (!wide) {
    J.a_mn = 0; J.b_mn = 0; J.P = S.P = (int)M; J.Q = S.Q = (int)N; J.s_by_row = S.s_by_row = 0;
    ta = X; ta_r = (int)m; ta_c = (int)n; tb = B; tb_r = (int)N; tb_c = (int)N;
    S.A = X; S.sa_p = n; S.sa_k = 1; S.B = B; S.sb_q = N; S.sb_k = 1;
  } else {
    J.a_mn = 0; J.b_mn = 1; J.P = S.P = (int)N; J.Q = S.Q = (int)M; J.s_by_row = S.s_by_row = 1;
    ta = B; ta_r = (int)N; ta_c = (int)N; tb = X; tb_r = (int)m; tb_c = (int)n;
    S.A = B; S.sa_p = N; S.sa_k = 1; S.B = X; S.sb_q = 1; S.sb_k = n;
  }
  finish_tiles(J, S);
  const bool simt = step_simt(dtype, m, n, {X, B, Out});
  return one_gemm(J, {ta, ta_r, ta_c}, {tb, tb_r, tb_c}, {Out, (int)m, (int)n}, {X, (int)m, (int)n}, S, simt, dtype,
                  reinterpret_cast<cudaStream_t>(stream), N);
}

ns_status nsx_precondition(void* A, int64_t N, ns_precond precond, const float* part, float* s, ns_dtype dtype,
                           void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  ns_status st;
  if ((st = validate_mat(A, N, N, dtype)) != NS_OK) return st;
  if (!s) return fail(NS_ERR_INVALID_VALUE, "s is NULL");
  if (precond != NS_PRECOND_FROBENIUS && precond != NS_PRECOND_AOL)
    return fail(NS_ERR_INVALID_VALUE, "precond must be FROBENIUS or AOL");
  DevCtx* dc = nullptr;
  if ((st = dev_ctx(&dc)) != NS_OK) return st;
  cudaStream_t strm = reinterpret_cast<cudaStream_t>(stream);
  const bool vec8 = dtype == NS_BF16 && N % 8 == 0 && !(reinterpret_cast<uintptr_t>(A) & 15);
  PrecondJob J;
  std::memset(&J, 0, sizeof(J));
  J.A = A; J.s = s; J.N = (int)N; J.precond = (int)precond;
  if (part) {
    if (precond != NS_PRECOND_AOL || dtype != NS_BF16)
      return fail(NS_ERR_INVALID_VALUE, "partials are AOL row sums of a bf16 Gram");
    J.part = part; J.part_ld = part_ld_for(N);
  }
  const bool lane_rows = part != nullptr;
  void* dmem = nullptr;
  CU_TRY(cudaMalloc(&dmem, 256 + sizeof(J)));
  CU_TRY(cudaMemset(dmem, 0, 256));  // grid-barrier words
  CU_TRY(cudaMemcpy(reinterpret_cast<uint8_t*>(dmem) + 256, &J, sizeof(J), cudaMemcpyHostToDevice));
  cudaError_t e = launch_precondition(reinterpret_cast<const PrecondJob*>(reinterpret_cast<uint8_t*>(dmem) + 256), 1,
                                      N, precond_segments((int)N, 0), vec8, dtype == NS_BF16,
                                      reinterpret_cast<unsigned*>(dmem), dc->flags,
                                      lane_rows ? 1 | precond_lane_kind(J.part_ld) : 0, strm);
  ++g_launches;
  cudaError_t e2 = cudaStreamSynchronize(strm);
  cudaFree(dmem);
  if (e != cudaSuccess) return fail(NS_ERR_CUDA, std::string("precond launch: ") + cudaGetErrorString(e));
  if (e2 != cudaSuccess) return fail(NS_ERR_CUDA, std::string("precond exec: ") + cudaGetErrorString(e2));
  return NS_OK;
}

}  // extern "C"
