// Work descriptors shared by the host planner (api.cu) and the kernels.
// One GemmJob = one matrix's share of one NS step launch; a launch walks a device
// array of jobs (grouped/batched launch).
#pragma once
#include <cstdint>

namespace tns {

enum GemmMode : int32_t {
  MODE_GRAM = 0,  // out = Xh^T Xh                          (Eq. 3 / Eq. 7)
  MODE_POLY = 1,  // out = (b aux + c acc) * s[col]         (Eq. 4; aux = A)
  MODE_XB = 2     // out = acc + a * aux * s[row|col]       (Eq. 5; aux = X_k)
};

// Tile geometry of the tcgen05 kernel (one CTA = one 128 x 256 output tile at a time).
constexpr int kBM = 128;  // UMMA M
constexpr int kBN = 256;  // UMMA N (default tile width; 128 for tile-starved plans)
constexpr int kBK = 64;   // K elements per pipeline stage = one 128-byte swizzle atom
constexpr int kSymBlock = 256;  // symmetric phases tile the lower triangle in 256 x 256 blocks
#ifndef TNS_GROUP_P
#define TNS_GROUP_P 16
#endif
constexpr int kGroupP = TNS_GROUP_P;  // XB raster: tiles grouped 16 row-blocks deep for L2 reuse

// One entry of a launch's tile list (built on the host in execution order):
//   bits [0,20) job index | [20,40) p0 / 128 | [40,60) q0 / bn | bit 63 mirrored store
// (bn = the launch's tile width, 256 or 128).
__host__ __device__ inline uint64_t pack_tile(uint32_t job, uint32_t p0, uint32_t q0, bool mirror, uint32_t bn = 256) {
  return (uint64_t)job | ((uint64_t)(p0 / 128) << 20) | ((uint64_t)(q0 / bn) << 40) |
         ((uint64_t)(mirror ? 1 : 0) << 63);
}

struct GemmJob {
  // Operand sources: D[p][q] = sum_k Aop[p][k] * Bop[q][k].
  const void* tmA;  // CUtensorMap (global memory) of the tensor holding Aop
  const void* tmB;  // CUtensorMap of the tensor holding Bop
  const void* tmOut;  // CUtensorMap of `out`, 32 x 32 boxes, 64-byte swizzle (epilogue stores)
  const void* tmAux;  // CUtensorMap of `aux`, 32 x 32 boxes, 64-byte swizzle (epilogue loads)
  int32_t a_mn;     // 1: Aop stored [k][p] (MN-major), 0: stored [p][k] (K-major)
  int32_t b_mn;
  int32_t mode;     // GemmMode
  int32_t sym;      // 1: lower-triangle 256-blocks, mirrored store (P == Q)
  int32_t P, Q, K;  // output rows/cols, contraction length
  int32_t tiles_q;  // number of 256-wide column tiles (rect jobs)
  int32_t tiles;    // tiles in this job
  int64_t tile_start;  // exclusive prefix over jobs of `tiles`
  void* out;           // output matrix, row-major, ld = ld
  const void* aux;     // POLY: A ; XB: X_k  (same [p][q] indexing, ld = ld)
  int64_t ld;
  const float* s;      // scaling vector or nullptr
  int32_t s_by_row;    // XB: scale a*aux by s[p] (1) or s[q] (0)
  float a, b, c;
  // GRAM with AOL (iteration 1): per-tile |A0| row-sum partials, written once each (no
  // atomics): part_ld slots per row -- [0, ceil(N/64)) direct 64-column blocks,
  // [ceil(N/64), + ceil(N/32)) mirrored 32-row blocks -- at part_at(); nullptr = not collected.
  float* part;
  int32_t part_ld;
  int32_t part_sm;  // 1: slot-major layout (see part_at)
  // XB of the last iteration, fused collective: also store every output tile into `npeer`
  // more destinations (peers' gather buffers over NVLink); tmPeer -> npeer consecutive
  // 32x32-box CUtensorMaps.
  const void* tmPeer;
  int32_t npeer;
  // Half-storage symmetric matrices: a_sym / b_sym = the operand is symmetric and stored
  // as its lower-triangle 256-blocks only (diagonal blocks whole); k-blocks in the upper
  // triangle are read transposed from the mirrored block (TMA coordinates swapped, UMMA
  // major bit flipped).  half = sym job stores only its lower-triangle tiles (no mirror).
  int32_t a_sym, b_sym, half;
  // POLY: added to diagonal elements before the column scaling, B' = bA + cA^2 + dI.  With
  // d = a_k the next XB needs no a*X term: X(aI + B) = aX + XB (Eq. 5 as one product).
  float diag_add;
  // Split-K GRAM (tile-starved launches, see SplitJob): the tile's fp32 partial over its
  // task's k-range goes to split_ws[(split - 1) * split_stride + p * split_ld + q], no epilogue.
  float* split_ws;
  int64_t split_stride;
  int32_t split_ld;
};

// CUDA-core (SIMT) variant of a GemmJob: operands by pointer + strides (elements),
// Aop[p][k] = A[p*sa_p + k*sa_k], Bop[q][k] = B[q*sb_q + k*sb_k].  Full (non-triangular)
// 64 x 64 tiles.  Used for the fp32 "exact" mode and for bf16 shapes TMA cannot address.
struct SimtJob {
  const void* A;
  const void* B;
  int64_t sa_p, sa_k, sb_q, sb_k;
  int32_t mode;
  int32_t P, Q, K;
  int32_t tiles_q;
  int32_t tiles;
  int64_t tile_start;
  void* out;
  const void* aux;
  int64_t ld;
  const float* s;
  int32_t s_by_row;
  float a, b, c;
};
constexpr int kSimtTile = 64;

// One matrix of a storage cast (muon.cu cast_kernel): fp32 -> bf16 (round to nearest even)
// before a mixed-precision call, bf16 -> fp32 after it.
struct CastJob {
  const void* src;
  void* dst;
  int64_t numel;
};

// Per-matrix descriptor for the preconditioning kernel (AOL / Frobenius).
// AOL rows with at most this many Gram-epilogue partial slots (N <= 1344) are summed by
// one lane in slot order; longer ones by four lanes or a warp (precond_rows.cuh
// kQuarterPartials).
constexpr int kSeqPartials = 64;
constexpr int kQuarterPartials = 256;  // four lanes per row up to here, a warp per row beyond
// Layout of a plan's partials (part_at): slot-major where the rows are summed by one or four
// lanes (consecutive rows in consecutive lanes), row-major for the warp-per-row sums.
__host__ __device__ inline int precond_part_sm(int part_ld) { return part_ld <= kQuarterPartials ? 1 : 0; }
// Slot t of row i of an N-row partial array: row-major part[i * part_ld + t], or slot-major
// part[t * N + i] (sm = 1: the plans' layout when part_ld <= kSeqPartials -- then the
// preconditioner reads one row per lane, and consecutive lanes read consecutive floats; the
// Gram epilogue's stores of a slot are coalesced the same way).  The single-step entry points
// (nsx_gram / nsx_precondition) keep row-major.
__host__ __device__ inline int64_t part_at(int part_ld, int sm, int N, int i, int t) {
  return sm ? (int64_t)t * N + i : (int64_t)i * part_ld + t;
}
struct PrecondJob {
  void* A;          // N x N symmetric Gram, in place -> A1
  float* s;         // N
  const float* part;  // row-sum partials from the Gram epilogue (GemmJob::part) or nullptr
  int32_t part_ld;
  int32_t part_sm;    // layout of part (part_at)
  int32_t half;       // A stored as lower-triangle 256-blocks: rescale only those
  int32_t N;
  int32_t precond;  // 1 Frobenius, 2 AOL
  int64_t row_start;  // prefix over jobs of N (phase 1: one warp per row)
  int64_t seg_start;  // prefix over jobs of precond_segments(N, half) (phase 2: one warp per segment)
};
// Phase-2 work units of one matrix (precond_rows.cuh): stored rows cut into 256-column
// segments; with half storage row i (in 256-block bi) holds columns [0, min(N, 256 (bi + 1))).
__host__ __device__ inline int64_t precond_segments(int N, int half) {
  const int64_t nb = (N + 255) / 256;
  if (!half) return (int64_t)N * nb;
  // full blocks 0..nb-2 have 256 rows of bi + 1 segments; the last block N - 256 (nb - 1) rows
  return 256 * (nb - 1) * nb / 2 + (int64_t)(N - 256 * (nb - 1)) * nb;
}


// One matrix of a Muon optimizer step (muon.cu).
struct MuonJob {
  float* M;        // momentum, fp32, numel
  const void* G;   // gradient (fp32 or bf16)
  void* U;         // bf16 staging: NS input, orthogonalised in place
  void* W;         // weight (fp32 or bf16)
  int64_t numel;
  float scale;     // max(1, m/n)^(1/2)
};

// One unit of work of a per-step launch (umma_gemm_kernel): a tile, or padding of the
// balanced per-worker task lists (api.cu balance_tasks).
enum TaskKind : uint32_t { TK_TILE = 0, TK_NONE = 3 };
enum StepKind : int32_t { PHK_GEMM = 0, PHK_PRE_S = 1, PHK_SPLIT = 2 };  // host-side step kinds (api.cu)
struct TaskDesc {
  uint64_t tile;        // TK_TILE: pack_tile(job, p0, q0, mirror)
  uint32_t kind;        // TaskKind
  uint32_t kb0, nkb;    // TK_TILE: k-blocks [kb0, kb0 + nkb) of the contraction (nkb = 0: all)
  uint32_t split;       // TK_TILE: 0, or 1 + index of this k-range's fp32 partial (split-K)
};

// Reduction of a split-K Gram (simt.cu): A = rnd(sum over s of ws[s]) in fixed order s = 0..S-1
// (deterministic), plus the AOL row sums of |A0| when part != nullptr (written to slot 0 of
// the row's part_ld slots; the others stay zero).  Only for N <= 256 (one symmetric block,
// stored whole).
struct SplitJob {
  const float* ws;
  int64_t stride;   // floats between consecutive partials
  int32_t ld;       // floats per partial row
  int32_t S, N;
  void* A;          // N x N, ld N, storage type of the plan
  float* part;
  int32_t part_ld;
  int32_t part_sm;    // layout of part (part_at)
  int64_t row_start;  // prefix over jobs of N (one warp per row)
};
constexpr int kSplitMaxN = 256;

// ------------------------------------------------------------------ cluster-resident NS
// Whole Newton-Schulz of one small matrix (short side N <= 128) inside one cluster of
// kClCtas CTAs (cluster_ns.cu).  Every CTA holds a full fp32 copy
// of Xh (M x N), A and B in shared memory; CTA r computes rows [r*Nr, r*Nr+Nr) of A and B
// and rows [r*Mr, r*Mr+Mr) of X_{k+1} and broadcasts them to its peers over DSMEM.
// Cluster size: 16 CTAs (non-portable) when every matrix of the launch fits the 16-CTA
// layout (half the rows per CTA: 128^2 fp32 82 -> 66 us), else the portable 8.
constexpr int kClCtas = 8;       // eligibility is decided with the 8-CTA layout
constexpr int kClCtasMax = 16;
#ifndef TNS_CL_THREADS
#define TNS_CL_THREADS 512
#endif
constexpr int kClThreads = TNS_CL_THREADS;
constexpr int kClMaxN = 128;
constexpr size_t kClMaxSmem = 227 * 1024;  // the sm_100 per-block maximum
constexpr int kClHdr = 64;                  // bytes before the float region (mbarriers)
struct ClusterJob {
  const void* x;  // input, caller layout (m x n row-major)
  void* out;      // output, caller layout (may equal x)
  float* xchg;    // cl_xchg_floats(M, N, C) floats of L2 scratch for the large row exchanges
  int32_t m, n, M, N, wide, pad;
};
struct ClLayout {
  int N4, Nr, Mr, ldx, lda;
  size_t offA, offB, offX, offXn, floats;  // in floats
};
__host__ __device__ inline ClLayout cl_layout(int M, int N, int C = kClCtas) {
  ClLayout L;
  L.N4 = (N + 3) & ~3;
  L.Nr = ((N + C - 1) / C + 3) & ~3;
  L.Mr = ((M + C - 1) / C + 3) & ~3;
  L.ldx = L.N4 + 4;  // X rows are also read with a row stride (XB): pad against bank conflicts
  L.lda = L.N4 + 4;  // A, B rows: padded too (the k-split lanes read 4 rows at once)
  size_t o = 0;
  L.offA = o; o += (size_t)L.N4 * L.lda;
  L.offB = o; o += (size_t)L.N4 * L.lda;
  L.offX = o; o += (size_t)C * L.Mr * L.ldx;
  L.offXn = o; o += (size_t)L.Mr * L.ldx;
  o += L.N4;  // s
  L.floats = o;
  return L;
}
// Row exchanges of the FFMA cluster kernel: a phase whose matrix (the rows every CTA must
// receive) has at least kClL2Bytes goes through an L2 buffer -- every CTA stores its rows once,
// cluster barrier, every CTA bulk-loads the whole matrix -- instead of one DSMEM bulk copy per
// peer (measured per SM: DSMEM ~13 B/cycle, L2 stores ~30, bulk L2 loads 55-65,
// tools/xfer_probe.cu); the small exchanges would lose the extra barrier + L2 round trip
// (64x27 bf16 33 -> 39 us all-L2), so only the large ones switch (graph replay, interleaved:
// 128^2 fp32 59.5 -> 58.6 us, 64x216 fp32 41.1 -> 39.2, 256x64 fp32 43.6 -> 41.0, small bf16
// unchanged).  Data movement only: the results are bitwise the same either way.
constexpr uint32_t kClL2Bytes = 32768;
__host__ __device__ inline size_t cl_xchg_floats(int M, int N, int C) {
  const ClLayout L = cl_layout(M, N, C);
  return 2 * (size_t)L.N4 * L.lda + (size_t)C * L.Mr * L.ldx;
}
__host__ __device__ inline bool cl_fits(int64_t M, int64_t N, int C = kClCtas) {
  return N >= 1 && N <= kClMaxN && M <= 4096 && cl_layout((int)M, (int)N, C).floats * 4 + kClHdr <= kClMaxSmem;
}

// ------------------------------------------------------------------ cluster-resident tcgen05 NS
// Whole Newton-Schulz of one mid-size bf16 matrix (short side N <= 256) in ONE launch of a
// C-CTA cluster (cluster_tc.cu): Xh in row slabs of R rows per CTA, N
// padded with zero columns to Np (128 or 256), A / B' copies in every CTA's shared memory.
// Gram all-reduce through an L2 scratch (`part`): each CTA's fp32 partial, lower-triangle
// 32 x 32 chunks only (tc_tri_chunks), then the bf16 A image (Np x Np, the shared-memory box
// layout) that the owners of its chunk ranges write and every CTA bulk-loads.  C is the
// smallest power of two (4..16) whose slabs fit -- a function of the shape alone, so a
// matrix's result never depends on the rest of its call; jobs are launched in groups of
// equal C.
constexpr int kTcCtas = 16;  // largest cluster (non-portable size)
constexpr size_t kTcMaxSmem = 227 * 1024;
struct TcJob {
  const void* tm_in;   // CUtensorMap (device) of the input X (m x n, 64 x 64 boxes, 128-byte swizzle)
  const void* tm_out;  // CUtensorMap of the output (may address the same buffer)
  float* part;         // tc_part_floats(Np, C) floats of scratch (partials, then the A image)
  int32_t m, n, M, N, wide, Np, R, C;
};
__host__ __device__ inline int tc_np(int64_t N) { return N <= 128 ? 128 : 256; }
// Lower-triangle 32 x 32 chunks (row block >= column block) of an Np x Np Gram partial.
__host__ __device__ inline int tc_tri_chunks(int Np) { return (Np / 32) * (Np / 32 + 1) / 2; }
__host__ __device__ inline size_t tc_part_floats(int Np, int C) {
  return (size_t)C * tc_tri_chunks(Np) * 1024 + (size_t)Np * Np / 2;
}
__host__ __device__ inline size_t tc_smem(int Np, int R, int /*C*/) {
  return (size_t)R * Np * 2 + (size_t)Np * Np * 2 + (size_t)Np * 4 + 64 + 1024;
}
// Slab rows per CTA for a C-CTA cluster: a multiple of 64, at least 128 (one M = 128 UMMA
// per update accumulator).
__host__ __device__ inline int tc_rows(int64_t M, int C) {
  const int64_t r = (M + C - 1) / C;
  const int64_t r64 = (r + 63) / 64 * 64;
  return (int)(r64 < 128 ? 128 : r64);
}
// Cluster size for an M x N matrix (0: does not fit): the smallest power of two C in 4..16
// that keeps the slabs at the minimum R = 128 rows (C >= M / 128); past M = 2048 it is 16 with
// taller slabs.  Measured (graph replay, profiles/r02_cluster_tc.log): a lone matrix is
// fastest with many CTAs and short slabs (64x576: 43 us at C = 16 or 8 with R = 128, 55 at 4
// with R = 192; C = 2 with 64 owned rows per CTA: 64x216 55 vs 47 at 4), but a call that also
// runs step-engine launches loses fewer SMs to small clusters (CIFAR set 103 us vs 108 at
// C = 16); R = 128 with the fewest CTAs keeps both.  A function of the shape alone.
__host__ __device__ inline int tc_cluster(int64_t M, int64_t N) {
  if (N < 1 || N > 256 || M < 1) return 0;
  const int Np = tc_np(N);
  for (int C = Np / 64 > 4 ? Np / 64 : 4; C <= kTcCtas; C *= 2) {  // C = 2 measured slower (64x216 55 vs 45 us)
    if ((int64_t)128 * C < M && C < kTcCtas) continue;
    const int R = tc_rows(M, C);
    if (R <= 256 && (int64_t)R * C >= M && tc_smem(Np, R, C) <= kTcMaxSmem) return C;
  }
  return 0;
}
__host__ __device__ inline bool tc_fits(int64_t M, int64_t N) { return tc_cluster(M, N) != 0; }

}  // namespace tns
