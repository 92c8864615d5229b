// tcgen05 (5th-gen tensor core) GEMM engine for the three matrix products of one
// Newton-Schulz step (Eqs. 3-5), bf16 in / fp32 accumulate in TMEM.
//
//   D[p][q] = sum_k Aop[p][k] * Bop[q][k]         (one 128 x 256 tile per CTA at a time)
//
//   MODE_GRAM : A  = Xh^T Xh          -- only lower-triangle 256x256 blocks are computed;
//                                        off-diagonal blocks are stored twice (mirrored),
//                                        "only one triangular part needs to be computed"
//                                        (P:L252).
//   MODE_POLY : B  = (b A + c A A) s   -- same triangular scheme (A A is symmetric), the
//                                        b*A term reads the stored bf16 A that the MMA
//                                        consumed; s folds the AOL column scaling of
//                                        iteration 1 (Alg. 2, X1 = X0 s never materialised).
//   MODE_XB   : X' = a X s + X B^T      -- fused AXPY epilogue: the a*X term is applied to
//                                        the accumulator in the epilogue, so X is not
//                                        re-read by a second kernel.
//
// Structure (persistent, warp-specialised, one CTA per SM, CTA pairs = clusters of 2):
//   warp 0      : TMA producer (one thread): 64x64 bf16 boxes, 128-byte swizzle, 5-stage
//                 smem ring (32 KB / CTA / stage); 2-CTA loads signal the leader's barrier
//   warp 1      : TMEM allocator + single-thread tcgen05.mma.cta_group::2 issuer (leader)
//   warps 4..11 : epilogue; each warp owns 32 TMEM lanes (rows) x 128 columns, in 32-column
//                 chunks: tcgen05.ld -> fused math in registers -> 64-byte-swizzled smem box
//                 -> TMA bulk store (mirrored blocks: a second, transposed box).  The aux
//                 operand (A for POLY, X for XB) arrives by TMA into smem, one chunk ahead.
//   The accumulator is double-buffered in TMEM (2 x 256 columns), so tile i's epilogue
//   overlaps tile i+1's MMAs.  Tiles come from a host-built list (one 8-byte word each).
// Operand tiles are moved as 64 x 64 bf16 boxes with 128-byte swizzle; K-major and
// MN-major operands use the same boxes (only the coordinate order and the UMMA
// descriptor differ), so X^T X on a row-major X needs no transpose copy.
// TNS_DBG (environment, measurement only) bits: 1 skip epilogue math/stores, 2 skip
// mirrored stores, 4 skip aux loads, 8 collect epilogue clock counters.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "jobs.h"
#include "kernels.h"
#include "ptx.cuh"

namespace tns {

// Per-CTA geometry.  CG = 1: one CTA computes a 128 x 256 tile (UMMA M=128, N=256).
// CG = 2: a CTA pair (cluster of 2, tcgen05 cta_group::2) computes a 256 x 256 tile
// (UMMA M=256, N=256); each CTA stages 128 rows of A and 128 rows of B per k-block and
// holds 128 rows x 256 fp32 columns of the accumulator in its TMEM.  The pair halves the
// L2->SM operand traffic per FLOP versus two independent 128 x 256 CTAs.
constexpr int kBoxBytes = 64 * 64 * 2;  // one 64 x 64 bf16 TMA box
constexpr int kNumEpiWarps = 8;
// Clock64 measurement counters (TNS_DBG bits 8 and 16) cost registers: compiled in only
// with -DTNS_MEASURE=1 (`TNS_MEASURE=1 python paper_2512_04632_b200/build.py`; tools/time_kernels.py,
// tools/one_case.py read them).
#ifndef TNS_MEASURE
#define TNS_MEASURE 0
#endif
constexpr bool kMeasure = TNS_MEASURE != 0;
constexpr int kEpiWarp0 = 2;                        // epilogue = warps 2..9 (TMEM lane quarter = warp % 4)
constexpr int kThreads = (kEpiWarp0 + kNumEpiWarps) * 32;  // 320: up to 204 registers per thread

// BN = tile width (UMMA N): 256, or 128 for tile-starved plans (small problems), where
// halving the tile halves each warp's epilogue chunks -- the epilogue is the longest part
// of a launch that has one tile per CTA pair.
template <int CG, int BN>
struct Geo {
  static constexpr uint32_t kTmemCols = 2 * BN;  // double-buffered accumulator
  static constexpr int kChunks = BN / 64;        // 32-column epilogue chunks per warp
  static constexpr int kARows = kBM;               // A rows staged per CTA
  static constexpr int kBRows = BN / CG;           // B rows staged per CTA
  static constexpr int kTileM = kBM * CG;          // output rows per tile
  static constexpr int kABytes = kARows * kBK * 2;
  static constexpr int kBBytes = kBRows * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
#ifndef TNS_STAGES2
#define TNS_STAGES2 4
#endif
  static constexpr int kStages = CG == 1 ? 2 : TNS_STAGES2;
  static constexpr int kEpiOff = kStages * kStageBytes;          // epilogue staging
  // per epilogue warp: 2 aux, 2 output and 2 mirror boxes (all double-buffered)
  static constexpr int kEpiBytes = kNumEpiWarps * 6 * 2048;
  static constexpr size_t kSmemBytes = (size_t)kEpiOff + kEpiBytes + 1024 + 512;
};

// Measurement counters (TNS_DBG bit 8): per-epilogue-warp clock64 deltas summed over tiles.
__device__ unsigned long long g_epi_prof[8];

struct TileInfo {
  int job;
  int p0, q0;
  bool mirror;
};

template <int BN>
__device__ __forceinline__ TileInfo decode_word(uint64_t w) {
  TileInfo ti;
  ti.job = (int)(w & 0xFFFFFu);
  ti.p0 = (int)((w >> 20) & 0xFFFFFu) * 128;
  ti.q0 = (int)((w >> 40) & 0xFFFFFu) * BN;
  ti.mirror = (w >> 63) != 0;
  return ti;
}

// Epilogue parameters of one job, held in registers for the whole tile.
struct Epi {
  const void* tmOut;
  const void* tmAux;
  int mode, P, Q, s_by_row;
  int64_t ld;
  uint16_t* out;
  const uint16_t* aux;
  const float* s;
  float a, b, c;
  float* part;
  int part_ld, part_sm;
  const uint8_t* tmPeer;
  int npeer;
  float diag_add;
  int half;
  float* split_ws;
  int64_t split_stride;
  int split_ld;
};
__device__ __forceinline__ Epi load_epi(const GemmJob* __restrict__ J) {
  Epi e;
  e.tmOut = J->tmOut; e.tmAux = J->tmAux;
  e.mode = J->mode; e.P = J->P; e.Q = J->Q; e.s_by_row = J->s_by_row;
  e.ld = J->ld;
  e.out = reinterpret_cast<uint16_t*>(J->out);
  e.aux = reinterpret_cast<const uint16_t*>(J->aux);
  e.s = J->s;
  e.a = J->a; e.b = J->b; e.c = J->c;
  e.part = J->part; e.part_ld = J->part_ld; e.part_sm = J->part_sm;
  e.tmPeer = reinterpret_cast<const uint8_t*>(J->tmPeer); e.npeer = J->npeer;
  e.diag_add = J->diag_add;
  e.half = J->half;
  e.split_ws = J->split_ws; e.split_stride = J->split_stride; e.split_ld = J->split_ld;
  return e;
}

__device__ __forceinline__ float bf2f(uint16_t h) {
  return __uint_as_float(((uint32_t)h) << 16);
}
__device__ __forceinline__ uint16_t f2bf(float f) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

// Epilogue staging: per warp three 32 x 32 bf16 boxes (2 KB each, 64-byte rows) in the
// 64-byte-swizzle layout the TMA uses (16-byte chunk c of row r lives at chunk
// c ^ ((r >> 1) & 3)), so one-row-per-lane and one-column-per-lane smem accesses are both
// bank-conflict free, and every global access is a coalesced bulk-tensor transfer.
__device__ __forceinline__ uint32_t sw64(uint32_t row, uint32_t byte) {
  return row * 64u + (byte ^ (((row >> 1) & 3u) << 4));
}

// Epilogue variants (warp-uniform, chosen once per tile; each is branch-free per element).
enum EpiVariant : int { V_GRAM = 0, V_POLY = 1, V_POLY_S = 2, V_XB = 3, V_XB_SROW = 4, V_XB_SCOL = 5 };
__device__ __forceinline__ int epi_variant(const Epi& E) {
  if (E.mode == MODE_GRAM) return V_GRAM;
  if (E.mode == MODE_POLY) return E.s ? V_POLY_S : V_POLY;
  if (E.s == nullptr && E.a == 0.f) return V_GRAM;  // a folded into B: plain store of X B'^T
  return E.s ? (E.s_by_row ? V_XB_SROW : V_XB_SCOL) : V_XB;
}
__device__ __forceinline__ bool epi_needs_aux(const Epi& E) {
  return E.mode == MODE_POLY || (E.mode == MODE_XB && (E.s != nullptr || E.a != 0.f));
}
__device__ __forceinline__ float lo_bf(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float hi_bf(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t pack_bf2(float a, float b) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b));
  return r;
}
// s[q .. q+32) as fp32 (the same for all lanes: broadcast loads; s is padded with zeros).
__device__ __forceinline__ void load_s32(const float* s, int q, float (&sv)[32]) {
  const float4* src = reinterpret_cast<const float4*>(s + q);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float4 f = __ldg(src + j);
    sv[4 * j] = f.x; sv[4 * j + 1] = f.y; sv[4 * j + 2] = f.z; sv[4 * j + 3] = f.w;
  }
}

// Math of one 32-column chunk of one output row.  r = fp32 accumulator D[p][q..q+32),
// x = aux row chunk (bf16 pairs).  o = bf16 pairs for out[p][q..], m = bf16 pairs for the
// mirrored out[q..][p] (only V_POLY_S differs from o: destination-column scaling).
// dg: warp-uniform, this chunk intersects the matrix diagonal and diag_add != 0.
__device__ __forceinline__ void epi_math(int var, const Epi& E, int p, int q, const uint32_t (&r)[32],
                                         const uint32_t (&x)[16], uint32_t (&o)[16], uint32_t (&m)[16],
                                         bool dg, bool& bad) {
  switch (var) {
    case V_GRAM:
#pragma unroll
      for (int i = 0; i < 16; ++i) o[i] = pack_bf2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
      break;
    case V_POLY: {
      const int d = p - q;  // this lane's diagonal element sits at column index d (if 0..31)
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float w0 = fmaf(E.c, __uint_as_float(r[2 * i]), E.b * lo_bf(x[i]));
        float w1 = fmaf(E.c, __uint_as_float(r[2 * i + 1]), E.b * hi_bf(x[i]));
        if (dg) { w0 += (d == 2 * i) ? E.diag_add : 0.f; w1 += (d == 2 * i + 1) ? E.diag_add : 0.f; }
        o[i] = pack_bf2(w0, w1);
      }
      break;
    }
    case V_POLY_S: {
      float sv[32];
      load_s32(E.s, q, sv);
      const float sp = __ldg(E.s + p);
      const int d = p - q;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float w0 = fmaf(E.c, __uint_as_float(r[2 * i]), E.b * lo_bf(x[i]));
        float w1 = fmaf(E.c, __uint_as_float(r[2 * i + 1]), E.b * hi_bf(x[i]));
        if (dg) { w0 += (d == 2 * i) ? E.diag_add : 0.f; w1 += (d == 2 * i + 1) ? E.diag_add : 0.f; }
        o[i] = pack_bf2(w0 * sv[2 * i], w1 * sv[2 * i + 1]);
        m[i] = pack_bf2(w0 * sp, w1 * sp);
      }
      break;
    }
    case V_XB:
#pragma unroll
      for (int i = 0; i < 16; ++i)
        o[i] = pack_bf2(fmaf(E.a, lo_bf(x[i]), __uint_as_float(r[2 * i])),
                        fmaf(E.a, hi_bf(x[i]), __uint_as_float(r[2 * i + 1])));
      break;
    case V_XB_SROW: {
      const float as = E.a * __ldg(E.s + p);
#pragma unroll
      for (int i = 0; i < 16; ++i)
        o[i] = pack_bf2(fmaf(as, lo_bf(x[i]), __uint_as_float(r[2 * i])),
                        fmaf(as, hi_bf(x[i]), __uint_as_float(r[2 * i + 1])));
      break;
    }
    default: {  // V_XB_SCOL
      float sv[32];
      load_s32(E.s, q, sv);
#pragma unroll
      for (int i = 0; i < 16; ++i)
        o[i] = pack_bf2(fmaf(E.a * sv[2 * i], lo_bf(x[i]), __uint_as_float(r[2 * i])),
                        fmaf(E.a * sv[2 * i + 1], hi_bf(x[i]), __uint_as_float(r[2 * i + 1])));
      break;
    }
  }
  // non-finite check of the 32 stored bf16 values: per half, (h & 0x7F80) + 0x80 reaches
  // bit 15 iff the exponent is all ones (Inf/NaN); OR over the words, one test at the end.
  // Only the update's outputs are checked: a non-finite A or B' always reaches X_{k+1}
  // (NaN and Inf propagate through the products; an overflowing Gram gives s = 0 and
  // 0 * Inf = NaN), so flag bit 1 is raised all the same, and the Gram / A^2 epilogues --
  // the ones as long as their short main loops -- save the instructions.
#ifndef TNS_CHECK_ALL_STEPS
  if (E.mode != MODE_XB) return;
#endif
  uint32_t nf = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) nf |= (o[i] & 0x7F807F80u) + 0x00800080u;
  bad |= (nf & 0x80008000u) != 0;
}

// SPLIT: the launch carries split-K tasks (k-ranges with fp32 partial stores, TaskDesc
// kb0/nkb/split); a separate instantiation so that the other launches keep the register
// allocation of the plain kernel.
template <int CG, bool SPLIT, int BN>
__global__ void __launch_bounds__(kThreads, 1)
    umma_gemm_kernel(const GemmJob* __restrict__ jobs, const TaskDesc* __restrict__ tasks, int64_t ntasks,
                     uint32_t* __restrict__ flags, int dbg) {
  using G = Geo<CG, BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + (size_t)G::kEpiOff + G::kEpiBytes);
  uint64_t* empty_bar = full_bar + G::kStages;
  uint64_t* tfull_bar = empty_bar + G::kStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* aux_bar = tempty_bar + 2;  // two per epilogue warp (double-buffered aux box)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aux_bar + 2 * kNumEpiWarps);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // TNS_DBG bit 16: latency timeline of CTA 0 (cycles since kernel entry, summed over launches)
  const bool tl = kMeasure && (dbg & 16) && blockIdx.x == 0 && lane == 0;
  const long long T0 = tl ? clock64() : 0;
#define TL(slot) do { if (tl) atomicAdd(&g_epi_prof[slot], (unsigned long long)(clock64() - T0)); } while (0)
  const uint32_t rank = (CG == 2) ? cluster_ctarank() : 0u;  // CTA rank within the pair
  const int64_t cid = blockIdx.x / CG;                         // CTA pair (tile worker) index
  const int64_t ncl = gridDim.x / CG;

  if (threadIdx.x == 0) {
    for (int i = 0; i < G::kStages; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], kNumEpiWarps * CG);
    }
    for (int i = 0; i < 2 * kNumEpiWarps; ++i) mbar_init(&aux_bar[i], 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc<CG>(tmem_slot, G::kTmemCols);
    tmem_relinquish<CG>();
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // everything above overlaps the previous kernel's tail (PDL).  Each role waits for it
  // (griddepcontrol.wait) right before its first access to data a previous launch writes or
  // reads -- operands, aux, outputs, step counters -- so the static task / job / tensormap
  // reads of its first tile overlap that tail too; the MMA issuer touches only smem and TMEM
  // and never waits.
  if (warp == 0) TL(0);  // setup done
  pdl_trigger();

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      int last_job = -1;
      bool waited = false;
      for (int64_t t = cid; t < ntasks; t += ncl) {
        const TaskDesc TD = tasks[t];
        if (TD.kind != TK_TILE) continue;
        const TileInfo ti = decode_word<BN>(TD.tile);
        const GemmJob* J = jobs + ti.job;
        const void* tmA = J->tmA;
        const void* tmB = J->tmB;
        const int a_mn = J->a_mn, b_mn = J->b_mn, K = J->K;
        const int a_sym = J->a_sym, b_sym = J->b_sym;
        if (ti.job != last_job) {
          if (!waited) { tma_prefetch_desc(tmA); tma_prefetch_desc(tmB); }
          tma_desc_acquire(tmA);
          tma_desc_acquire(tmB);
          last_job = ti.job;
        }
        if (!waited) {  // operands come from the previous launch
          pdl_wait();
          waited = true;
          TL(1);  // dependency resolved
        }
        const int pa = ti.p0 + (int)rank * G::kARows;  // this CTA's A rows
        const int qb = ti.q0 + (int)rank * G::kBRows;  // this CTA's B rows
        const int kbeg = SPLIT ? (int)TD.kb0 : 0;
        const int kend = (SPLIT && TD.nkb) ? kbeg + (int)TD.nkb : (K + kBK - 1) / kBK;
        for (int kb = kbeg; kb < kend; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + (size_t)stage * G::kStageBytes;
          uint8_t* sb = sa + G::kABytes;
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], G::kStageBytes * CG);
          const int k0 = kb * kBK;
          // half-storage symmetric operand: an upper-triangle block is read transposed
          const int a_e = a_mn ^ (a_sym && (k0 >> 8) > (pa >> 8));
          const int b_e = b_mn ^ (b_sym && (k0 >> 8) > (qb >> 8));
#pragma unroll
          for (int i = 0; i < G::kARows / 64; ++i) {
            const int c0 = a_e ? pa + 64 * i : k0, c1 = a_e ? k0 : pa + 64 * i;
            if constexpr (CG == 2) tma_load_2d_cg2(sa + i * kBoxBytes, tmA, &full_bar[stage], c0, c1);
            else tma_load_2d(sa + i * kBoxBytes, tmA, &full_bar[stage], c0, c1);
          }
#pragma unroll
          for (int i = 0; i < G::kBRows / 64; ++i) {
            const int c0 = b_e ? qb + 64 * i : k0, c1 = b_e ? k0 : qb + 64 * i;
            if constexpr (CG == 2) tma_load_2d_cg2(sb + i * kBoxBytes, tmB, &full_bar[stage], c0, c1);
            else tma_load_2d(sb + i * kBoxBytes, tmB, &full_bar[stage], c0, c1);
          }
          if (++stage == G::kStages) { stage = 0; phase ^= 1; }
          if (kb == kbeg && t == cid) TL(2);  // first loads issued
        }
      }
      // tail: wait until the MMA released every stage, so no commit-arrive is still in
      // flight towards this CTA's barriers when it exits
      for (int i = 0; i < G::kStages; ++i) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        if (++stage == G::kStages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer (leader)
    if (lane == 0 && rank == 0) {
      uint32_t stage = 0, phase = 0, as = 0, aphase = 0;
      for (int64_t t = cid; t < ntasks; t += ncl) {
        const TaskDesc TD = tasks[t];
        if (TD.kind != TK_TILE) continue;
        const TileInfo ti = decode_word<BN>(TD.tile);
        const GemmJob* J = jobs + ti.job;
        const uint32_t a_mn = (uint32_t)J->a_mn, b_mn = (uint32_t)J->b_mn;
        const int K = J->K;
        const int a_sym = J->a_sym, b_sym = J->b_sym;
        const int pblk = ti.p0 >> 8, qblk = ti.q0 >> 8;  // both CTAs' rows share the block
        // TNS_MEASURE builds, TNS_DBG bit 64: MMA-issuer stall cycles (slot 0 tiles, 1 waiting
        // for a free accumulator = epilogue-bound, 2 waiting for operands = feed-bound, 3 busy)
        // (bits 256 / 512 / 1024 restrict the counting to GRAM / POLY / XB tiles)
        const bool mprof = kMeasure && (dbg & 64) && (!(dbg & 1792) || (dbg & (256 << J->mode)));
        long long m0 = mprof ? clock64() : 0;
        mbar_wait(&tempty_bar[as], aphase ^ 1);
        if (mprof) { const long long m1 = clock64(); atomicAdd(&g_epi_prof[1], (unsigned long long)(m1 - m0)); m0 = m1;
                     atomicAdd(&g_epi_prof[0], 1ull); }
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + as * BN;
        const int kbeg = SPLIT ? (int)TD.kb0 : 0;
        const int kend = (SPLIT && TD.nkb) ? kbeg + (int)TD.nkb : (K + kBK - 1) / kBK;
        for (int kb = kbeg; kb < kend; ++kb) {
          if (mprof) {
            const long long m1 = clock64();
            atomicAdd(&g_epi_prof[3], (unsigned long long)(m1 - m0));
            m0 = m1;
          }
          mbar_wait(&full_bar[stage], phase);
          if (mprof) {
            const long long m1 = clock64();
            atomicAdd(&g_epi_prof[2], (unsigned long long)(m1 - m0));
            m0 = m1;
          }
          tc_fence_after();
          if (kb == kbeg && t == cid) TL(3);  // first operands landed
          const uint32_t sa = smem_u32(smem + (size_t)stage * G::kStageBytes);
          const uint32_t sb = sa + G::kABytes;
          const int kblk = (kb * kBK) >> 8;
          const uint32_t a_e = a_mn ^ (uint32_t)(a_sym && kblk > pblk);
          const uint32_t b_e = b_mn ^ (uint32_t)(b_sym && kblk > qblk);
          const uint32_t idesc = make_idesc_bf16(kBM * CG, BN, a_e, b_e);
          const uint32_t a_lbo = a_e ? 8192u : 16u, a_step = a_e ? 2048u : 32u;
          const uint32_t b_lbo = b_e ? 8192u : 16u, b_step = b_e ? 2048u : 32u;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint64_t adesc = make_sdesc(sa + kk * a_step, a_lbo, 1024u);
            const uint64_t bdesc = make_sdesc(sb + kk * b_step, b_lbo, 1024u);
            umma_bf16<CG>(d_tmem, adesc, bdesc, idesc, (kb != kbeg || kk != 0) ? 1u : 0u);
          }
          umma_commit<CG>(&empty_bar[stage]);
          if (++stage == G::kStages) { stage = 0; phase ^= 1; }
        }
        umma_commit<CG>(&tfull_bar[as]);
        if (++as == 2) { as = 0; aphase ^= 1; }
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ------------------------------------------------------------------ epilogue
    const int ew = warp - kEpiWarp0;
    const int quad = warp & 3;  // TMEM lanes [32*quad, 32*quad + 32)
    const int half = ew >> 2;   // 128-column half of the 256-wide tile
    // staging (2 KB boxes): aux[0..1] @ 0, 2K; out[0..1] @ 4K, 6K; mirror[0..1] @ 8K, 10K
    uint8_t* s_aux = smem + G::kEpiOff + ew * 12288;
    uint8_t* s_out = s_aux + 4096;
    uint8_t* s_mir = s_aux + 8192;
    uint64_t* abar = aux_bar + 2 * ew;
    const uint32_t sa_aux = smem_u32(s_aux), sa_out = smem_u32(s_out), sa_mir = smem_u32(s_mir);
    uint32_t as = 0, aphase = 0, xph = 0;  // xph bit b: parity of aux buffer b
    bool bad = false;
    // measurement counters (TNS_DBG bit 8): accumulated straight into g_epi_prof so that no
    // register array stays live in production
#define EPC(i, v) atomicAdd(&g_epi_prof[i], (unsigned long long)(v))
    bool waited = false;
    for (int64_t t = cid; t < ntasks; t += ncl) {
      const TaskDesc TD = tasks[t];
      if (!waited) {  // aux and outputs: after the previous launch
        pdl_wait();
        waited = true;
      }
      if (TD.kind == TK_NONE) continue;  // schedule padding (balanced per-step task lists)
      const TileInfo ti = decode_word<BN>(TD.tile);
      const Epi E = load_epi(jobs + ti.job);
      const int var = epi_variant(E);
      const bool has_aux = epi_needs_aux(E) && !(dbg & 4);
      const int prow = ti.p0 + (int)rank * kBM + quad * 32;  // first of this warp's 32 rows
      const int p = prow + lane;
      const int qh = ti.q0 + half * (BN / 2);
      float rsum = 0.f, rsum1 = 0.f;  // |A0| row sums of columns [qh, qh+64) and [qh+64, qh+128)
      if (has_aux && lane == 0) {  // prefetch aux chunks 0 and 1 before the accumulator is ready
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          mbar_arrive_expect_tx(abar + b, 2048);
          tma_load_2d(s_aux + b * 2048, E.tmAux, abar + b, qh + 32 * b, prow);
        }
      }
      const bool prof = kMeasure && (dbg & 8) && lane == 0 && (!(dbg & 1792) || (dbg & (256 << E.mode)));
      long long t0 = prof ? clock64() : 0, t1;
      mbar_wait(&tfull_bar[as], aphase);
      tc_fence_after();
      if (ew == 0 && t == cid) TL(4);  // first accumulator ready
      if (prof) { t1 = clock64(); EPC(1, t1 - t0); t0 = t1; EPC(0, 1); }
#pragma unroll 1
      for (int c = 0; c < G::kChunks; ++c) {
        const int q = qh + c * 32;
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(quad * 32) << 16) + as * BN + (uint32_t)(q - ti.q0), r);
        uint32_t x[16];
        const int xb = c & 1;  // aux / output buffer of this chunk
        if (has_aux) {
          mbar_wait(abar + xb, (xph >> xb) & 1u);
          if (prof) { t1 = clock64(); EPC(3, t1 - t0); t0 = t1; }
          xph ^= 1u << xb;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint4 u;
            asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
                         : "r"(sa_aux + 2048u * xb + sw64((uint32_t)lane, 16u * j)));
            x[4 * j] = u.x; x[4 * j + 1] = u.y; x[4 * j + 2] = u.z; x[4 * j + 3] = u.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) x[j] = 0u;
        }
        tmem_ld_wait();
        if (prof) { t1 = clock64(); EPC(2, t1 - t0); t0 = t1; }
        if (c == G::kChunks - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (CG == 2) mbar_arrive_cluster(&tempty_bar[as], 0);
            else mbar_arrive_relaxed(&tempty_bar[as]);
          }
        }
        if (has_aux && c + 2 < G::kChunks) {  // refill this aux buffer with chunk c + 2
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive_expect_tx(abar + xb, 2048);
            tma_load_2d(s_aux + 2048 * xb, E.tmAux, abar + xb, q + 64, prow);
          }
        }
        if (SPLIT && TD.split) {  // split-K: this k-range's fp32 partial, no epilogue math
          float4* dst = reinterpret_cast<float4*>(E.split_ws + (int64_t)(TD.split - 1) * E.split_stride +
                                                  (int64_t)p * E.split_ld + q);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            dst[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                 __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
          continue;
        }
        if (dbg & 1) continue;
        // mirrored block: transposed box in smem for the mirrored store (full storage) and/or
        // the AOL column sums (iteration-1 Gram); half storage skips the store
        const bool mir_store = ti.mirror && !E.half && !(dbg & 2);
        const bool mir = mir_store || (ti.mirror && E.part != nullptr);
        uint32_t o[16], m[16];
        // chunk rows [prow, prow+32) x cols [q, q+32) contain diagonal elements iff they overlap
        const bool dg = (E.diag_add != 0.f) && !ti.mirror && (q < prow + 32) && (prow < q + 32);
        epi_math(var, E, p, q, r, x, o, m, dg, bad);
        if (E.part != nullptr) {  // AOL row sums of |A0| per 64-column slot (Eq. 8)
          float cs = 0.f;
#pragma unroll
          for (int i = 0; i < 16; ++i) cs += fabsf(lo_bf(o[i])) + fabsf(hi_bf(o[i]));
          if (c < 2) rsum += cs; else rsum1 += cs;
        }
        if (prof) { t1 = clock64(); EPC(4, t1 - t0); t0 = t1; }
        // the bulk stores that last read these staging boxes (chunk c - 2's group) must be
        // done with them
        if (lane == 0) bulk_wait_read<1>();
        __syncwarp();
        if (prof) { t1 = clock64(); EPC(5, t1 - t0); t0 = t1; }
#pragma unroll
        for (int j = 0; j < 4; ++j)
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(sa_out + 2048u * xb + sw64((uint32_t)lane, 16u * j)),
                       "r"(o[4 * j]), "r"(o[4 * j + 1]), "r"(o[4 * j + 2]), "r"(o[4 * j + 3])
                       : "memory");
        if (mir) {
          const bool sep = (var == V_POLY_S);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const uint32_t w = sep ? m[i >> 1] : o[i >> 1];
            const uint16_t h = (uint16_t)(i & 1 ? (w >> 16) : (w & 0xFFFFu));
            asm volatile("st.shared.u16 [%0], %1;" ::"r"(sa_mir + 2048u * xb + sw64((uint32_t)i, 2u * lane)), "h"(h)
                         : "memory");
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          uint8_t* so = s_out + 2048 * xb;
          tma_store_2d(E.tmOut, so, q, prow);             // rows prow.., cols q..
          if (mir_store) tma_store_2d(E.tmOut, s_mir + 2048 * xb, prow, q);  // rows q.., cols prow..
          // fused all-gather: the same box to every peer's buffer (NVLink), tile by tile
          for (int r = 0; r < E.npeer; ++r) tma_store_2d(E.tmPeer + 128 * r, so, q, prow);
          bulk_commit();
        }
        if (E.part != nullptr && mir) {
          // mirrored block: row q+lane of A0 gets the |.| sum over this warp's 32 rows,
          // read back from the transposed staging box (row `lane` of it)
          float cs = 0.f;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint4 u;
            asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
                         : "r"(sa_mir + 2048u * xb + sw64((uint32_t)lane, 16u * j)));
            cs += fabsf(lo_bf(u.x)) + fabsf(hi_bf(u.x)) + fabsf(lo_bf(u.y)) + fabsf(hi_bf(u.y)) +
                  fabsf(lo_bf(u.z)) + fabsf(hi_bf(u.z)) + fabsf(lo_bf(u.w)) + fabsf(hi_bf(u.w));
          }
          if (q + lane < E.Q && prow < E.P)
            E.part[part_at(E.part_ld, E.part_sm, E.P, q + lane, (E.Q + 63) / 64 + prow / 32)] = cs;
        }
        if (prof) { t1 = clock64(); EPC(6, t1 - t0); t0 = t1; }
      }
      if (E.part != nullptr && p < E.P) {
        if (qh < E.Q) E.part[part_at(E.part_ld, E.part_sm, E.P, p, qh / 64)] = rsum;
        if (G::kChunks > 2 && qh + 64 < E.Q) E.part[part_at(E.part_ld, E.part_sm, E.P, p, qh / 64 + 1)] = rsum1;
      }
      if (++as == 2) { as = 0; aphase ^= 1; }
    }
    if (lane == 0) bulk_wait<0>();
    if (ew == 0) TL(5);  // epilogue stores complete
#undef EPC
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, 2u);
  }

  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<CG>(tmem_base, G::kTmemCols);
    TL(6);
    if (tl) atomicAdd(&g_epi_prof[7], 1ull);
  }
#undef TL
}

template <int CG, bool SPLIT, int BN>
static cudaError_t launch_cg(const GemmJob* d_jobs, const TaskDesc* d_tasks, int64_t ntasks, int64_t max_tiles,
                             int num_sms, uint32_t* d_flags, cudaStream_t stream) {
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  auto kern = umma_gemm_kernel<CG, SPLIT, BN>;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Geo<CG, BN>::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  if (!attr_set[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)Geo<CG, BN>::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set[dev & 63] = true;
  }
  // persistent: one CTA (pair) per SM (pair), or one per tile when there are fewer tiles
  const int64_t workers = num_sms / CG;
  const int64_t nclusters = max_tiles > workers ? workers : max_tiles;
  cfg.gridDim = dim3((unsigned)(nclusters * CG));
  static int dbg = -1;
  if (dbg < 0) {  // measurement knob (never set in production): TNS_DBG bits 1 skip epilogue,
    const char* e = getenv("TNS_DBG");  // 2 skip mirrored stores, 4 skip aux prefetch, 8 counters, 16 timeline
    dbg = e ? atoi(e) : 0;
  }
  return cudaLaunchKernelEx(&cfg, kern, d_jobs, d_tasks, ntasks, d_flags, dbg);
}

cudaError_t launch_umma_gemm(const GemmJob* d_jobs, const TaskDesc* d_tasks, int64_t ntasks, int64_t max_tiles,
                             int cg, int num_sms, uint32_t* d_flags, bool split, int bn, cudaStream_t stream) {
  if (ntasks <= 0) return cudaSuccess;
#define TNS_LAUNCH(CG_, SP_, BN_) \
  launch_cg<CG_, SP_, BN_>(d_jobs, d_tasks, ntasks, max_tiles, num_sms, d_flags, stream)
  if (cg == 2) {
    if (bn == 128) return split ? TNS_LAUNCH(2, true, 128) : TNS_LAUNCH(2, false, 128);
    return split ? TNS_LAUNCH(2, true, 256) : TNS_LAUNCH(2, false, 256);
  }
  return split ? TNS_LAUNCH(1, true, 256) : TNS_LAUNCH(1, false, 256);
#undef TNS_LAUNCH
}

cudaError_t umma_epi_prof(unsigned long long* out, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_epi_prof, sizeof(g_epi_prof));
  if (e == cudaSuccess && reset) {
    unsigned long long z[8] = {};
    e = cudaMemcpyToSymbol(g_epi_prof, z, sizeof(z));
  }
  return e;
}

// Tiles of one job in execution order (host).  Symmetric jobs: lower-triangle 256 x 256
// blocks row by row, (2 / cg) row parts each.  Rectangular jobs: grouped raster, kGroupP
// tile-rows deep, so concurrently running tiles share operand rows/columns in L2.
void umma_tile_list(const GemmJob& J, uint32_t job, int cg, int bn, std::vector<uint64_t>& out) {
  if (J.sym) {
    const int nb = (J.P + kSymBlock - 1) / kSymBlock;
    for (int bi = 0; bi < nb; ++bi)
      for (int bj = 0; bj <= bi; ++bj)
        for (int h = 0; h < 2 / cg; ++h)
          for (int qq = 0; qq < kSymBlock / bn; ++qq) {
            const int p0 = bi * kSymBlock + h * kBM, q0 = bj * kSymBlock + qq * bn;
            if (p0 < J.P && q0 < J.Q) out.push_back(pack_tile(job, p0, q0, bi != bj, bn));
          }
    return;
  }
  const int tm = kBM * cg;
  const int tp = (J.P + tm - 1) / tm, tq = (J.Q + bn - 1) / bn;
  for (int g0 = 0; g0 < tp; g0 += kGroupP) {
    const int gsz = tp - g0 < kGroupP ? tp - g0 : kGroupP;
    for (int qb = 0; qb < tq; ++qb)
      for (int i = 0; i < gsz; ++i) out.push_back(pack_tile(job, (g0 + i) * tm, qb * bn, false, bn));
  }
}

}  // namespace tns
