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
// Structure (persistent, warp-specialised, one CTA per SM):
//   warp 0      : TMA producer (one thread) -> 4-stage smem ring (48 KB / stage)
//   warp 1      : TMEM allocator + single-thread tcgen05.mma issuer
//   warps 4..11 : epilogue, TMEM -> registers -> global (two 128-column halves x four
//                 32-lane TMEM quadrants); the accumulator is double-buffered in TMEM
//                 (2 x 256 columns) so the epilogue of tile i overlaps the MMAs of tile i+1.
// Operand tiles are moved as 64 x 64 bf16 boxes with 128-byte swizzle; K-major and
// MN-major operands use the same boxes (only the coordinate order and the UMMA
// descriptor differ), so X^T X on a row-major X needs no transpose copy.
#include <cuda_runtime.h>

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
constexpr int kThreads = (4 + kNumEpiWarps) * 32;  // 384
constexpr uint32_t kTmemCols = 2 * kBN;            // double-buffered accumulator

template <int CG>
struct Geo {
  static constexpr int kARows = kBM;               // A rows staged per CTA
  static constexpr int kBRows = kBN / CG;          // B rows staged per CTA
  static constexpr int kTileM = kBM * CG;          // output rows per tile
  static constexpr int kABytes = kARows * kBK * 2;
  static constexpr int kBBytes = kBRows * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = CG == 1 ? 4 : 6;
  static constexpr size_t kSmemBytes = (size_t)kStages * kStageBytes + 1024 + 256;
};

struct TileInfo {
  int job;
  int p0, q0;
  bool mirror;
  bool valid;
};

__device__ __forceinline__ int find_job(const GemmJob* __restrict__ jobs, int njobs, int64_t t) {
  int lo = 0, hi = njobs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].tile_start <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

template <int CG>
__device__ __forceinline__ TileInfo decode_tile(const GemmJob* __restrict__ jobs, int njobs,
                                                int64_t t) {
  TileInfo ti;
  ti.job = find_job(jobs, njobs, t);
  const GemmJob& J = jobs[ti.job];
  const int local = (int)(t - J.tile_start);
  if (J.sym) {
    // lower-triangle 256 x 256 block L = bi(bi+1)/2 + bj; (2 / CG) row parts per block
    constexpr int parts = 2 / CG;
    const int L = local / parts, h = local % parts;
    int bi = (int)((sqrtf(8.0f * (float)L + 1.0f) - 1.0f) * 0.5f);
    while ((bi + 1) * (bi + 2) / 2 <= L) ++bi;
    while (bi * (bi + 1) / 2 > L) --bi;
    const int bj = L - bi * (bi + 1) / 2;
    ti.p0 = bi * kSymBlock + h * kBM;
    ti.q0 = bj * kSymBlock;
    ti.mirror = (bi != bj);
    ti.valid = ti.p0 < J.P;
  } else {
    // grouped raster: kGroupP row-blocks deep, column-block index slowest within a group
    constexpr int TM = kBM * CG;
    const int tiles_p = (J.P + TM - 1) / TM;
    const int tq = J.tiles_q;
    const int group = local / (kGroupP * tq);
    const int first_p = group * kGroupP;
    const int gsz = min(tiles_p - first_p, kGroupP);
    const int r = local - group * kGroupP * tq;
    ti.p0 = (first_p + r % gsz) * TM;
    ti.q0 = (r / gsz) * kBN;
    ti.mirror = false;
    ti.valid = true;
  }
  return ti;
}

__device__ __forceinline__ float bf2f(uint16_t h) {
  return __uint_as_float(((uint32_t)h) << 16);
}
__device__ __forceinline__ uint16_t f2bf(float f) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

// One 32-column chunk of one output row, values v[0..31] = D[p][q..q+31].
__device__ __forceinline__ void epilogue_chunk(const GemmJob& J, int p, int q, const uint32_t (&r)[32],
                                               bool mirror, bool& bad) {
  const bool rowok = p < J.P;
  const int64_t ld = J.ld;
  uint16_t* __restrict__ out = reinterpret_cast<uint16_t*>(J.out);
  const uint16_t* __restrict__ aux = reinterpret_cast<const uint16_t*>(J.aux);
  const bool full = (q + 32 <= J.Q);
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);

  // direct-tile values w[i] (before any per-destination scaling)
  if (J.mode != MODE_GRAM && rowok) {
    float x[32];
    if (full) {
      const uint4* src = reinterpret_cast<const uint4*>(aux + (int64_t)p * ld + q);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint4 u = __ldg(src + j);
        const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          x[8 * j + 2 * e] = bf2f((uint16_t)(w4[e] & 0xFFFFu));
          x[8 * j + 2 * e + 1] = bf2f((uint16_t)(w4[e] >> 16));
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) x[i] = (q + i < J.Q) ? bf2f(aux[(int64_t)p * ld + q + i]) : 0.f;
    }
    if (J.mode == MODE_POLY) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = fmaf(J.c, v[i], J.b * x[i]);
    } else {  // MODE_XB
      if (J.s == nullptr) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = fmaf(J.a, x[i], v[i]);
      } else if (J.s_by_row) {
        const float as = J.a * J.s[p];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = fmaf(as, x[i], v[i]);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float sq = (q + i < J.Q) ? J.s[q + i] : 0.f;
          v[i] = fmaf(J.a * sq, x[i], v[i]);
        }
      }
    }
  }

  // direct store: out[p][q + i]
  if (rowok) {
    const bool colscale = (J.mode == MODE_POLY && J.s != nullptr);
    uint16_t o[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      float w = v[i];
      if (colscale) w *= (q + i < J.Q) ? J.s[q + i] : 0.f;
      o[i] = f2bf(w);
      bad |= !isfinite(w) && (q + i < J.Q);
    }
    if (full) {
      uint4* dst = reinterpret_cast<uint4*>(out + (int64_t)p * ld + q);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint4 u;
        u.x = (uint32_t)o[8 * j + 0] | ((uint32_t)o[8 * j + 1] << 16);
        u.y = (uint32_t)o[8 * j + 2] | ((uint32_t)o[8 * j + 3] << 16);
        u.z = (uint32_t)o[8 * j + 4] | ((uint32_t)o[8 * j + 5] << 16);
        u.w = (uint32_t)o[8 * j + 6] | ((uint32_t)o[8 * j + 7] << 16);
        dst[j] = u;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (q + i < J.Q) out[(int64_t)p * ld + q + i] = o[i];
    }
    // mirrored store: out[q + i][p]  (coalesced across the warp: consecutive p)
    if (mirror) {
      const float sp = (J.mode == MODE_POLY && J.s != nullptr) ? J.s[p] : 1.f;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        if (q + i < J.Q) out[(int64_t)(q + i) * ld + p] = f2bf(v[i] * sp);
      }
    }
  }
}

template <int CG>
__global__ void __launch_bounds__(kThreads, 1)
    umma_gemm_kernel(const GemmJob* __restrict__ jobs, int njobs, int64_t total_tiles,
                     uint32_t* __restrict__ flags) {
  using G = Geo<CG>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + (size_t)G::kStages * G::kStageBytes);
  uint64_t* empty_bar = full_bar + G::kStages;
  uint64_t* tfull_bar = empty_bar + G::kStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = (CG == 2) ? cluster_ctarank() : 0u;  // CTA rank within the pair
  const int64_t cid = blockIdx.x / CG;                       // cluster (tile worker) index
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
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc<CG>(tmem_slot, kTmemCols);
    tmem_relinquish<CG>();
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      int last_job = -1;
      for (int64_t t = cid; t < total_tiles; t += ncl) {
        const TileInfo ti = decode_tile<CG>(jobs, njobs, t);
        if (!ti.valid) continue;
        const GemmJob& J = jobs[ti.job];
        if (ti.job != last_job) {
          tma_desc_acquire(J.tmA);
          tma_desc_acquire(J.tmB);
          last_job = ti.job;
        }
        const int pa = ti.p0 + (int)rank * G::kARows;  // this CTA's A rows
        const int qb = ti.q0 + (int)rank * G::kBRows;  // this CTA's B rows
        const int nk = (J.K + kBK - 1) / kBK;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + (size_t)stage * G::kStageBytes;
          uint8_t* sb = sa + G::kABytes;
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], G::kStageBytes * CG);
          const int k0 = kb * kBK;
#pragma unroll
          for (int i = 0; i < G::kARows / 64; ++i) {
            const int c0 = J.a_mn ? pa + 64 * i : k0, c1 = J.a_mn ? k0 : pa + 64 * i;
            if constexpr (CG == 2) tma_load_2d_cg2(sa + i * kBoxBytes, J.tmA, &full_bar[stage], c0, c1);
            else tma_load_2d(sa + i * kBoxBytes, J.tmA, &full_bar[stage], c0, c1);
          }
#pragma unroll
          for (int i = 0; i < G::kBRows / 64; ++i) {
            const int c0 = J.b_mn ? qb + 64 * i : k0, c1 = J.b_mn ? k0 : qb + 64 * i;
            if constexpr (CG == 2) tma_load_2d_cg2(sb + i * kBoxBytes, J.tmB, &full_bar[stage], c0, c1);
            else tma_load_2d(sb + i * kBoxBytes, J.tmB, &full_bar[stage], c0, c1);
          }
          if (++stage == G::kStages) { stage = 0; phase ^= 1; }
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
      for (int64_t t = cid; t < total_tiles; t += ncl) {
        const TileInfo ti = decode_tile<CG>(jobs, njobs, t);
        if (!ti.valid) continue;
        const GemmJob& J = jobs[ti.job];
        const uint32_t idesc = make_idesc_bf16(kBM * CG, kBN, (uint32_t)J.a_mn, (uint32_t)J.b_mn);
        const uint32_t a_lbo = J.a_mn ? 8192u : 16u, a_step = J.a_mn ? 2048u : 32u;
        const uint32_t b_lbo = J.b_mn ? 8192u : 16u, b_step = J.b_mn ? 2048u : 32u;
        mbar_wait(&tempty_bar[as], aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + as * kBN;
        const int nk = (J.K + kBK - 1) / kBK;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + (size_t)stage * G::kStageBytes);
          const uint32_t sb = sa + G::kABytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint64_t adesc = make_sdesc(sa + kk * a_step, a_lbo, 1024u);
            const uint64_t bdesc = make_sdesc(sb + kk * b_step, b_lbo, 1024u);
            umma_bf16<CG>(d_tmem, adesc, bdesc, idesc, (kb | kk) != 0 ? 1u : 0u);
          }
          umma_commit<CG>(&empty_bar[stage]);
          if (++stage == G::kStages) { stage = 0; phase ^= 1; }
        }
        umma_commit<CG>(&tfull_bar[as]);
        if (++as == 2) { as = 0; aphase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ epilogue
    const int quad = warp & 3;         // TMEM lanes [32*quad, 32*quad + 32)
    const int half = (warp - 4) >> 2;  // 128-column half of the 256-wide tile
    uint32_t as = 0, aphase = 0;
    bool bad = false;
    for (int64_t t = cid; t < total_tiles; t += ncl) {
      const TileInfo ti = decode_tile<CG>(jobs, njobs, t);
      if (!ti.valid) continue;
      const GemmJob& J = jobs[ti.job];
      mbar_wait(&tfull_bar[as], aphase);
      tc_fence_after();
      const int p = ti.p0 + (int)rank * kBM + quad * 32 + lane;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        const int cl = half * 128 + c * 32;
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(quad * 32) << 16) + as * kBN + (uint32_t)cl, r);
        tmem_ld_wait();
        if (c == 3) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (CG == 2) mbar_arrive_cluster(&tempty_bar[as], 0);
            else mbar_arrive(&tempty_bar[as]);
          }
        }
        epilogue_chunk(J, p, ti.q0 + cl, r, ti.mirror, bad);
      }
      if (++as == 2) { as = 0; aphase ^= 1; }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, 2u);
  }

  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<CG>(tmem_base, kTmemCols);
  }
}

template <int CG>
static cudaError_t launch_cg(const GemmJob* d_jobs, int njobs, int64_t total_tiles, int num_sms,
                             uint32_t* d_flags, cudaStream_t stream) {
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  auto kern = umma_gemm_kernel<CG>;
  if (!attr_set[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)Geo<CG>::kSmemBytes);
    if (e != cudaSuccess) return e;
    if (CG == 2) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    attr_set[dev & 63] = true;
  }
  const int64_t workers = num_sms / CG;  // persistent: one CTA (pair) per SM (pair)
  const int64_t nclusters = total_tiles < workers ? total_tiles : workers;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nclusters * CG));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Geo<CG>::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, d_jobs, njobs, total_tiles, d_flags);
}

cudaError_t launch_umma_gemm(const GemmJob* d_jobs, int njobs, int64_t total_tiles, int cg, int num_sms,
                             uint32_t* d_flags, cudaStream_t stream) {
  if (total_tiles <= 0) return cudaSuccess;
  return cg == 2 ? launch_cg<2>(d_jobs, njobs, total_tiles, num_sms, d_flags, stream)
                 : launch_cg<1>(d_jobs, njobs, total_tiles, num_sms, d_flags, stream);
}

int umma_tiles(int sym, int P, int Q, int cg) {
  if (sym) {
    const int nb = (P + kSymBlock - 1) / kSymBlock;
    return nb * (nb + 1) / 2 * (2 / cg);
  }
  const int tm = kBM * cg;
  return ((P + tm - 1) / tm) * ((Q + kBN - 1) / kBN);
}

}  // namespace tns
