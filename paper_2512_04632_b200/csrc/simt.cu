// CUDA-core kernels:
//   * simt_gemm_kernel  -- the three NS products (Eqs. 3-5) with the same fused epilogues
//     as the tcgen05 engine, for the fp32 "exact" mode (fp32 storage, fp32 FFMA) and for
//     bf16 shapes that TMA cannot address (row pitch not a multiple of 16 bytes).
//   * precondition_kernel -- the fused AOL preconditioner (Eqs. 7-9, Alg. 2 l.2-4):
//     phase 1: one warp per row of A0, s_i = rsqrt(sum_j |A0_ij|) (Eq. 8) with vectorised
//     16-byte loads and a fixed-order warp-shuffle reduction (deterministic); Frobenius:
//     s = rsqrt(trace A0) = 1/||X||_F (Eq. 10);  grid barrier;  phase 2: A1 = s_i A0_ij s_j
//     in place (Alg. 2 l.4, "Update A to avoid recomputation"), one warp per 256-column
//     segment of a stored row (equal bytes per warp under half storage).  HBM-bound.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cuda_runtime.h>

#include "jobs.h"
#include "kernels.h"
#include "precond_rows.cuh"

namespace tns {

// ------------------------------------------------------------------------------ SIMT GEMM
template <typename T>
__global__ void __launch_bounds__(256)
    simt_gemm_kernel(const SimtJob* __restrict__ jobs, int njobs, int64_t total_tiles,
                     uint32_t* __restrict__ flags) {
  // KT = 64: one global round trip per 64 k (the fp32 path is latency-bound at small sizes)
  constexpr int TILE = kSimtTile, KT = 64;
  __shared__ float As[KT][TILE + 4];
  __shared__ float Bs[KT][TILE + 4];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  bool bad = false;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");  // operands come from the previous step
  for (int64_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
    int lo = 0, hi = njobs - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (jobs[mid].tile_start <= t) lo = mid; else hi = mid - 1;
    }
    const SimtJob& J = jobs[lo];
    const int local = (int)(t - J.tile_start);
    const int p0 = (local / J.tiles_q) * TILE, q0 = (local % J.tiles_q) * TILE;
    const T* __restrict__ A = reinterpret_cast<const T*>(J.A);
    const T* __restrict__ B = reinterpret_cast<const T*>(J.B);
    float acc[4][4] = {};
    for (int k0 = 0; k0 < J.K; k0 += KT) {
      float ra[16], rb[16];  // issue all 32 loads before any smem store (one round trip)
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int idx = tid + e * 256;
        int pp, kk;
        if (J.sa_p == 1) { pp = idx & 63; kk = idx >> 6; } else { kk = idx & 63; pp = idx >> 6; }
        const int gp = p0 + pp, gk = k0 + kk;
        ra[e] = (gp < J.P && gk < J.K) ? ld_val<T>(A + gp * J.sa_p + gk * J.sa_k) : 0.f;
        int qq, kq;
        if (J.sb_q == 1) { qq = idx & 63; kq = idx >> 6; } else { kq = idx & 63; qq = idx >> 6; }
        const int gq = q0 + qq, gk2 = k0 + kq;
        rb[e] = (gq < J.Q && gk2 < J.K) ? ld_val<T>(B + gq * J.sb_q + gk2 * J.sb_k) : 0.f;
      }
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int idx = tid + e * 256;
        if (J.sa_p == 1) As[idx >> 6][idx & 63] = ra[e]; else As[idx & 63][idx >> 6] = ra[e];
        if (J.sb_q == 1) Bs[idx >> 6][idx & 63] = rb[e]; else Bs[idx & 63][idx >> 6] = rb[e];
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < KT; ++kk) {
        float a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) { a[i] = As[kk][ty * 4 + i]; b[i] = Bs[kk][tx * 4 + i]; }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
    }
    T* __restrict__ out = reinterpret_cast<T*>(J.out);
    const T* __restrict__ aux = reinterpret_cast<const T*>(J.aux);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int p = p0 + ty * 4 + i;
      if (p >= J.P) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int q = q0 + tx * 4 + j;
        if (q >= J.Q) continue;
        float v = acc[i][j];
        const int64_t off = (int64_t)p * J.ld + q;
        if (J.mode == MODE_POLY) {
          v = fmaf(J.c, v, J.b * ld_val<T>(aux + off));
          if (J.s) v *= J.s[q];
        } else if (J.mode == MODE_XB) {
          const float sc = J.s ? (J.s_by_row ? J.s[p] : J.s[q]) : 1.f;
          v = fmaf(J.a * sc, ld_val<T>(aux + off), v);
        }
        bad |= !isfinite(v);
        out[off] = st_conv<T>(v);
      }
    }
  }
  if (__syncthreads_or(bad) && tid == 0) atomicOr(flags, 2u);
}

cudaError_t launch_simt_gemm(const SimtJob* d_jobs, int njobs, int64_t total_tiles, int num_sms,
                             bool is_bf16, uint32_t* d_flags, cudaStream_t stream) {
  if (total_tiles <= 0) return cudaSuccess;
  const int64_t cap = (int64_t)num_sms * 8;
  const int grid = (int)(total_tiles < cap ? total_tiles : cap);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (is_bf16) return cudaLaunchKernelEx(&cfg, simt_gemm_kernel<uint16_t>, d_jobs, njobs, total_tiles, d_flags);
  return cudaLaunchKernelEx(&cfg, simt_gemm_kernel<float>, d_jobs, njobs, total_tiles, d_flags);
}

// ------------------------------------------------------------------------------ preconditioner
// Self-resetting grid barrier (all CTAs co-resident: cooperative launch).  bar[0] counts
// arrivals, bar[1] is a generation number; the last arriver resets the count and bumps the
// generation, so no host-side reset (memset) is needed between launches.
__device__ __forceinline__ int find_seg_job(const PrecondJob* __restrict__ jobs, int njobs, int64_t g) {
  int lo = 0, hi = njobs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].seg_start <= g) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g0 = *gen;
    __threadfence();
    const unsigned old = atomicAdd(bar, 1u);
    if (old == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g0) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

template <typename T, bool VEC8>
__global__ void __launch_bounds__(256, 3)
    precondition_kernel(const PrecondJob* __restrict__ jobs, int njobs, int64_t total_rows,
                        int64_t total_segs, unsigned* barrier, uint32_t* __restrict__ flags, int mode) {
  // mode bit 0: AOL from the Gram partials (lane loops), bits 3 / 4 / 5: the launch has rows
  // summed by four lanes / a warp / one lane (host flags); bits 1 / 2 (TNS_PRE_DBG, measurement
  // only): skip phase 1 / phase 2
  const int lane_rows = mode & 1;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");  // A0 comes from the preceding Gram launch
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint32_t fl = 0;
  // ---- phase 1: scaling vector s (Eq. 8 / Eq. 10); each warp owns a contiguous run of rows
  const int64_t per = (total_rows + nwarps - 1) / nwarps;
  const int64_t r_beg = gwarp * per, r_end = min(total_rows, r_beg + per);
  if (mode & 2) {
  } else if (lane_rows) {  // AOL from the Gram epilogue's partials (every job)
    // Short partial rows (part_ld <= kSeqPartials, N <= 1344): one LANE per row, 32 rows per
    // warp at a time -- the row sums are short, so rows, not columns, carry the parallelism.
    // Longer ones: four lanes per row or a warp per row (precond_rows.cuh kQuarterPartials).
    // Which summation a row gets depends on its matrix's N alone (reading R11); the host
    // flags which kinds the launch holds (bit 5 one lane, bit 3 four lanes, bit 4 a warp per
    // row), and only those loops run.
    if (mode & 32) {
      for (int64_t row0 = r_beg; row0 < r_end; row0 += 32) {
        const int64_t row = row0 + lane;
        if (row < r_end) {
          const int jb = find_pjob(jobs, njobs, row);
          const PrecondJob& J = jobs[jb];
          if (J.part_ld <= kSeqPartials) {
            const int i = (int)(row - J.row_start);
            const float r = aol_rowsum_partials(J, i);
            J.s[i] = r > 0.f ? rsqrtf(r) : 0.f;
            if (!(r > 0.f)) fl |= 1u;
            if (!isfinite(r)) fl |= 2u;
          }
        }
      }
    }
    const unsigned kinds = ((mode & 8) ? 1u : 0u) | ((mode & 16) ? 2u : 0u);
    if (kinds & 1u) {  // four lanes per row, 8 rows at a time
      const int qt = lane >> 3;
      for (int64_t row0 = r_beg; row0 < r_end; row0 += 8) {
        const int64_t row = row0 + (lane & 7);
        float v = 0.f;
        bool mine = false;
        int jb = 0, i = 0;
        if (row < r_end) {
          jb = find_pjob(jobs, njobs, row);
          mine = jobs[jb].part_ld > kSeqPartials && jobs[jb].part_ld <= kQuarterPartials;
          i = (int)(row - jobs[jb].row_start);
          if (mine) v = aol_rowsum_quarter(jobs[jb], i, qt);
        }
        const float q1 = __shfl_sync(0xffffffffu, v, (lane & 7) + 8);   // quarters 1..3 of
        const float q2 = __shfl_sync(0xffffffffu, v, (lane & 7) + 16);  // this lane's row,
        const float q3 = __shfl_sync(0xffffffffu, v, (lane & 7) + 24);  // added in order
        if (mine && qt == 0) {
          const float r = ((v + q1) + q2) + q3;
          const PrecondJob& J = jobs[jb];
          J.s[i] = r > 0.f ? rsqrtf(r) : 0.f;
          if (!(r > 0.f)) fl |= 1u;
          if (!isfinite(r)) fl |= 2u;
        }
      }
    }
    if (kinds & 2u) {  // one warp per row (two rows of a matrix at a time)
      int jb = find_pjob(jobs, njobs, r_beg);
      for (int64_t row = r_beg; row < r_end;) {
        while (jb + 1 < njobs && jobs[jb + 1].row_start <= row) ++jb;
        const PrecondJob& J = jobs[jb];
        if (J.part_ld <= kQuarterPartials) { ++row; continue; }
        const int i = (int)(row - J.row_start);
        float r[2];
        int nr = 1;
        if (row + 1 < r_end && i + 1 < J.N) {
          aol_rowsum_tree2(J, i, i + 1, lane, r[0], r[1]);
          nr = 2;
        } else {
          r[0] = aol_rowsum_tree(J, i, lane);
        }
        if (lane == 0)
          for (int u = 0; u < nr; ++u) {
            J.s[i + u] = r[u] > 0.f ? rsqrtf(r[u]) : 0.f;
            if (!(r[u] > 0.f)) fl |= 1u;
            if (!isfinite(r[u])) fl |= 2u;
          }
        row += nr;
      }
    }
  } else if (r_beg < r_end) {
    int jb = find_pjob(jobs, njobs, r_beg);
    for (int64_t row = r_beg; row < r_end; ++row) {
      while (jb + 1 < njobs && jobs[jb + 1].row_start <= row) ++jb;
      precond_row_s<T, VEC8>(jobs[jb], (int)(row - jobs[jb].row_start), lane, fl);
    }
  }
  grid_barrier(barrier);
  // ---- phase 2: A1 = diag(s) A0 diag(s)  (Alg. 2 l.4).  Work is counted in 256-column
  // segments of stored rows (precond_segments): each warp takes an equal contiguous run of
  // segments -- equal bytes per warp under half storage, whatever the mix of matrix sizes --
  // ordered down 256-column strips (precond_seg_pos), 8 rows per lane in flight.
  const int64_t sper = (mode & 4) ? 0 : (total_segs + nwarps - 1) / nwarps;
  int64_t g = gwarp * sper;
  const int64_t g_end = min(total_segs, g + sper);
  if (g < g_end) {
    int jb = find_seg_job(jobs, njobs, g);
    SegPos sp;
    int r;
    precond_seg_pos(jobs[jb].N, jobs[jb].half, g - jobs[jb].seg_start, sp, r);
    while (g < g_end) {
      const PrecondJob& J = jobs[jb];
      const int cnt = (int)min((int64_t)(sp.rows - r), g_end - g);
      precond_strip<T, VEC8>(J, sp, r, cnt, lane);
      g += cnt;
      r += cnt;
      if (g < g_end && r >= sp.rows) {  // next strip (or the next matrix)
        if (g >= jobs[jb].seg_start + precond_segments(J.N, J.half)) ++jb;
        precond_seg_pos(jobs[jb].N, jobs[jb].half, g - jobs[jb].seg_start, sp, r);
      }
    }
  }
  if (fl) atomicOr(flags, fl);
}

template <typename T, bool V>
static cudaError_t launch_precond_t(const PrecondJob* d_jobs, int njobs, int64_t total_rows,
                                    int64_t total_segs, unsigned* d_barrier, uint32_t* d_flags,
                                    int lane_rows, cudaStream_t stream) {
  auto kern = precondition_kernel<T, V>;
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, 0);
  if (occ < 1) occ = 1;
  static const int occ_cap = [] { const char* e = getenv("TNS_PRE_OCC"); return e ? atoi(e) : 0; }();  // A/B knob
  if (occ_cap > 0 && occ_cap < occ) occ = occ_cap;
  // one warp per row (phase 1) and per 4 segments (phase 2), at most the co-resident grid
  // (cooperative launch: the grid barrier needs every CTA resident)
  const int64_t warps = std::max<int64_t>(total_rows, (total_segs + 3) / 4);
  const int64_t want = (warps * 32 + 255) / 256;
  int64_t cap = (int64_t)sms * occ;
  int grid = (int)(want < cap ? (want < 1 ? 1 : want) : cap);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  static const int dbg = [] { const char* e = getenv("TNS_PRE_DBG"); return e ? atoi(e) : 0; }();
  const int lr = lane_rows;
  return cudaLaunchKernelEx(&cfg, kern, d_jobs, njobs, total_rows, total_segs, d_barrier, d_flags,
                            lr | (dbg & 6));
}

// ------------------------------------------------------------------------------ split-K Gram
// A = rnd(sum_s ws[s]) for the split-K Gram of tile-starved launches (SplitJob, jobs.h): one
// warp per row, lanes over 8-column groups (N <= 256: one pass), partials summed in the
// fixed order s = 0..S-1 (deterministic); AOL row sums of the rounded |A0| (Eq. 8) from the
// same registers.  L2-resident: the partials were written by the immediately preceding Gram.
__global__ void __launch_bounds__(256)
    split_reduce_kernel(const SplitJob* __restrict__ jobs, int njobs, int64_t total_rows,
                        uint32_t* __restrict__ flags) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the partials come from the Gram launch
  const int lane = threadIdx.x & 31;
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= total_rows) return;
  int lo = 0, hi = njobs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].row_start <= row) lo = mid; else hi = mid - 1;
  }
  const SplitJob& J = jobs[lo];
  const int i = (int)(row - J.row_start);
  float rs = 0.f;
  bool bad = false;
  for (int c0 = lane * 8; c0 < J.N; c0 += 256) {
    float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const float* src = J.ws + (int64_t)i * J.ld + c0;
    for (int sp = 0; sp < J.S; ++sp) {
      const float4 u0 = __ldcg(reinterpret_cast<const float4*>(src + sp * J.stride));
      const float4 u1 = __ldcg(reinterpret_cast<const float4*>(src + sp * J.stride + 4));
      v[0] += u0.x; v[1] += u0.y; v[2] += u0.z; v[3] += u0.w;
      v[4] += u1.x; v[5] += u1.y; v[6] += u1.z; v[7] += u1.w;
    }
    uint16_t h[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      h[e] = __bfloat16_as_ushort(__float2bfloat16_rn(v[e]));
      const float r = __uint_as_float((uint32_t)h[e] << 16);
      rs += fabsf(r);
      bad |= !isfinite(r);
    }
    uint4 w;
    w.x = h[0] | ((uint32_t)h[1] << 16); w.y = h[2] | ((uint32_t)h[3] << 16);
    w.z = h[4] | ((uint32_t)h[5] << 16); w.w = h[6] | ((uint32_t)h[7] << 16);
    *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(J.A) + (int64_t)i * J.N + c0) = w;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);
  if (J.part != nullptr && lane == 0) J.part[part_at(J.part_ld, J.part_sm, J.N, i, 0)] = rs;
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, 2u);
}

cudaError_t launch_split_reduce(const SplitJob* d_jobs, int njobs, int64_t total_rows, uint32_t* d_flags,
                                cudaStream_t stream) {
  if (total_rows <= 0) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((total_rows + 7) / 8));
  cfg.blockDim = dim3(256);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, split_reduce_kernel, d_jobs, njobs, total_rows, d_flags);
}

cudaError_t launch_precondition(const PrecondJob* d_jobs, int njobs, int64_t total_rows,
                                int64_t total_segs, bool vec8, bool is_bf16, unsigned* d_barrier,
                                uint32_t* d_flags, int lane_mode, cudaStream_t stream) {
  const int lr = lane_mode & (1 | 8 | 16 | 32);
  if (is_bf16) {
    return vec8 ? launch_precond_t<uint16_t, true>(d_jobs, njobs, total_rows, total_segs, d_barrier, d_flags, lr, stream)
                : launch_precond_t<uint16_t, false>(d_jobs, njobs, total_rows, total_segs, d_barrier, d_flags, lr, stream);
  }
  return launch_precond_t<float, false>(d_jobs, njobs, total_rows, total_segs, d_barrier, d_flags, lr, stream);
}

}  // namespace tns
