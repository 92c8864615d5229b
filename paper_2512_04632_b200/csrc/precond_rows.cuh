// Work units of the AOL / Frobenius preconditioner kernel (simt.cu; Eqs. 7-11,
// Alg. 2 l.2-4).  Phase 1 (scaling vector s): one warp per row of one matrix.  Phase 2
// (A1 = diag(s) A0 diag(s)): one warp per 256-column segment of a stored row, so every warp
// moves the same bytes whatever the matrix sizes and the half storage.
#pragma once
#include <cuda_bf16.h>

#include "jobs.h"

namespace tns {

template <typename T> __device__ __forceinline__ float ld_val(const T* p);
template <> __device__ __forceinline__ float ld_val<float>(const float* p) { return *p; }
template <> __device__ __forceinline__ float ld_val<uint16_t>(const uint16_t* p) {
  return __uint_as_float(((uint32_t)*p) << 16);
}
template <typename T> __device__ __forceinline__ T st_conv(float f);
template <> __device__ __forceinline__ float st_conv<float>(float f) { return f; }
template <> __device__ __forceinline__ uint16_t st_conv<uint16_t>(float f) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

__device__ __forceinline__ int find_pjob(const PrecondJob* __restrict__ jobs, int njobs, int64_t v) {
  int lo = 0, hi = njobs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].row_start <= v) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// AOL row sum of |A0| for row i from the Gram epilogue's partials: direct 64-column slots
// of the blocks <= bi, mirrored 32-row slots of the blocks > bi (each |A0_ij| counted once),
// summed sequentially in slot order (independent loads, fixed order: deterministic).
__device__ __forceinline__ float aol_rowsum_partials(const PrecondJob& J, int i) {
  const int N = J.N, bi = i / 256;
  const int n1 = (N + 63) / 64, n2 = (N + 31) / 32;
  const int d_end = min(4 * (bi + 1), n1), m_beg = min(8 * (bi + 1), n2);
  // the row's slots as one list (direct ones, then mirrored ones), loaded up to 32 at a time and
  // added in list order (the zeros past the end add nothing): the same sum, bitwise, as a
  // plain sequential loop -- in one L2 round trip for N <= 1024 instead of one per slot
  const int nd = d_end, nt = d_end + (n2 - m_beg);
  float acc = 0.f;
  for (int t0 = 0; t0 < nt; t0 += 32) {
    float v[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      const int t = t0 + e;
      v[e] = t < nd ? J.part[part_at(J.part_ld, J.part_sm, N, i, t)]
                    : (t < nt ? J.part[part_at(J.part_ld, J.part_sm, N, i, n1 + m_beg + (t - nd))] : 0.f);
    }
#pragma unroll
    for (int e = 0; e < 32; ++e) acc += v[e];
  }
  return acc;
}

// How the AOL row sums of a matrix are formed from its partials (a function of N alone,
// reading R11): part_ld <= kSeqPartials (N <= 1344) one lane per row, slots in order;
// <= kQuarterPartials (N <= 5440) four lanes per row, a contiguous quarter of the slot list
// each, the quarters added in order (both slot-major: consecutive rows in consecutive lanes);
// beyond, one warp per row over the row-major slots, lane-strided and a fixed tree.  (Measured:
// four lanes beat the warp tree at 2048^2 / 4096^2, lose at 8192^2, where every row is long
// and a warp per row keeps its loads in whole 128-byte lines.)
// (kQuarterPartials, precond_part_sm: jobs.h)
// Quarter qt of the slot list of row i (kSeqPartials < part_ld <= kQuarterPartials): list
// positions [qt c, min(nt, (qt + 1) c)), c = ceil(nt / 4), summed in order, 32 loads in flight.
__device__ __forceinline__ float aol_rowsum_quarter(const PrecondJob& J, int i, int qt) {
  const int N = J.N, bi = i / 256;
  const int n1 = (N + 63) / 64, n2 = (N + 31) / 32;
  const int d_end = min(4 * (bi + 1), n1), m_beg = min(8 * (bi + 1), n2);
  const int nd = d_end, nt = d_end + (n2 - m_beg);
  const int c = (nt + 3) / 4, t_beg = qt * c, t_end = min(nt, t_beg + c);
  float acc = 0.f;
  for (int t0 = t_beg; t0 < t_end; t0 += 32) {
    float v[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      const int t = t0 + e;
      v[e] = t < t_end ? (t < nd ? J.part[part_at(J.part_ld, J.part_sm, N, i, t)]
                                 : J.part[part_at(J.part_ld, J.part_sm, N, i, n1 + m_beg + (t - nd))])
                       : 0.f;
    }
#pragma unroll
    for (int e = 0; e < 32; ++e) acc += v[e];
  }
  return acc;
}
// Warp-wide row sum (part_ld > kQuarterPartials, row-major partials): lane k sums slots k,
// k + 32, ... of the list in that order, then a fixed xor tree; every lane returns the sum.
__device__ __forceinline__ float aol_rowsum_tree(const PrecondJob& J, int i, int lane) {
  const int bi = i / 256;
  const int n1 = (J.N + 63) / 64, n2 = (J.N + 31) / 32;
  const float* pr = J.part + (int64_t)i * J.part_ld;
  const int d_end = min(4 * (bi + 1), n1), m_beg = min(8 * (bi + 1), n2);
  float acc = 0.f;
  for (int k0 = lane; k0 < d_end; k0 += 256) {
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = (k0 + 32 * e < d_end) ? pr[k0 + 32 * e] : 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc += v[e];
  }
  for (int k0 = m_beg + lane; k0 < n2; k0 += 256) {
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = (k0 + 32 * e < n2) ? pr[n1 + k0 + 32 * e] : 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc += v[e];
  }
  return warp_sum(acc);
}

// Two rows of one matrix at once (the loads of both in flight together); each row's sum is
// formed exactly as aol_rowsum_tree forms it (same per-lane order, same tree).
__device__ __forceinline__ void aol_rowsum_tree2(const PrecondJob& J, int i0, int i1, int lane, float& r0, float& r1) {
  const int n1 = (J.N + 63) / 64, n2 = (J.N + 31) / 32;
  const float* p0 = J.part + (int64_t)i0 * J.part_ld;
  const float* p1 = J.part + (int64_t)i1 * J.part_ld;
  const int b0 = i0 / 256, b1 = i1 / 256;
  const int d0 = min(4 * (b0 + 1), n1), m0 = min(8 * (b0 + 1), n2);
  const int d1 = min(4 * (b1 + 1), n1), m1 = min(8 * (b1 + 1), n2);
  float a0 = 0.f, a1 = 0.f;
  for (int k0 = lane; k0 < max(d0, d1); k0 += 256) {
    float v0[8], v1[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      v0[e] = (k0 + 32 * e < d0) ? p0[k0 + 32 * e] : 0.f;
      v1[e] = (k0 + 32 * e < d1) ? p1[k0 + 32 * e] : 0.f;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) { a0 += v0[e]; a1 += v1[e]; }
  }
  // the mirrored slots: each row walks its own range m.. n2 in steps of 256 from m + lane
  for (int j = 0; m0 + lane + j < n2 || m1 + lane + j < n2; j += 256) {
    float v0[8], v1[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int k0 = m0 + lane + j + 32 * e, k1 = m1 + lane + j + 32 * e;
      v0[e] = (k0 < n2) ? p0[n1 + k0] : 0.f;
      v1[e] = (k1 < n2) ? p1[n1 + k1] : 0.f;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) { a0 += v0[e]; a1 += v1[e]; }
  }
  r0 = warp_sum(a0);
  r1 = warp_sum(a1);
}

// Phase 1 for row i: s_i (AOL, Eq. 8) or, for row 0, the whole Frobenius s (Eq. 10).
// Fixed-order reductions: deterministic.
template <typename T, bool VEC8>
__device__ __forceinline__ void precond_row_s(const PrecondJob& J, int i, int lane, uint32_t& fl) {
  const T* __restrict__ A = reinterpret_cast<const T*>(J.A);
  const int N = J.N;
  // (AOL from the Gram epilogue's partials runs in the kernel's lane loop instead:
  // aol_rowsum_partials / aol_rowsum_quarter / aol_rowsum_tree)
  if (J.precond == 2) {  // AOL from A0 itself: s_i = (sum_j |A0_ij|)^(-1/2)
    float acc = 0.f;
    const T* Ai = A + (int64_t)i * N;
    if (VEC8 && sizeof(T) == 2) {
      for (int j = lane * 8; j < N; j += 256) {
        const uint4 u = *reinterpret_cast<const uint4*>(Ai + j);
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          acc += fabsf(__uint_as_float(w[e] << 16));
          acc += fabsf(__uint_as_float(w[e] & 0xFFFF0000u));
        }
      }
    } else {
      for (int j = lane; j < N; j += 32) acc += fabsf(ld_val<T>(Ai + j));
    }
    const float r = warp_sum(acc);
    if (lane == 0) {
      J.s[i] = r > 0.f ? rsqrtf(r) : 0.f;
      if (!(r > 0.f)) fl |= 1u;
      if (!isfinite(r)) fl |= 2u;
    }
  } else if (i == 0) {  // Frobenius: s = 1/sqrt(trace A0) = 1/||X||_F, one warp per matrix
    float acc = 0.f;
    for (int j = lane; j < N; j += 32) acc += ld_val<T>(A + (int64_t)j * N + j);
    const float tr = warp_sum(acc);
    const float sv = tr > 0.f ? rsqrtf(tr) : 0.f;
    for (int j = lane; j < N; j += 32) J.s[j] = sv;
    if (lane == 0 && !(tr > 0.f)) fl |= 1u;
    if (lane == 0 && !isfinite(tr)) fl |= 2u;
  }
}

// Phase 2 work order.  A stored row is cut into 256-column segments; with half storage
// row i (in 256-block bi) holds columns [0, min(N, 256 (bi + 1))), i.e. bi + 1 segments, else
// ceil(N / 256) (precond_segments, jobs.h).  Segments are numbered strip by strip: block row
// bi (half storage; the whole matrix otherwise), then column segment cb, then the row -- so a
// warp's run of consecutive segments walks DOWN a 256-column strip: s_j of its columns is
// loaded once per strip and each row of the strip is one coalesced 512-byte access.
struct SegPos { int row0, rows, cb; };  // strip = rows [row0, row0 + rows) x segment cb
__device__ __forceinline__ void precond_seg_pos(int N, int half, int64_t g, SegPos& sp, int& r) {
  if (!half) {
    sp.row0 = 0; sp.rows = N;
    sp.cb = (int)(g / N);
    r = (int)(g % N);
    return;
  }
  // block row bi starts at segment 128 bi (bi + 1) (all earlier block rows are full)
  int bi = (int)((sqrtf(1.f + (float)g / 32.f) - 1.f) * 0.5f);
  while (bi > 0 && 128 * (int64_t)bi * (bi + 1) > g) --bi;
  while (128 * (int64_t)(bi + 1) * (bi + 2) <= g) ++bi;
  const int64_t q = g - 128 * (int64_t)bi * (bi + 1);
  sp.row0 = 256 * bi;
  sp.rows = min(256, N - 256 * bi);
  sp.cb = (int)(q / sp.rows);
  r = (int)(q % sp.rows);
}

// Phase 2 for rows [r, r + cnt) of a strip: A1[i][c..c+256) = s_i A0[i][c..c+256) s_c..
// (Alg. 2 l.4).  Lane owns columns c + 8 lane .. + 8 (one 16-byte vector in bf16) with their
// s_j in registers; 8 rows in flight (all loads of a batch before any store).
template <typename T, bool VEC8>
__device__ __forceinline__ void precond_strip(const PrecondJob& J, const SegPos& sp, int r, int cnt, int lane) {
  const int c0 = sp.cb * 256;
  const int lim = J.half ? min(J.N, sp.row0 + 256) : J.N;  // stored columns of these rows
  if (VEC8 && sizeof(T) == 2) {
    const int j = c0 + lane * 8;
    if (j >= lim) return;
    const float4 s0 = *reinterpret_cast<const float4*>(J.s + j);
    const float4 s1 = *reinterpret_cast<const float4*>(J.s + j + 4);
    const float sj[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
    uint16_t* base = reinterpret_cast<uint16_t*>(J.A) + j;
#ifndef TNS_PRE_ROWS
#define TNS_PRE_ROWS 6
#endif
    constexpr int kR = TNS_PRE_ROWS;
    for (int i0 = sp.row0 + r; i0 < sp.row0 + r + cnt; i0 += kR) {
      const int n = min(kR, sp.row0 + r + cnt - i0);
      uint4 u[kR];
      float si[kR];
#pragma unroll
      for (int v = 0; v < kR; ++v)
        if (v < n) {
          u[v] = *reinterpret_cast<const uint4*>(base + (int64_t)(i0 + v) * J.N);
          si[v] = J.s[i0 + v];
        }
#pragma unroll
      for (int v = 0; v < kR; ++v)
        if (v < n) {
          uint32_t w[4] = {u[v].x, u[v].y, u[v].z, u[v].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float lo = (si[v] * __uint_as_float(w[e] << 16)) * sj[2 * e];
            const float hi = (si[v] * __uint_as_float(w[e] & 0xFFFF0000u)) * sj[2 * e + 1];
            w[e] = (uint32_t)st_conv<uint16_t>(lo) | ((uint32_t)st_conv<uint16_t>(hi) << 16);
          }
          *reinterpret_cast<uint4*>(base + (int64_t)(i0 + v) * J.N) = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
  } else {
    T* A = reinterpret_cast<T*>(J.A);
    for (int i = sp.row0 + r; i < sp.row0 + r + cnt; ++i) {
      const float si = J.s[i];
      for (int jj = c0 + lane; jj < min(c0 + 256, lim); jj += 32)
        A[(int64_t)i * J.N + jj] = st_conv<T>((si * ld_val<T>(A + (int64_t)i * J.N + jj)) * J.s[jj]);
    }
  }
}

}  // namespace tns
