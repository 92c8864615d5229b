// CUDA-core kernels:
//   * simt_gemm_kernel  -- the three NS products (Eqs. 3-5) with the same fused epilogues
//     as the tcgen05 engine, for the fp32 "exact" mode (fp32 storage, fp32 FFMA) and for
//     bf16 shapes that TMA cannot address (row pitch not a multiple of 16 bytes).
//   * precondition_kernel -- the fused AOL preconditioner (Eqs. 7-9, Alg. 2 l.2-4):
//     phase 1: one warp per row of A0, s_i = rsqrt(sum_j |A0_ij|) (Eq. 8) with vectorised
//     16-byte loads and a fixed-order warp-shuffle reduction (deterministic); Frobenius:
//     s = rsqrt(trace A0) = 1/||X||_F (Eq. 10);  grid barrier;  phase 2: A1 = s_i A0_ij s_j
//     in place (Alg. 2 l.4, "Update A to avoid recomputation").  HBM-bound.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "jobs.h"
#include "kernels.h"

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

// ------------------------------------------------------------------------------ SIMT GEMM
template <typename T>
__global__ void __launch_bounds__(256)
    simt_gemm_kernel(const SimtJob* __restrict__ jobs, int njobs, int64_t total_tiles,
                     uint32_t* __restrict__ flags) {
  constexpr int TILE = kSimtTile, KT = 16;
  __shared__ float As[KT][TILE + 4];
  __shared__ float Bs[KT][TILE + 4];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  bool bad = false;
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
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int idx = tid + e * 256;
        int pp, kk;
        if (J.sa_p == 1) { pp = idx & 63; kk = idx >> 6; } else { kk = idx & 15; pp = idx >> 4; }
        const int gp = p0 + pp, gk = k0 + kk;
        As[kk][pp] = (gp < J.P && gk < J.K) ? ld_val<T>(A + gp * J.sa_p + gk * J.sa_k) : 0.f;
        int qq, kq;
        if (J.sb_q == 1) { qq = idx & 63; kq = idx >> 6; } else { kq = idx & 15; qq = idx >> 4; }
        const int gq = q0 + qq, gk2 = k0 + kq;
        Bs[kq][qq] = (gq < J.Q && gk2 < J.K) ? ld_val<T>(B + gq * J.sb_q + gk2 * J.sb_k) : 0.f;
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
  if (is_bf16)
    simt_gemm_kernel<uint16_t><<<grid, 256, 0, stream>>>(d_jobs, njobs, total_tiles, d_flags);
  else
    simt_gemm_kernel<float><<<grid, 256, 0, stream>>>(d_jobs, njobs, total_tiles, d_flags);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------ preconditioner
__device__ __forceinline__ int find_pjob(const PrecondJob* __restrict__ jobs, int njobs,
                                         int64_t v, bool by_row) {
  int lo = 0, hi = njobs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    const int64_t st = by_row ? jobs[mid].row_start : jobs[mid].vec_start;
    if (st <= v) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Self-resetting grid barrier (all CTAs co-resident: cooperative launch).  bar[0] counts
// arrivals, bar[1] is a generation number; the last arriver resets the count and bumps the
// generation, so no host-side reset (memset) is needed between launches.
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
__global__ void __launch_bounds__(256)
    precondition_kernel(const PrecondJob* __restrict__ jobs, int njobs, int64_t total_rows,
                        int64_t total_items, unsigned* barrier, uint32_t* __restrict__ flags) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");  // A0 comes from the preceding Gram launch
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint32_t fl = 0;

  (void)total_items;
  // ---- phase 1: scaling vector s (Eq. 8 / Eq. 10)
  for (int64_t row = gwarp; row < total_rows; row += nwarps) {
    const PrecondJob& J = jobs[find_pjob(jobs, njobs, row, true)];
    const int i = (int)(row - J.row_start);
    const T* __restrict__ A = reinterpret_cast<const T*>(J.A);
    const int N = J.N;
    if (J.precond == 2 && J.part != nullptr) {
      // AOL from the Gram epilogue's partials: direct 128-column slots of blocks <= bi,
      // mirrored 32-row slots of blocks > bi (each |A0_ij| counted exactly once)
      const int bi = i / 256;
      const int n1 = (N + 127) / 128, n2 = (N + 31) / 32;
      const float* pr = J.part + (int64_t)i * J.part_ld;
      const int d_end = min(2 * (bi + 1), n1), m_beg = min(8 * (bi + 1), n2);
      float acc = 0.f;
      for (int k = lane; k < d_end; k += 32) acc += pr[k];
      for (int k = m_beg + lane; k < n2; k += 32) acc += pr[n1 + k];
      const float r = warp_sum(acc);
      if (lane == 0) {
        J.s[i] = r > 0.f ? rsqrtf(r) : 0.f;
        if (!(r > 0.f)) fl |= 1u;
        if (!isfinite(r)) fl |= 2u;
      }
    } else if (J.precond == 2) {  // AOL: s_i = (sum_j |A0_ij|)^(-1/2)
      float acc = 0.f;
      const T* Ai = A + (int64_t)i * N;
      if (VEC8 && sizeof(T) == 2) {
        for (int j = lane * 8; j < N; j += 256) {
          const uint4 u = __ldg(reinterpret_cast<const uint4*>(Ai + j));
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

  grid_barrier(barrier);

  // ---- phase 2: A1 = diag(s) A0 diag(s)  (Alg. 2 l.4), one warp per row: s_i once,
  // 16-byte vectors of A and float4 pairs of s along the row (coalesced, no divisions)
  for (int64_t row = gwarp; row < total_rows; row += nwarps) {
    const PrecondJob& J = jobs[find_pjob(jobs, njobs, row, true)];
    const int i = (int)(row - J.row_start);
    const int N = J.N;
    const float si = J.s[i];
    T* Ai = reinterpret_cast<T*>(J.A) + (int64_t)i * N;
    if (VEC8 && sizeof(T) == 2) {
      for (int j = lane * 8; j < N; j += 256) {
        uint4* pv = reinterpret_cast<uint4*>(Ai + j);
        uint4 u = *pv;
        const float4 s0 = *reinterpret_cast<const float4*>(J.s + j);
        const float4 s1 = *reinterpret_cast<const float4*>(J.s + j + 4);
        const float sj[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
        uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float lo = (si * __uint_as_float(w[e] << 16)) * sj[2 * e];
          const float hi = (si * __uint_as_float(w[e] & 0xFFFF0000u)) * sj[2 * e + 1];
          w[e] = (uint32_t)st_conv<uint16_t>(lo) | ((uint32_t)st_conv<uint16_t>(hi) << 16);
        }
        u.x = w[0]; u.y = w[1]; u.z = w[2]; u.w = w[3];
        *pv = u;
      }
    } else {
      for (int j = lane; j < N; j += 32) Ai[j] = st_conv<T>((si * ld_val<T>(Ai + j)) * J.s[j]);
    }
  }
  if (fl) atomicOr(flags, fl);
}

template <typename T, bool V>
static cudaError_t launch_precond_t(const PrecondJob* d_jobs, int njobs, int64_t total_rows,
                                    int64_t total_items, unsigned* d_barrier, uint32_t* d_flags,
                                    cudaStream_t stream) {
  auto kern = precondition_kernel<T, V>;
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, 0);
  if (occ < 1) occ = 1;
  const int64_t want = (total_rows * 32 + 255) / 256;  // one warp per row
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
  return cudaLaunchKernelEx(&cfg, kern, d_jobs, njobs, total_rows, total_items, d_barrier, d_flags);
}

cudaError_t launch_precondition(const PrecondJob* d_jobs, int njobs, int64_t total_rows,
                                int64_t total_items, bool vec8, bool is_bf16, unsigned* d_barrier,
                                uint32_t* d_flags, cudaStream_t stream) {
  if (is_bf16) {
    return vec8 ? launch_precond_t<uint16_t, true>(d_jobs, njobs, total_rows, total_items, d_barrier, d_flags, stream)
                : launch_precond_t<uint16_t, false>(d_jobs, njobs, total_rows, total_items, d_barrier, d_flags, stream);
  }
  return launch_precond_t<float, false>(d_jobs, njobs, total_rows, total_items, d_barrier, d_flags, stream);
}

}  // namespace tns
