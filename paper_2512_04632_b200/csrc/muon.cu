// The Muon optimizer step around the NS path (PAPER.md P:L16, L97,
// L311-315: "momentum -> orthogonalize -> update" with Turbo-Muon as a drop-in NS):
//   muon_momentum_kernel : G <- gscale G (1/world: the data-parallel mean folded in) ;
//                          M <- beta M + (1-beta) G ;  U <- nesterov ? (1-beta) G + beta M : M
//                          (U in bf16 = the NS input, orthogonalised in place afterwards)
//   muon_apply_kernel    : W <- W (1 - lr wd) - lr * max(1, m/n)^(1/2) * U
// Both are HBM-bound elementwise passes, grouped over all matrices of a step (blockIdx.y =
// matrix), 8 elements per thread with 16-byte vector accesses when aligned.  Reading R13.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"

namespace tns {

__device__ __forceinline__ float bfv(uint16_t h) { return __uint_as_float(((uint32_t)h) << 16); }
__device__ __forceinline__ uint16_t tobf(float f) { return __bfloat16_as_ushort(__float2bfloat16_rn(f)); }

template <typename T> __device__ __forceinline__ float ldf(const T* p, int64_t i);
template <> __device__ __forceinline__ float ldf<float>(const float* p, int64_t i) { return p[i]; }
template <> __device__ __forceinline__ float ldf<uint16_t>(const uint16_t* p, int64_t i) { return bfv(p[i]); }
template <typename T> __device__ __forceinline__ void stf(T* p, int64_t i, float v);
template <> __device__ __forceinline__ void stf<float>(float* p, int64_t i, float v) { p[i] = v; }
template <> __device__ __forceinline__ void stf<uint16_t>(uint16_t* p, int64_t i, float v) { p[i] = tobf(v); }

// 8 consecutive elements as fp32 (16-byte vector loads / stores; the caller checks alignment)
__device__ __forceinline__ void ld8(const float* p, float (&v)[8]) {
  const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void ld8(const uint16_t* p, float (&v)[8]) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    v[2 * e] = __uint_as_float(w[e] << 16);
    v[2 * e + 1] = __uint_as_float(w[e] & 0xFFFF0000u);
  }
}
__device__ __forceinline__ void st8(float* p, const float (&v)[8]) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
}
__device__ __forceinline__ void st8(uint16_t* p, const float (&v)[8]) {
  uint32_t w[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) w[e] = (uint32_t)tobf(v[2 * e]) | ((uint32_t)tobf(v[2 * e + 1]) << 16);
  *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
}

// Grid-stride over 8-element groups (vec: every buffer of the job is 16-byte aligned and
// numel % 8 == 0; otherwise element by element).  Elementwise, HBM-bound.
template <typename TG>
__global__ void __launch_bounds__(256) muon_momentum_kernel(const MuonJob* __restrict__ jobs, float beta,
                                                            float gscale, int nesterov) {
  const MuonJob J = jobs[blockIdx.y];
  const TG* G = reinterpret_cast<const TG*>(J.G);
  uint16_t* U = reinterpret_cast<uint16_t*>(J.U);
  const float ob = 1.0f - beta;
  const bool vec = ((J.numel & 7) == 0) && !((reinterpret_cast<uintptr_t>(J.G) | reinterpret_cast<uintptr_t>(J.M) |
                                               reinterpret_cast<uintptr_t>(J.U)) & 15);
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  if (vec) {
    for (int64_t i = t0 * 8; i < J.numel; i += nt * 8) {
      float g[8], m[8], u[8];
      ld8(G + i, g);
      ld8(J.M + i, m);
#pragma unroll
      for (int e = 0; e < 8; ++e) g[e] *= gscale;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        m[e] = fmaf(beta, m[e], ob * g[e]);
        u[e] = nesterov ? fmaf(ob, g[e], beta * m[e]) : m[e];
      }
      st8(J.M + i, m);
      st8(U + i, u);
    }
    return;
  }
  for (int64_t i = t0; i < J.numel; i += nt) {
    const float g = ldf<TG>(G, i) * gscale;
    const float m = fmaf(beta, J.M[i], ob * g);
    J.M[i] = m;
    U[i] = tobf(nesterov ? fmaf(ob, g, beta * m) : m);
  }
}

template <typename TW>
__global__ void __launch_bounds__(256) muon_apply_kernel(const MuonJob* __restrict__ jobs, float lr, float wd) {
  const MuonJob J = jobs[blockIdx.y];
  TW* W = reinterpret_cast<TW*>(J.W);
  const uint16_t* O = reinterpret_cast<const uint16_t*>(J.U);
  const float keep = 1.0f - lr * wd, step = lr * J.scale;
  const bool vec = ((J.numel & 7) == 0) && !((reinterpret_cast<uintptr_t>(J.W) | reinterpret_cast<uintptr_t>(J.U)) & 15);
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  if (vec) {
    for (int64_t i = t0 * 8; i < J.numel; i += nt * 8) {
      float w[8], o[8];
      ld8(W + i, w);
      ld8(O + i, o);
#pragma unroll
      for (int e = 0; e < 8; ++e) w[e] = fmaf(-step, o[e], w[e] * keep);
      st8(W + i, w);
    }
    return;
  }
  for (int64_t i = t0; i < J.numel; i += nt) stf<TW>(W, i, fmaf(-step, bfv(O[i]), ldf<TW>(W, i) * keep));
}

__device__ __forceinline__ uint32_t pack_rn(float lo, float hi) {
  return (uint32_t)tobf(lo) | ((uint32_t)tobf(hi) << 16);
}

// fp32 <-> bf16 storage casts of a mixed-precision call, all matrices in one launch
// (blockIdx.y strides over matrices, 8 elements per thread; 16-byte aligned buffers).
template <bool TO_BF16>
__global__ void __launch_bounds__(256) cast_kernel(const CastJob* __restrict__ jobs, int count) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous launch's results
  for (int jb = blockIdx.y; jb < count; jb += gridDim.y) {
    const CastJob J = jobs[jb];
    const int64_t nt = (int64_t)gridDim.x * blockDim.x, t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(J.src) | reinterpret_cast<uintptr_t>(J.dst)) & 15) == 0;
    const int64_t nv = vec ? J.numel / 8 : 0;
    for (int64_t v = t0; v < nv; v += nt) {
      if constexpr (TO_BF16) {
        const float4 a = reinterpret_cast<const float4*>(J.src)[2 * v];
        const float4 b = reinterpret_cast<const float4*>(J.src)[2 * v + 1];
        uint4 w;
        w.x = pack_rn(a.x, a.y); w.y = pack_rn(a.z, a.w); w.z = pack_rn(b.x, b.y); w.w = pack_rn(b.z, b.w);
        reinterpret_cast<uint4*>(J.dst)[v] = w;
      } else {
        const uint4 w = reinterpret_cast<const uint4*>(J.src)[v];
        float4* d = reinterpret_cast<float4*>(J.dst) + 2 * v;
        d[0] = make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xFFFF0000u),
                           __uint_as_float(w.y << 16), __uint_as_float(w.y & 0xFFFF0000u));
        d[1] = make_float4(__uint_as_float(w.z << 16), __uint_as_float(w.z & 0xFFFF0000u),
                           __uint_as_float(w.w << 16), __uint_as_float(w.w & 0xFFFF0000u));
      }
    }
    for (int64_t e = nv * 8 + t0; e < J.numel; e += nt) {
      if constexpr (TO_BF16)
        reinterpret_cast<uint16_t*>(J.dst)[e] =
            __bfloat16_as_ushort(__float2bfloat16_rn(reinterpret_cast<const float*>(J.src)[e]));
      else
        reinterpret_cast<float*>(J.dst)[e] = __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(J.src)[e] << 16);
    }
  }
}

cudaError_t launch_cast(const CastJob* d_jobs, int count, int64_t max_numel, bool to_bf16, int sms,
                        cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  int64_t want = (max_numel + 2047) / 2048;
  const int64_t cap = (int64_t)sms * 8 / count + 1;
  if (want > cap) want = cap;
  if (want < 1) want = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)want, (unsigned)(count < 65535 ? count : 65535));
  cfg.blockDim = dim3(256);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (to_bf16) return cudaLaunchKernelEx(&cfg, cast_kernel<true>, d_jobs, count);
  return cudaLaunchKernelEx(&cfg, cast_kernel<false>, d_jobs, count);
}

static dim3 muon_grid(int64_t max_numel, int count, int sms) {
  int64_t want = (max_numel + 2047) / 2048;  // 8 elements per thread
  const int64_t cap = (int64_t)sms * 8 / (count > 0 ? count : 1) + 1;
  if (want > cap) want = cap;
  if (want < 1) want = 1;
  return dim3((unsigned)want, (unsigned)count);
}

cudaError_t launch_muon_momentum(const MuonJob* d_jobs, int count, int64_t max_numel, bool g_bf16, float beta, float gscale,
                                 int nesterov, int sms, cudaStream_t stream) {
  const dim3 grid = muon_grid(max_numel, count, sms);
  if (g_bf16) muon_momentum_kernel<uint16_t><<<grid, 256, 0, stream>>>(d_jobs, beta, gscale, nesterov);
  else muon_momentum_kernel<float><<<grid, 256, 0, stream>>>(d_jobs, beta, gscale, nesterov);
  return cudaGetLastError();
}

cudaError_t launch_muon_apply(const MuonJob* d_jobs, int count, int64_t max_numel, bool w_bf16, float lr, float wd,
                              int sms, cudaStream_t stream) {
  const dim3 grid = muon_grid(max_numel, count, sms);
  if (w_bf16) muon_apply_kernel<uint16_t><<<grid, 256, 0, stream>>>(d_jobs, lr, wd);
  else muon_apply_kernel<float><<<grid, 256, 0, stream>>>(d_jobs, lr, wd);
  return cudaGetLastError();
}

}  // namespace tns
