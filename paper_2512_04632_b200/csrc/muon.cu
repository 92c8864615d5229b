// The Muon optimizer step around the NS path (PAPER.md P:L16, L97,
// L311-315: "momentum -> orthogonalize -> update" with Turbo-Muon as a drop-in NS):
//   muon_momentum_kernel : M <- beta M + (1-beta) G ;  U <- nesterov ? (1-beta) G + beta M : M
//                          (U in bf16 = the NS input, orthogonalised in place afterwards)
//   muon_apply_kernel    : W <- W (1 - lr wd) - lr * max(1, m/n)^(1/2) * U
// Both are HBM-bound elementwise passes, grouped over all matrices of a step (blockIdx.y =
// matrix), 4 elements per thread with vector loads when aligned.  Reading R13.
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

template <typename TG>
__global__ void __launch_bounds__(256) muon_momentum_kernel(const MuonJob* __restrict__ jobs, float beta,
                                                            int nesterov) {
  const MuonJob J = jobs[blockIdx.y];
  const TG* G = reinterpret_cast<const TG*>(J.G);
  uint16_t* U = reinterpret_cast<uint16_t*>(J.U);
  const float ob = 1.0f - beta;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < J.numel; i += stride) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (i + e >= J.numel) break;
      const float g = ldf<TG>(G, i + e);
      const float m = fmaf(beta, J.M[i + e], ob * g);
      J.M[i + e] = m;
      U[i + e] = tobf(nesterov ? fmaf(ob, g, beta * m) : m);
    }
  }
}

template <typename TW>
__global__ void __launch_bounds__(256) muon_apply_kernel(const MuonJob* __restrict__ jobs, float lr, float wd) {
  const MuonJob J = jobs[blockIdx.y];
  TW* W = reinterpret_cast<TW*>(J.W);
  const uint16_t* O = reinterpret_cast<const uint16_t*>(J.U);
  const float keep = 1.0f - lr * wd, step = lr * J.scale;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < J.numel; i += stride) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (i + e >= J.numel) break;
      stf<TW>(W, i + e, fmaf(-step, bfv(O[i + e]), ldf<TW>(W, i + e) * keep));
    }
  }
}

static dim3 muon_grid(int64_t max_numel, int count, int sms) {
  int64_t want = (max_numel + 1023) / 1024;
  const int64_t cap = (int64_t)sms * 8 / (count > 0 ? count : 1) + 1;
  if (want > cap) want = cap;
  if (want < 1) want = 1;
  return dim3((unsigned)want, (unsigned)count);
}

cudaError_t launch_muon_momentum(const MuonJob* d_jobs, int count, int64_t max_numel, bool g_bf16, float beta,
                                 int nesterov, int sms, cudaStream_t stream) {
  const dim3 grid = muon_grid(max_numel, count, sms);
  if (g_bf16) muon_momentum_kernel<uint16_t><<<grid, 256, 0, stream>>>(d_jobs, beta, nesterov);
  else muon_momentum_kernel<float><<<grid, 256, 0, stream>>>(d_jobs, beta, nesterov);
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
