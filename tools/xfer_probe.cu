// Measurement only (not part of the library): per-SM transfer rates inside one thread-block
// cluster, to choose how the cluster-resident NS kernel (csrc/cluster_tc.cu) moves its Gram
// partials and A rows.  One cluster of C CTAs (256 threads, like the kernel); each CTA moves
// `bytes` and the cycles from a cluster barrier to completion are recorded (max over CTAs).
//   mode 0  st.global.cg.v4, each warp 512 contiguous bytes per instruction (the kernel's drain)
//   mode 1  smem -> global bulk copies (cp.async.bulk.global.shared::cta), 8 threads x 16 KB pieces
//   mode 2  ld.global.cg.v4 of C slices (the kernel's reduce), 16 loads in flight per thread
//   mode 3  global -> smem bulk copies (C slices, complete_tx), two rounds through 128 KB
//   mode 4  DSMEM bulk copies: bytes / (C - 1) to each peer (the kernel's broadcast)
//   mode 5  global -> smem bulk copies of one shared 128 KB block (every CTA reads the same)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xfer_probe tools/xfer_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t rank_in_cluster() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(a), "r"(par) : "memory");
}

__global__ void __launch_bounds__(256, 1) probe(int mode, int C, uint32_t bytes, float4* gbuf, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t rank = rank_in_cluster();
  const int cl = blockIdx.x / C;
  float4* mine = gbuf + ((size_t)blockIdx.x * bytes) / 16;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (uint32_t i = threadIdx.x; i < 128 * 1024 / 16; i += 256) reinterpret_cast<float4*>(sm)[i] = make_float4(i, 1, 2, 3);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  csync();
  const long long t0 = clock64();
  float acc = 0.f;
  if (mode == 0) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t n = bytes / 512;  // warp-instructions of 512 B
    for (uint32_t i = warp; i < n; i += 8) __stcg(mine + (size_t)i * 32 + lane, make_float4(i, lane, 0, 1));
  } else if (mode == 1) {
    if (threadIdx.x < 8) {
      for (uint32_t off = threadIdx.x * 16384; off < bytes; off += 8 * 16384)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"((uint8_t*)mine + off),
                     "r"(su32(sm + (off & (128 * 1024 - 1)))), "r"(16384u) : "memory");
      asm volatile("cp.async.bulk.commit_group;\n\tcp.async.bulk.wait_group 0;" ::: "memory");
    }
  } else if (mode == 2) {
    // my slice of every CTA's region: bytes / C per source, read in 16-deep batches
    const uint32_t slice = bytes / C;
    const float4* base = gbuf + ((size_t)cl * C * bytes) / 16;
    for (uint32_t u = threadIdx.x; u < slice / 16; u += 256) {
      float4 v[16];
#pragma unroll
      for (int t = 0; t < 16; ++t)
        v[t] = t < C ? __ldcg(base + ((size_t)t * bytes + (size_t)rank * slice) / 16 + u) : make_float4(0, 0, 0, 0);
#pragma unroll
      for (int t = 0; t < 16; ++t) acc += v[t].x + v[t].y + v[t].z + v[t].w;
    }
  } else if (mode == 3 || mode == 5) {
    const uint32_t slice = mode == 3 ? bytes / C : 0;
    const uint8_t* base = reinterpret_cast<const uint8_t*>(gbuf) + (size_t)cl * C * bytes;
    uint32_t par = 0;
    for (uint32_t done = 0; done < bytes; done += 128 * 1024) {
      const uint32_t chunk = bytes - done < 128 * 1024 ? bytes - done : 128 * 1024;
      if (threadIdx.x == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(chunk) : "memory");
      __syncthreads();
      if (threadIdx.x < 8) {
        for (uint32_t off = threadIdx.x * 8192; off < chunk; off += 8 * 8192) {
          const uint32_t g = done + off;  // mode 3: C slices of bytes / C; mode 5: one shared block
          const uint8_t* src = mode == 3 ? base + (size_t)(g / slice) * bytes + rank * slice + g % slice : base + g;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           su32(sm + off)), "l"(src), "r"(8192u), "r"(su32(&bar)) : "memory");
        }
      }
      mbar_wait(su32(&bar), par);
      par ^= 1;
    }
  } else if (mode == 4) {
    const uint32_t per = bytes / (C - 1) / 16 * 16;
    if (threadIdx.x == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(per * (C - 1)) : "memory");
    csync();
    if (threadIdx.x >= 1 && (int)threadIdx.x < C) {
      const uint32_t peer = (rank + threadIdx.x) % C;
      uint32_t rb, dst;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(su32(&bar)), "r"(peer));
      // each sender writes its own region of the receiver's buffer
      const uint32_t src = su32(sm) + rank * (per & ~15u) % (120 * 1024);
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst) : "r"(src), "r"(peer));
      for (uint32_t off = 0; off < per; off += 8192) {
        const uint32_t n = per - off < 8192 ? per - off : 8192;
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         dst + off % 8192), "r"(src + off % 8192), "r"(n), "r"(rb) : "memory");
      }
    }
    mbar_wait(su32(&bar), 0);
  }
  __syncthreads();
  const long long t1 = clock64();
  if (acc == 12345.f) out[1023] = 1;
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  csync();
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int C = argc > 1 ? atoi(argv[1]) : 16;
  const int nclusters = argc > 2 ? atoi(argv[2]) : 1;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  float4* gbuf;
  long long* out;
  const uint32_t maxb = 256 * 1024;
  cudaMalloc(&gbuf, (size_t)maxb * C * nclusters);
  cudaMemset(gbuf, 0, (size_t)maxb * C * nclusters);
  cudaMallocManaged(&out, 1024 * sizeof(long long));
  const char* names[] = {"st.global.cg.v4 drain", "bulk smem->global", "ld.global.cg.v4 x16 reduce",
                         "bulk global->smem slices", "DSMEM bulk to C-1 peers", "bulk global->smem shared block"};
  const uint32_t sizes[] = {64 * 1024, 128 * 1024, 256 * 1024};
  for (int mode = 0; mode < 6; ++mode)
    for (uint32_t b : sizes) {
      if (mode == 4 && b > 120 * 1024) continue;
      if (mode == 5 && b > 128 * 1024) continue;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(C * nclusters);
      cfg.blockDim = dim3(256);
      cfg.dynamicSmemBytes = 200 * 1024;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = C;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      long long best = -1;
      double mean_best = 0;
      for (int rep = 0; rep < 5; ++rep) {
        cudaError_t e = cudaLaunchKernelEx(&cfg, probe, mode, C, b, gbuf, out);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("mode %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
        long long mx = 0;
        double mean = 0;
        for (int i = 0; i < C * nclusters; ++i) { mx = out[i] > mx ? out[i] : mx; mean += out[i]; }
        if (best < 0 || mx < best) { best = mx; mean_best = mean / (C * nclusters); }
      }
      printf("C=%2d clusters=%d %-32s %7u B/CTA: max %7lld cyc (mean %7.0f) = %6.1f B/cyc/SM\n", C, nclusters,
             names[mode], b, best, mean_best, (double)b / best);
    }
  return 0;
}
