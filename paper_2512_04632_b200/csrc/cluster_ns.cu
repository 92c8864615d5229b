// Cluster-resident Newton-Schulz for small matrices (
// small matrices are latency/communication-bound, not FLOP-bound).
//
// One thread-block cluster of C (8 or 16) CTAs runs ALL steps of Alg. 2 for one
// matrix in ONE launch, with every operand resident in shared memory:
//   load Xh (every CTA keeps a full fp32 copy, M x N, of the short-side orientation)
//   for k = 1..T:
//     G: CTA r computes rows R_r of A_k = Xh^T Xh                          (Eq. 3)
//        -> DSMEM broadcast of the rows to every CTA of the cluster, cluster barrier
//        k = 1: s from the full A0 (AOL Eq. 8 row sums / Frobenius Eq. 10 trace),
//               A1 = diag(s) A0 diag(s), X1 = X0 diag(s)     (Alg. 2 l.2-4)
//     P: CTA r computes rows R_r of B_k = b A_k + c A_k A_k                 (Eq. 4)
//        -> DSMEM broadcast, cluster barrier
//     X: CTA r computes its rows of X_{k+1} = a X_k + X_k B_k               (Eq. 5)
//        -> DSMEM broadcast into every CTA's Xh copy, cluster barrier
//   store this CTA's rows of X_{T+1} (caller layout, transposed back for m < n)
// A phase whose full matrix is at least kClL2Bytes (jobs.h) exchanges through an L2 buffer
// instead of DSMEM (each CTA stores its rows once, cluster barrier, every CTA bulk-loads the
// matrix): the same data, measured faster for the larger matrices only.
// Arithmetic is fp32 FFMA; in bf16 mode every stored X, A, B value is rounded to bf16
// (the same storage points as the tcgen05 path, reading R7).  In fp32 mode, when a CTA's own
// rows of X fit its B buffer, P and X fuse into X' = aX + b(XA) + c((XA)A) per row (reading
// R16): B is never formed, one exchange per iteration fewer.  The symmetric operands are
// read through their transposes (A_ik = A_ki, bitwise: the products are computed in the
// same order for (i, k) and (k, i)), so every shared-memory operand load is a 16-byte
// vector along a row.  Reductions have a fixed order: results are deterministic.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "jobs.h"
#include "kernels.h"
#include "ptx.cuh"

namespace tns {

__device__ unsigned long long g_cl_tl[9];  // TNS_DBG bit 128: phase timeline of cluster 0, CTA 0

namespace {

template <typename S> __device__ __forceinline__ float cl_ld(const S* p, int64_t i);
template <> __device__ __forceinline__ float cl_ld<float>(const float* p, int64_t i) { return p[i]; }
template <> __device__ __forceinline__ float cl_ld<uint16_t>(const uint16_t* p, int64_t i) {
  return __uint_as_float(((uint32_t)p[i]) << 16);
}
template <typename S> __device__ __forceinline__ void cl_st(S* p, int64_t i, float v);
template <> __device__ __forceinline__ void cl_st<float>(float* p, int64_t i, float v) { p[i] = v; }
template <> __device__ __forceinline__ void cl_st<uint16_t>(uint16_t* p, int64_t i, float v) {
  p[i] = __bfloat16_as_ushort(__float2bfloat16_rn(v));
}
// storage rounding of an intermediate (bf16 mode: round to nearest even)
template <typename S> __device__ __forceinline__ float rnd(float v);
template <> __device__ __forceinline__ float rnd<float>(float v) { return v; }
template <> __device__ __forceinline__ float rnd<uint16_t>(float v) {
  return __bfloat162float(__float2bfloat16_rn(v));
}

__device__ __forceinline__ uint32_t dsmem_addr(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
// Bulk copy (TMA engine) of a contiguous block of this CTA's shared memory into a peer
// CTA's shared memory; the peer's mbarrier counts the bytes when they land (no cluster-wide
// barrier and no GPU-scope fence on the data path).
__device__ __forceinline__ void dsmem_bulk(uint32_t dst, uint32_t src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "r"(src), "r"(bytes), "r"(bar)
               : "memory");
}
// Bulk copy (TMA engine) global -> this CTA's shared memory, counted on mbarrier `bar`.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void cl_wait(const uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ float cl_warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// C[i][j..j+4) = sum_k L(i, k) R[k][j..j+4) for rows i < rows (in groups of 4) and
// column groups j/4 < cols4, handed to epi(i, j, float4) for i < rows.
//   LT = true : L(i, k) = Lp[k * ldl + i]  (k-major: 16-byte vector over i)
//   LT = false: L(i, k) = Lp[i * ldl + k]  (row-major: 4 scalar loads)
// Thread tiles are 4 x 4; when there are fewer tiles than threads the K range is split
// across up to 8 adjacent lanes (interleaved k) and reduced with a fixed xor tree.
template <bool LT, class Epi>
__device__ __forceinline__ void cl_gemm(const float* __restrict__ Lp, int ldl, const float* __restrict__ R, int ldr,
                                        int rows, int cols4, int K, Epi epi, int dbg) {
  if (dbg & 64) K = 0;
  const int rt = (rows + 3) >> 2;
  const int tiles = rt * cols4;
  if (tiles == 0) return;
  int ks = 1;
  while (ks < 8 && tiles * ks * 2 <= kClThreads) ks <<= 1;
  const int nthr = tiles * ks;
  for (int base = 0; base < nthr; base += kClThreads) {
    const int t = base + (int)threadIdx.x;
    const bool active = t < nthr;
    const int tile = t / ks, part = t % ks;
    const int ti = tile / cols4, tj = tile % cols4;
    float acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] = 0.f;
    if (active) {
      const float* lp = LT ? Lp + ti * 4 : Lp + (size_t)ti * 4 * ldl;
      const float* rp = R + tj * 4;
#pragma unroll 4
      for (int k = part; k < K; k += ks) {
        float l[4];
        if (LT) {
          const float4 lv = *reinterpret_cast<const float4*>(lp + (size_t)k * ldl);
          l[0] = lv.x; l[1] = lv.y; l[2] = lv.z; l[3] = lv.w;
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) l[u] = lp[(size_t)u * ldl + k];
        }
        const float4 rv = *reinterpret_cast<const float4*>(rp + (size_t)k * ldr);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          acc[u][0] = fmaf(l[u], rv.x, acc[u][0]);
          acc[u][1] = fmaf(l[u], rv.y, acc[u][1]);
          acc[u][2] = fmaf(l[u], rv.z, acc[u][2]);
          acc[u][3] = fmaf(l[u], rv.w, acc[u][3]);
        }
      }
    }
    for (int o = 1; o < ks; o <<= 1)
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] += __shfl_xor_sync(0xffffffffu, acc[u][v], o);
    if (active && part == 0) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (ti * 4 + u < rows) epi(ti * 4 + u, tj * 4, make_float4(acc[u][0], acc[u][1], acc[u][2], acc[u][3]));
    }
  }
}

template <typename S, int C>
__global__ void __launch_bounds__(kClThreads, 1)
    cluster_ns_kernel(const ClusterJob* __restrict__ jobs, const float* __restrict__ coeffs, int iters, int precond,
                      uint32_t* __restrict__ flags, int dbg) {
  extern __shared__ float4 cl_smem4[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(cl_smem4);  // data-arrival barriers: 0 A, 1 B, 2 X
  float* sm = reinterpret_cast<float*>(cl_smem4) + kClHdr / 4;
  const ClusterJob J = jobs[blockIdx.x / C];
  const uint32_t rank = cluster_ctarank();
  const ClLayout L = cl_layout(J.M, J.N, C);
  const int M = J.M, N = J.N, lda = L.lda, ldx = L.ldx, C4 = L.N4 / 4;
  float* A = sm + L.offA;
  float* B = sm + L.offB;
  float* Xf = sm + L.offX;
  float* Xn = sm + L.offXn;
  float* s = Xn + (size_t)L.Mr * L.ldx;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kWarps = kClThreads / 32;
  const bool tl = (dbg & 128) && blockIdx.x == 0 && tid == 0;
  const long long T0 = tl ? clock64() : 0;
#define CL_TL(i) do { if (tl) atomicAdd(&g_cl_tl[i], (unsigned long long)(clock64() - T0)); } while (0)
  const int r0 = (int)rank * L.Nr, nr = max(0, min(L.Nr, N - r0));  // this CTA's rows of A, B
  const int o = (int)rank * L.Mr, mr = max(0, min(L.Mr, M - o));    // this CTA's rows of Xh
  uint32_t peer[C], peer_bar[C];
  const uint32_t sm_u32 = smem_u32(sm), bar_u32 = smem_u32(bars);
#pragma unroll
  for (int d = 0; d < C; ++d) {
    peer[d] = dsmem_addr(sm_u32, (uint32_t)d);
    peer_bar[d] = dsmem_addr(bar_u32, (uint32_t)d);
  }
  // After every thread wrote its part of a block: make it visible to the async proxy, then
  // one thread copies the block to sm[dst_off..) of every peer, counted on their barrier b.
  auto publish = [&](int b, size_t dst_off, const float* src, uint32_t bytes) {
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0 && bytes > 0)
      for (int d = 0; d < C; ++d)
        if (d != (int)rank) dsmem_bulk(peer[d] + (uint32_t)(dst_off * 4), smem_u32(src), bytes, peer_bar[d] + 8u * b);
  };
  // bytes each CTA receives per phase: the other CTAs' rows
  const uint32_t bytes_ab = (uint32_t)(N - nr) * lda * 4, bytes_x = (uint32_t)(M - mr) * ldx * 4;
  // Large phases go through L2 instead (kClL2Bytes): every thread stores its share of this
  // CTA's rows [row0, row0 + nrows) into the buffer g; after a cluster barrier the whole
  // matrix [0, total_rows) is bulk-loaded into dst (the own rows included: identical values),
  // completing on barrier b.  A function of the shape: the same choice in every CTA.
  const bool l2_ab = (uint32_t)N * lda * 4 >= kClL2Bytes, l2_x = (uint32_t)M * ldx * 4 >= kClL2Bytes;
  // fp32 mode whose own X rows fit the B buffer: no B phase (reading R16, below)
  constexpr bool kF32 = sizeof(S) == 4;
  const bool reassoc = kF32 && L.Mr <= L.N4;
  auto exchange = [&](int b, float* g, float* dst, const float* src, int row0, int nrows, int total_rows, int ld,
                      uint32_t par) {
    __syncthreads();  // every thread's epilogue rows are in src
    const int n4 = nrows * ld / 4;
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* g4 = reinterpret_cast<float4*>(g + (size_t)row0 * ld);
    for (int e = tid; e < n4; e += kClThreads) __stcg(g4 + e, s4[e]);
    asm volatile("fence.proxy.async.global;" ::: "memory");  // read back by the async proxy
    cluster_sync();  // every CTA's rows are in L2 (release / acquire); all reads of dst are done
    asm volatile("fence.proxy.async.global;" ::: "memory");
    const uint32_t bytes = (uint32_t)total_rows * ld * 4;
    if (tid == 0) mbar_arrive_expect_tx(&bars[b], bytes);
    __syncthreads();  // the expected byte count is registered before any copy can complete
    constexpr uint32_t kPiece = 16384;
    for (uint32_t off = (uint32_t)tid * kPiece; off < bytes; off += kClThreads * kPiece)
      bulk_g2s(smem_u32(dst) + off, reinterpret_cast<const uint8_t*>(g) + off, min(kPiece, bytes - off),
               smem_u32(&bars[b]));
    cl_wait(&bars[b], par);
  };
  float* gA = J.xchg;
  float* gB = gA + (size_t)L.N4 * lda;
  float* gX = gB + (size_t)L.N4 * lda;

  if (tid == 0) {
    for (int b = 0; b < 3; ++b) mbar_init(&bars[b], 1);
    fence_mbar_init();
  }
  // zero everything (padding rows / columns must stay zero), then load the full Xh
  for (size_t i = tid; i < L.floats / 4; i += kClThreads) cl_smem4[kClHdr / 16 + i] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();
  const S* x = reinterpret_cast<const S*>(J.x);
  // flat, coalesced over the caller layout; 8 loads in flight per thread before the stores
  {
    const int total = J.m * J.n, n = J.n;
    const int dr = kClThreads / n, dc = kClThreads % n;  // (row, col) step of one stride
    int sr = tid / n, sc = tid % n;
    for (int e0 = 0; e0 < total; e0 += 8 * kClThreads) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * kClThreads + tid;
        v[u] = e < total ? cl_ld<S>(x, e) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (e0 + u * kClThreads + tid < total)
          Xf[J.wide ? (size_t)sc * ldx + sr : (size_t)sr * ldx + sc] = v[u];
        sr += dr; sc += dc;
        if (sc >= n) { sc -= n; ++sr; }
      }
    }
  }
  cluster_sync();  // every CTA initialised (buffers, barriers) before any DSMEM store reaches it
  CL_TL(0);

  uint32_t fl = 0;
  for (int k = 0; k < iters; ++k) {
    const float a = coeffs[3 * k], b = coeffs[3 * k + 1], c = coeffs[3 * k + 2];
    const uint32_t par = (uint32_t)k & 1u;
    // ---- G: rows [r0, r0+nr) of A = Xh^T Xh  (L(i, kk) = Xh[kk][r0+i]: k-major)
    if (tid == 0 && !l2_ab) mbar_arrive_expect_tx(&bars[0], bytes_ab);
    cl_gemm<true>(Xf + r0, ldx, Xf, ldx, nr, C4, M, [&](int i, int j, float4 v) {
      v.x = rnd<S>(v.x); v.y = rnd<S>(v.y); v.z = rnd<S>(v.z); v.w = rnd<S>(v.w);
      *reinterpret_cast<float4*>(A + (size_t)(r0 + i) * lda + j) = v;
    }, dbg);
    if (l2_ab) {
      exchange(0, gA, A, A + (size_t)r0 * lda, r0, nr, N, lda, par);
    } else {
      publish(0, L.offA + (size_t)r0 * lda, A + (size_t)r0 * lda, (uint32_t)nr * lda * 4);
      cl_wait(&bars[0], par);
    }
    if (k == 0) CL_TL(1);
    if (k == 0 && precond != 0) {
      // A0 is rescaled IN PLACE below, including this CTA's own rows, which the bulk copies
      // of the G phase may still be reading.  Every CTA has received all of A0 once it gets
      // here, so after a cluster barrier all those copies are complete: arrive now, rescale
      // everything but the own rows, wait, then rescale the own rows (the data itself came
      // with complete_tx, so the barrier needs no release fence).
      cluster_arrive_relaxed();
      // every CTA derives the same s from its full copy of A0 (fixed order: identical)
      if (precond == 2) {  // AOL, Eq. 8: s_i = (sum_j |A0_ij|)^(-1/2), 0 for a zero row
        // one thread per row, columns in order (row stride lda: conflict-free 16-byte reads)
        for (int i = tid; i < N; i += kClThreads) {
          const float4* row = reinterpret_cast<const float4*>(A + (size_t)i * lda);
          float s0 = 0.f, s1 = 0.f;
#pragma unroll 4
          for (int q = 0; q < C4; ++q) {
            const float4 v = row[q];
            s0 += fabsf(v.x) + fabsf(v.y);
            s1 += fabsf(v.z) + fabsf(v.w);
          }
          const float rs = s0 + s1;
          s[i] = rs > 0.f ? rsqrtf(rs) : 0.f;
          if (!(rs > 0.f)) fl |= 1u;
          if (!isfinite(rs)) fl |= 2u;
        }
      } else if (warp == 0) {  // Frobenius, Eq. 10: s = 1/sqrt(trace A0) = 1/||X||_F
        float acc = 0.f;
        for (int j = lane; j < N; j += 32) acc += A[(size_t)j * lda + j];
        const float tr = cl_warp_sum(acc);
        const float sv = tr > 0.f ? rsqrtf(tr) : 0.f;
        for (int j = lane; j < N; j += 32) s[j] = sv;
        if (lane == 0 && !(tr > 0.f)) fl |= 1u;
        if (lane == 0 && !isfinite(tr)) fl |= 2u;
      }
      __syncthreads();
      // A1 = diag(s) A0 diag(s) (symmetric product: bitwise symmetric), X1 = X0 diag(s);
      // s is zero beyond N, so the padding stays zero.  Flat over (row, 16-byte column group).
      auto scale4 = [&](float* p, float f, float4 sj) {
        float4 v = *reinterpret_cast<float4*>(p);
        v.x = rnd<S>(v.x * (f * sj.x)); v.y = rnd<S>(v.y * (f * sj.y));
        v.z = rnd<S>(v.z * (f * sj.z)); v.w = rnd<S>(v.w * (f * sj.w));
        *reinterpret_cast<float4*>(p) = v;
      };
      // X: column scaling only (f = 1 keeps the products exact: v * (1 * s_j) = v * s_j)
#pragma unroll 4
      for (int e = tid; e < M * C4; e += kClThreads) {
        const int i = e / C4, q = e - i * C4;
        scale4(Xf + (size_t)i * ldx + 4 * q, 1.f, *reinterpret_cast<const float4*>(s + 4 * q));
      }
      // A: the peers' rows (rows [0, N) minus [r0, r0 + nr))
      const int nother = N - nr;
#pragma unroll 4
      for (int e = tid; e < nother * C4; e += kClThreads) {
        int i = e / C4;
        const int q = e - i * C4;
        i += i >= r0 ? nr : 0;
        scale4(A + (size_t)i * lda + 4 * q, s[i], *reinterpret_cast<const float4*>(s + 4 * q));
      }
      cluster_wait();
      for (int e = tid; e < nr * C4; e += kClThreads) {
        const int i = r0 + e / C4, q = e % C4;
        scale4(A + (size_t)i * lda + 4 * q, s[i], *reinterpret_cast<const float4*>(s + 4 * q));
      }
      __syncthreads();
    }
    if (k == 0) CL_TL(2);
    if (reassoc) {
      // fp32 mode (reading R16): X_{k+1} = a X_k + b (X_k A_k) + c ((X_k A_k) A_k), Eq. 4-5 with
      // the product associated per row -- this CTA's rows need only A_k, so B_k is never
      // formed or exchanged (one row exchange per iteration fewer; no storage rounding in fp32)
      if (tid == 0 && !l2_x) mbar_arrive_expect_tx(&bars[2], bytes_x);
      cl_gemm<false>(Xf + (size_t)o * ldx, ldx, A, lda, mr, C4, N, [&](int i, int j, float4 v) {
        *reinterpret_cast<float4*>(B + (size_t)i * lda + j) = v;  // Y = X_k A_k (own rows)
      }, dbg);
      __syncthreads();
      if (k == 0) CL_TL(3);
      cl_gemm<false>(B, lda, A, lda, mr, C4, N, [&](int i, int j, float4 v) {
        const float4 xv = *reinterpret_cast<const float4*>(Xf + (size_t)(o + i) * ldx + j);
        const float4 yv = *reinterpret_cast<const float4*>(B + (size_t)i * lda + j);
        v.x = fmaf(a, xv.x, fmaf(b, yv.x, c * v.x)); v.y = fmaf(a, xv.y, fmaf(b, yv.y, c * v.y));
        v.z = fmaf(a, xv.z, fmaf(b, yv.z, c * v.z)); v.w = fmaf(a, xv.w, fmaf(b, yv.w, c * v.w));
        *reinterpret_cast<float4*>(Xn + (size_t)i * ldx + j) = v;
      }, dbg);
    } else {
    // ---- P: rows [r0, r0+nr) of B = b A + c A A  (L(i, kk) = A[i][kk] = A[kk][i])
    if (tid == 0 && !l2_ab) mbar_arrive_expect_tx(&bars[1], bytes_ab);
    cl_gemm<true>(A + r0, lda, A, lda, nr, C4, N, [&](int i, int j, float4 v) {
      const float4 av = *reinterpret_cast<const float4*>(A + (size_t)(r0 + i) * lda + j);
      v.x = rnd<S>(fmaf(c, v.x, b * av.x)); v.y = rnd<S>(fmaf(c, v.y, b * av.y));
      v.z = rnd<S>(fmaf(c, v.z, b * av.z)); v.w = rnd<S>(fmaf(c, v.w, b * av.w));
      *reinterpret_cast<float4*>(B + (size_t)(r0 + i) * lda + j) = v;
    }, dbg);
    if (l2_ab) {
      exchange(1, gB, B, B + (size_t)r0 * lda, r0, nr, N, lda, par);
    } else {
      publish(1, L.offB + (size_t)r0 * lda, B + (size_t)r0 * lda, (uint32_t)nr * lda * 4);
      cl_wait(&bars[1], par);
    }
    if (k == 0) CL_TL(3);
    // ---- X: rows [o, o+mr) of X_{k+1} = a X_k + X_k B_k  (L = X_k rows, row-major)
    if (tid == 0 && !l2_x) mbar_arrive_expect_tx(&bars[2], bytes_x);
    cl_gemm<false>(Xf + (size_t)o * ldx, ldx, B, lda, mr, C4, N, [&](int i, int j, float4 v) {
      const float4 xv = *reinterpret_cast<const float4*>(Xf + (size_t)(o + i) * ldx + j);
      v.x = rnd<S>(fmaf(a, xv.x, v.x)); v.y = rnd<S>(fmaf(a, xv.y, v.y));
      v.z = rnd<S>(fmaf(a, xv.z, v.z)); v.w = rnd<S>(fmaf(a, xv.w, v.w));
      *reinterpret_cast<float4*>(Xn + (size_t)i * ldx + j) = v;
    }, dbg);
    }
    if (l2_x) {  // (the exchange's cluster barrier also ends every read of this CTA's X_k rows)
      exchange(2, gX, Xf, Xn, o, mr, M, ldx, par);
      if (k == 0) CL_TL(4);
    } else {
      // (publish's barrier also ends every read of this CTA's X_k rows)
      publish(2, L.offX + (size_t)o * ldx, Xn, (uint32_t)mr * ldx * 4);
      if (k == 0) CL_TL(4);
      for (int e = tid; e < mr * C4; e += kClThreads) {  // own rows: local copy
        const int i = e / C4, j = (e % C4) * 4;
        *reinterpret_cast<float4*>(Xf + (size_t)(o + i) * ldx + j) = *reinterpret_cast<const float4*>(Xn + (size_t)i * ldx + j);
      }
      __syncthreads();
      cl_wait(&bars[2], par);
    }
    if (k == 0) CL_TL(5);
  }
  CL_TL(6);

  // this CTA's rows of the result, in the caller's layout
  S* out = reinterpret_cast<S*>(J.out);
  bool bad = false;
  if (!J.wide) {  // warp per row, lanes along it
    for (int i = warp; i < mr; i += kWarps)
      for (int j = lane; j < N; j += 32) {
        const float v = Xf[(size_t)(o + i) * ldx + j];
        bad |= !isfinite(v);
        cl_st<S>(out, (int64_t)(o + i) * J.n + j, v);
      }
  } else {  // out row j holds column j of Xh: lanes along this CTA's rows of Xh
    for (int j = warp; j < N; j += kWarps)
      for (int i = lane; i < mr; i += 32) {
        const float v = Xf[(size_t)(o + i) * ldx + j];
        bad |= !isfinite(v);
        cl_st<S>(out, (int64_t)j * J.n + (o + i), v);
      }
  }
  if (bad) fl |= 2u;
  if (rank == 0 || (fl & 2u)) {
    if (fl) atomicOr(flags, fl);
  }
  __syncthreads();
  CL_TL(7);
  if (tl) atomicAdd(&g_cl_tl[8], 1ull);
#undef CL_TL
}

}  // namespace

cudaError_t cluster_timeline(unsigned long long* out9, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out9, g_cl_tl, sizeof(g_cl_tl));
  if (e == cudaSuccess && reset) {
    unsigned long long z[9] = {};
    e = cudaMemcpyToSymbol(g_cl_tl, z, sizeof(z));
  }
  return e;
}

template <int C>
static cudaError_t launch_cl(const ClusterJob* d_jobs, int njobs, const float* d_coeffs, int iters, int precond,
                             bool is_bf16, size_t smem_bytes, uint32_t* d_flags, cudaStream_t stream) {
  static bool attr_set[64][2] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  auto kern = is_bf16 ? cluster_ns_kernel<uint16_t, C> : cluster_ns_kernel<float, C>;
  if (!attr_set[dev & 63][is_bf16]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kClMaxSmem);
    if (e != cudaSuccess) return e;
    if (C > 8) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    attr_set[dev & 63][is_bf16] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(njobs * C));
  cfg.blockDim = dim3(kClThreads);
  cfg.dynamicSmemBytes = smem_bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static int dbg = -1;
  if (dbg < 0) {  // measurement knob (never set in production): TNS_DBG bits
    const char* e = getenv("TNS_DBG");  // 64 = skip the K loops (wrong results), 128 = timeline
    dbg = e ? atoi(e) : 0;
  }
  return cudaLaunchKernelEx(&cfg, kern, d_jobs, d_coeffs, iters, precond, d_flags, dbg);
}

cudaError_t launch_cluster_ns(const ClusterJob* d_jobs, int njobs, const float* d_coeffs, int iters, int precond,
                              bool is_bf16, size_t smem_bytes, int ctas, uint32_t* d_flags, cudaStream_t stream) {
  if (njobs <= 0) return cudaSuccess;
  return ctas == 16 ? launch_cl<16>(d_jobs, njobs, d_coeffs, iters, precond, is_bf16, smem_bytes, d_flags, stream)
                    : launch_cl<8>(d_jobs, njobs, d_coeffs, iters, precond, is_bf16, smem_bytes, d_flags, stream);
}

}  // namespace tns
