// Cluster-resident tcgen05 Newton-Schulz for mid-size matrices (PAPER.md
// small and mid-size matrices are latency/communication-bound, and P:L327: the CIFAR
// conv weights reshaped to 2-D, e.g. 256 x 2304).
//
// One thread-block cluster of C CTAs (a power of two, 2..16, set by the shape: tc_cluster)
// runs ALL steps of Alg. 2 for one matrix in ONE launch.  Xh (M x N, the short-side orientation, N padded with zero columns to
// Np in {128, 256}) is split into row slabs of R in {128, 192, 256} rows, one per CTA,
// resident in shared memory for the whole call in the 64 x 64-box / 128-byte-swizzle layout
// the TMA loads it in (X itself, not a transposed copy: wide inputs are oriented by the UMMA
// major bits, as in the step engine).  Every CTA also holds a full copy of A (Np x Np bf16),
// which the polynomial step turns into B' in place.  Per iteration k (Eqs. 3-5):
//   Gram  : each CTA P_r = slab_r^T slab_r (tcgen05, fp32 in TMEM), written to an fp32
//           scratch in L2; cluster barrier; CTA r sums rows [r Np/C, (r+1) Np/C) of the C
//           partials in a fixed order (deterministic), rounds them to bf16 -- A_k rows -- and
//           broadcasts them to every CTA's A copy by bulk DSMEM copies (mbarrier complete_tx).
//           k = 1: the owner also forms s_i = (sum_j |A0_ij|)^(-1/2) (AOL, Eq. 8) or the
//           trace (Frobenius, Eq. 10) for its rows and broadcasts it; every CTA then forms
//           A1 = diag(s) A0 diag(s) and X1 = X0 diag(s) in its own copies (Alg. 2 l.3-4).
//   Poly  : every CTA computes B' = a_k I + b_k A + c_k A^2 for the full matrix (tcgen05, A
//           as both operands; redundant per CTA, no communication), in place over A (Eq. 4
//           with Eq. 5's a_k folded in, reading R15).
//   Update: slab_r <- slab_r B'^T (tcgen05), written back over the slab in place (Eq. 5).
// After T iterations each CTA TMA-stores its slab.  Rounding: bf16 storage of X, A, B' (every
// stored value rounded once, RNE), fp32 accumulation and fp32 scaling -- reading R6; X1 is
// materialised here (Alg. 2 l.3 literally), where the step engine folds diag(s) into B'1, so
// the two engines agree to bf16 rounding, not bitwise (routing is shape-only: a matrix always
// takes the same engine, batching never changes its result).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "jobs.h"
#include "kernels.h"
#include "ptx.cuh"

namespace tns {

__device__ long long g_tc_tl[64];  // TNS_DBG bit 4096: phase stamps of CTA 0 (measurement only)

namespace {

constexpr int kBox = 64 * 64 * 2;  // one 64 x 64 bf16 box, 128-byte rows, 128-byte swizzle
constexpr int kTcThreads = 256;    // 8 warps: TMEM lane quarter = warp % 4

__device__ __forceinline__ uint32_t tc_mapa(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void tc_bulk_s2s(uint32_t dst, uint32_t src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "r"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void tc_wait_cluster(uint64_t* bar, uint32_t parity) {
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
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t pk_bf2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ uint16_t to_bf(float f) { return __bfloat16_as_ushort(__float2bfloat16_rn(f)); }
// byte offset of element column c (0..63) of row r (0..63) inside a 128-byte-swizzled box
__device__ __forceinline__ uint32_t swz(uint32_t r, uint32_t c) {
  return r * 128u + ((((c >> 3) ^ (r & 7u)) << 4) | ((c & 7u) << 1));
}
__device__ __forceinline__ bool bad16(uint32_t w) {  // either bf16 of the pair non-finite
  return (((w & 0x7F807F80u) + 0x00800080u) & 0x80008000u) != 0;
}

struct TcGeo {
  int Np, R, nb, rb;     // padded short side, slab rows, Np / 64, R / 64
  int rows;              // rows of A owned per CTA in the reduction: Np / C (<= 64)
  int C;                 // CTAs in the cluster
  uint32_t slab, abuf;   // smem offsets (relative to the 1024-aligned base)
  uint32_t svec, trbuf, diag, bars;  // diag: tc_diag_floats (Frobenius diagonal / AOL per-warp row sums)
};
__device__ __forceinline__ TcGeo tc_geo(const TcJob& J) {
  TcGeo g;
  g.Np = J.Np; g.R = J.R; g.nb = J.Np / 64; g.rb = J.R / 64; g.C = J.C; g.rows = J.Np / J.C;
  g.slab = 0;
  g.abuf = (uint32_t)J.R * J.Np * 2;
  g.svec = g.abuf + (uint32_t)J.Np * J.Np * 2;
  g.trbuf = g.svec + (uint32_t)J.Np * 4;
  g.diag = g.trbuf + kTcCtas * 16;
  g.bars = g.diag + (uint32_t)tc_diag_floats(J.Np, J.C) * 4;  // 3 mbarriers + the TMEM address slot (tc_smem() budgets 64 bytes)
  return g;
}

}  // namespace

// Slab box (slab row block i, N block j): tall inputs keep row blocks fastest (K-major for
// the update's A operand needs its two 64-row blocks adjacent), wide inputs N blocks fastest
// (K-major for the Gram's operands).
__device__ __forceinline__ uint32_t slab_box(const TcGeo& g, int wide, int i, int j) {
  return g.slab + (uint32_t)(wide ? (i * g.nb + j) : (j * g.rb + i)) * kBox;
}
// A box (row block i, column block j): row blocks fastest (K-major operands, 64-row blocks
// adjacent).
__device__ __forceinline__ uint32_t a_box(const TcGeo& g, int i, int j) {
  return g.abuf + (uint32_t)(j * g.nb + i) * kBox;
}

__global__ void __launch_bounds__(kTcThreads, 1)
    cluster_tc_ns_kernel(const TcJob* __restrict__ jobs, const float* __restrict__ coeffs, int iters, int precond,
                         uint32_t* __restrict__ flags, int dbg) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t base = smem_u32(sm);
  const TcJob& J = jobs[blockIdx.x / jobs[0].C];  // every job of a launch has the same C
  const uint32_t rank = cluster_ctarank();
  const TcGeo g = tc_geo(J);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, qd = warp & 3;
  const int wide = J.wide;
  uint64_t* bar_load = reinterpret_cast<uint64_t*>(sm + g.bars);
  uint64_t* bar_mma = bar_load + 1;
  uint64_t* bar_rx = bar_load + 2;
  uint64_t* bar_mma1 = bar_load + 3;  // second accumulator of a batch (its epilogue overlaps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_load + 4);
  float* svec = reinterpret_cast<float*>(sm + g.svec);
  float* trbuf = reinterpret_cast<float*>(sm + g.trbuf);
  float* diag = reinterpret_cast<float*>(sm + g.diag);
  bool bad = false, zero = false;
  // TNS_DBG bit 4096 (measurement only): cycle stamps of CTA 0 of the first cluster, printed
  const bool tl = (dbg & 4096) && blockIdx.x == 0 && threadIdx.x == 0;
  int ntl = 0;
  const long long T0 = tl ? clock64() : 0;
#define TC_TL() do { if (tl && ntl < 64) g_tc_tl[ntl++] = clock64() - T0; } while (0)

  if (threadIdx.x == 0) {
    mbar_init(bar_load, 1);
    mbar_init(bar_mma, 1);
    mbar_init(bar_rx, 1);
    mbar_init(bar_mma1, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc<1>(tmem_slot, 512);
    tmem_relinquish<1>();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();

  // ---- load this CTA's slab of Xh (rows [rank R, rank R + R)); TMA fills rows past M and
  //      columns past N with zeros, which the iteration keeps at zero
  if (threadIdx.x == 0) {
    pdl_wait();  // X may come from the previous kernel in the stream
    tma_prefetch_desc(J.tm_in);
    mbar_arrive_expect_tx(bar_load, (uint32_t)(g.rb * g.nb) * kBox);
    for (int i = 0; i < g.rb; ++i)
      for (int j = 0; j < g.nb; ++j) {
        const int mrow = (int)rank * g.R + 64 * i, ncol = 64 * j;
        // tall: X rows are Xh rows (c0 = column, c1 = row); wide: X rows are Xh columns
        tma_load_2d(sm + slab_box(g, wide, i, j), J.tm_in, bar_load, wide ? mrow : ncol, wide ? ncol : mrow);
      }
  }
  mbar_wait(bar_load, 0);
  TC_TL();

  uint32_t ph0 = 0, ph1 = 0;  // parities of bar_mma / bar_mma1
  const int nacc_g = g.Np > 128 ? 2 : 1;            // Gram / A^2 accumulators of 128 rows
  const int nacc_x = g.R > 128 ? 2 : 1;             // update accumulators (R = 192: rows 64..191)
  const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
  const float* cf = coeffs;

  for (int k = 0; k < iters; ++k) {
    const float ca = cf[3 * k], cb = cf[3 * k + 1], cc = cf[3 * k + 2];
    // ===================================================== Gram partial  P_r = slab^T slab
    __syncthreads();
    if (threadIdx.x == 0) {
      tc_fence_after();
      const uint32_t idesc = make_idesc_bf16(128, (uint32_t)g.Np, wide ? 0u : 1u, wide ? 0u : 1u);
      for (int a = 0; a < nacc_g; ++a) {
        for (int ks = 0; ks < g.R / 16; ++ks) {
          const int kb = ks >> 2, kk = ks & 3;
          uint64_t ad, bd;
          if (!wide) {  // Aop[p][k] = slab[k][p]: MN-major, 64-wide p chunks one N block apart
            const uint32_t lbo = (uint32_t)g.rb * kBox;
            ad = make_sdesc(base + slab_box(g, 0, kb, 2 * a) + kk * 2048, lbo, 1024);
            bd = make_sdesc(base + slab_box(g, 0, kb, 0) + kk * 2048, lbo, 1024);
          } else {      // Aop[p][k] = X[p][k]: K-major, the slab's N blocks adjacent
            ad = make_sdesc(base + slab_box(g, 1, kb, 2 * a) + kk * 32, 16, 1024);
            bd = make_sdesc(base + slab_box(g, 1, kb, 0) + kk * 32, 16, 1024);
          }
          umma_bf16<1>(tmem + (uint32_t)(a * g.Np), ad, bd, idesc, ks ? 1u : 0u);
        }
        umma_commit<1>(a ? bar_mma1 : bar_mma);  // accumulator a done: its epilogue may start
      }
    }
    {  // TMEM -> fp32 partial in L2, in the TMEM-natural order pidx(): every store instruction
       // of a warp writes 32 consecutive float4 (512 contiguous bytes).  Accumulator 0 drains
       // while accumulator 1 is still being computed; two TMEM loads in flight per wait.
      float* P = J.part + (size_t)rank * g.Np * g.Np;
      const int nch = g.Np / 32;
#ifdef TNS_TC_NO_OVERLAP
      mbar_wait(bar_mma, ph0);
      if (nacc_g > 1) mbar_wait(bar_mma1, ph1);
#endif
      for (int a = 0; a < nacc_g; ++a) {
#ifndef TNS_TC_NO_OVERLAP
        mbar_wait(a ? bar_mma1 : bar_mma, a ? ph1 : ph0);
#endif
        if (a == 0) TC_TL();
        tc_fence_after();
        for (int c = warp >> 2; c < nch; c += 4) {
          uint32_t r[2][32];
          tmem_ld_32x32b_x32(tmem + lane_base + (uint32_t)(a * g.Np + c * 32), r[0]);
          tmem_ld_32x32b_x32(tmem + lane_base + (uint32_t)(a * g.Np + (c + 2) * 32), r[1]);
          tmem_ld_wait_regs(r[0]);
          tmem_ld_wait_regs(r[1]);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float4* dst = reinterpret_cast<float4*>(P) + (size_t)(((a * 4 + qd) * nch + c + 2 * h) * 8) * 32 + lane;
#pragma unroll
            for (int v = 0; v < 8; ++v)
              __stcg(dst + v * 32, make_float4(__uint_as_float(r[h][4 * v]), __uint_as_float(r[h][4 * v + 1]),
                                               __uint_as_float(r[h][4 * v + 2]), __uint_as_float(r[h][4 * v + 3])));
          }
        }
      }
      ph0 ^= 1;
      if (nacc_g > 1) ph1 ^= 1;
    }
    tc_fence_before();
    TC_TL();
    cluster_sync();  // every partial of this iteration is in L2 (release / acquire)
    TC_TL();
    // ===================================================== reduce my rows of A_k, broadcast
    const int o0 = (int)rank * g.rows;
    if (threadIdx.x == 0) {
      uint32_t bytes = (uint32_t)(g.C - 1) * g.rows * 128u * g.nb;
      if (k == 0 && precond == 2) bytes += (uint32_t)(g.C - 1) * g.rows * 4u;
      if (k == 0 && precond == 1) bytes += (uint32_t)(g.C - 1) * 16u;
      mbar_arrive_expect_tx(bar_rx, bytes);
    }
    {
      // The partials are stored as float4 units pidx(p, q) = ((((a*4 + qd)*nch + c)*8 + v)*32 + l),
      // p = 128 a + 32 qd + l, q = 32 c + 4 v.  My rows [o0, o0 + rows) share (a, qd); a lane
      // takes one row (l) of one column unit (c, v): loads of consecutive lanes are consecutive.
      const int nch = g.Np / 32, units = nch * 8;
      const int rl = g.rows < 32 ? g.rows : 32;   // lanes per column unit (one row each)
      const int per = 32 / rl;                     // column units per warp pass
      const int r0 = lane % rl, sub = lane / rl;
      float rs[2] = {0.f, 0.f};
#pragma unroll
      for (int gi = 0; gi < 2; ++gi) {             // rows > 32 (C = 2 or 4): two row groups
        if (gi * rl >= g.rows) break;
        const int r = gi * rl + r0, i = o0 + r;
        const int a0 = i >> 7, qd0 = (i >> 5) & 3, l0 = i & 31;
        for (int u0 = warp * per; u0 < units; u0 += 8 * per) {
          const int unit = u0 + sub;
          const int c = unit >> 3, v = unit & 7;
          const float4* src = reinterpret_cast<const float4*>(J.part) +
                              (size_t)(((a0 * 4 + qd0) * nch + c) * 8 + v) * 32 + l0;
          float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int t0 = 0; t0 < g.C; t0 += 8) {  // partials 0..C-1 summed in order, 8 loads in flight
            float4 pv[8];
#pragma unroll
            for (int t = 0; t < 8; ++t)
              pv[t] = (t0 + t < g.C) ? __ldcg(src + (size_t)(t0 + t) * g.Np * g.Np / 4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int t = 0; t < 8; ++t) { acc.x += pv[t].x; acc.y += pv[t].y; acc.z += pv[t].z; acc.w += pv[t].w; }
          }
          const int q = c * 32 + v * 4;
          const uint32_t w0 = pk_bf2(acc.x, acc.y), w1 = pk_bf2(acc.z, acc.w);
          bad |= bad16(w0) | bad16(w1);
          rs[gi] += fabsf(bf_lo(w0)) + fabsf(bf_hi(w0)) + fabsf(bf_lo(w1)) + fabsf(bf_hi(w1));
          if (k == 0 && precond == 1 && q <= i && i < q + 4) {  // the diagonal element of row i
            const float dv[4] = {bf_lo(w0), bf_hi(w0), bf_lo(w1), bf_hi(w1)};
            diag[i - o0] = dv[i - q];
          }
          *reinterpret_cast<uint2*>(sm + a_box(g, i >> 6, q >> 6) + swz((uint32_t)(i & 63), (uint32_t)(q & 63))) =
              make_uint2(w0, w1);
        }
      }
      if (k == 0 && precond == 2) {  // Eq. 8 on the stored bf16 A0 row: fixed-order reduction
#pragma unroll
        for (int gi = 0; gi < 2; ++gi) {
          if (gi * rl >= g.rows) break;
          float v = rs[gi];
          for (int o = rl; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if (lane < rl) diag[warp * g.rows + gi * rl + lane] = v;  // per-warp row sums (scratch)
        }
        __syncthreads();
        if (threadIdx.x < g.rows) {
          float t = 0.f;
          for (int w = 0; w < 8; ++w) t += diag[w * g.rows + threadIdx.x];
          const int ii = o0 + (int)threadIdx.x;
          svec[ii] = t > 0.f ? rsqrtf(t) : 0.f;
          if (!(t > 0.f) && ii < J.N) zero = true;
        }
      }
    }
    // my rows were written by generic stores and go out through the async proxy (bulk copies)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    TC_TL();
    if (threadIdx.x == 0 && k == 0 && precond == 1) {  // my rows' share of tr(A0), in row order
      float tr = 0.f;
      for (int i = 0; i < g.rows; ++i) tr += diag[i];
      trbuf[4 * rank] = tr;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (k == 0 && precond == 1) __syncthreads();
    if (threadIdx.x >= 1 && (int)threadIdx.x < g.C) {  // one thread per peer issues its copies
      const uint32_t peer = (rank + threadIdx.x) % g.C;
      const uint32_t rbar = tc_mapa(smem_u32(bar_rx), peer);
      for (int j = 0; j < g.nb; ++j) {
        const uint32_t src = base + a_box(g, o0 >> 6, j) + (uint32_t)(o0 & 63) * 128u;
        tc_bulk_s2s(tc_mapa(src, peer), src, (uint32_t)g.rows * 128u, rbar);
      }
      if (k == 0 && precond == 2) {
        const uint32_t src = base + g.svec + (uint32_t)o0 * 4u;
        tc_bulk_s2s(tc_mapa(src, peer), src, (uint32_t)g.rows * 4u, rbar);
      }
      if (k == 0 && precond == 1) {
        const uint32_t src = base + g.trbuf + rank * 16u;
        tc_bulk_s2s(tc_mapa(src, peer), src, 16u, rbar);
      }
    }
    tc_wait_cluster(bar_rx, (uint32_t)(k & 1));
    // My bulk copies to the peers read my rows of A, which the preconditioner (k = 1) or the
    // A^2 epilogue overwrites next: every peer having received everything (its rx wait) is
    // the only completion signal, so a split cluster barrier -- arrive here, wait before the
    // first store into A -- orders them (the A^2 MMAs in between hide its latency).
    cluster_arrive_relaxed();
    bool a_pending = true;
    TC_TL();
    // ===================================================== k = 1: the preconditioner
    if (k == 0 && precond != 0) {
      cluster_wait();
      a_pending = false;
      if (precond == 1) {
        float tr = 0.f;
        for (int r = 0; r < g.C; ++r) tr += trbuf[4 * r];
        const float s = tr > 0.f ? rsqrtf(tr) : 0.f;
        if (!(tr > 0.f) && rank == 0 && threadIdx.x == 0) zero = true;
        for (int i = threadIdx.x; i < g.Np; i += kTcThreads) svec[i] = s;
        __syncthreads();
      }
      // A1 = diag(s) A0 diag(s) (Alg. 2 l.4), X1 = X0 diag(s) (Alg. 2 l.3): 16-byte chunks
      const int achunks = g.Np * g.Np / 8;
      for (int t = threadIdx.x; t < achunks; t += kTcThreads) {
        const int bx = t >> 9, w = t & 511, r = w >> 3, ch = w & 7;  // 512 chunks per box
        const int bi = bx % g.nb, bj = bx / g.nb;                    // a_box order
        const int row = bi * 64 + r, col0 = bj * 64 + ((ch ^ (r & 7)) << 3);
        uint4* p = reinterpret_cast<uint4*>(sm + g.abuf + (uint32_t)bx * kBox + r * 128 + ch * 16);
        uint4 u = *p;
        uint32_t wv[4] = {u.x, u.y, u.z, u.w};
        const float si = svec[row];
#pragma unroll
        for (int e = 0; e < 4; ++e)
          wv[e] = pk_bf2((si * bf_lo(wv[e])) * svec[col0 + 2 * e], (si * bf_hi(wv[e])) * svec[col0 + 2 * e + 1]);
        *p = make_uint4(wv[0], wv[1], wv[2], wv[3]);
      }
      const int xchunks = g.R * g.Np / 8;
      for (int t = threadIdx.x; t < xchunks; t += kTcThreads) {
        const int bx = t >> 9, w = t & 511, r = w >> 3, ch = w & 7;
        const int cpos = (ch ^ (r & 7)) << 3;
        uint4* p = reinterpret_cast<uint4*>(sm + g.slab + (uint32_t)bx * kBox + r * 128 + ch * 16);
        uint4 u = *p;
        uint32_t wv[4] = {u.x, u.y, u.z, u.w};
        if (!wide) {  // box (i, j) at j * rb + i: columns are N indices
          const int n0 = (bx / g.rb) * 64 + cpos;
#pragma unroll
          for (int e = 0; e < 4; ++e) wv[e] = pk_bf2(bf_lo(wv[e]) * svec[n0 + 2 * e], bf_hi(wv[e]) * svec[n0 + 2 * e + 1]);
        } else {      // box (i, j) at i * nb + j: box rows are N indices
          const float sn = svec[(bx % g.nb) * 64 + r];
#pragma unroll
          for (int e = 0; e < 4; ++e) wv[e] = pk_bf2(bf_lo(wv[e]) * sn, bf_hi(wv[e]) * sn);
        }
        *p = make_uint4(wv[0], wv[1], wv[2], wv[3]);
      }
    }
    // ===================================================== B' = a I + b A + c A^2 (in place)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    TC_TL();
    if (threadIdx.x == 0) {
      tc_fence_after();
      const uint32_t idesc = make_idesc_bf16(128, (uint32_t)g.Np, 0u, 0u);
      for (int a = 0; a < nacc_g; ++a) {
        for (int ks = 0; ks < g.Np / 16; ++ks) {
          const int kb = ks >> 2, kk = ks & 3;
          const uint64_t ad = make_sdesc(base + a_box(g, 2 * a, kb) + kk * 32, 16, 1024);
          const uint64_t bd = make_sdesc(base + a_box(g, 0, kb) + kk * 32, 16, 1024);
          umma_bf16<1>(tmem + (uint32_t)(a * g.Np), ad, bd, idesc, ks ? 1u : 0u);
        }
        umma_commit<1>(a ? bar_mma1 : bar_mma);
      }
    }
    {
      // B' overwrites A in place, and A is the B operand of both accumulators' UMMAs: wait
      // for all of them before the first store, and for every peer to hold my rows of A
      mbar_wait(bar_mma, ph0);
      if (nacc_g > 1) mbar_wait(bar_mma1, ph1);
      if (a_pending) cluster_wait();
      TC_TL();
      tc_fence_after();
      const int nch = g.Np / 32;
      for (int a = 0; a < nacc_g; ++a) {
        const int p = a * 128 + qd * 32 + lane;
        for (int c = warp >> 2; c < nch; c += 4) {
          uint32_t r[2][32];
          tmem_ld_32x32b_x32(tmem + lane_base + (uint32_t)(a * g.Np + c * 32), r[0]);
          tmem_ld_32x32b_x32(tmem + lane_base + (uint32_t)(a * g.Np + (c + 2) * 32), r[1]);
          tmem_ld_wait_regs(r[0]);
          tmem_ld_wait_regs(r[1]);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int q0 = (c + 2 * hh) * 32;
#pragma unroll
            for (int h = 0; h < 4; ++h) {  // 8 columns per 16-byte chunk
              const int q = q0 + 8 * h;
              uint4* ptr = reinterpret_cast<uint4*>(sm + a_box(g, p >> 6, q >> 6) + swz((uint32_t)(p & 63), (uint32_t)(q & 63)));
              const uint4 u4 = *ptr;
              const uint32_t x[4] = {u4.x, u4.y, u4.z, u4.w};
              uint32_t o[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                float w0 = fmaf(cc, __uint_as_float(r[hh][8 * h + 2 * e]), cb * bf_lo(x[e]));
                float w1 = fmaf(cc, __uint_as_float(r[hh][8 * h + 2 * e + 1]), cb * bf_hi(x[e]));
                if (q + 2 * e == p) w0 += ca;
                if (q + 2 * e + 1 == p) w1 += ca;
                o[e] = pk_bf2(w0, w1);
                bad |= bad16(o[e]);
              }
              *ptr = make_uint4(o[0], o[1], o[2], o[3]);
            }
          }
        }
      }
      ph0 ^= 1;
      if (nacc_g > 1) ph1 ^= 1;
    }
    // ===================================================== slab <- slab B'^T (in place)
    tc_fence_before();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    TC_TL();
    if (threadIdx.x == 0) {
      tc_fence_after();
      const uint32_t idesc = make_idesc_bf16(128, (uint32_t)g.Np, wide ? 1u : 0u, 0u);
      for (int a = 0; a < nacc_x; ++a) {
        const int rb0 = (a == 0) ? 0 : (g.R == 192 ? 1 : 2);  // first 64-row block of the accumulator
        for (int ks = 0; ks < g.Np / 16; ++ks) {
          const int kb = ks >> 2, kk = ks & 3;
          uint64_t ad;
          if (!wide)  // Aop[p][k] = slab[p][k]: K-major, row blocks adjacent
            ad = make_sdesc(base + slab_box(g, 0, rb0, kb) + kk * 32, 16, 1024);
          else        // Aop[p][k] = X[k][p]: MN-major, 64-wide p chunks one slab block apart
            ad = make_sdesc(base + slab_box(g, 1, rb0, kb) + kk * 2048, (uint32_t)g.nb * kBox, 1024);
          const uint64_t bd = make_sdesc(base + a_box(g, 0, kb) + kk * 32, 16, 1024);
          umma_bf16<1>(tmem + (uint32_t)(a * g.Np), ad, bd, idesc, ks ? 1u : 0u);
        }
        umma_commit<1>(a ? bar_mma1 : bar_mma);
      }
    }
    {
      // X' overwrites the slab in place, which both accumulators' UMMAs read (R = 192: their
      // rows overlap): wait for all of them
      mbar_wait(bar_mma, ph0);
      if (nacc_x > 1) mbar_wait(bar_mma1, ph1);
      TC_TL();
      tc_fence_after();
      const int nch = g.Np / 32;
      for (int a = 0; a < nacc_x; ++a) {
        const int prow0 = (a == 0) ? 0 : (g.R == 192 ? 64 : 128);  // slab row of TMEM lane 0
        const int p = prow0 + qd * 32 + lane;
        if (a == 1 && g.R == 192 && qd < 2) continue;  // R = 192: rows 64..127 belong to accumulator 0
        for (int c = warp >> 2; c < nch; c += 2) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem + lane_base + (uint32_t)(a * g.Np + c * 32), r);
        tmem_ld_wait_regs(r);
        const int q0 = c * 32;
        if (!wide) {
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int q = q0 + 8 * h;
            uint32_t o[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              o[e] = pk_bf2(__uint_as_float(r[8 * h + 2 * e]), __uint_as_float(r[8 * h + 2 * e + 1]));
              bad |= bad16(o[e]);
            }
            *reinterpret_cast<uint4*>(sm + slab_box(g, 0, p >> 6, q >> 6) + swz((uint32_t)(p & 63), (uint32_t)(q & 63))) =
                make_uint4(o[0], o[1], o[2], o[3]);
          }
        } else {  // wide: the slab stores [n][m] boxes: element (p, q) at row q, column p
          const uint32_t bx = slab_box(g, 1, p >> 6, q0 >> 6);
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const uint16_t h = to_bf(__uint_as_float(r[e]));
            bad |= ((h & 0x7F80u) == 0x7F80u);
            *reinterpret_cast<uint16_t*>(sm + bx + swz((uint32_t)((q0 + e) & 63), (uint32_t)(p & 63))) = h;
          }
        }
        }
      }
      ph0 ^= 1;
      if (nacc_x > 1) ph1 ^= 1;
    }
    tc_fence_before();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the next Gram's MMAs read the slab
    __syncthreads();
    TC_TL();
  }

  // ---- store the slab (TMA clips rows past M and columns past N)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    tma_prefetch_desc(J.tm_out);
    for (int i = 0; i < g.rb; ++i)
      for (int j = 0; j < g.nb; ++j) {
        const int mrow = (int)rank * g.R + 64 * i, ncol = 64 * j;
        if (mrow >= J.M || ncol >= J.N) continue;
        tma_store_2d(J.tm_out, sm + slab_box(g, wide, i, j), wide ? mrow : ncol, wide ? ncol : mrow);
      }
    bulk_commit();
    bulk_wait<0>();
    TC_TL();
    if (tl) {
      printf("tc timeline (cycles since entry, CTA 0): load %lld |", g_tc_tl[0]);
      for (int i = 1; i < ntl; ++i) printf(" %lld", g_tc_tl[i] - g_tc_tl[i - 1]);
      printf("\n");
    }
  }
#undef TC_TL
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, 2u);
  if (__any_sync(0xffffffffu, zero) && lane == 0) atomicOr(flags, 1u);
  tc_fence_before();
  cluster_sync();  // no CTA leaves while a peer's bulk copies into it may be in flight
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, 512);
  }
}

cudaError_t launch_cluster_tc_ns(const TcJob* d_jobs, int njobs, int ctas, const float* d_coeffs, int iters,
                                 int precond, size_t smem_bytes, uint32_t* d_flags, cudaStream_t stream) {
  if (njobs <= 0) return cudaSuccess;
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  auto kern = cluster_tc_ns_kernel;
  if (!attr_set[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcMaxSmem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    attr_set[dev & 63] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(njobs * ctas));
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = smem_bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)ctas;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  static const int dbg = [] { const char* e = getenv("TNS_DBG"); return e ? atoi(e) : 0; }();
  return cudaLaunchKernelEx(&cfg, kern, d_jobs, d_coeffs, iters, precond, d_flags, dbg);
}

}  // namespace tns
