// Cluster-resident tcgen05 Newton-Schulz for mid-size matrices (PAPER.md
// small and mid-size matrices are latency/communication-bound, and P:L327: the CIFAR
// conv weights reshaped to 2-D, e.g. 256 x 2304).
//
// One thread-block cluster of C CTAs (a power of two, 4..16, set by the shape: tc_cluster)
// runs ALL steps of Alg. 2 for one matrix in ONE launch.  Xh (M x N, the
// short-side orientation, N padded with zero columns to Np in {128, 256}) is split into row
// slabs of R in {128, 192, 256} rows, one per CTA,
// resident in shared memory for the whole call in the 64 x 64-box / 128-byte-swizzle layout
// the TMA loads it in (X itself, not a transposed copy: wide inputs are oriented by the UMMA
// major bits, as in the step engine).  Every CTA also holds a full copy of A (Np x Np bf16),
// which the polynomial step turns into B' in place.  Per iteration k (Eqs. 3-5):
//   Gram  : each CTA P_r = slab_r^T slab_r (tcgen05, fp32 in TMEM); its lower-triangle 32 x 32
//           chunks go to an fp32 scratch in L2; cluster barrier; CTA r sums an equal share of
//           the chunk elements over the C partials in a fixed order (deterministic), rounds them
//           to bf16 -- A_k -- and writes them, mirrored, into a global A image laid out like the
//           shared-memory A buffer; cluster barrier; every CTA bulk-loads the whole image
//           (measured on B200, tools/xfer_probe.cu: L2 stores ~30 B/cycle/SM, bulk L2 loads
//           55-65, DSMEM bulk copies ~13 -- so the triangle halves the dominant store traffic
//           and the L2 image replaces a DSMEM broadcast).
//           k = 1: every CTA forms s_i = (sum_j |A0_ij|)^(-1/2) (AOL, Eq. 8) or tr(A0)^(-1/2)
//           (Frobenius, Eq. 10) from its copy of A0, then A1 = diag(s) A0 diag(s) in its own
//           copy (Alg. 2 l.4); X1 = X0 diag(s) (l.3) is never formed: diag(s) is folded into
//           B'1 (its columns), as in the step engine (reading R15).
//   Poly  : every CTA computes B' = a_k I + b_k A + c_k A^2 for the full matrix (tcgen05, A
//           as both operands; redundant per CTA, no communication), in place over A (Eq. 4
//           with Eq. 5's a_k folded in, reading R15; k = 1: times diag(s) on the right).
//   Update: slab_r <- slab_r B'^T (tcgen05; wide inputs: X_r <- B' X_r, the same product with
//           the slab as the B operand), written back over the slab in place (Eq. 5).
// After T iterations each CTA TMA-stores its slab.  Rounding: bf16 storage of X, A, B' (every
// stored value rounded once, RNE), fp32 accumulation and fp32 scaling -- readings R6 / R15,
// the same roundings as the step engine; the two engines still agree to bf16 rounding only,
// not bitwise (their fp32 sums run in different orders), and routing is shape-only: a matrix
// always takes the same engine, batching never changes its result.
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
// byte offset of element column c (0..63) of row r (0..63) inside a 128-byte-swizzled box
__device__ __forceinline__ uint32_t swz(uint32_t r, uint32_t c) {
  return r * 128u + ((((c >> 3) ^ (r & 7u)) << 4) | ((c & 7u) << 1));
}
__device__ __forceinline__ bool bad16(uint32_t w) {  // either bf16 of the pair non-finite
  return (((w & 0x7F807F80u) + 0x00800080u) & 0x80008000u) != 0;
}

struct TcGeo {
  int Np, R, nb, rb;     // padded short side, slab rows, Np / 64, R / 64
  int C;                 // CTAs in the cluster
  int L;                 // lower-triangle 32 x 32 chunks of a Gram partial (tc_tri_chunks)
  uint32_t slab, abuf;   // smem offsets (relative to the 1024-aligned base)
  uint32_t svec, bars;
};
__device__ __forceinline__ TcGeo tc_geo(const TcJob& J) {
  TcGeo g;
  g.Np = J.Np; g.R = J.R; g.nb = J.Np / 64; g.rb = J.R / 64; g.C = J.C; g.L = tc_tri_chunks(J.Np);
  g.slab = 0;
  g.abuf = (uint32_t)J.R * J.Np * 2;
  g.svec = g.abuf + (uint32_t)J.Np * J.Np * 2;
  g.bars = g.svec + (uint32_t)J.Np * 4;  // 4 mbarriers + the TMEM address slot (tc_smem() budgets 64 bytes)
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
// adjacent).  The global A image (TcJob::part) has the same layout, offsets relative to abuf.
__device__ __forceinline__ uint32_t a_box(const TcGeo& g, int i, int j) {
  return g.abuf + (uint32_t)(j * g.nb + i) * kBox;
}
// byte offset of element (i, j) of A in the image / relative to abuf
__device__ __forceinline__ uint32_t a_img(const TcGeo& g, int i, int j) {
  return (uint32_t)((j >> 6) * g.nb + (i >> 6)) * kBox + swz((uint32_t)(i & 63), (uint32_t)(j & 63));
}

// The Gram all-reduce, owner side: float4 units [rank per, (rank + 1) per) of the lower-triangle
// chunk order, summed over the CC partials in order 0..CC-1 (16 loads in flight per thread:
// 16 / CC units per batch), rounded to bf16 once, written into the A image with their mirrors.
template <int CC>
__device__ __forceinline__ void reduce_share(const TcGeo& g, float* part, uint32_t rank, bool& bad) {
  constexpr int kUpb = 16 / CC;
  const int U = g.L * 256, per = U / CC;
  const float4* Pb = reinterpret_cast<const float4*>(part);
  uint8_t* img = reinterpret_cast<uint8_t*>(part + (size_t)CC * g.L * 1024);
  for (int w0 = (int)threadIdx.x; w0 < per; w0 += kTcThreads * kUpb) {
    float4 pv[kUpb][CC];
#pragma unroll
    for (int i = 0; i < kUpb; ++i) {
      const int w = w0 + i * kTcThreads;
#pragma unroll
      for (int t = 0; t < CC; ++t)
        pv[i][t] = w < per ? __ldcg(Pb + (size_t)t * U + (size_t)rank * per + w) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < kUpb; ++i) {
      const int w = w0 + i * kTcThreads;
      if (w >= per) break;
      float4 a4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int t = 0; t < CC; ++t) { a4.x += pv[i][t].x; a4.y += pv[i][t].y; a4.z += pv[i][t].z; a4.w += pv[i][t].w; }
      const int u = (int)rank * per + w;
      const int ci = u >> 8, v = (u >> 5) & 7, l = u & 31;
      int rb = 0;
      while ((rb + 1) * (rb + 2) / 2 <= ci) ++rb;
      const int row = rb * 32 + l, col = (ci - rb * (rb + 1) / 2) * 32 + v * 4;
      const uint32_t w0b = pk_bf2(a4.x, a4.y), w1b = pk_bf2(a4.z, a4.w);
      bad |= bad16(w0b) | bad16(w1b);
      const uint16_t hv[4] = {(uint16_t)(w0b & 0xFFFFu), (uint16_t)(w0b >> 16), (uint16_t)(w1b & 0xFFFFu), (uint16_t)(w1b >> 16)};
      if (col + 3 <= row) {
        *reinterpret_cast<uint2*>(img + a_img(g, row, col)) = make_uint2(w0b, w1b);
      } else {  // a diagonal chunk: the elements on or below the diagonal only
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (col + e <= row) *reinterpret_cast<uint16_t*>(img + a_img(g, row, col + e)) = hv[e];
      }
#pragma unroll
      for (int e = 0; e < 4; ++e)  // mirrored: A_k is stored symmetric, bit for bit
        if (col + e < row) *reinterpret_cast<uint16_t*>(img + a_img(g, col + e, row)) = hv[e];
    }
  }
}

// B' = a_k I + b_k A + c_k A^2 for 32 columns [q0, q0 + 32) of row p, in place over the bf16
// A row (Eq. 4 with Eq. 5's a_k folded in, reading R15), two columns per packed fp32x2
// FMUL2 / FFMA2 (the same fp32 roundings as fmaf(c, r, b * x) per element).  No non-finite
// test here: a non-finite A or B' always reaches X_{k+1}, whose stores are checked.
__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
  uint64_t d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
  return d;
}
template <bool DIAG, bool SCALE>
__device__ __forceinline__ void poly_chunk(uint8_t* sm, const TcGeo& g, int p, int q0, const uint32_t (&r)[32],
                                           const uint4 (&xv)[4], float ca, float cb, float cc, const float* sv) {
  const uint64_t cb2 = pk2(cb, cb), cc2 = pk2(cc, cc);
#pragma unroll
  for (int h = 0; h < 4; ++h) {  // 8 columns per 16-byte swizzle chunk
    const int q = q0 + 8 * h;
    const uint32_t x[4] = {xv[h].x, xv[h].y, xv[h].z, xv[h].w};
    float sc[8];
    if (SCALE) {  // k = 1: B'1 diag(s) -- column q scaled by s_q (X1 = X0 diag(s) never formed)
      const float4 a0 = *reinterpret_cast<const float4*>(sv + q), a1 = *reinterpret_cast<const float4*>(sv + q + 4);
      sc[0] = a0.x; sc[1] = a0.y; sc[2] = a0.z; sc[3] = a0.w; sc[4] = a1.x; sc[5] = a1.y; sc[6] = a1.z; sc[7] = a1.w;
    }
    uint32_t o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint64_t t, w;
      asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(cb2), "l"(pk2(bf_lo(x[e]), bf_hi(x[e]))));
      asm("fma.rn.f32x2 %0, %1, %2, %3;"
          : "=l"(w)
          : "l"(cc2), "l"(pk2(__uint_as_float(r[8 * h + 2 * e]), __uint_as_float(r[8 * h + 2 * e + 1]))), "l"(t));
      float w0, w1;
      asm("mov.b64 {%0, %1}, %2;" : "=f"(w0), "=f"(w1) : "l"(w));
      if (DIAG) {
        w0 = (q + 2 * e == p) ? w0 + ca : w0;
        w1 = (q + 2 * e + 1 == p) ? w1 + ca : w1;
      }
      if (SCALE) {
        w0 *= sc[2 * e];
        w1 *= sc[2 * e + 1];
      }
      o[e] = pk_bf2(w0, w1);
    }
    *reinterpret_cast<uint4*>(sm + a_box(g, p >> 6, q >> 6) + swz((uint32_t)(p & 63), (uint32_t)(q & 63))) =
        make_uint4(o[0], o[1], o[2], o[3]);
  }
}

__global__ void __launch_bounds__(kTcThreads, 1)
    cluster_tc_ns_kernel(const TcJob* __restrict__ jobs, const float* __restrict__ coeffs, int iters, int precond,
                         uint32_t* __restrict__ flags, int dbg) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned by pointer arithmetic on the __shared__ array (not through an integer
  // cast), so the compiler keeps the shared state space: LDS / STS, not generic LD / ST
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
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
    {
      // TMEM -> fp32 partial in L2: only the lower-triangle 32 x 32 chunks (A is symmetric),
      // chunk (rb, c) at index rb (rb + 1) / 2 + c, inside a chunk float4 unit v * 32 + lane =
      // row 32 rb + lane, columns 32 c + 4 v .. + 3 (every store instruction of a warp writes
      // 512 contiguous bytes).  Accumulator 0 drains while accumulator 1 is being computed;
      // two TMEM loads in flight per wait.
      float4* P = reinterpret_cast<float4*>(J.part) + (size_t)rank * g.L * 256;
      const int h = warp >> 2;
      for (int a = 0; a < nacc_g; ++a) {
        mbar_wait(a ? bar_mma1 : bar_mma, a ? ph1 : ph0);
        if (a == 0) TC_TL();
        tc_fence_after();
        const int rb = a * 4 + qd;  // this warp's 32-row block
        for (int c = h; c <= rb; c += 4) {  // chunks c and c + 2 of the row block
          const bool two = c + 2 <= rb;       // warp-uniform
          uint32_t r[2][32];
          tmem_ld_32x32b_x32(tmem + lane_base + (uint32_t)(a * g.Np + c * 32), r[0]);
          if (two) tmem_ld_32x32b_x32(tmem + lane_base + (uint32_t)(a * g.Np + (c + 2) * 32), r[1]);
          tmem_ld_wait_regs(r[0]);
          if (two) tmem_ld_wait_regs(r[1]);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            if (hh && !two) break;
            float4* dst = P + (size_t)(rb * (rb + 1) / 2 + c + 2 * hh) * 256 + lane;
#pragma unroll
            for (int v = 0; v < 8; ++v)
              __stcg(dst + v * 32, make_float4(__uint_as_float(r[hh][4 * v]), __uint_as_float(r[hh][4 * v + 1]),
                                               __uint_as_float(r[hh][4 * v + 2]), __uint_as_float(r[hh][4 * v + 3])));
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
    // ===================================================== reduce my share of A_k into the image
    {
      // CTA r owns float4 units [r U / C, (r + 1) U / C) of the chunk order (equal shares of the
      // triangle); it sums them over the C partials in the fixed order 0..C-1 (deterministic),
      // rounds to bf16 once and writes the elements, and the mirrored ones, into the A image.
      // (Staging the slices in shared memory by bulk copies measured slower: 8.3 vs 5.3 k cycles.)
      if (g.C == 16) reduce_share<16>(g, J.part, rank, bad);
      else if (g.C == 8) reduce_share<8>(g, J.part, rank, bad);
      else reduce_share<4>(g, J.part, rank, bad);
      // generic stores, read next by the bulk (async-proxy) copies of every CTA
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    TC_TL();
    cluster_sync();  // the A_k image is complete
    asm volatile("fence.proxy.async.global;" ::: "memory");
    if (threadIdx.x == 0) {  // every CTA loads the whole image into its A buffer
      const uint32_t bytes = (uint32_t)g.Np * g.Np * 2, piece = bytes / 16;
      const uint8_t* img = reinterpret_cast<const uint8_t*>(J.part + (size_t)g.C * g.L * 1024);
      mbar_arrive_expect_tx(bar_rx, bytes);
      for (uint32_t o = 0; o < bytes; o += piece)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         base + g.abuf + o), "l"(img + o), "r"(piece), "r"(smem_u32(bar_rx))
                     : "memory");
    }
    tc_wait_cluster(bar_rx, (uint32_t)(k & 1));
    TC_TL();
    // ===================================================== k = 1: the preconditioner
    if (k == 0 && precond != 0) {
      // s from the bf16 A0 every CTA now holds (no communication): AOL s_i = (sum_j |A0_ij|)^(-1/2)
      // (Eq. 8, columns in order), Frobenius s = tr(A0)^(-1/2) (Eq. 10)
      if (precond == 2) {
        if ((int)threadIdx.x < g.Np) {
          const int i = threadIdx.x;
          float t = 0.f;
          for (int jb = 0; jb < g.nb; ++jb)
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) {
              const uint4 u4 = *reinterpret_cast<const uint4*>(sm + a_box(g, i >> 6, jb) + (uint32_t)(i & 63) * 128u +
                                                               (uint32_t)((ch ^ (i & 7)) << 4));
              t += fabsf(bf_lo(u4.x)) + fabsf(bf_hi(u4.x)) + fabsf(bf_lo(u4.y)) + fabsf(bf_hi(u4.y)) +
                   fabsf(bf_lo(u4.z)) + fabsf(bf_hi(u4.z)) + fabsf(bf_lo(u4.w)) + fabsf(bf_hi(u4.w));
            }
          svec[i] = t > 0.f ? rsqrtf(t) : 0.f;
          if (!(t > 0.f) && i < J.N) zero = true;
        }
      } else {
        if ((int)threadIdx.x < g.Np) {
          const int i = threadIdx.x;
          svec[i] = bf_lo(*reinterpret_cast<const uint16_t*>(sm + g.abuf + a_img(g, i, i)));
        }
        __syncthreads();
        float tr = 0.f;
        if (warp == 0) {  // fixed order: lane sums its strided diagonal entries, then a fixed tree
          for (int i = lane; i < g.Np; i += 32) tr += svec[i];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
        }
        __syncthreads();
        if (warp == 0 && lane == 0) {
          const float s = tr > 0.f ? rsqrtf(tr) : 0.f;
          if (!(tr > 0.f)) zero = true;
          for (int i = 0; i < g.Np; ++i) svec[i] = s;
        }
      }
      __syncthreads();
      // A1 = diag(s) A0 diag(s) (Alg. 2 l.4) in this CTA's copy, box by box (no index division:
      // the box walk gives row and column blocks), two boxes x two 16-byte chunks per thread in
      // flight (all loads of a group before its stores).  X1 = X0 diag(s) (l.3) is never formed:
      // s goes into the k = 1 A^2 epilogue (B'1 diag(s), as in the step engine, reading R15).
      for (int bj = 0; bj < g.nb; ++bj)
        for (int bi = 0; bi < g.nb; bi += 2) {
          uint4 u[4];
          float si[4];
          float4 s0[4], s1[4];
          uint4* pp[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int w = (int)threadIdx.x + (j & 1) * kTcThreads, r = w >> 3, ch = w & 7;  // 512 chunks per box
            const int bx = bj * g.nb + bi + (j >> 1);
            const int col0 = bj * 64 + ((ch ^ (r & 7)) << 3);
            pp[j] = reinterpret_cast<uint4*>(sm + g.abuf + (uint32_t)bx * kBox + r * 128 + ch * 16);
            u[j] = *pp[j];
            si[j] = svec[(bi + (j >> 1)) * 64 + r];
            s0[j] = *reinterpret_cast<const float4*>(svec + col0);
            s1[j] = *reinterpret_cast<const float4*>(svec + col0 + 4);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t wv[4] = {u[j].x, u[j].y, u[j].z, u[j].w};
            const float sc[8] = {s0[j].x, s0[j].y, s0[j].z, s0[j].w, s1[j].x, s1[j].y, s1[j].z, s1[j].w};
            uint32_t o[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
              o[e] = pk_bf2((si[j] * bf_lo(wv[e])) * sc[2 * e], (si[j] * bf_hi(wv[e])) * sc[2 * e + 1]);
            *pp[j] = make_uint4(o[0], o[1], o[2], o[3]);
          }
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
      // for all of them before the first store
      mbar_wait(bar_mma, ph0);
      if (nacc_g > 1) mbar_wait(bar_mma1, ph1);
      TC_TL();
      tc_fence_after();
      const int nch = g.Np / 32;
      const bool scale1 = k == 0 && precond != 0;  // B'1 diag(s): X1 = X0 diag(s) folded in
      for (int a = 0; a < nacc_g; ++a) {
        const int p = a * 128 + qd * 32 + lane;
        for (int c = warp >> 2; c < nch; c += 4) {
          uint32_t r[2][32];
          tmem_ld_32x32b_x32(tmem + lane_base + (uint32_t)(a * g.Np + c * 32), r[0]);
          tmem_ld_32x32b_x32(tmem + lane_base + (uint32_t)(a * g.Np + (c + 2) * 32), r[1]);
          uint4 xv[2][4];  // the b_k A term's bf16 A, loaded while the TMEM loads are in flight
#pragma unroll
          for (int hh = 0; hh < 2; ++hh)
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const int q = (c + 2 * hh) * 32 + 8 * h;
              xv[hh][h] = *reinterpret_cast<const uint4*>(sm + a_box(g, p >> 6, q >> 6) + swz((uint32_t)(p & 63), (uint32_t)(q & 63)));
            }
          tmem_ld_wait_regs(r[0]);
          tmem_ld_wait_regs(r[1]);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int q0 = (c + 2 * hh) * 32;
            // the chunk holds this warp's diagonal elements iff its 32 columns are the warp's
            // 32 rows (warp-uniform): only then the a_k I term needs per-element selects
            const bool dg = q0 == p - lane;
            if (!scale1) {
              if (dg) poly_chunk<true, false>(sm, g, p, q0, r[hh], xv[hh], ca, cb, cc, svec);
              else poly_chunk<false, false>(sm, g, p, q0, r[hh], xv[hh], ca, cb, cc, svec);
            } else {
              if (dg) poly_chunk<true, true>(sm, g, p, q0, r[hh], xv[hh], ca, cb, cc, svec);
              else poly_chunk<false, true>(sm, g, p, q0, r[hh], xv[hh], ca, cb, cc, svec);
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
      if (!wide) {  // D[p][q] = sum_k slab[p][k] B'[q][k]: R slab rows in 128-row accumulators
        const uint32_t idesc = make_idesc_bf16(128, (uint32_t)g.Np, 0u, 0u);
        for (int a = 0; a < nacc_x; ++a) {
          const int rb0 = (a == 0) ? 0 : (g.R == 192 ? 1 : 2);  // first 64-row block of the accumulator
          for (int ks = 0; ks < g.Np / 16; ++ks) {
            const int kb = ks >> 2, kk = ks & 3;
            // Aop[p][k] = slab[p][k]: K-major, row blocks adjacent
            const uint64_t ad = make_sdesc(base + slab_box(g, 0, rb0, kb) + kk * 32, 16, 1024);
            const uint64_t bd = make_sdesc(base + a_box(g, 0, kb) + kk * 32, 16, 1024);
            umma_bf16<1>(tmem + (uint32_t)(a * g.Np), ad, bd, idesc, ks ? 1u : 0u);
          }
          umma_commit<1>(a ? bar_mma1 : bar_mma);
        }
      } else {
        // wide: the slab holds X itself ([n][m] boxes), and X' = B' X (B' symmetric): D[n][m] =
        // sum_j B'[n][j] X[j][m] -- A operand B' (K-major), B operand the slab (MN-major, UMMA
        // N = R), so the accumulator rows are slab box rows (vector stores, no 64-row overlap)
        const uint32_t idesc = make_idesc_bf16(128, (uint32_t)g.R, 0u, 1u);
        for (int a = 0; a < nacc_g; ++a) {
          for (int ks = 0; ks < g.Np / 16; ++ks) {
            const int kb = ks >> 2, kk = ks & 3;
            const uint64_t ad = make_sdesc(base + a_box(g, 2 * a, kb) + kk * 32, 16, 1024);
            const uint64_t bd = make_sdesc(base + slab_box(g, 1, 0, kb) + kk * 2048, (uint32_t)g.nb * kBox, 1024);
            umma_bf16<1>(tmem + (uint32_t)(a * 256), ad, bd, idesc, ks ? 1u : 0u);
          }
          umma_commit<1>(a ? bar_mma1 : bar_mma);
        }
      }
    }
    if (!wide) {
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
          uint32_t nf = 0;
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int q = q0 + 8 * h;
            uint32_t o[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              o[e] = pk_bf2(__uint_as_float(r[8 * h + 2 * e]), __uint_as_float(r[8 * h + 2 * e + 1]));
              nf |= (o[e] & 0x7F807F80u) + 0x00800080u;
            }
            *reinterpret_cast<uint4*>(sm + slab_box(g, 0, p >> 6, q >> 6) + swz((uint32_t)(p & 63), (uint32_t)(q & 63))) =
                make_uint4(o[0], o[1], o[2], o[3]);
          }
          bad |= (nf & 0x80008000u) != 0;
        }
      }
      ph0 ^= 1;
      if (nacc_x > 1) ph1 ^= 1;
    } else {
      mbar_wait(bar_mma, ph0);  // the slab is the B operand of both accumulators
      if (nacc_g > 1) mbar_wait(bar_mma1, ph1);
      TC_TL();
      tc_fence_after();
      for (int a = 0; a < nacc_g; ++a) {
        const int n = a * 128 + qd * 32 + lane;
        for (int c = warp >> 2; c < g.R / 32; c += 2) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem + lane_base + (uint32_t)(a * 256 + c * 32), r);
          tmem_ld_wait_regs(r);
          uint32_t nf = 0;
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int m = c * 32 + 8 * h;
            uint32_t o[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              o[e] = pk_bf2(__uint_as_float(r[8 * h + 2 * e]), __uint_as_float(r[8 * h + 2 * e + 1]));
              nf |= (o[e] & 0x7F807F80u) + 0x00800080u;
            }
            *reinterpret_cast<uint4*>(sm + slab_box(g, 1, m >> 6, n >> 6) + swz((uint32_t)(n & 63), (uint32_t)(m & 63))) =
                make_uint4(o[0], o[1], o[2], o[3]);
          }
          bad |= (nf & 0x80008000u) != 0;
        }
      }
      ph0 ^= 1;
      if (nacc_g > 1) ph1 ^= 1;
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
