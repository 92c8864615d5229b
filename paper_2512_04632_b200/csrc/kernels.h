// Host-side launch wrappers for the device kernels (implemented in *.cu).
#pragma once
#include <cuda_runtime.h>

#include "jobs.h"

namespace tns {

// tcgen05 bf16 engine (umma_gemm.cu).  One persistent launch over all jobs' tiles.
// cg = 1: 128 x 256 tiles per CTA; cg = 2: 256 x 256 tiles per CTA pair (cta_group::2).
cudaError_t launch_umma_gemm(const GemmJob* d_jobs, int njobs, int64_t total_tiles, int cg,
                             int num_sms, uint32_t* d_flags, cudaStream_t stream);
// Number of tiles of one job for the given cta group (host side).
int umma_tiles(int sym, int P, int Q, int cg);

// CUDA-core engine (simt.cu); is_bf16 selects the storage type.
cudaError_t launch_simt_gemm(const SimtJob* d_jobs, int njobs, int64_t total_tiles, int num_sms,
                             bool is_bf16, uint32_t* d_flags, cudaStream_t stream);

// Fused AOL / Frobenius preconditioner (simt.cu): row-abs-sum (or trace) + rsqrt, grid
// barrier, then A <- diag(s) A diag(s).  `barrier` must point at a zeroed uint32 (the
// wrapper zeroes it on `stream`).  vec8 = all N are multiples of 8 (16-byte vectors).
cudaError_t launch_precondition(const PrecondJob* d_jobs, int njobs, int64_t total_rows,
                                int64_t total_elems_or_vecs, bool vec8, bool is_bf16,
                                unsigned* d_barrier, uint32_t* d_flags, cudaStream_t stream);

}  // namespace tns
