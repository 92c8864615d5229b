// Host-side launch wrappers for the device kernels (implemented in *.cu).
#pragma once
#include <cuda_runtime.h>

#include <utility>
#include <vector>

#include "jobs.h"

namespace tns {

// tcgen05 bf16 engine (umma_gemm.cu).  One persistent launch over all jobs' tiles.
// cg = 1: 128 x 256 tiles per CTA; cg = 2: 256 x 256 tiles per CTA pair (cta_group::2).
// d_tasks: the launch's task list (TaskDesc, TK_TILE or TK_NONE padding) in execution
// order; max_tiles = tiles of the step (grid sizing).  split: the task list holds split-K
// tasks (TaskDesc::split != 0).  bn: tile width 256, or 128 (cg = 2 only) -- the tile list
// must have been built with the same bn.
cudaError_t launch_umma_gemm(const GemmJob* d_jobs, const TaskDesc* d_tasks, int64_t ntasks, int64_t max_tiles,
                             int cg, int num_sms, uint32_t* d_flags, bool split, int bn, cudaStream_t stream);
// Read (and optionally reset) the epilogue clock counters (TNS_DBG bit 8 measurement).
cudaError_t umma_epi_prof(unsigned long long* out, bool reset);
// Append the tiles of job `job` (host side), bn = tile width (256 or 128).
void umma_tile_list(const GemmJob& J, uint32_t job, int cg, int bn, std::vector<uint64_t>& out);

// CUDA-core engine (simt.cu); is_bf16 selects the storage type.
cudaError_t launch_simt_gemm(const SimtJob* d_jobs, int njobs, int64_t total_tiles, int num_sms,
                             bool is_bf16, uint32_t* d_flags, cudaStream_t stream);

// Fused AOL / Frobenius preconditioner (simt.cu): row-abs-sum (or trace) + rsqrt, grid
// barrier, then A <- diag(s) A diag(s).  `barrier` points at two zero-initialised uint32
// words (arrival count, generation) owned by the caller; the barrier resets itself.
// total_segs = sum of precond_segments(N, half) over jobs (PrecondJob::seg_start prefix);
// vec8 = all N are multiples of 8 and A 16-byte aligned (16-byte vectors).
// lane_rows: AOL from Gram partials with part_ld <= kSeqPartials for every job -> phase 1
// runs one lane per row (precond_rows.cuh).
cudaError_t launch_precondition(const PrecondJob* d_jobs, int njobs, int64_t total_rows,
                                int64_t total_segs, bool vec8, bool is_bf16,
                                unsigned* d_barrier, uint32_t* d_flags, int lane_mode, cudaStream_t stream);
// lane_mode: bit 0 = AOL from the Gram partials for every job (lane loops); with it, bits
// 3 / 4 / 5 = some job's rows are summed by four lanes / a warp / one lane (precond_rows.cuh)
__host__ __device__ inline int precond_lane_kind(int part_ld) {
  return part_ld <= kSeqPartials ? 32 : (part_ld <= kQuarterPartials ? 8 : 16);
}

// Split-K Gram reduction (simt.cu): one warp per row of every job (bf16 storage).
cudaError_t launch_split_reduce(const SplitJob* d_jobs, int njobs, int64_t total_rows, uint32_t* d_flags,
                                cudaStream_t stream);

// Whole NS of `njobs` small matrices, one cluster of `ctas` (8 or 16) CTAs each (cluster_ns.cu).
// d_coeffs: 3*iters floats in device memory; smem_bytes: max cl_layout(..).floats * 4.
cudaError_t launch_cluster_ns(const ClusterJob* d_jobs, int njobs, const float* d_coeffs, int iters, int precond,
                              bool is_bf16, size_t smem_bytes, int ctas, uint32_t* d_flags, cudaStream_t stream);
// TNS_DBG bit 128 measurement: per-phase clock64 offsets of cluster 0 summed over launches
// (8 phase marks + launch count).
cudaError_t cluster_timeline(unsigned long long* out9, bool reset);

// Whole NS of `njobs` mid-size bf16 matrices on the tensor cores, one cluster of `ctas` CTAs
// each (every job's C == ctas; cluster_tc.cu); smem_bytes = max tc_smem(Np, R) over the jobs;
// d_coeffs: 3*iters floats.
cudaError_t launch_cluster_tc_ns(const TcJob* d_jobs, int njobs, int ctas, const float* d_coeffs, int iters,
                                 int precond, size_t smem_bytes, uint32_t* d_flags, cudaStream_t stream);

// fp32 <-> bf16 storage casts of a mixed-precision call (muon.cu), one launch for all jobs.
cudaError_t launch_cast(const CastJob* d_jobs, int count, int64_t max_numel, bool to_bf16, int sms,
                        cudaStream_t stream);

// Muon step around the path (muon.cu): momentum + nesterov -> bf16 U; W update from U.
cudaError_t launch_muon_momentum(const MuonJob* d_jobs, int count, int64_t max_numel, bool g_bf16, float beta, float gscale,
                                 int nesterov, int sms, cudaStream_t stream);
cudaError_t launch_muon_apply(const MuonJob* d_jobs, int count, int64_t max_numel, bool w_bf16, float lr, float wd,
                              int sms, cudaStream_t stream);

}  // namespace tns
