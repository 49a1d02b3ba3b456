// bo_ep.cu - row-block permutation used by the expert-parallel exchange.
//
// Under expert parallelism rows arrive from every source rank
// ordered (source, executor, expert, token); the grouped GEMMs need them
// ordered (executor, source, expert, token), and the results go back the
// other way.  Both are block permutations whose block tables the host derives
// from the all-gathered counts; this kernel moves the rows (16-byte vectors,
// warp per row) and the per-row gate weight that travels with them.
#include "bo_kernels.h"
#include "bo_ptx.cuh"

namespace bo {

__global__ void __launch_bounds__(256) k_block_copy(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                    int vec_per_row, const float* __restrict__ w_src,
                                                    float* __restrict__ w_dst, int n_blocks,
                                                    const int32_t* __restrict__ src_off,
                                                    const int32_t* __restrict__ dst_start, int64_t total_rows) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = gw; i < total_rows; i += nw) {
    int lo = 0, hi = n_blocks;   // dst_start[lo] <= i < dst_start[hi]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (dst_start[mid] <= i) lo = mid; else hi = mid;
    }
    const int64_t srow = static_cast<int64_t>(src_off[lo]) + (i - dst_start[lo]);
    const uint4* sp = src + srow * vec_per_row;
    uint4* dp = dst + i * vec_per_row;
    for (int c = lane; c < vec_per_row; c += 32) dp[c] = __ldg(sp + c);
    if (w_src && lane == 0) w_dst[i] = w_src[srow];
  }
}

cudaError_t launch_block_copy(const void* src, void* dst, int row_bytes, const float* w_src, float* w_dst,
                              int n_blocks, const int32_t* src_off, const int32_t* dst_start, int64_t total_rows,
                              int num_sms, cudaStream_t s) {
  if (total_rows <= 0 || n_blocks <= 0) return cudaSuccess;
  int64_t blocks = (total_rows + 7) / 8;
  if (blocks > num_sms * 8) blocks = num_sms * 8;
  k_block_copy<<<static_cast<int>(blocks), 256, 0, s>>>(static_cast<const uint4*>(src), static_cast<uint4*>(dst),
                                                        row_bytes / 16, w_src, w_dst, n_blocks, src_off, dst_start,
                                                        total_rows);
  return cudaGetLastError();
}

}  // namespace bo
