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

// ----------------------------------------------------------------------------
// Row de-duplication of united experts (oracle
// permutation_dedup).  Under Eq. 5-6 a token whose slots s1, s2 are delegated to
// the same united expert contributes q1 F_u(x) + q2 F_u(x) = (q1 + q2) F_u(x),
// so one row with the summed weight replaces the duplicates.  Alg. 1 itself is
// unchanged (it runs on the assignment counts); only the rows are recounted.
namespace bo {

// Per token tile: rows per executor after merging (first occurrence of each
// executor among the token's K slots).
__global__ void __launch_bounds__(256) k_dedup_count(const int32_t* __restrict__ topk_id, int T, int K, int tile,
                                                     int E, const int32_t* __restrict__ exec_of,
                                                     int32_t* __restrict__ tile_xcnt) {
  __shared__ int hist[kMaxExec];
  for (int i = threadIdx.x; i < E; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const int t0 = blockIdx.x * tile;
  const int t1 = min(t0 + tile, T);
  for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
    int xs[16];
    for (int s = 0; s < K; ++s) {
      const int x = exec_of[__ldg(topk_id + static_cast<int64_t>(t) * K + s)];
      xs[s] = x;
      bool dup = false;
      for (int q = 0; q < s; ++q) dup |= xs[q] == x;
      if (x >= 0 && !dup) atomicAdd(&hist[x], 1);   // integer count: order-independent
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < E; i += blockDim.x) tile_xcnt[static_cast<int64_t>(blockIdx.x) * E + i] = hist[i];
}

// One CTA: per-executor prefix over tiles, executor row offsets, m-tile prefix,
// and the row statistics of the merged layout.
__global__ void __launch_bounds__(512) k_dedup_plan(const int32_t* __restrict__ tile_xcnt, int ntiles, int m, int E,
                                                    int32_t* __restrict__ tile_xbase, int32_t* __restrict__ exec_off,
                                                    int32_t* __restrict__ mtile_off, int64_t* __restrict__ stats) {
  __shared__ int s_rows[kMaxExec];
  __shared__ int s_scan[kMaxExec + 1];
  __shared__ int s_scan2[kMaxExec + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int x = warp; x < E; x += 16) {   // warp per executor, lanes over tiles
    int carry = 0;
    for (int t0 = 0; t0 < ntiles; t0 += 32) {
      const int t = t0 + lane;
      const int v = t < ntiles ? __ldg(tile_xcnt + static_cast<int64_t>(t) * E + x) : 0;
      int incl = v;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
      }
      if (t < ntiles) tile_xbase[static_cast<int64_t>(t) * E + x] = carry + incl - v;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) s_rows[x] = carry;
  }
  __syncthreads();
  if (threadIdx.x == 0) {   // E <= 512: a short serial scan
    int a = 0, b = 0;
    for (int x = 0; x < E; ++x) {
      s_scan[x] = a;
      s_scan2[x] = b;
      a += s_rows[x];
      b += (s_rows[x] + kBM - 1) / kBM;
    }
    s_scan[E] = a;
    s_scan2[E] = b;
    long long r_orig = 0;
    for (int x = 0; x < m; ++x) r_orig += s_rows[x];
    stats[4] = r_orig;
    stats[5] = a - r_orig;                         // united rows after merging
    stats[6] = stats[7] - a;                       // assignments without a row of their own (dropped + merged)
  }
  __syncthreads();
  for (int x = threadIdx.x; x <= E; x += blockDim.x) {
    exec_off[x] = s_scan[x];
    mtile_off[x] = s_scan2[x];
  }
}

// Per token tile: stable rank of each (token, executor) first occurrence inside
// its executor (token order), row = exec_off + tile prefix + rank; the row carries
// the summed gate weight of the token's slots on that executor (slot order).
__global__ void __launch_bounds__(256) k_permute_dedup(const int32_t* __restrict__ topk_id,
                                                       const float* __restrict__ topk_w, int T, int K, int tile,
                                                       int E, const int32_t* __restrict__ exec_of,
                                                       const int32_t* __restrict__ tile_xbase,
                                                       const int32_t* __restrict__ exec_off,
                                                       int32_t* __restrict__ row_of, int32_t* __restrict__ row_tok,
                                                       float* __restrict__ row_w) {
  __shared__ int wcnt[8][kMaxExec];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 8 * kMaxExec; i += blockDim.x) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const int64_t a0 = static_cast<int64_t>(blockIdx.x) * tile * K;
  const int64_t a1 = min(static_cast<int64_t>(blockIdx.x + 1) * tile, static_cast<int64_t>(T)) * K;
  const int n = static_cast<int>(a1 - a0);
  const int per_warp = ((n + 8 * 32 - 1) / (8 * 32)) * 32;
  const int w0 = warp * per_warp;
  const int w1 = min(w0 + per_warp, n);
  // key of an assignment: its executor if it is the token's first slot on that executor, else -1
  auto key_of = [&](int i) -> int {
    if (i >= w1) return -1;
    const int64_t a = a0 + i;
    const int64_t t = a / K;
    const int s = static_cast<int>(a - t * K);
    const int x = exec_of[__ldg(topk_id + a)];
    if (x < 0) return -1;
    for (int q = 0; q < s; ++q)
      if (exec_of[__ldg(topk_id + t * K + q)] == x) return -1;
    return x;
  };
  for (int base = w0; base < w1; base += 32) {
    const int x = key_of(base + lane);
    const uint32_t peers = __match_any_sync(0xffffffffu, x);
    const int leader = __ffs(peers) - 1;
    if (lane == leader && x >= 0) wcnt[warp][x] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (int x = threadIdx.x; x < E; x += blockDim.x) {
    int run = 0;
    for (int w = 0; w < 8; ++w) {
      const int c = wcnt[w][x];
      wcnt[w][x] = run;
      run += c;
    }
  }
  __syncthreads();
  const uint32_t lt = lanemask_lt();
  for (int base = w0; base < w1; base += 32) {
    const int i = base + lane;
    const int x = key_of(i);
    const uint32_t peers = __match_any_sync(0xffffffffu, x);
    const int leader = __ffs(peers) - 1;
    const int start = x >= 0 ? wcnt[warp][x] : 0;
    __syncwarp();
    if (lane == leader && x >= 0) wcnt[warp][x] = start + __popc(peers);
    __syncwarp();
    if (i < w1) {
      const int64_t a = a0 + i;
      if (x >= 0) {
        const int64_t t = a / K;
        const int r = exec_off[x] + tile_xbase[static_cast<int64_t>(blockIdx.x) * E + x] + start + __popc(peers & lt);
        float w = 0.0f;
        for (int q = 0; q < K; ++q)   // merged weight, slot order
          if (exec_of[__ldg(topk_id + t * K + q)] == x) w += __ldg(topk_w + t * K + q);
        row_of[a] = r;
        row_tok[r] = static_cast<int32_t>(t);
        row_w[r] = w;
      } else {
        row_of[a] = -1;
      }
    }
  }
}

cudaError_t launch_dedup(int stage, const int32_t* topk_id, const float* topk_w, int T, int K, int tile, int m,
                         int E, const int32_t* exec_of, int32_t* tile_xcnt, int32_t* tile_xbase, int32_t* exec_off,
                         int32_t* mtile_off, int64_t* stats, int32_t* row_of, int32_t* row_tok, float* row_w,
                         cudaStream_t s) {
  const int ntiles = (T + tile - 1) / tile;
  if (ntiles == 0) return cudaSuccess;
  if (stage == 0) k_dedup_count<<<ntiles, 256, 0, s>>>(topk_id, T, K, tile, E, exec_of, tile_xcnt);
  else if (stage == 1) k_dedup_plan<<<1, kMaxExec, 0, s>>>(tile_xcnt, ntiles, m, E, tile_xbase, exec_off, mtile_off,
                                                            stats);
  else k_permute_dedup<<<ntiles, 256, 0, s>>>(topk_id, topk_w, T, K, tile, E, exec_of, tile_xbase, exec_off, row_of,
                                              row_tok, row_w);
  return cudaGetLastError();
}

}  // namespace bo
