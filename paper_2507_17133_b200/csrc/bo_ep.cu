// bo_ep.cu - device side of the expert-parallel exchange:
// the per-forward exchange tables computed from the all-gathered counts (no host
// round trip), and the row-block permutation between the exchange layout
// (source, executor, expert, token) and the grouped GEMMs' layout (executor,
// source, expert, token).
#include "bo_kernels.h"
#include "bo_ptx.cuh"

namespace bo {

// Exclusive scan of in[0, n) into out[0, n) by one warp (chunks of 32, shuffle scan
// plus carry); returns the total.  in / out may alias.
__device__ int warp_excl_scan(const int* in, int* out, int n, int lane) {
  int carry = 0;
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    const int v = i < n ? in[i] : 0;
    int incl = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int o = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += o;
    }
    __syncwarp();
    if (i < n) out[i] = carry + incl - v;
    carry += __shfl_sync(0xffffffffu, incl, 31);
    __syncwarp();
  }
  return carry;
}

// One CTA.  gathered [R, ld] count rows (this forward's counts of every rank, D18),
// exec_of_expert [m] of the global plan.  Writes the tables of EpTables (bo_kernels.h).
__global__ void __launch_bounds__(512) k_ep_tables(const __grid_constant__ EpStatic st,
                                                   const int32_t* __restrict__ gathered, int ld,
                                                   const int32_t* __restrict__ exec_of, EpTables tb) {
  __shared__ int s_exec[kMaxExperts];
  __shared__ int s_rows[kEpMaxRanks * kEpMaxV];   // rows[r][v]
  __shared__ int s_pre[kEpMaxV];                  // send prefix over v (this rank as source)
  __shared__ int s_base[kEpMaxV];
  __shared__ int s_flat[kEpMaxRanks * kEpMaxV];   // scratch for (i, r) / (r, i) scans
  const int R = st.R, m = st.m, V = st.V, nl = st.nl, me = st.rank;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < m; e += blockDim.x) s_exec[e] = exec_of[e];
  __syncthreads();
  // rows[r][v]: assignments of source r's batch that virtual executor v processes
  for (int i = tid; i < R * V; i += blockDim.x) {
    const int r = i / V, v = i - r * V;
    const int code = st.vexec[v];
    const int idx = code & 0xffff;
    int rows = 0;
    if (((code >> 23) & 1) == 0) {   // original expert idx: its own rows when it executes as itself
      rows = s_exec[idx] == idx ? gathered[r * ld + idx] : 0;
    } else {                          // slice of united expert idx: every member delegated to it
      const int e1 = min((idx + 1) * st.way, m);
      for (int e = idx * st.way; e < e1; ++e)
        if (s_exec[e] == m + idx) rows += gathered[r * ld + e];
    }
    s_rows[i] = rows;
  }
  __syncthreads();
  // source side (r = me): segment of each v in the send buffer
  if (warp == 0) {
    warp_excl_scan(s_rows + me * V, s_pre, V, lane);
    for (int v = lane; v < V; v += 32) {
      const int q = (st.vexec[v] >> 24) & 0xff;
      s_base[v] = st.padded ? static_cast<int>(q * st.cap) + s_pre[v] - s_pre[st.vfirst[q]] : s_pre[v];
    }
  }
  if (warp == 1) {   // rows this rank sends to q
    for (int q = lane; q < R; q += 32) {
      int n = 0;
      for (int v = st.vfirst[q]; v < st.vfirst[q + 1]; ++v) n += s_rows[me * V + v];
      tb.send_rows[q] = n;
      tb.splits[q] = n;
    }
  }
  if (warp == 2) {   // rows q receives from each source r (this rank as destination)
    for (int r = lane; r < R; r += 32) {
      int n = 0;
      for (int i = 0; i < nl; ++i) n += s_rows[r * V + st.local_v[i]];
      tb.recv_rows[r] = n;
      tb.splits[R + r] = n;
    }
  }
  __syncthreads();
  // row_base[e * nrep + rep] (dispatch of this rank's assignments)
  for (int e = tid; e < m; e += blockDim.x) {
    const int x = s_exec[e];
    for (int rep = 0; rep < st.nrep; ++rep) tb.row_base[e * st.nrep + rep] = -1;
    if (x >= 0 && x < m) {
      tb.row_base[e * st.nrep] = s_base[st.v_of_orig[e]];
    } else if (x >= m) {
      const int j = x - m;
      int acc = 0;   // earlier members of the same united executor (member order, D11)
      for (int e2 = j * st.way; e2 < e; ++e2)
        if (s_exec[e2] == x) acc += gathered[me * ld + e2];
      for (int sl = 0; sl < st.nslices; ++sl) tb.row_base[e * st.nrep + sl] = s_base[st.v_of_slice[j * st.nrep + sl]] + acc;
    }
  }
  // destination side: receive offsets recv_blk[r][i] (r, i order) and grouped offsets (i, r order)
  __shared__ int s_rbase[kEpMaxRanks + 1];
  if (warp == 0) {
    // source segment starts: exact = prefix of recv_rows, padded = r * cap
    int run = 0;
    for (int r = 0; r < R; ++r) {
      if (lane == 0) s_rbase[r] = st.padded ? static_cast<int>(r * st.cap) : run;
      int n = 0;
      for (int i = lane; i < nl; i += 32) n += s_rows[r * V + st.local_v[i]];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) n += __shfl_xor_sync(0xffffffffu, n, off);
      run += n;
    }
    if (lane == 0) s_rbase[R] = st.padded ? static_cast<int>(R * st.cap) : run;
  }
  __syncthreads();
  // (r, i) order: inverse-table destinations = receive layout
  for (int k = tid; k < R * nl; k += blockDim.x) {
    const int r = k / nl, i = k - r * nl;
    s_flat[k] = s_rows[r * V + st.local_v[i]];
  }
  __syncthreads();
  if (warp == 0) {
    for (int r = 0; r < R; ++r) warp_excl_scan(s_flat + r * nl, s_flat + r * nl, nl, lane);
  }
  __syncthreads();
  for (int k = tid; k < R * nl; k += blockDim.x) {
    const int r = k / nl, i = k - r * nl;
    tb.inv_dst[k] = s_rbase[r] + s_flat[k];       // recv_blk[r][i]
    tb.fwd_src[i * R + r] = s_rbase[r] + s_flat[k];
    const int len = s_rows[r * V + st.local_v[i]];
    tb.inv_len[k] = len;
    tb.fwd_len[i * R + r] = len;
  }
  __syncthreads();
  // (i, r) order: grouped layout (executor-major, then source)
  for (int k = tid; k < R * nl; k += blockDim.x) {
    const int i = k / R, r = k - i * R;
    s_flat[k] = s_rows[r * V + st.local_v[i]];
  }
  __syncthreads();
  int total = 0;
  if (warp == 0) total = warp_excl_scan(s_flat, s_flat, R * nl, lane);
  __syncthreads();
  for (int k = tid; k < R * nl; k += blockDim.x) {
    const int i = k / R, r = k - i * R;
    tb.fwd_dst[k] = s_flat[k];
    tb.inv_src[r * nl + i] = s_flat[k];
  }
  if (warp == 0) {
    // executor row offsets and the m-tile prefix of the local grouped GEMMs
    int carry = 0, mcarry = 0;
    for (int i0 = 0; i0 < nl; i0 += 32) {
      const int i = i0 + lane;
      int rows = 0;
      if (i < nl)
        for (int r = 0; r < R; ++r) rows += s_rows[r * V + st.local_v[i]];
      int a = rows, b = (rows + kBM - 1) / kBM;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int oa = __shfl_up_sync(0xffffffffu, a, off), ob = __shfl_up_sync(0xffffffffu, b, off);
        if (lane >= off) { a += oa; b += ob; }
      }
      if (i < nl) {
        tb.exec_off[i] = carry + a - rows;
        tb.mtile_off[i] = mcarry + b - (rows + kBM - 1) / kBM;
      }
      carry += __shfl_sync(0xffffffffu, a, 31);
      mcarry += __shfl_sync(0xffffffffu, b, 31);
    }
    if (lane == 0) {
      tb.exec_off[nl] = carry;
      tb.mtile_off[nl] = mcarry;
      tb.fwd_dst[R * nl] = total;
      tb.inv_dst[R * nl] = s_rbase[R];
      tb.totals[0] = total;         // grouped rows
      tb.totals[1] = s_rbase[R];    // receive-layout extent
    }
  }
}

cudaError_t launch_ep_tables(const EpStatic& st, const int32_t* gathered, int ld, const int32_t* exec_of,
                             const EpTables& tb, cudaStream_t s) {
  k_ep_tables<<<1, 512, 0, s>>>(st, gathered, ld, exec_of, tb);
  return cudaGetLastError();
}

// Row-block copy: block b moves len[b] rows src_off[b] + k -> dst_start[b] + k
// (dst_start ascending; rows of the destination no block covers are left alone),
// with the float weight that travels with each row when w_src != nullptr.  The
// destination extent is read on the device (*extent, capped at extent_max).
__global__ void __launch_bounds__(256) k_block_copy(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                    int vec_per_row, const float* __restrict__ w_src,
                                                    float* __restrict__ w_dst, int n_blocks,
                                                    const int32_t* __restrict__ dst_start,
                                                    const int32_t* __restrict__ len,
                                                    const int32_t* __restrict__ src_off,
                                                    const int32_t* __restrict__ extent, int64_t extent_max) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  int64_t total = extent ? static_cast<int64_t>(*extent) : extent_max;
  total = total < extent_max ? total : extent_max;
  for (int64_t i = gw; i < total; i += nw) {
    int lo = 0, hi = n_blocks;   // last block with dst_start[lo] <= i
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (dst_start[mid] <= i) lo = mid; else hi = mid;
    }
    const int64_t k = i - dst_start[lo];
    if (k < 0 || k >= len[lo]) continue;
    const int64_t srow = static_cast<int64_t>(src_off[lo]) + k;
    const uint4* sp = src + srow * vec_per_row;
    uint4* dp = dst + i * vec_per_row;
    for (int c = lane; c < vec_per_row; c += 32) dp[c] = __ldg(sp + c);
    if (w_src && lane == 0) w_dst[i] = w_src[srow];
  }
}

cudaError_t launch_block_copy(const void* src, void* dst, int row_bytes, const float* w_src, float* w_dst,
                              int n_blocks, const int32_t* dst_start, const int32_t* len, const int32_t* src_off,
                              const int32_t* extent, int64_t extent_max, int num_sms, cudaStream_t s) {
  if (extent_max <= 0 || n_blocks <= 0) return cudaSuccess;
  int64_t blocks = (extent_max + 7) / 8;
  if (blocks > num_sms * 8) blocks = num_sms * 8;
  k_block_copy<<<static_cast<int>(blocks), 256, 0, s>>>(static_cast<const uint4*>(src), static_cast<uint4*>(dst),
                                                        row_bytes / 16, w_src, w_dst, n_blocks, dst_start, len,
                                                        src_off, extent, extent_max);
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
  // per-warp counts without atomics: the lanes holding the same executor meet in
  // __match_any_sync and the lowest of them adds the group's size to its warp's row
  __shared__ int hist[8][kMaxExec];
  for (int i = threadIdx.x; i < 8 * kMaxExec; i += blockDim.x) (&hist[0][0])[i] = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = blockIdx.x * tile;
  const int t1 = min(t0 + tile, T);
  for (int tb = t0; tb < t1; tb += blockDim.x) {   // warp-uniform trip count
    const int t = tb + threadIdx.x;
    int xs[16];
    for (int s = 0; s < K; ++s) {
      const int x = t < t1 ? exec_of[__ldg(topk_id + static_cast<int64_t>(t) * K + s)] : -1;
      xs[s] = x;
      bool dup = false;
      for (int q = 0; q < s; ++q) dup |= xs[q] == x;
      const int key = (x >= 0 && !dup) ? x : -1;
      const uint32_t peers = __match_any_sync(0xffffffffu, key);
      if (key >= 0 && lane == __ffs(peers) - 1) hist[warp][key] += __popc(peers);
      __syncwarp();
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < E; i += blockDim.x) {
    int c = 0;
    for (int w = 0; w < 8; ++w) c += hist[w][i];
    tile_xcnt[static_cast<int64_t>(blockIdx.x) * E + i] = c;
  }
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
