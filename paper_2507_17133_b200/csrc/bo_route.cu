// bo_route.cu - routing, Algorithm-1 plan, permutation, gather, combine, united init.
//
// Kernels (all deterministic, no floating-point atomics):
//   k_topk_hist   Eq. 7: per token, K largest fp32 logits (ties ->
//                 lower id, reading D8) by warp-shuffle argmax; softmax over the
//                 K selected; per-tile expert histogram (Alg. 1 cnt_i).
//   k_plan        Alg. 1 on one CTA: counts, rank-by-counting sort
//                 (cnt desc, id asc, D5), exclusive prefix in sorted order,
//                 S1 iff prefix < T = S * (1 - ratio) in fp64 (D1, D3), S2
//                 grouped by floor(e / way), special case, executor
//                 map, row offsets (executor, expert, token order, D11).
//   k_permute     stable in-expert rank of every (token, slot) assignment via
//                 __match_any_sync + popc (no atomics) -> row_of / row_tok / row_w.
//   k_gather      concat_tokens: Xp[row] = x[token], 16-byte vectors,
//                 each token read once and written to its K rows.
//   k_combine     Eq. 5 sum: y[t] = [x_t] + sum_s Yp[row_of(t,s)], fp32,
//                 slot order.
//   k_united_mean united-expert init (D14): fp64 group mean, one RNE rounding.
#include <float.h>

#include <atomic>

#include <cooperative_groups.h>

#include "bo_kernels.h"
#include "bo_ptx.cuh"

namespace bo {

namespace cg = cooperative_groups;

// ----------------------------------------------------------------- top-k
// Warp-cooperative Eq. 7 for one token whose m logits are spread over the
// lanes (expert e = lane + 32*j in v[j]).  K rounds of a shuffle argmax over
// (logit desc, id asc) (reading D8; -0 == +0 by IEEE comparison), then the
// softmax over the K selected.  Lane s < K returns slot s (id, weight).
template <int VPL>
__device__ __forceinline__ void warp_topk_softmax(const float (&v)[VPL], int m, int K, int lane, int& my_id,
                                                  float& my_w) {
  uint32_t taken = 0;
  my_id = -1;
  float my_v = 0.0f;
  for (int s = 0; s < K; ++s) {
    float bv = -FLT_MAX;
    int bi = 0x7fffffff;
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int e = lane + 32 * j;
      if (e < m && !((taken >> j) & 1u) && (bi == 0x7fffffff || v[j] > bv)) { bv = v[j]; bi = e; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      const bool better = oi != 0x7fffffff && (bi == 0x7fffffff || ov > bv || (ov == bv && oi < bi));
      if (better) { bv = ov; bi = oi; }
    }
    if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
    if (lane == s) { my_id = bi; my_v = bv; }
  }
  const float vmax = __shfl_sync(0xffffffffu, my_v, 0);   // slot 0 holds the maximum
  const float ex = lane < K ? expf(my_v - vmax) : 0.0f;
  float sum = ex;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
  my_w = ex / sum;
}

// Top-K of given fp32 logits (parity entry / injected logits) + per-tile histogram.
template <int VPL>
__global__ void __launch_bounds__(512) k_topk_hist(const float* __restrict__ logits, int T, int m, int K, int tile,
                                                   int32_t* __restrict__ topk_id, float* __restrict__ topk_w,
                                                   int32_t* __restrict__ tile_cnt) {
  // per-warp expert counts (a token's K ids are distinct, so lane writes never collide;
  // no atomics), summed over the warps in a fixed order at the end
  __shared__ int hist[16][kMaxExperts];
  for (int i = threadIdx.x; i < 16 * kMaxExperts; i += blockDim.x) (&hist[0][0])[i] = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = blockIdx.x * tile;
  const int t1 = min(t0 + tile, T);
  const int nw = blockDim.x >> 5;
  for (int t = t0 + warp; t < t1; t += nw) {
    float v[VPL];
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int e = lane + 32 * j;
      v[j] = e < m ? __ldg(logits + static_cast<int64_t>(t) * m + e) : 0.0f;
    }
    int id;
    float w;
    warp_topk_softmax<VPL>(v, m, K, lane, id, w);
    if (lane < K) {
      topk_id[static_cast<int64_t>(t) * K + lane] = id;
      topk_w[static_cast<int64_t>(t) * K + lane] = w;
      hist[warp][id] += 1;
    }
    __syncwarp();
  }
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    int c = 0;
    for (int w = 0; w < nw; ++w) c += hist[w][i];
    tile_cnt[static_cast<int64_t>(blockIdx.x) * m + i] = c;
  }
}

cudaError_t launch_topk_hist(const float* logits, int T, int m, int K, int tile, int32_t* topk_id, float* topk_w,
                             int32_t* tile_cnt, cudaStream_t s) {
  const int ntiles = (T + tile - 1) / tile;
  if (ntiles == 0) return cudaSuccess;
  const int vpl = (m + 31) / 32;
  const int threads = tile >= 128 ? 512 : 256;   // a warp per token, tokens of the tile over 8-16 warps
  switch (vpl) {
#define BO_TOPK_CASE(N) \
  case N: k_topk_hist<N><<<ntiles, threads, 0, s>>>(logits, T, m, K, tile, topk_id, topk_w, tile_cnt); break;
    BO_TOPK_CASE(1) BO_TOPK_CASE(2) BO_TOPK_CASE(3) BO_TOPK_CASE(4)
    BO_TOPK_CASE(5) BO_TOPK_CASE(6) BO_TOPK_CASE(7) BO_TOPK_CASE(8)
#undef BO_TOPK_CASE
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// ------------------------------------------------------- small-m router
// Eq. 8 + Eq. 7 + histogram in one pass for m <= 32 (Mixtral: 8 experts):
// the contraction has N = m, far too narrow for a tensor-core tile, and the
// step is bound by reading x once (HBM), so it runs on the CUDA cores with
// the router centroids staged in shared memory by cp.async.  Warp per token,
// 16-byte loads of x issued in batches of 8 per lane (memory-level
// parallelism), fp32 accumulation, one shuffle all-reduce per expert, then the
// warp top-K.  A CTA covers `tile` tokens (8 warps x tile/8 tokens).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <typename T>
__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[16 / sizeof(T)]) {
  if constexpr (sizeof(T) == 2) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 t = __bfloat1622float2(h[i]);
      f[2 * i] = t.x;
      f[2 * i + 1] = t.y;
    }
  } else {
    f[0] = __uint_as_float(v.x);
    f[1] = __uint_as_float(v.y);
    f[2] = __uint_as_float(v.z);
    f[3] = __uint_as_float(v.w);
  }
}

template <typename T, int MAXM, int TPW>
__global__ void __launch_bounds__(256) k_router_small(const T* __restrict__ x, const T* __restrict__ Wr, int Tn,
                                                      int d, int m, int K, float* __restrict__ logits,
                                                      int32_t* __restrict__ topk_id, float* __restrict__ topk_w,
                                                      int32_t* __restrict__ tile_cnt) {
  extern __shared__ uint4 s_wr[];
  __shared__ int hist[8][32];   // per-warp expert counts (no atomics), summed in warp order
  constexpr int EPV = 16 / sizeof(T);         // elements per 16-byte vector
  constexpr int BATCH = TPW >= 4 ? 4 : (TPW == 2 ? 8 : 16);   // 16-byte loads per token in flight per lane
  const int nvec = d / EPV;
  {
    const uint4* src = reinterpret_cast<const uint4*>(Wr);
    for (int i = threadIdx.x; i < m * nvec; i += blockDim.x) cp_async16(s_wr + i, src + i);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  hist[warp][lane] = 0;
  const int tbase = blockIdx.x * (8 * TPW) + warp * TPW;   // this warp's TPW consecutive tokens
  float acc[TPW][MAXM];
#pragma unroll
  for (int i = 0; i < TPW; ++i)
#pragma unroll
    for (int e = 0; e < MAXM; ++e) acc[i][e] = 0.0f;
  bool waited = false;
  for (int c0 = 0; c0 < nvec; c0 += 32 * BATCH) {
    uint4 xv[TPW][BATCH];
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
      const int t = tbase + i;
#pragma unroll
      for (int b = 0; b < BATCH; ++b) {
        const int c = c0 + b * 32 + lane;
        xv[i][b] = (t < Tn && c < nvec) ? __ldg(reinterpret_cast<const uint4*>(x + static_cast<int64_t>(t) * d) + c)
                                        : make_uint4(0, 0, 0, 0);
      }
    }
    if (!waited) {   // centroids land in shared memory while the first x batch is in flight
      cp_async_wait_all();
      __syncthreads();
      waited = true;
    }
#pragma unroll
    for (int b = 0; b < BATCH; ++b) {
      const int c = c0 + b * 32 + lane;
      if (c < nvec) {
        float xf[TPW][EPV];
#pragma unroll
        for (int i = 0; i < TPW; ++i) unpack8<T>(xv[i][b], xf[i]);
#pragma unroll
        for (int e = 0; e < MAXM; ++e) {
          if (e < m) {
            float wf[EPV];
            unpack8<T>(s_wr[e * nvec + c], wf);   // one shared load feeds TPW tokens
#pragma unroll
            for (int i = 0; i < TPW; ++i)
#pragma unroll
              for (int k = 0; k < EPV; ++k) acc[i][e] = fmaf(xf[i][k], wf[k], acc[i][e]);
          }
        }
      }
    }
  }
  if (!waited) {
    cp_async_wait_all();
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TPW; ++i) {
    const int t = tbase + i;
    float v[1];
    v[0] = 0.0f;
#pragma unroll
    for (int e = 0; e < MAXM; ++e) {
      if (e < m) {
        float a = acc[i][e];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
        if (lane == e) v[0] = a;
      }
    }
    if (t < Tn) {   // warp-uniform
      if (lane < m) logits[static_cast<int64_t>(t) * m + lane] = v[0];
      int id;
      float w;
      warp_topk_softmax<1>(v, m, K, lane, id, w);
      if (lane < K) {
        topk_id[static_cast<int64_t>(t) * K + lane] = id;
        topk_w[static_cast<int64_t>(t) * K + lane] = w;
        hist[warp][id] += 1;   // a token's K ids are distinct
      }
      __syncwarp();
    }
  }
  __syncthreads();
  if (threadIdx.x < m) {
    int c = 0;
    for (int w = 0; w < 8; ++w) c += hist[w][threadIdx.x];
    tile_cnt[static_cast<int64_t>(blockIdx.x) * m + threadIdx.x] = c;
  }
}

// Decode-sized batches (T < 8 * #SM): k_router_small would run one warp per
// token on T/8 CTAs, latency-bound on the FMA chain of each warp.  Here the
// hidden dimension of each token is split over 8/tpc warps of a CTA (tpc
// tokens per CTA, >= #SM CTAs), centroids read through L1 (no shared-memory
// staging), partial logits reduced in a fixed order through shared memory.
// One token tile (tpc tokens, 256 threads) of the split-warp router; also the
// first phase of the fused decode routing kernel (k_route_fused).
// BULK: the tile's x rows and all of Wr are first brought into (dynamic) shared memory by
// TMA bulk copies on one mbarrier (Wr at offset 0, then the tpc rows): per-thread global
// loads keep only ~10-16 KB in flight per SM (the phase probe put this tile at 7.5 us on C3),
// the copy engine the whole 80 KB at once.
template <typename T, int MAXM, bool BULK = false>
__device__ __forceinline__ void router_split_tile(const T* __restrict__ x, const T* __restrict__ Wr, int Tn, int d,
                                                  int m, int K, int tpc, float* __restrict__ logits,
                                                  int32_t* __restrict__ topk_id, float* __restrict__ topk_w,
                                                  int32_t* __restrict__ tile_cnt, int tile_idx) {
  __shared__ float s_part[8][MAXM];
  __shared__ int hist[8][32];   // per-warp expert counts (no atomics)
  constexpr int EPV = 16 / sizeof(T);
  constexpr int U = 4;   // 16-byte x loads per lane in flight
  const int nvec = d / EPV;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpt = 8 / tpc;
  const int tl = warp / wpt, q = warp - tl * wpt;
  const int t = tile_idx * tpc + tl;
  const int nvw = nvec / wpt;
  const int v0 = q * nvw, v1 = v0 + nvw;
  hist[warp][lane] = 0;
  float acc[MAXM];
#pragma unroll
  for (int e = 0; e < MAXM; ++e) acc[e] = 0.0f;
  const uint4* xsrc = reinterpret_cast<const uint4*>(x + static_cast<int64_t>(t) * d);
  const uint4* wsrc = reinterpret_cast<const uint4*>(Wr);
  if constexpr (BULK) {
    extern __shared__ __align__(128) uint8_t rs_dyn[];
    __shared__ __align__(8) uint64_t rs_bar;
    const uint32_t wbytes = static_cast<uint32_t>(m) * d * sizeof(T);
    const uint32_t rbytes = static_cast<uint32_t>(d) * sizeof(T);
    if (threadIdx.x == 0) {
      mbar_init(&rs_bar, 1);
      fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int t0 = tile_idx * tpc;
      const int nt = Tn - t0 < tpc ? Tn - t0 : tpc;
      mbar_arrive_expect_tx(&rs_bar, wbytes + static_cast<uint32_t>(nt) * rbytes);
      bulk_g2s(rs_dyn, Wr, wbytes, &rs_bar);
      for (int i = 0; i < nt; ++i)
        bulk_g2s(rs_dyn + wbytes + i * rbytes, x + static_cast<int64_t>(t0 + i) * d, rbytes, &rs_bar);
    }
    mbar_wait(&rs_bar, 0);
    xsrc = reinterpret_cast<const uint4*>(rs_dyn + wbytes + tl * rbytes);
    wsrc = reinterpret_cast<const uint4*>(rs_dyn);
  }
  auto ldv = [](const uint4* p) { return BULK ? *p : __ldg(p); };
  if (t < Tn) {
    const uint4* xr = xsrc;
    const uint4* wr = wsrc;
    for (int c0 = v0 + lane; c0 < v1; c0 += 32 * U) {
      uint4 xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + 32 * u;
        xv[u] = c < v1 ? ldv(xr + c) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int e0 = 0; e0 < MAXM; e0 += 8) {
        if (e0 < m) {
          uint4 wv[U][8];
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int c = c0 + 32 * u;
              wv[u][j] = (c < v1 && e0 + j < m) ? ldv(wr + static_cast<int64_t>(e0 + j) * nvec + c)
                                                : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            float xf[EPV];
            unpack8<T>(xv[u], xf);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float wf[EPV];
              unpack8<T>(wv[u][j], wf);
#pragma unroll
              for (int k = 0; k < EPV; ++k) acc[e0 + j] = fmaf(xf[k], wf[k], acc[e0 + j]);
            }
          }
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < MAXM; ++e) {
    if (e < m) {
      float a = acc[e];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
      if (lane == 0) s_part[warp][e] = a;
    }
  }
  __syncthreads();
  if (q == 0 && t < Tn) {   // warp-uniform: the token's first warp finishes Eq. 8 and does Eq. 7
    float v[1];
    v[0] = 0.0f;
    if (lane < m)
      for (int qq = 0; qq < wpt; ++qq) v[0] += s_part[tl * wpt + qq][lane];
    if (lane < m) logits[static_cast<int64_t>(t) * m + lane] = v[0];
    int id;
    float w;
    warp_topk_softmax<1>(v, m, K, lane, id, w);
    if (lane < K) {
      topk_id[static_cast<int64_t>(t) * K + lane] = id;
      topk_w[static_cast<int64_t>(t) * K + lane] = w;
      hist[warp][id] += 1;   // one token per warp here: its K ids are distinct
    }
  }
  __syncthreads();
  if (threadIdx.x < m) {
    int c = 0;
    for (int w = 0; w < 8; ++w) c += hist[w][threadIdx.x];
    tile_cnt[static_cast<int64_t>(tile_idx) * m + threadIdx.x] = c;
  }
}

template <typename T, int MAXM, bool BULK>
__global__ void __launch_bounds__(256) k_router_split(const T* __restrict__ x, const T* __restrict__ Wr, int Tn,
                                                      int d, int m, int K, int tpc, float* __restrict__ logits,
                                                      int32_t* __restrict__ topk_id, float* __restrict__ topk_w,
                                                      int32_t* __restrict__ tile_cnt) {
  router_split_tile<T, MAXM, BULK>(x, Wr, Tn, d, m, K, tpc, logits, topk_id, topk_w, tile_cnt, blockIdx.x);
}

template <typename K>
static cudaError_t smem_attr_once(K kern, int bytes, std::atomic<uint64_t>& done);
static int router_bulk_bytes(int dtype, int m, int d, int tpc);

// Prefill-sized batches, m <= 32, bf16: Eq. 8 on the tensor cores with
// mma.sync m16n8k16 (bf16 x bf16 -> fp32).  N = m is far too narrow for a
// tcgen05 tile, but one m16n8k16 per 8 experts x 16 tokens x 16 k replaces
// 2 x 16 x 8 x 16 FMAs.  CTA = 16 tokens x 4 warps, warp w reduces over the
// w-th quarter of d; operands come straight from global memory in 16-byte
// loads: within every 32-wide k chunk, thread (r = lane/4, q = lane%4) holds
// x[r][8q..8q+7], x[r+8][8q..8q+7] and Wr[n][8q..8q+7]; the two MMAs of the
// chunk take elements {0,1},{2,3} and {4,5},{6,7} as their k-pairs (the same
// k permutation on both operands, so the dot products are unchanged).  Partial
// logits of the 4 warps are summed in a fixed order through shared memory,
// then the warp top-K of Eq. 7.
__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int NB, int NW>
__global__ void __launch_bounds__(32 * NW) k_router_mma(const __nv_bfloat16* __restrict__ x,
                                                    const __nv_bfloat16* __restrict__ Wr, int Tn, int d, int m, int K,
                                                    float* __restrict__ logits, int32_t* __restrict__ topk_id,
                                                    float* __restrict__ topk_w, int32_t* __restrict__ tile_cnt) {
  constexpr int U = 4;   // 32-wide k chunks in flight per thread
  __shared__ float s_c[NW][16][NB * 8 + 1];
  __shared__ int hist[NW][32];   // per-warp expert counts (no atomics)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane >> 2, q = lane & 3;
  const int t0 = blockIdx.x * 16;
  const int nk = d / NW, k0 = warp * nk;
  hist[warp][lane] = 0;
  const bool va = t0 + r < Tn, vb = t0 + r + 8 < Tn;
  const uint4* xa = reinterpret_cast<const uint4*>(x + static_cast<int64_t>(va ? t0 + r : 0) * d + k0 + 8 * q);
  const uint4* xb = reinterpret_cast<const uint4*>(x + static_cast<int64_t>(vb ? t0 + r + 8 : 0) * d + k0 + 8 * q);
  const uint4* wp[NB];
  bool vw[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    vw[j] = 8 * j + r < m;
    wp[j] = reinterpret_cast<const uint4*>(Wr + static_cast<int64_t>(vw[j] ? 8 * j + r : 0) * d + k0 + 8 * q);
  }
  float c[NB][4];
#pragma unroll
  for (int j = 0; j < NB; ++j) c[j][0] = c[j][1] = c[j][2] = c[j][3] = 0.0f;
  const uint4 z = make_uint4(0, 0, 0, 0);
  // register double buffer: the loads of chunk group i+1 are issued before the MMAs of group i
  uint4 a[2][U], b[2][U], w[2][U][NB];
  auto load = [&](int buf, int kc) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool in = kc + 32 * u < nk;
      const int off = (kc + 32 * u) / 8;      // in 16-byte units
      a[buf][u] = (in && va) ? __ldg(xa + off) : z;
      b[buf][u] = (in && vb) ? __ldg(xb + off) : z;
#pragma unroll
      for (int j = 0; j < NB; ++j) w[buf][u][j] = (in && vw[j]) ? __ldg(wp[j] + off) : z;
    }
  };
  auto compute = [&](int buf) {
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        mma_bf16_16816(c[j], a[buf][u].x, b[buf][u].x, a[buf][u].y, b[buf][u].y, w[buf][u][j].x, w[buf][u][j].y);
        mma_bf16_16816(c[j], a[buf][u].z, b[buf][u].z, a[buf][u].w, b[buf][u].w, w[buf][u][j].z, w[buf][u][j].w);
      }
  };
  load(0, 0);
  for (int kc = 0; kc < nk; kc += 64 * U) {   // nk is a multiple of 32 (d % 128 == 0)
    load(1, kc + 32 * U);
    compute(0);
    if (kc + 32 * U >= nk) break;
    load(0, kc + 64 * U);
    compute(1);
  }
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    s_c[warp][r][8 * j + 2 * q] = c[j][0];
    s_c[warp][r][8 * j + 2 * q + 1] = c[j][1];
    s_c[warp][r + 8][8 * j + 2 * q] = c[j][2];
    s_c[warp][r + 8][8 * j + 2 * q + 1] = c[j][3];
  }
  __syncthreads();
  // warp w finishes tokens (16 / NW) w ..: fixed-order sum over the K slices, Eq. 7, histogram
  for (int i = 0; i < 16 / NW; ++i) {
    const int tt = (16 / NW) * warp + i;
    const int t = t0 + tt;
    if (t >= Tn) break;   // warp-uniform
    float v[1];
    v[0] = 0.0f;
    if (lane < m)
      for (int ww = 0; ww < NW; ++ww) v[0] += s_c[ww][tt][lane];
    if (lane < m) logits[static_cast<int64_t>(t) * m + lane] = v[0];
    int id;
    float wgt;
    warp_topk_softmax<1>(v, m, K, lane, id, wgt);
    if (lane < K) {
      topk_id[static_cast<int64_t>(t) * K + lane] = id;
      topk_w[static_cast<int64_t>(t) * K + lane] = wgt;
      hist[warp][id] += 1;   // a token's K ids are distinct
    }
    __syncwarp();
  }
  __syncthreads();
  if (threadIdx.x < m) {
    int c = 0;
    for (int w = 0; w < NW; ++w) c += hist[w][threadIdx.x];
    tile_cnt[static_cast<int64_t>(blockIdx.x) * m + threadIdx.x] = c;
  }
}

bool router_mma_ok(int dtype, int m, int d, int T, int num_sms) {
  // decode-sized batches keep the split-warp router: its 1-token tiles give the
  // permutation one CTA per token (mma router: 16-token tiles, permute 2.4x slower at T = 256)
  return dtype == 0 && m <= 32 && d % 128 == 0 && T >= 8 * num_sms;
}
constexpr int kRouterMmaWarps = 8;   // K slices per 16-token tile (d % 256 == 0), else 4

cudaError_t launch_router_mma(const void* x, const void* Wr, int T, int d, int m, int K, float* logits,
                              int32_t* topk_id, float* topk_w, int32_t* tile_cnt, cudaStream_t s) {
  const int ntiles = (T + 15) / 16;
  if (ntiles == 0) return cudaSuccess;
  const auto* xb = static_cast<const __nv_bfloat16*>(x);
  const auto* wb = static_cast<const __nv_bfloat16*>(Wr);
  const int nb = (m + 7) / 8;
#define BO_RM(NB, NW) \
  k_router_mma<NB, NW><<<ntiles, 32 * NW, 0, s>>>(xb, wb, T, d, m, K, logits, topk_id, topk_w, tile_cnt)
  if (d % (32 * kRouterMmaWarps) == 0) {
    if (nb == 1) BO_RM(1, kRouterMmaWarps); else if (nb == 2) BO_RM(2, kRouterMmaWarps); else BO_RM(4, kRouterMmaWarps);
  } else {
    if (nb == 1) BO_RM(1, 4); else if (nb == 2) BO_RM(2, 4); else BO_RM(4, 4);
  }
#undef BO_RM
  return cudaGetLastError();
}

int router_split_tpc(int T, int num_sms) {
  if (T >= 8 * num_sms) return 0;   // k_router_small
  return T >= 4 * num_sms ? 4 : (T >= 2 * num_sms ? 2 : 1);
}

cudaError_t launch_router_split(int dtype, const void* x, const void* Wr, int T, int d, int m, int K, int tpc,
                                float* logits, int32_t* topk_id, float* topk_w, int32_t* tile_cnt, cudaStream_t s) {
  const int ntiles = (T + tpc - 1) / tpc;
  if (ntiles == 0) return cudaSuccess;
  const int bulk = router_bulk_bytes(dtype, m, d, tpc);
#define BO_RS(TYPE, M)                                                                                         \
  do {                                                                                                         \
    if (bulk) {                                                                                                \
      static std::atomic<uint64_t> done{0};                                                                    \
      const cudaError_t e = smem_attr_once(k_router_split<TYPE, M, true>, 176 * 1024, done);                   \
      if (e != cudaSuccess) return e;                                                                          \
      k_router_split<TYPE, M, true><<<ntiles, 256, bulk, s>>>(static_cast<const TYPE*>(x),                     \
                                                              static_cast<const TYPE*>(Wr), T, d, m, K, tpc,   \
                                                              logits, topk_id, topk_w, tile_cnt);              \
    } else {                                                                                                   \
      k_router_split<TYPE, M, false><<<ntiles, 256, 0, s>>>(static_cast<const TYPE*>(x),                       \
                                                            static_cast<const TYPE*>(Wr), T, d, m, K, tpc,     \
                                                            logits, topk_id, topk_w, tile_cnt);                \
    }                                                                                                          \
  } while (0)
  if (dtype == 0) {
    if (m <= 8) BO_RS(__nv_bfloat16, 8); else if (m <= 16) BO_RS(__nv_bfloat16, 16); else BO_RS(__nv_bfloat16, 32);
  } else {
    if (m <= 8) BO_RS(float, 8); else if (m <= 16) BO_RS(float, 16); else BO_RS(float, 32);
  }
#undef BO_RS
  return cudaGetLastError();
}

bool router_small_ok(int dtype, int m, int d) {
  const int eb = dtype == 0 ? 2 : 4;
  return m <= 32 && static_cast<int64_t>(m) * d * eb <= 160 * 1024;
}

int router_small_tile(int T, int num_sms) {
  const int tpw = T >= 4 * 8 * num_sms ? 4 : (T >= 2 * 8 * num_sms ? 2 : 1);   // tokens per warp, SMs stay full
  return 8 * tpw;
}

// cudaFuncSetAttribute applies to the current device's context: set it once per device
template <typename K>
static cudaError_t smem_attr_once(K kern, int bytes, std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = dev < 64 ? (uint64_t(1) << dev) : 0;
  if (bit && (done.load(std::memory_order_acquire) & bit)) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && bit) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

cudaError_t launch_router_small(int dtype, const void* x, const void* Wr, int T, int d, int m, int K, int tile,
                                float* logits, int32_t* topk_id, float* topk_w, int32_t* tile_cnt, cudaStream_t s) {
  const int ntiles = (T + tile - 1) / tile;
  if (ntiles == 0) return cudaSuccess;
  const int eb = dtype == 0 ? 2 : 4;
  const int smem = m * d * eb;
  cudaError_t e = cudaSuccess;
#define BO_ROUTER_CASE(TYPE, M, TPW)                                                                           \
  {                                                                                                            \
    auto k = k_router_small<TYPE, M, TPW>;                                                                     \
    static std::atomic<uint64_t> done{0};   /* per device ordinal (the attribute is per context) */            \
    e = smem_attr_once(k, 160 * 1024, done);                                                                   \
    if (e != cudaSuccess) return e;                                                                            \
    k<<<ntiles, 256, smem, s>>>(static_cast<const TYPE*>(x), static_cast<const TYPE*>(Wr), T, d, m, K, logits,  \
                                topk_id, topk_w, tile_cnt);                                                    \
  }
#define BO_ROUTER_M(TYPE, TPW)                      \
  if (m <= 8) BO_ROUTER_CASE(TYPE, 8, TPW)          \
  else if (m <= 16) BO_ROUTER_CASE(TYPE, 16, TPW)   \
  else BO_ROUTER_CASE(TYPE, 32, TPW)
  const int tpw = tile / 8;
  if (dtype == 0) {
    if (tpw == 1) { BO_ROUTER_M(__nv_bfloat16, 1) }
    else if (tpw == 2) { BO_ROUTER_M(__nv_bfloat16, 2) }
    else { BO_ROUTER_M(__nv_bfloat16, 4) }
  } else {
    if (tpw == 1) { BO_ROUTER_M(float, 1) }
    else if (tpw == 2) { BO_ROUTER_M(float, 2) }
    else { BO_ROUTER_M(float, 4) }
  }
#undef BO_ROUTER_M
#undef BO_ROUTER_CASE
  return cudaGetLastError();
}

// ------------------------------------------------------------ Algorithm 1
// Exclusive scan of one int per thread over the whole block (16 warps):
// warp shuffle scan, warp totals through shared memory.  Returns the
// exclusive prefix; *total receives the block sum.
__device__ __forceinline__ long long block_excl_scan(long long v, long long* s_warp, long long* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  long long incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const long long o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    long long w = lane < nw ? s_warp[lane] : 0;
    long long wi = w;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const long long o = __shfl_up_sync(0xffffffffu, wi, off);
      if (lane >= off) wi += o;
    }
    if (lane < nw) s_warp[lane] = wi - w;            // exclusive warp offsets
    if (lane == 31) s_warp[32] = wi;                 // block total
  }
  __syncthreads();
  const long long r = s_warp[warp] + incl - v;
  *total = s_warp[32];
  __syncthreads();   // s_warp reusable after return
  return r;
}

constexpr int kPlanStage = 8192;    // tile histograms staged in shared memory when ntiles*m fits

__global__ void __launch_bounds__(512) k_plan(const int32_t* __restrict__ tile_cnt, int ntiles, int m, int way,
                                              double ratio, int mode, int32_t* __restrict__ tile_base,
                                              int32_t* __restrict__ counts, int32_t* __restrict__ exec_of_expert,
                                              int32_t* __restrict__ expert_row_off, int32_t* __restrict__ exec_off,
                                              int32_t* __restrict__ mtile_off, int64_t* __restrict__ stats,
                                              int n_shared, int shared_rows, PlanExt ext) {
  // Expert parallelism (ext.knob_in): the knob travels with the all-gathered count rows
  // [R, m + 4] (tail [T, mode, ratio lo, ratio hi]); every rank plans with rank 0's, so
  // ranks whose host knobs differ (a per-rank SALC loop) still agree on the global plan.
  if (ext.knob_in) {
    mode = ext.knob_in[1];
    ratio = __hiloint2double(ext.knob_in[3], ext.knob_in[2]);
  }
  if (ext.row_tail && threadIdx.x == 0) {   // this rank's gather row tail
    ext.row_tail[0] = ext.row_T;
    ext.row_tail[1] = mode;
    ext.row_tail[2] = __double2loint(ratio);
    ext.row_tail[3] = __double2hiint(ratio);
  }
  const int ld = ext.ld > 0 ? ext.ld : m;   // row stride of tile_cnt
  __shared__ __align__(16) int s_tc[kPlanStage];
  __shared__ int s_cnt[kMaxExperts];
  __shared__ int s_sorted[kMaxExperts];
  __shared__ long long s_excl[kMaxExperts];
  __shared__ int s_gsize[kMaxExperts];
  __shared__ int s_exec[kMaxExperts];
  __shared__ int s_xoff[kMaxExec];
  __shared__ long long s_warp[33];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int G = (m + way - 1) / way;
  const int E = m + G;
  const int n_tc = ntiles * m;
  const bool staged = n_tc <= kPlanStage;
  // 16-byte cp.async needs a 16-byte-aligned source; a caller's counts row (bo_plan_counts /
  // bo_plan_from_counts take any int32 pointer) may be only 4-byte aligned
  const bool vec16 = (reinterpret_cast<uintptr_t>(tile_cnt) & 15u) == 0 && ld == m;

  // 1. cnt_i (Alg. 1 input) and the per-tile exclusive prefix used by
  //    the permutation.  Histograms are staged with coalesced loads, then a
  //    warp per expert scans over tiles (lanes over tiles, shuffle scan + carry).
  if (staged) {   // all loads in flight at once (cp.async), not one dependent load per iteration
    const int n16 = vec16 ? n_tc / 4 : 0;
    for (int i = tid; i < n16; i += blockDim.x) cp_async16(s_tc + 4 * i, tile_cnt + 4 * i);
    for (int i = 4 * n16 + tid; i < n_tc; i += blockDim.x) s_tc[i] = __ldg(tile_cnt + (i / m) * ld + i % m);
    cp_async_wait_all();
  }
  __syncthreads();
  if (staged && m >= 32) {
    // many experts: thread (chunk c, expert e) walks its chunk of tiles sequentially
    // (consecutive threads read consecutive experts: no shared-memory bank conflicts;
    // the lane-over-tiles scan below strides by m, a 32-way conflict for m = 128)
    __shared__ int s_chunk[kMaxExec];
    const int nch = blockDim.x / m;                      // >= 1 (m <= 256 < 512)
    const int e = tid % m, ch = tid / m;
    const int per = (ntiles + nch - 1) / nch;
    const int t0 = ch * per, t1 = min(ntiles, t0 + per);
    int sum = 0;
    if (ch < nch)
      for (int t = t0; t < t1; ++t) sum += s_tc[t * m + e];
    if (ch < nch) s_chunk[ch * m + e] = sum;
    __syncthreads();
    if (ch < nch) {
      int carry = 0;
      for (int c2 = 0; c2 < ch; ++c2) carry += s_chunk[c2 * m + e];
      if (tile_base)
        for (int t = t0; t < t1; ++t) {
          const int v = s_tc[t * m + e];
          s_tc[t * m + e] = carry;
          carry += v;
        }
      if (ch == nch - 1) {
        int tot = 0;
        for (int c2 = 0; c2 < nch; ++c2) tot += s_chunk[c2 * m + e];
        s_cnt[e] = tot;
        counts[e] = tot;
      }
    }
  } else
  for (int e = warp; e < m; e += 16) {
    int carry = 0;
    for (int t0 = 0; t0 < ntiles; t0 += 32) {
      const int t = t0 + lane;
      const int v = t < ntiles ? (staged ? s_tc[t * m + e] : __ldg(tile_cnt + static_cast<int64_t>(t) * ld + e)) : 0;
      int incl = v;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
      }
      if (tile_base && t < ntiles) {
        if (staged) s_tc[t * m + e] = carry + incl - v;   // written back coalesced below
        else tile_base[static_cast<int64_t>(t) * m + e] = carry + incl - v;
      }
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) {
      s_cnt[e] = carry;
      counts[e] = carry;
    }
  }
  __syncthreads();
  if (tile_base && staged) {   // per-tile prefixes: 16-byte coalesced stores instead of m-strided ones
    const int n16 = n_tc / 4;
    for (int i = tid; i < n16; i += blockDim.x)
      reinterpret_cast<int4*>(tile_base)[i] = reinterpret_cast<const int4*>(s_tc)[i];
    for (int i = 4 * n16 + tid; i < n_tc; i += blockDim.x) tile_base[i] = s_tc[i];
  }
  // 2. Alg. 1 line 5: order by (cnt desc, id asc) (D5) -- rank by counting
  const int c_me = tid < m ? s_cnt[tid] : 0;
  if (tid < m) {
    int pos = 0;
#pragma unroll 8
    for (int j = 0; j < m; ++j) {   // independent shared loads: unrolled so they overlap
      const int cj = s_cnt[j];
      pos += (cj > c_me) | ((cj == c_me) & (j < tid));
    }
    s_sorted[pos] = tid;
  }
  __syncthreads();
  // 3. lines 6-15: S and the exclusive prefix sum_partial in sorted order
  long long S;
  const long long excl = block_excl_scan(tid < m ? s_cnt[s_sorted[tid]] : 0, s_warp, &S);
  if (tid < m) s_excl[s_sorted[tid]] = excl;
  __syncthreads();
  const double threshold = 1.0 - ratio;                // D2
  const double Tcov = static_cast<double>(S) * threshold;   // line 7, fp64 (D3)
  bool in_s1 = false, in_s2 = false;
  if (tid < m) {
    const bool active = c_me > 0;                                 // D6
    in_s1 = active && static_cast<double>(s_excl[tid]) < Tcov;    // D1
    in_s2 = active && !in_s1;
    s_exec[tid] = in_s2 ? 1 : 0;                                  // S2 flags (s_exec reused below)
  }
  __syncthreads();
  if (tid < G) {   // group_experts (line 23): |M_j| = S2 members of group j, counted by its own thread
    int n = 0;
    for (int e = tid * way; e < min((tid + 1) * way, m); ++e) n += s_exec[e];
    s_gsize[tid] = n;
  }
  __syncthreads();
  // 4. executor of each expert (lines 16-30)
  int x_me = -1;
  if (tid < m) {
    if (in_s1) x_me = tid;                               // original expert
    else if (!in_s2) x_me = -1;                          // inactive
    else if (mode == 1) x_me = -2;                       // full brownout: ignored
    else if (s_gsize[tid / way] == 1) x_me = tid;        // special case
    else x_me = m + tid / way;                           // united expert of group tid / way
    s_exec[tid] = x_me;
    exec_of_expert[tid] = x_me;
  }
  __syncthreads();
  // 5. rows per executor, exec_off / mtile_off = exclusive scans over executors;
  //    the N_s shared experts of Eq. 5 follow the routed executors (all tokens each)
  int rows = 0;
  if (tid >= E && tid < E + n_shared) rows = shared_rows;
  if (tid < E) {
    if (tid < m) {
      rows = s_exec[tid] == tid ? s_cnt[tid] : 0;
    } else {
      const int j = tid - m;
      const int e1 = min((j + 1) * way, m);
      for (int e = j * way; e < e1; ++e)
        if (s_exec[e] == tid) rows += s_cnt[e];
    }
  }
  long long R_total;
  const long long xoff = block_excl_scan(rows, s_warp, &R_total);
  long long MT_total;
  const long long moff = block_excl_scan((rows + kBM - 1) / kBM, s_warp, &MT_total);
  const int Et = E + n_shared;
  if (tid < Et) {
    exec_off[tid] = static_cast<int>(xoff);
    mtile_off[tid] = static_cast<int>(moff);
  }
  if (tid < E) s_xoff[tid] = static_cast<int>(xoff);
  if (tid == 0) {
    exec_off[Et] = static_cast<int>(R_total);
    mtile_off[Et] = static_cast<int>(MT_total);
  }
  R_total -= static_cast<long long>(n_shared) * shared_rows;   // routed rows only, for the statistics
  __syncthreads();
  // 6. expert_row_off: executor start + earlier members of the same executor (D11)
  if (tid < m) {
    int off = -1;
    if (x_me >= 0) {
      off = s_xoff[x_me];
      if (x_me >= m)
        for (int e = (x_me - m) * way; e < tid; ++e)
          if (s_exec[e] == x_me) off += s_cnt[e];
    }
    expert_row_off[tid] = off;
  }
  // 7. statistics (P:173 / P:194 access counts, rows per class)
  const int n_acc = __syncthreads_count(tid < E && rows > 0);
  const int n_uni = __syncthreads_count(tid >= m && tid < E && rows > 0);
  const int n_s1 = __syncthreads_count(in_s1);
  const int n_single = __syncthreads_count(in_s2 && x_me == tid);
  long long r_orig;
  block_excl_scan(tid < m ? rows : 0, s_warp, &r_orig);
  if (tid == 0) {
    stats[0] = n_acc;
    stats[1] = n_s1;
    stats[2] = n_uni;
    stats[3] = n_single;
    stats[4] = r_orig;
    stats[5] = R_total - r_orig;
    stats[6] = S - R_total;
    stats[7] = S;
  }
}

cudaError_t launch_plan(const int32_t* tile_cnt, int ntiles, int m, int way, double ratio, int mode,
                        int32_t* tile_base, int32_t* counts, int32_t* exec_of_expert, int32_t* expert_row_off,
                        int32_t* exec_off, int32_t* mtile_off, int64_t* stats, cudaStream_t s, int n_shared,
                        int shared_rows, PlanExt ext) {
  k_plan<<<1, kMaxExec, 0, s>>>(tile_cnt, ntiles, m, way, ratio, mode, tile_base, counts, exec_of_expert,
                                expert_row_off, exec_off, mtile_off, stats, n_shared, shared_rows, ext);
  return cudaGetLastError();
}

// ----------------------------------------------------------- permutation
// One CTA per token tile (the tile of the histogram that produced tile_base).
// Assignments a = t*K + s of the tile are split into 8 contiguous warp ranges;
// pass 1 counts per (warp, expert), a prefix over warps gives each warp's
// start, pass 2 assigns ranks in order (stable: token ascending, D11).
// Row of (assignment, rep) = row_base[e*nrep + rep] + tile_base[tile][e] + rank
// (row_base < 0: no row, e.g. dropped in full brownout).  nrep = 1 on one GPU;
// under expert parallelism an assignment delegated to an f-sliced united
// expert has one row per slice.
// One token tile (256 threads); tb_row = the tile's per-expert exclusive prefix
// (global memory in k_permute, shared memory in k_route_fused).
__device__ __forceinline__ void permute_tile(const int32_t* __restrict__ topk_id, const float* __restrict__ topk_w,
                                             int T, int K, int m, int tile, int tile_idx, const int32_t* tb_row,
                                             const int32_t* row_base, int nrep, int32_t* __restrict__ row_of,
                                             int32_t* __restrict__ row_tok, float* __restrict__ row_w,
                                             const uint4* __restrict__ x, uint4* __restrict__ xp, int vec_per_row,
                                             int n_shared, const int32_t* shared_off) {
  // row_of is [T, KR] with KR = K*nrep + n_shared: slot s replica rep at
  // s*nrep + rep, the shared experts' rows (Eq. 5 second term) after them.
  const int KR = K * nrep + n_shared;
  __shared__ int wcnt[8][kMaxExperts];
  // the tile's rows for the fused gather below (the gather's row reads then come from shared
  // memory instead of an L2 round trip per (vector, slot) on row_of just written)
  __shared__ int s_rows[kPermRowsSmem];
  const bool rows_smem = xp != nullptr && tile * KR <= kPermRowsSmem;
  const int t0_tile = tile_idx * tile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 8 * kMaxExperts; i += blockDim.x) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const int64_t a0 = static_cast<int64_t>(tile_idx) * tile * K;
  const int64_t a1 = min(static_cast<int64_t>(tile_idx + 1) * tile, static_cast<int64_t>(T)) * K;
  const int n = static_cast<int>(a1 - a0);
  const int per_warp = ((n + 8 * 32 - 1) / (8 * 32)) * 32;
  const int w0 = warp * per_warp;
  const int w1 = min(w0 + per_warp, n);
  // pass 1: per-warp counts
  for (int base = w0; base < w1; base += 32) {
    const int i = base + lane;
    const int e = i < w1 ? topk_id[a0 + i] : -1;
    const uint32_t peers = __match_any_sync(0xffffffffu, e);
    const int leader = __ffs(peers) - 1;
    if (lane == leader && e >= 0) wcnt[warp][e] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  if (threadIdx.x < m) {
    int run = 0;
    for (int w = 0; w < 8; ++w) {
      const int c = wcnt[w][threadIdx.x];
      wcnt[w][threadIdx.x] = run;
      run += c;
    }
  }
  __syncthreads();
  // pass 2: ranks in assignment order
  const uint32_t lt = lanemask_lt();
  for (int base = w0; base < w1; base += 32) {
    const int i = base + lane;
    const int e = i < w1 ? topk_id[a0 + i] : -1;
    const uint32_t peers = __match_any_sync(0xffffffffu, e);
    const int leader = __ffs(peers) - 1;
    const int start = e >= 0 ? wcnt[warp][e] : 0;
    __syncwarp();
    if (lane == leader && e >= 0) wcnt[warp][e] = start + __popc(peers);
    __syncwarp();
    if (e >= 0) {
      const int64_t a = a0 + i;
      const int rank = tb_row[e] + start + __popc(peers & lt);
      const float w = topk_w[a];
      const int64_t t = a / K;
      const int64_t slot0 = t * KR + (a - t * K) * nrep;
      for (int rep = 0; rep < nrep; ++rep) {
        const int base_r = row_base[e * nrep + rep];
        const int r = base_r >= 0 ? base_r + rank : -1;
        row_of[slot0 + rep] = r;
        if (rows_smem) s_rows[(t - t0_tile) * KR + (a - t * K) * nrep + rep] = r;
        if (r >= 0) {
          if (row_tok) row_tok[r] = static_cast<int32_t>(t);
          row_w[r] = w;
        }
      }
    }
  }
  // shared-expert rows of this tile: token t -> row shared_off[i] + t, weight 1
  if (n_shared > 0) {
    const int t0 = tile_idx * tile;
    const int nt = min(tile, T - t0);
    for (int i = threadIdx.x; i < nt * n_shared; i += blockDim.x) {
      const int tt = i / n_shared, j = i - tt * n_shared;
      const int64_t t = t0 + tt;
      const int r = shared_off[j] + static_cast<int>(t);
      row_of[t * KR + K * nrep + j] = r;
      if (rows_smem) s_rows[tt * KR + K * nrep + j] = r;
      if (row_tok) row_tok[r] = static_cast<int32_t>(t);
      row_w[r] = 1.0f;
    }
  }
  // concat_tokens for this tile: copy each token's x row to its rows,
  // flattened over (token, 16-byte vector); row_of of the tile was written by
  // this CTA and is visible after the barrier.
  if (xp) {
    __syncthreads();
    const int t0 = tile_idx * tile;
    const int nt = min(tile, T - t0);
    const int total = nt * vec_per_row;
    constexpr int U = 4;   // loads in flight per thread before the stores (the copy is latency-bound)
    for (int i0 = threadIdx.x; i0 < total; i0 += U * blockDim.x) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * blockDim.x;
        if (i < total) {
          const int tt = i / vec_per_row;
          v[u] = __ldg(x + (t0 + tt) * static_cast<int64_t>(vec_per_row) + (i - tt * vec_per_row));
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * blockDim.x;
        if (i < total) {
          const int tt = i / vec_per_row;
          const int c = i - tt * vec_per_row;
          const int64_t t = t0 + tt;
          for (int s = 0; s < KR; ++s) {
            const int r = rows_smem ? s_rows[tt * KR + s] : row_of[t * KR + s];
            if (r >= 0) xp[static_cast<int64_t>(r) * vec_per_row + c] = v[u];
          }
        }
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_permute(const int32_t* __restrict__ topk_id,
                                                 const float* __restrict__ topk_w, int T, int K, int m, int tile,
                                                 const int32_t* __restrict__ tile_base,
                                                 const int32_t* __restrict__ row_base, int nrep,
                                                 int32_t* __restrict__ row_of, int32_t* __restrict__ row_tok,
                                                 float* __restrict__ row_w, const uint4* __restrict__ x,
                                                 uint4* __restrict__ xp, int vec_per_row, int n_shared,
                                                 const int32_t* __restrict__ shared_off) {
  permute_tile(topk_id, topk_w, T, K, m, tile, blockIdx.x, tile_base + static_cast<int64_t>(blockIdx.x) * m,
               row_base, nrep, row_of, row_tok, row_w, x, xp, vec_per_row, n_shared, shared_off);
}

cudaError_t launch_permute(const int32_t* topk_id, const float* topk_w, int T, int K, int m, int tile,
                           const int32_t* tile_base, const int32_t* row_base, int nrep, int32_t* row_of,
                           int32_t* row_tok, float* row_w, cudaStream_t s, int dtype, const void* x, void* xp,
                           int d, int n_shared, const int32_t* shared_off) {
  const int ntiles = (T + tile - 1) / tile;
  if (ntiles == 0) return cudaSuccess;
  const int vec = xp ? d * (dtype == 0 ? 2 : 4) / 16 : 0;
  k_permute<<<ntiles, 256, 0, s>>>(topk_id, topk_w, T, K, m, tile, tile_base, row_base, nrep, row_of, row_tok,
                                   row_w, static_cast<const uint4*>(x), static_cast<uint4*>(xp), vec, n_shared,
                                   shared_off);
  return cudaGetLastError();
}

// ------------------------------------------------- fused decode routing
// Decode-sized batches (m <= 32 on the split-warp router): Eq. 8 + Eq. 7 + histogram,
// Algorithm 1, the permutation (and concat_tokens, when the gather rides in the
// permute) in ONE cooperative launch instead of three (Alg. 1 is
// "negligible", so its launch and dependency gaps should not cost a kernel).
// Phase 1 = one k_router_split tile per CTA; a grid barrier (every tile histogram is
// needed); phase 2: every CTA runs Algorithm 1 itself, warp-synchronously on warp 0
// (lane = expert), on the same histograms (identical results, ntiles * m ints from L2,
// no second barrier); CTA 0 also writes the plan's global outputs; phase 3 = k_permute's
// tile with the tile prefix, expert row offsets and shared-expert offsets from the
// CTA's own copy of the plan.

// Algorithm 1 for m <= 32 experts and Et = m + G + N_s <= 64 executors on one
// warp: lane e < m holds cnt_e (Alg. 1 input).  The same steps, readings and
// outputs as k_plan: order by (cnt desc, id asc) (D5), exclusive prefix in that order,
// S1 iff prefix < Tcov = S (1 - ratio) in fp64 (D1-D3), inactive experts nowhere (D6), S2
// grouped by floor(e / way), single-member groups keep the original, full mode
// drops S2 (-2), rows in (executor, expert, token) order (D11), the N_s shared executors
// last with shared_rows rows each.  s_row_off[m], s_xoff[Et + 1] receive expert_row_off /
// exec_off; write_global: also the global plan arrays.
__device__ __forceinline__ void plan_small_warp(int cnt, int m, int way, double ratio, int mode, int n_shared,
                                                int shared_rows, int32_t* s_row_off, int32_t* s_xoff,
                                                bool write_global, int32_t* __restrict__ counts,
                                                int32_t* __restrict__ exec_of_expert,
                                                int32_t* __restrict__ expert_row_off, int32_t* __restrict__ exec_off,
                                                int32_t* __restrict__ mtile_off, int64_t* __restrict__ stats) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int e = lane;
  const bool ve = e < m;
  const int G = (m + way - 1) / way, E = m + G, Et = E + n_shared;
  const int c = ve ? cnt : 0;
  // line 5: rank by (cnt desc, id asc); exclusive prefix in that order; S
  int pos = 0;
  for (int j = 0; j < m; ++j) {
    const int cj = __shfl_sync(FULL, c, j);
    pos += (cj > c) | ((cj == c) & (j < e));
  }
  long long excl = 0, S = 0;
  for (int j = 0; j < m; ++j) {
    const int cj = __shfl_sync(FULL, c, j);
    const int pj = __shfl_sync(FULL, pos, j);
    excl += pj < pos ? cj : 0;
    S += cj;
  }
  // lines 6-15: S1 / S2 against Tcov in fp64
  const double Tcov = static_cast<double>(S) * (1.0 - ratio);
  const bool active = ve && c > 0;
  const bool in_s1 = active && static_cast<double>(excl) < Tcov;
  const bool in_s2 = active && !in_s1;
  // line 23: |M_j| = S2 members of e's group
  int gsize = 0;
  for (int j = 0; j < m; ++j) {
    const int s2j = __shfl_sync(FULL, static_cast<int>(in_s2), j);
    gsize += (s2j && j / way == e / way) ? 1 : 0;
  }
  // lines 16-30: executor of each expert
  int x_e = -1;
  if (ve) {
    if (in_s1) x_e = e;
    else if (!in_s2) x_e = -1;
    else if (mode == 1) x_e = -2;
    else if (gsize == 1) x_e = e;
    else x_e = m + e / way;
  }
  // rows of executors x0 = lane and x1 = lane + 32
  const int x0 = lane, x1 = lane + 32;
  int r0 = 0, r1 = 0;
  for (int j = 0; j < m; ++j) {
    const int xj = __shfl_sync(FULL, x_e, j);
    const int cj = __shfl_sync(FULL, c, j);
    r0 += xj == x0 ? cj : 0;
    r1 += xj == x1 ? cj : 0;
  }
  if (x0 >= E && x0 < Et) r0 = shared_rows;
  if (x1 >= E && x1 < Et) r1 = shared_rows;
  if (x0 >= Et) r0 = 0;
  if (x1 >= Et) r1 = 0;
  // exclusive scans over the executors (rows and 128-row m-tiles)
  auto scan2 = [&](int v0, int v1, int& ex0, int& ex1, int& total) {
    int i0 = v0, i1 = v1;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int o0 = __shfl_up_sync(FULL, i0, off);
      const int o1 = __shfl_up_sync(FULL, i1, off);
      if (lane >= off) { i0 += o0; i1 += o1; }
    }
    const int t0 = __shfl_sync(FULL, i0, 31);
    ex0 = i0 - v0;
    ex1 = t0 + i1 - v1;
    total = t0 + __shfl_sync(FULL, i1, 31);
  };
  int xo0, xo1, R_all, mo0, mo1, MT_all;
  scan2(r0, r1, xo0, xo1, R_all);
  scan2((r0 + kBM - 1) / kBM, (r1 + kBM - 1) / kBM, mo0, mo1, MT_all);
  if (x0 <= Et) s_xoff[x0] = x0 == Et ? R_all : xo0;
  if (x1 <= Et) s_xoff[x1] = x1 == Et ? R_all : xo1;
  // expert_row_off: executor start + earlier members of the same executor (D11)
  const int xs = x_e >= 0 ? x_e : 0;
  const int st0 = __shfl_sync(FULL, xo0, xs & 31), st1 = __shfl_sync(FULL, xo1, xs & 31);
  int off = x_e >= 0 ? (x_e < 32 ? st0 : st1) : -1;
  int before = 0;   // rows of the same united executor's earlier members
  for (int j = 0; j < m; ++j) {
    const int xj = __shfl_sync(FULL, x_e, j);
    const int cj = __shfl_sync(FULL, c, j);
    before += (j < e && xj == x_e) ? cj : 0;
  }
  if (x_e >= m) off += before;
  if (ve) s_row_off[e] = off;
  // statistics (P:173 / P:194 access counts, rows per class)
  const int n_acc = __popc(__ballot_sync(FULL, x0 < E && r0 > 0)) + __popc(__ballot_sync(FULL, x1 < E && r1 > 0));
  const int n_uni = __popc(__ballot_sync(FULL, x0 >= m && x0 < E && r0 > 0)) +
                    __popc(__ballot_sync(FULL, x1 >= m && x1 < E && r1 > 0));
  const int n_s1 = __popc(__ballot_sync(FULL, in_s1));
  const int n_single = __popc(__ballot_sync(FULL, in_s2 && x_e == e));
  long long r_orig = (x0 < m ? r0 : 0) + (x1 < m ? r1 : 0);
  long long r_routed = (x0 < E ? r0 : 0) + (x1 < E ? r1 : 0);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    r_orig += __shfl_xor_sync(FULL, r_orig, o);
    r_routed += __shfl_xor_sync(FULL, r_routed, o);
  }
  if (write_global) {
    if (ve) {
      counts[e] = c;
      exec_of_expert[e] = x_e;
      expert_row_off[e] = off;
    }
    if (x0 < Et) { exec_off[x0] = xo0; mtile_off[x0] = mo0; }
    if (x1 < Et) { exec_off[x1] = xo1; mtile_off[x1] = mo1; }
    if (lane == 0) {
      exec_off[Et] = R_all;
      mtile_off[Et] = MT_all;
      stats[0] = n_acc;
      stats[1] = n_s1;
      stats[2] = n_uni;
      stats[3] = n_single;
      stats[4] = r_orig;
      stats[5] = r_routed - r_orig;
      stats[6] = S - r_routed;
      stats[7] = S;
    }
  }
}

#ifdef BO_PROBE
// Instrumentation build only: globaltimer stamps of each CTA's phases in the last
// k_route_fused launch [entry, router tile done, grid barrier passed, histograms staged,
// plan done, permute done].
__device__ unsigned long long g_rf_probe[1024][6];
#define BO_RF_STAMP(k)                                                                \
  do {                                                                                \
    if (threadIdx.x == 0 && blockIdx.x < 1024) {                                      \
      unsigned long long t_;                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                          \
      g_rf_probe[blockIdx.x][k] = t_;                                                 \
    }                                                                                 \
  } while (0)
#else
#define BO_RF_STAMP(k) \
  do {                 \
  } while (0)
#endif

template <typename T, int MAXM, bool BULK>
__global__ void __launch_bounds__(256)
    k_route_fused(const T* __restrict__ x, const T* __restrict__ Wr, int Tn, int d, int m, int K, int tpc,
                  float* __restrict__ logits, int32_t* __restrict__ topk_id, float* __restrict__ topk_w,
                  int32_t* __restrict__ tile_cnt, int way, double ratio, int mode, int32_t* __restrict__ counts,
                  int32_t* __restrict__ exec_of_expert, int32_t* __restrict__ expert_row_off,
                  int32_t* __restrict__ exec_off, int32_t* __restrict__ mtile_off, int64_t* __restrict__ stats,
                  int n_shared, int32_t* __restrict__ row_of, int32_t* __restrict__ row_tok,
                  float* __restrict__ row_w, uint4* __restrict__ xp, int vec_per_row) {
  __shared__ __align__(16) int32_t s_tc[kRouteFusedStage];   // every tile histogram [ntiles, m]
  __shared__ int32_t s_sum[2][8][MAXM];   // per-warp partial column sums: all tiles / tiles before mine
  __shared__ int32_t s_row_off[MAXM];
  __shared__ int32_t s_xoff[kRouteFusedMaxExec + 1];
  __shared__ int32_t s_tb[MAXM];
  BO_RF_STAMP(0);
  router_split_tile<T, MAXM, BULK>(x, Wr, Tn, d, m, K, tpc, logits, topk_id, topk_w, tile_cnt, blockIdx.x);
  BO_RF_STAMP(1);
  cg::this_grid().sync();   // every tile histogram written (and visible)
  BO_RF_STAMP(2);
  // Alg. 1 input cnt_e = sum over tiles; this tile's exclusive prefix = sum over the tiles before
  // it.  All ntiles * m counts are staged with one round of L2-coherent 16-byte loads (written
  // in this kernel: no .nc path), then warp w sums tiles w, w + 8, ... per expert (lane).
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = gridDim.x, me = blockIdx.x;
  const int n_tc = ntiles * m;
  for (int i = threadIdx.x; i < n_tc / 4; i += blockDim.x)
    reinterpret_cast<int4*>(s_tc)[i] = __ldcg(reinterpret_cast<const int4*>(tile_cnt) + i);
  for (int i = (n_tc & ~3) + threadIdx.x; i < n_tc; i += blockDim.x) s_tc[i] = __ldcg(tile_cnt + i);
  __syncthreads();
  BO_RF_STAMP(3);
  if (lane < m) {
    int all = 0, bef = 0;
    for (int t = warp; t < ntiles; t += 8) {
      const int v = s_tc[t * m + lane];
      all += v;
      bef += t < me ? v : 0;
    }
    s_sum[0][warp][lane] = all;
    s_sum[1][warp][lane] = bef;
  }
  __syncthreads();
  if (warp == 0) {
    int cnt = 0, base = 0;
    if (lane < m)
      for (int w = 0; w < 8; ++w) {
        cnt += s_sum[0][w][lane];
        base += s_sum[1][w][lane];
      }
    if (lane < m) s_tb[lane] = base;
    plan_small_warp(cnt, m, way, ratio, mode, n_shared, Tn, s_row_off, s_xoff, me == 0, counts, exec_of_expert,
                    expert_row_off, exec_off, mtile_off, stats);
  }
  __syncthreads();
  BO_RF_STAMP(4);
  const int E = m + (m + way - 1) / way;
  // BULK: the tile's x rows are already in shared memory (router phase); concat_tokens
  // then leaves as one TMA bulk store per (token, row) instead of the permute's
  // per-thread copy loop
  permute_tile(topk_id, topk_w, Tn, K, m, tpc, me, s_tb, s_row_off, 1, row_of, row_tok, row_w,
               reinterpret_cast<const uint4*>(x), BULK ? nullptr : xp, vec_per_row, n_shared, s_xoff + E);
  if constexpr (BULK) {
    if (xp) {
      __syncthreads();   // row_of of the tile written (this CTA)
      extern __shared__ __align__(128) uint8_t rs_dyn[];
      const int KR = K + n_shared;
      const uint32_t rbytes = static_cast<uint32_t>(vec_per_row) * 16u;
      const uint8_t* xs = rs_dyn + static_cast<size_t>(m) * rbytes;   // after Wr (m rows)
      const int t0 = me * tpc;
      const int nt = Tn - t0 < tpc ? Tn - t0 : tpc;
      if (threadIdx.x < nt * KR) {
        const int i = threadIdx.x / KR, sl = threadIdx.x - i * KR;
        const int r = row_of[static_cast<int64_t>(t0 + i) * KR + sl];
        if (r >= 0) {
          bulk_s2g(reinterpret_cast<uint8_t*>(xp) + static_cast<int64_t>(r) * rbytes, xs + i * rbytes, rbytes);
          bulk_commit();
          bulk_wait_all();   // complete before the grid ends (the next kernel's TMA reads Xp)
        }
      }
    }
  }
  __syncthreads();
  BO_RF_STAMP(5);
}

#ifdef BO_PROBE
extern "C" __attribute__((visibility("default"))) int bo_probe_rf_copy(void* stamps) {
  return cudaMemcpyFromSymbol(stamps, g_rf_probe, sizeof(g_rf_probe)) != cudaSuccess;
}
#endif

// Co-resident CTAs of the cooperative grid (resident CTAs per SM x #SM), queried once per
// device and kept (the forward is on the host's per-call path).
template <typename T, int MAXM>
static int route_fused_capacity(int num_sms) {
  static std::atomic<int> per_sm[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  int nb = dev < 64 ? per_sm[dev].load(std::memory_order_relaxed) : 0;
  if (nb <= 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_route_fused<T, MAXM, false>, 256, 0) != cudaSuccess)
      return 0;
    if (dev < 64) per_sm[dev].store(nb, std::memory_order_relaxed);
  }
  return nb * num_sms;
}

int route_fused_tpc(int T, int num_sms) {
  for (int tpc = 1; tpc <= 8; tpc *= 2)
    if ((T + tpc - 1) / tpc <= num_sms) return tpc;   // one CTA per SM at most: a cheap grid barrier
  return 0;
}

bool route_fused_ok(int dtype, int m, int way, int T, int tpc, int n_shared, int num_sms) {
  if (m > 32 || tpc <= 0 || T <= 0) return false;
  const int ntiles = (T + tpc - 1) / tpc;
  if (m + (m + way - 1) / way + n_shared > kRouteFusedMaxExec || ntiles * m > kRouteFusedStage) return false;
  int cap;
  if (dtype == 0) cap = m <= 8 ? route_fused_capacity<__nv_bfloat16, 8>(num_sms)
                               : (m <= 16 ? route_fused_capacity<__nv_bfloat16, 16>(num_sms)
                                          : route_fused_capacity<__nv_bfloat16, 32>(num_sms));
  else cap = m <= 8 ? route_fused_capacity<float, 8>(num_sms)
                    : (m <= 16 ? route_fused_capacity<float, 16>(num_sms) : route_fused_capacity<float, 32>(num_sms));
  return ntiles <= cap;   // a cooperative grid must be co-resident (the BULK variant's dynamic
                          // shared memory still fits one CTA per SM: ntiles <= #SM by route_fused_tpc)
}

// Dynamic shared memory of the BULK router tile (Wr + the tile's x rows), or 0 when it does
// not fit next to the static arrays (the tile then loads from global memory directly).
static int router_bulk_bytes(int dtype, int m, int d, int tpc) {
  const int64_t eb = dtype == 0 ? 2 : 4;
  const int64_t b = (static_cast<int64_t>(m) + tpc) * d * eb;
  return b <= 176 * 1024 ? static_cast<int>(b) : 0;
}

cudaError_t launch_route_fused(int dtype, const void* x, const void* Wr, int T, int d, int m, int K, int tpc,
                               float* logits, int32_t* topk_id, float* topk_w, int32_t* tile_cnt, int way,
                               double ratio, int mode, int32_t* counts, int32_t* exec_of_expert,
                               int32_t* expert_row_off, int32_t* exec_off, int32_t* mtile_off, int64_t* stats,
                               int n_shared, int32_t* row_of, int32_t* row_tok, float* row_w, void* xp,
                               cudaStream_t s) {
  const int ntiles = (T + tpc - 1) / tpc;
  const int vec = d * (dtype == 0 ? 2 : 4) / 16;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(ntiles));
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  uint4* xpv = static_cast<uint4*>(xp);
  const int bulk = router_bulk_bytes(dtype, m, d, tpc);
  cfg.dynamicSmemBytes = static_cast<size_t>(bulk);
#define BO_RF(TYPE, M)                                                                                         \
  do {                                                                                                         \
    if (bulk) {                                                                                                \
      static std::atomic<uint64_t> done{0};                                                                    \
      const cudaError_t e = smem_attr_once(k_route_fused<TYPE, M, true>, 176 * 1024, done);                    \
      if (e != cudaSuccess) return e;                                                                          \
    }                                                                                                          \
    return cudaLaunchKernelEx(&cfg, bulk ? k_route_fused<TYPE, M, true> : k_route_fused<TYPE, M, false>,      \
                              static_cast<const TYPE*>(x), static_cast<const TYPE*>(Wr), T, d, m, K, tpc, logits, \
                              topk_id, topk_w, tile_cnt, way, ratio, mode, counts, exec_of_expert,             \
                              expert_row_off, exec_off, mtile_off, stats, n_shared, row_of, row_tok, row_w, xpv, \
                              vec);                                                                            \
  } while (0)
  if (dtype == 0) {
    if (m <= 8) BO_RF(__nv_bfloat16, 8); else if (m <= 16) BO_RF(__nv_bfloat16, 16); else BO_RF(__nv_bfloat16, 32);
  } else {
    if (m <= 8) BO_RF(float, 8); else if (m <= 16) BO_RF(float, 16); else BO_RF(float, 32);
  }
#undef BO_RF
}

// ----------------------------------------------------------------- gather
// Flattened over (token, 16-byte vector): consecutive threads copy consecutive
// vectors of the same token (coalesced), each x vector is loaded once and
// stored to all of the token's rows (KR = K * nrep row slots).  UNROLL
// independent items per thread keep several loads in flight; the flat index
// space fills every SM even for a few hundred (decode) tokens.
template <int UNROLL>
__global__ void __launch_bounds__(256) k_gather(const uint4* __restrict__ x, int T, int vec_per_row, int KR,
                                                const int32_t* __restrict__ row_of, uint4* __restrict__ xp) {
  const int64_t total = static_cast<int64_t>(T) * vec_per_row;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; base < total;
       base += stride * UNROLL) {
    uint4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t i = base + u * stride;
      if (i < total) v[u] = __ldg(x + i);
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t i = base + u * stride;
      if (i < total) {
        const int64_t t = i / vec_per_row;
        const int c = static_cast<int>(i - t * vec_per_row);
        for (int s = 0; s < KR; ++s) {
          const int r = __ldg(row_of + t * KR + s);
          if (r >= 0) xp[static_cast<int64_t>(r) * vec_per_row + c] = v[u];
        }
      }
    }
  }
}

cudaError_t launch_gather(int dtype, const void* x, int T, int d, int KR, const int32_t* row_of, void* xp,
                          int num_sms, cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  const int vec = d * (dtype == 0 ? 2 : 4) / 16;
  const int64_t total = static_cast<int64_t>(T) * vec;
  int64_t blocks = (total + 4 * 256 - 1) / (4 * 256);
  if (blocks > num_sms * 8) blocks = num_sms * 8;
  k_gather<4><<<static_cast<int>(blocks), 256, 0, s>>>(static_cast<const uint4*>(x), T, vec, KR, row_of,
                                                      static_cast<uint4*>(xp));
  return cudaGetLastError();
}

// ---------------------------------------------------------------- combine
template <typename T>
struct Vec8;
template <>
struct Vec8<__nv_bfloat16> {
  static constexpr int kElems = 8;
  __device__ static void load(const void* p, float (&f)[8]) {
    const uint4 u = __ldg(static_cast<const uint4*>(p));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 t = __bfloat1622float2(h[i]);
      f[2 * i] = t.x;
      f[2 * i + 1] = t.y;
    }
  }
  __device__ static void store(void* p, const float (&f)[8]) {
    uint4 u;
    u.x = pack_bf16x2(f[0], f[1]);
    u.y = pack_bf16x2(f[2], f[3]);
    u.z = pack_bf16x2(f[4], f[5]);
    u.w = pack_bf16x2(f[6], f[7]);
    *static_cast<uint4*>(p) = u;
  }
};
template <>
struct Vec8<float> {
  static constexpr int kElems = 8;
  __device__ static void load(const void* p, float (&f)[8]) {
    const float4 a = __ldg(static_cast<const float4*>(p));
    const float4 b = __ldg(static_cast<const float4*>(p) + 1);
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
    f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  }
  __device__ static void store(void* p, const float (&f)[8]) {
    static_cast<float4*>(p)[0] = make_float4(f[0], f[1], f[2], f[3]);
    static_cast<float4*>(p)[1] = make_float4(f[4], f[5], f[6], f[7]);
  }
};

// Flattened over (token, 8-element vector) like the gather; fp32 sum of the
// token's rows in slot order (then slice order), plus the residual if asked.
template <typename T>
__global__ void __launch_bounds__(256) k_combine(const T* __restrict__ yp, const T* __restrict__ x, int Tn, int d,
                                                 int KR, const int32_t* __restrict__ row_of, int add_residual,
                                                 T* __restrict__ y) {
  const int nvec = d / 8;
  const int64_t total = static_cast<int64_t>(Tn) * nvec;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int64_t t = i / nvec;
    const int c = static_cast<int>(i - t * nvec);
    float acc[8];
    if (add_residual) {
      Vec8<T>::load(x + t * d + c * 8, acc);
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = 0.0f;
    }
    for (int s = 0; s < KR; ++s) {   // slot order, then slice order (Eq. 5 sum)
      const int r = __ldg(row_of + t * KR + s);
      if (r >= 0) {
        float v[8];
        Vec8<T>::load(yp + static_cast<int64_t>(r) * d + c * 8, v);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] += v[k];
      }
    }
    Vec8<T>::store(y + t * d + c * 8, acc);
  }
}

cudaError_t launch_combine(int dtype, const void* yp, const void* x, int T, int d, int KR, const int32_t* row_of,
                           int add_residual, void* y, int num_sms, cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  const int64_t total = static_cast<int64_t>(T) * (d / 8);
  int64_t blocks = (total + 255) / 256;
  if (blocks > num_sms * 8) blocks = num_sms * 8;
  if (dtype == 0)
    k_combine<__nv_bfloat16><<<static_cast<int>(blocks), 256, 0, s>>>(
        static_cast<const __nv_bfloat16*>(yp), static_cast<const __nv_bfloat16*>(x), T, d, KR, row_of, add_residual,
        static_cast<__nv_bfloat16*>(y));
  else
    k_combine<float><<<static_cast<int>(blocks), 256, 0, s>>>(static_cast<const float*>(yp),
                                                              static_cast<const float*>(x), T, d, KR, row_of,
                                                              add_residual, static_cast<float*>(y));
  return cudaGetLastError();
}

// Split-K combine: rows' fp32 partials (already gate-weighted) summed over the
// splits in split order, then over the token's slots in slot order.
template <typename T>
__global__ void __launch_bounds__(256) k_combine_partials(const float* __restrict__ part,
                                                          const int* __restrict__ ks_dev, int64_t R,
                                                          const T* __restrict__ x, int Tn, int d, int KR,
                                                          const int32_t* __restrict__ row_of, int add_residual,
                                                          T* __restrict__ y) {
  const int ks = *ks_dev;
  const int nvec = d / 8;
  const int64_t total = static_cast<int64_t>(Tn) * nvec;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int64_t t = i / nvec;
    const int c = static_cast<int>(i - t * nvec);
    float acc[8];
    if (add_residual) {
      Vec8<T>::load(x + t * d + c * 8, acc);
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = 0.0f;
    }
    for (int s = 0; s < KR; ++s) {
      const int r = __ldg(row_of + t * KR + s);
      if (r < 0) continue;
      float row[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) row[k] = 0.0f;
      for (int sp = 0; sp < ks; ++sp) {
        float v[8];
        Vec8<float>::load(part + (sp * R + r) * d + c * 8, v);
#pragma unroll
        for (int k = 0; k < 8; ++k) row[k] += v[k];
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] += row[k];
    }
    Vec8<T>::store(y + t * d + c * 8, acc);
  }
}

cudaError_t launch_combine_partials(int dtype, const float* partial, const int* ks, int64_t R, const void* x, int T,
                                    int d, int KR, const int32_t* row_of, int add_residual, void* y, int num_sms,
                                    cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  const int64_t total = static_cast<int64_t>(T) * (d / 8);
  int64_t blocks = (total + 255) / 256;
  if (blocks > num_sms * 8) blocks = num_sms * 8;
  if (dtype == 0)
    k_combine_partials<__nv_bfloat16><<<static_cast<int>(blocks), 256, 0, s>>>(
        partial, ks, R, static_cast<const __nv_bfloat16*>(x), T, d, KR, row_of, add_residual,
        static_cast<__nv_bfloat16*>(y));
  else
    k_combine_partials<float><<<static_cast<int>(blocks), 256, 0, s>>>(partial, ks, R, static_cast<const float*>(x),
                                                                        T, d, KR, row_of, add_residual,
                                                                        static_cast<float*>(y));
  return cudaGetLastError();
}

// ------------------------------------------------------------ united init
// Round an fp64 value to bf16, ties to even, directly from the fp64 bits.
__device__ __forceinline__ uint16_t f64_to_bf16_rne(double v) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  const unsigned long long sign = b >> 63;
  const long long exp = static_cast<long long>((b >> 52) & 0x7ff);
  if (exp == 0x7ff) {   // inf / nan
    const unsigned long long mant = b & 0xfffffffffffffull;
    return static_cast<uint16_t>((sign << 15) | 0x7f80u | (mant ? 0x40u : 0u));
  }
  if (v == 0.0) return static_cast<uint16_t>(sign << 15);
  // bf16 significand has 8 bits; drop 45 of the 53 fp64 significand bits.
  const unsigned long long low = b & ((1ull << 45) - 1);
  unsigned long long kept = b >> 45;                  // sign | exp(11) | mant(7)
  const unsigned long long half = 1ull << 44;
  if (low > half || (low == half && (kept & 1ull))) ++kept;
  // re-bias the exponent from 1023 to 127 (normal range only; generators stay inside it)
  const long long e11 = static_cast<long long>((kept >> 7) & 0x7ff);
  const unsigned long long mant7 = kept & 0x7f;
  const long long e8 = e11 - 1023 + 127;
  if (e8 >= 0xff) return static_cast<uint16_t>((sign << 15) | 0x7f80u);
  if (e8 <= 0) return static_cast<uint16_t>(sign << 15);   // flush (outside the generated range)
  return static_cast<uint16_t>((sign << 15) | (static_cast<unsigned long long>(e8) << 7) | mant7);
}

template <typename T>
__global__ void k_united_mean(const T* __restrict__ W, int m, int way, int64_t per_expert, T* __restrict__ U) {
  const int G = (m + way - 1) / way;
  const int64_t total = static_cast<int64_t>(G) * per_expert;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(i / per_expert);
    const int64_t o = i - static_cast<int64_t>(j) * per_expert;
    const int e0 = j * way, e1 = min((j + 1) * way, m);
    double acc = 0.0;
    for (int e = e0; e < e1; ++e) {   // members ascending
      double w;
      if constexpr (sizeof(T) == 2) w = static_cast<double>(__bfloat162float(W[static_cast<int64_t>(e) * per_expert + o]));
      else w = static_cast<double>(W[static_cast<int64_t>(e) * per_expert + o]);
      acc += w;
    }
    const double mean = acc / static_cast<double>(e1 - e0);
    if constexpr (sizeof(T) == 2) {
      const uint16_t bits = f64_to_bf16_rne(mean);
      U[i] = *reinterpret_cast<const __nv_bfloat16*>(&bits);
    } else {
      U[i] = __double2float_rn(mean);
    }
  }
}

cudaError_t launch_build_united(int dtype, const void* W, int m, int way, int64_t per_expert, void* U,
                                cudaStream_t s) {
  const int G = (m + way - 1) / way;
  const int64_t total = static_cast<int64_t>(G) * per_expert;
  if (total == 0) return cudaSuccess;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (dtype == 0)
    k_united_mean<__nv_bfloat16><<<static_cast<int>(blocks), 256, 0, s>>>(
        static_cast<const __nv_bfloat16*>(W), m, way, per_expert, static_cast<__nv_bfloat16*>(U));
  else
    k_united_mean<float><<<static_cast<int>(blocks), 256, 0, s>>>(static_cast<const float*>(W), m, way,
                                                                  per_expert, static_cast<float*>(U));
  return cudaGetLastError();
}

}  // namespace bo
