// bo_distill.cu - element-wise kernels of united-expert distillation
// (BrownoutServe §4.2, Eq. 4).  The contractions (teacher FFNs,
// student forward, backward, weight gradients with the fused SGD update) run
// on the tcgen05 grouped GEMM (bo_gemm.cu); these kernels hold the
// element-wise steps between them.  Every reduction is a fixed-order tree
// (no atomics), so a step is bitwise reproducible.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "bo_kernels.h"

namespace bo {
namespace {

__device__ __forceinline__ float bf(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ __nv_bfloat16 tobf(float v) { return __float2bfloat16_rn(v); }

__device__ __forceinline__ double block_sum_d(double v, double* sh) {
  // 256 threads (1-D): fixed-order tree; the result is valid in thread 0
  const int tid = threadIdx.x;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((tid & 31) == 0) sh[tid >> 5] = v;
  __syncthreads();
  double r = 0.0;
  if (tid == 0)
    for (int w = 0; w < 8; ++w) r += sh[w];
  return r;
}

__global__ void k_fill_offsets(int32_t* off, int n, int stride) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x) off[i] = i * stride;
}

// Hbar[j, t] = (1/k_j) sum_{i in group j} Yo[i, t]  (the pointwise minimiser of
// Eq. 4) and the per-block partial of sum_t sum_i ||Yo[i, t] - Hbar[j, t]||^2.
// grid (nb, G), 256 threads; one thread per float4 of the [N, d] slab.
__global__ void __launch_bounds__(256) k_group_mean(const float4* __restrict__ Yo, int m, int way, int64_t N,
                                                    int d4, float4* __restrict__ Hbar, double* __restrict__ part) {
  __shared__ double sh[8];
  const int j = blockIdx.y;
  const int e0 = j * way;
  const int e1 = min(e0 + way, m);
  const float inv_k = 1.0f / static_cast<float>(e1 - e0);
  const int64_t n4 = N * d4;
  double acc = 0.0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * 256) {
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int e = e0; e < e1; ++e) {
      const float4 v = Yo[static_cast<int64_t>(e) * n4 + i];
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    s.x *= inv_k; s.y *= inv_k; s.z *= inv_k; s.w *= inv_k;
    Hbar[static_cast<int64_t>(j) * n4 + i] = s;
    for (int e = e0; e < e1; ++e) {
      const float4 v = Yo[static_cast<int64_t>(e) * n4 + i];
      const double a = static_cast<double>(v.x) - s.x, b = static_cast<double>(v.y) - s.y;
      const double c = static_cast<double>(v.z) - s.z, dd = static_cast<double>(v.w) - s.w;
      acc += a * a + b * b + c * c + dd * dd;
    }
  }
  const double r = block_sum_d(acc, sh);
  if (threadIdx.x == 0) part[static_cast<int64_t>(j) * gridDim.x + blockIdx.x] = r;
}

// out[j] = base[j] + scale_j * sum_b part[j, b] (fixed-order: strided per-thread
// sums, then a tree), scale_j = 1 / (N k_j) or 1 / N.  One 256-thread block per group.
__global__ void __launch_bounds__(256) k_reduce_groups(const double* __restrict__ part, int nb, int m, int way,
                                                       int64_t N, int divide_by_k, const double* __restrict__ base,
                                                       double* __restrict__ out) {
  __shared__ double sh[8];
  const int j = blockIdx.x;
  double s = 0.0;
  for (int b = threadIdx.x; b < nb; b += 256) s += part[static_cast<int64_t>(j) * nb + b];
  s = block_sum_d(s, sh);
  if (threadIdx.x == 0) {
    const int k = min(way, m - j * way);
    double v = s / static_cast<double>(N);
    if (divide_by_k) v /= static_cast<double>(k);
    out[j] = (base ? base[j] : 0.0) + v;
  }
}

// ---- 64 x 64 tiles over a batch of [R, C] matrices (R, C multiples of 64):
//      element-wise op with normal and / or transposed ([C, R]) outputs.
//      256 threads; each thread owns 2 adjacent columns of 8 rows (bf16x2 /
//      float2 accesses, 128-256 B per warp row) and, for the transposed store,
//      2 adjacent rows of 8 output rows.
enum TileOp { OP_SWIGLU_FWD = 0, OP_MSE_GRAD = 1, OP_SWIGLU_BWD = 2, OP_CAST = 3 };

__device__ __forceinline__ float2 ld_bf2(const void* p, int64_t i) {
  const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(static_cast<const __nv_bfloat16*>(p) + i);
  return __bfloat1622float2(v);
}
__device__ __forceinline__ void st_bf2(__nv_bfloat16* p, int64_t i, float a, float b) {
  *reinterpret_cast<__nv_bfloat162*>(p + i) = __floats2bfloat162_rn(a, b);
}
__device__ __forceinline__ float silu_bwd_a(float g, float a, float q) {
  const float s = __fdividef(1.0f, 1.0f + __expf(-a));   // fast division (see silu_f in bo_gemm.cu)
  return g * q * (s + a * s * (1.0f - s));
}

template <int OP>
__global__ void __launch_bounds__(256) k_tile(const void* __restrict__ in0, const void* __restrict__ in1,
                                              const void* __restrict__ in2, __nv_bfloat16* __restrict__ out,
                                              __nv_bfloat16* __restrict__ outT, __nv_bfloat16* __restrict__ outT2,
                                              int64_t R, int64_t C, float scale, double* __restrict__ part) {
  constexpr int NT = OP == OP_SWIGLU_BWD ? 2 : 1;
  __shared__ float t[NT][64][65];
  __shared__ double sh[8];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int64_t b = blockIdx.z;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 64, c0 = static_cast<int64_t>(blockIdx.x) * 64;
  const int64_t base = b * R * C;
  const int cc = 2 * l;
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int rr = w + 8 * k;
    const int64_t i = base + (r0 + rr) * C + c0 + cc;
    float2 v0, v1 = make_float2(0.f, 0.f);
    if constexpr (OP == OP_SWIGLU_FWD) {
      // Hs = silu(P) * Q (D24); Hs and Hs^T
      const float2 a = ld_bf2(in0, i), q = ld_bf2(in1, i);
      const __nv_bfloat162 h = __floats2bfloat162_rn(__fdividef(a.x, 1.0f + __expf(-a.x)) * q.x,
                                                     __fdividef(a.y, 1.0f + __expf(-a.y)) * q.y);
      *reinterpret_cast<__nv_bfloat162*>(out + i) = h;
      v0 = __bfloat1622float2(h);
    } else if constexpr (OP == OP_MSE_GRAD) {
      // dL/dY = (2/N) (Y - Hbar) (Eq. 4, D21); dY and dY^T; sum of squares
      const float2 y = *reinterpret_cast<const float2*>(static_cast<const float*>(in0) + i);
      const float2 hb = *reinterpret_cast<const float2*>(static_cast<const float*>(in1) + i);
      const float ex = y.x - hb.x, ey = y.y - hb.y;
      acc += static_cast<double>(ex) * ex + static_cast<double>(ey) * ey;
      const __nv_bfloat162 g = __floats2bfloat162_rn(ex * scale, ey * scale);
      *reinterpret_cast<__nv_bfloat162*>(out + i) = g;
      v0 = __bfloat1622float2(g);
    } else if constexpr (OP == OP_SWIGLU_BWD) {
      // dP = dHs * Q * silu'(P), dQ = dHs * silu(P); transposed outputs only
      const float2 g = ld_bf2(in0, i), a = ld_bf2(in1, i), q = ld_bf2(in2, i);
      v0 = make_float2(silu_bwd_a(g.x, a.x, q.x), silu_bwd_a(g.y, a.y, q.y));
      v1 = make_float2(g.x * __fdividef(a.x, 1.0f + __expf(-a.x)), g.y * __fdividef(a.y, 1.0f + __expf(-a.y)));
    } else {
      // fp32 master -> bf16 copy and / or transposed copy
      v0 = *reinterpret_cast<const float2*>(static_cast<const float*>(in0) + i);
      if (out) st_bf2(out, i, v0.x, v0.y);
    }
    t[0][rr][cc] = v0.x;
    t[0][rr][cc + 1] = v0.y;
    if constexpr (NT == 2) {
      t[1][rr][cc] = v1.x;
      t[1][rr][cc + 1] = v1.y;
    }
  }
  if constexpr (OP == OP_MSE_GRAD) {
    const double r = block_sum_d(acc, sh);
    if (threadIdx.x == 0) {
      const int64_t nbx = gridDim.x, nby = gridDim.y;
      part[b * nbx * nby + static_cast<int64_t>(blockIdx.y) * nbx + blockIdx.x] = r;
    }
  }
  if (!outT) return;
  __syncthreads();
  // transposed: element (r, c) -> outT[b][c][r]; this thread: rows 2l, 2l+1 of output rows w + 8k
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int c = w + 8 * k;
    const int64_t o = base + (c0 + c) * R + r0 + cc;
    st_bf2(outT, o, t[0][cc][c], t[0][cc + 1][c]);
    if constexpr (NT == 2) st_bf2(outT2, o, t[1][cc][c], t[1][cc + 1][c]);
  }
}

__global__ void k_widen(const __nv_bfloat16* __restrict__ in, float* __restrict__ out, int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = bf(in[i]);
}

template <int OP>
cudaError_t tile_launch(const void* a, const void* b, const void* c, void* out, void* outT, void* outT2, int64_t B,
                        int64_t R, int64_t C, float scale, double* part, cudaStream_t s) {
  if (B == 0 || R == 0 || C == 0) return cudaSuccess;
  if (R % 64 || C % 64) return cudaErrorInvalidValue;
  dim3 grid(static_cast<unsigned>(C / 64), static_cast<unsigned>(R / 64), static_cast<unsigned>(B));
  k_tile<OP><<<grid, 256, 0, s>>>(a, b, c, static_cast<__nv_bfloat16*>(out),
                                          static_cast<__nv_bfloat16*>(outT), static_cast<__nv_bfloat16*>(outT2), R, C,
                                          scale, part);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_fill_offsets(int32_t* off, int n, int stride, cudaStream_t s) {
  k_fill_offsets<<<(n + 256) / 256, 256, 0, s>>>(off, n, stride);
  return cudaGetLastError();
}

int group_mean_blocks(int64_t N, int d, int num_sms) {
  const int64_t n4 = N * (d / 4);
  int64_t nb = (n4 + 255) / 256;
  const int64_t cap = 2 * static_cast<int64_t>(num_sms);
  return static_cast<int>(nb < cap ? (nb < 1 ? 1 : nb) : cap);
}

cudaError_t launch_group_mean(const float* Yo, int m, int way, int64_t N, int d, float* Hbar, double* part,
                              double* floor_out, int num_sms, cudaStream_t s) {
  const int G = (m + way - 1) / way;
  const int nb = group_mean_blocks(N, d, num_sms);
  k_group_mean<<<dim3(nb, G), 256, 0, s>>>(reinterpret_cast<const float4*>(Yo), m, way, N, d / 4,
                                           reinterpret_cast<float4*>(Hbar), part);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_reduce_groups<<<G, 256, 0, s>>>(part, nb, m, way, N, 1, nullptr, floor_out);
  return cudaGetLastError();
}

cudaError_t launch_swiglu_fwd(const void* P, const void* Q, void* Hs, void* HsT, int64_t G, int64_t N, int64_t f,
                              cudaStream_t s) {
  return tile_launch<OP_SWIGLU_FWD>(P, Q, nullptr, Hs, HsT, nullptr, G, N, f, 0.f, nullptr, s);
}

int mse_grad_blocks(int64_t N, int64_t d) { return static_cast<int>((d / 64) * (N / 64)); }

cudaError_t launch_mse_grad(const float* Y, const float* Hbar, void* dY, void* dYT, int64_t G, int64_t N, int64_t d,
                            double* part, const double* floor_in, int m, int way, double* loss_out, cudaStream_t s) {
  cudaError_t e = tile_launch<OP_MSE_GRAD>(Y, Hbar, nullptr, dY, dYT, nullptr, G, N, d,
                                           2.0f / static_cast<float>(N), part, s);
  if (e != cudaSuccess) return e;
  const int nb = mse_grad_blocks(N, d);
  k_reduce_groups<<<static_cast<int>(G), 256, 0, s>>>(part, nb, m, way, N, 0, floor_in, loss_out);
  return cudaGetLastError();
}

cudaError_t launch_swiglu_bwd(const void* dHs, const void* P, const void* Q, void* dPT, void* dQT, int64_t G,
                              int64_t N, int64_t f, cudaStream_t s) {
  return tile_launch<OP_SWIGLU_BWD>(dHs, P, Q, nullptr, dPT, dQT, G, N, f, 0.f, nullptr, s);
}

cudaError_t launch_cast_master(const float* W, void* Wb, void* WbT, int64_t G, int64_t R, int64_t C, cudaStream_t s) {
  return tile_launch<OP_CAST>(W, nullptr, nullptr, Wb, WbT, nullptr, G, R, C, 0.f, nullptr, s);
}

cudaError_t launch_widen(const void* Wb, float* W, int64_t n, int num_sms, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 8 * num_sms) blocks = 8 * num_sms;
  k_widen<<<static_cast<int>(blocks), 256, 0, s>>>(static_cast<const __nv_bfloat16*>(Wb), W, n);
  return cudaGetLastError();
}

}  // namespace bo
