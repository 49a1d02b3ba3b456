// Microbenchmark: DRAM read bandwidth of the GEMM weight-tile access pattern
// (boxes of R rows x 128 B at a row stride of S bytes) vs contiguous chunks.
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

// each block reads `boxes` boxes; box b: rows [0,R) at base + b_off + r*S, 128 B each (8 x uint4)
__global__ void k_box(const uint4* __restrict__ p, int64_t nbox_total, int R, int64_t stride16, int64_t boxes_per_row_band, uint4* sink) {
  uint4 acc = make_uint4(0,0,0,0);
  for (int64_t b = blockIdx.x; b < nbox_total; b += gridDim.x) {
    // box b -> (row band, k column): k fastest like the GEMM mainloop of one tile
    const int64_t band = b / boxes_per_row_band, kcol = b % boxes_per_row_band;
    const uint4* base = p + band * R * stride16 + kcol * 8;
    for (int i = threadIdx.x; i < R * 8; i += blockDim.x) {
      const int r = i >> 3, c = i & 7;
      uint4 v = __ldcs(base + r * stride16 + c);
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}
// box of R rows x (W*128 B): k window W (consecutive k-blocks of the same rows at once)
__global__ void k_boxw(const uint4* __restrict__ p, int64_t nbox_total, int R, int W, int64_t stride16,
                       int64_t boxes_per_row_band, uint4* sink) {
  uint4 acc = make_uint4(0,0,0,0);
  for (int64_t b = blockIdx.x; b < nbox_total; b += gridDim.x) {
    const int64_t band = b / boxes_per_row_band, kcol = b % boxes_per_row_band;
    const uint4* base = p + band * R * stride16 + kcol * 8 * W;
    for (int i = threadIdx.x; i < R * 8 * W; i += blockDim.x) {
      const int r = i / (8 * W), c = i % (8 * W);
      uint4 v = __ldcs(base + r * stride16 + c);
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}
__global__ void k_lin(const uint4* __restrict__ p, int64_t n16, uint4* sink) {
  uint4 acc = make_uint4(0,0,0,0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(p + i);
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}
int main() {
  const int64_t rows = 8 * 2 * 14336, cols = 4096;   // Mixtral Wg+Wu stacks: 1.88 GB bf16
  const int64_t bytes = rows * cols * 2;
  uint4 *p, *sink;
  cudaMalloc(&p, bytes); cudaMalloc(&sink, 64);
  cudaMemset(p, 1, bytes);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int64_t stride16 = cols * 2 / 16;
  for (int R : {112, 128}) {
    const int64_t bands = rows / R, kb = cols * 2 / 128;
    for (int blocks : {148, 296, 592, 1184}) {
      for (int it = 0; it < 2; ++it) {
        cudaEventRecord(a);
        k_box<<<blocks, 512>>>(p, bands * kb, R, stride16, kb, sink);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (it) printf("box R=%d blocks=%d: %.0f GB/s\n", R, blocks, bands * R * 128.0 * kb / ms / 1e6);
      }
    }
  }
  for (int W : {2, 4, 8}) {
    const int R = 128;
    const int64_t bands = rows / R, kb = cols * 2 / (128 * W);
    for (int blocks : {592, 1184}) {
      for (int it = 0; it < 2; ++it) {
        cudaEventRecord(a);
        k_boxw<<<blocks, 512>>>(p, bands * kb, R, W, stride16, kb, sink);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (it) printf("box R=%d window=%d B blocks=%d: %.0f GB/s\n", R, 128 * W, blocks, bands * R * 128.0 * W * kb / ms / 1e6);
      }
    }
  }
  for (int blocks : {148, 592, 1184, 2368}) {
    for (int it = 0; it < 2; ++it) {
      cudaEventRecord(a);
      k_lin<<<blocks, 512>>>(p, bytes / 16, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (it) printf("linear blocks=%d: %.0f GB/s\n", blocks, bytes / ms / 1e6);
    }
  }
  return 0;
}
