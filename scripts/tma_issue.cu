// Microbenchmark: producer-thread cost of issuing TMA tile loads vs box size.
// One thread per CTA loads 32 KB per round as 32 KB / box boxes of `box` rows x 128 B
// (SWIZZLE_128B, the GEMM operand format), then waits on the mbarrier.  Reports the
// cycles spent issuing and the cycles until the round's bytes have landed, for one
// CTA alone and for 148 CTAs at once (one per SM), from an L2-resident 2 MB tensor
// and from a 1 GB tensor (DRAM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2507_17133_b200/csrc \
//        scripts/tma_issue.cu -lcuda -o /tmp/tma_issue && /tmp/tma_issue
#include "bo_ptx.cuh"

#include <vector>

using namespace bo;

__global__ void k_issue(const __grid_constant__ CUtensorMap m, int box, int rows, int reps, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int nl = 256 / box;   // 32 KB per round
  const uint64_t pol = policy_evict_normal();
  uint32_t phase = 0;
  long long ti = 0, tt = 0;
  int row = (blockIdx.x * 256) % rows;
  for (int r = 0; r < reps; ++r) {
    const long long t0 = clock64();
    mbar_arrive_expect_tx(&bar, 32768);
    for (int i = 0; i < nl; ++i) {
      tma_load_2d(smem + i * box * 128, &m, &bar, 0, row, pol);
      row += box;
      if (row + box > rows) row = 0;
    }
    const long long t1 = clock64();
    mbar_wait(&bar, phase);
    phase ^= 1;
    const long long t2 = clock64();
    if (r > 0) {   // round 0 warms the descriptor
      ti += t1 - t0;
      tt += t2 - t0;
    }
    row = (row + 148 * 256) % rows;
  }
  out[2 * blockIdx.x] = ti / (reps - 1);
  out[2 * blockIdx.x + 1] = tt / (reps - 1);
}

typedef CUresult (*PFN_encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  PFN_encode enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  if (!enc) {
    printf("no cuTensorMapEncodeTiled\n");
    return 1;
  }
  const long long big_rows = (1LL << 30) / 128;   // 1 GB of 128-byte rows (64 bf16 per row, K-major)
  void* buf;
  cudaMalloc(&buf, big_rows * 128);
  cudaMemset(buf, 0, big_rows * 128);
  long long* d_out;
  cudaMalloc(&d_out, 148 * 2 * sizeof(long long));
  cudaFuncSetAttribute(k_issue, cudaFuncAttributeMaxDynamicSharedMemorySize, 34 * 1024);
  printf("{\"unit\": \"cycles per 32 KB round\", \"rows\": [\n");
  bool first = true;
  for (long long rows : {16384LL, big_rows}) {   // 2 MB (L2-resident) / 1 GB
    for (int box : {16, 32, 64, 128, 256}) {
      CUtensorMap m;
      cuuint64_t dims[2] = {64, static_cast<cuuint64_t>(rows)};
      cuuint64_t strides[1] = {128};
      cuuint32_t boxd[2] = {64, static_cast<cuuint32_t>(box)};
      cuuint32_t estr[2] = {1, 1};
      if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, boxd, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("encode failed\n");
        return 1;
      }
      for (int grid : {1, 148}) {
        k_issue<<<grid, 32, 34 * 1024>>>(m, box, static_cast<int>(rows), 65, d_out);
        if (cudaDeviceSynchronize() != cudaSuccess) {
          printf("kernel failed\n");
          return 1;
        }
        std::vector<long long> h(2 * grid);
        cudaMemcpy(h.data(), d_out, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
        double ti = 0, tt = 0;
        for (int b = 0; b < grid; ++b) {
          ti += h[2 * b];
          tt += h[2 * b + 1];
        }
        printf("%s {\"tensor\": \"%s\", \"box_rows\": %d, \"boxes\": %d, \"ctas\": %d, \"issue\": %.0f, "
               "\"issue_per_box\": %.1f, \"round\": %.0f}",
               first ? " " : ",\n ", rows == 16384 ? "L2 2MB" : "DRAM 1GB", box, 256 / box, grid, ti / grid,
               ti / grid / (256 / box), tt / grid);
        first = false;
      }
    }
  }
  printf("\n]}\n");
  return 0;
}
