/*
 * c_forward.c - a plain C client of the brownout C ABI (include/brownout.h),
 * no Python or PyTorch: load fp32 inputs from files, convert to bf16 on the
 * host, cudaMalloc / cudaMemcpy them, build the united experts, set the
 * brownout ratio and run moe_forward(tokens, router, experts, united) (B:5),
 * then write y (bf16 bits) and the plan statistics.
 *
 *   c_forward <dir> d f m K way T ratio
 *     reads  <dir>/{x,Wr,Wg,Wu,Wd}.f32 (row-major fp32, exactly bf16-representable)
 *     writes <dir>/y_c.bf16 (uint16 bits [T, d]) and prints "stats ..." / "kernels ..."
 * Exit code 0 on success; on any bo_status error prints bo_last_error() and exits 1.
 *
 * Build: gcc -O2 -I include examples/c_forward.c -L paper_2507_17133_b200 -lbrownout
 *            -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,... -o c_forward
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "brownout.h"

#define CHECK_BO(call)                                                                     \
  do {                                                                                     \
    bo_status s_ = (call);                                                                 \
    if (s_ != BO_OK) {                                                                     \
      fprintf(stderr, "%s -> %s: %s\n", #call, bo_status_string(s_), bo_last_error());    \
      return 1;                                                                            \
    }                                                                                      \
  } while (0)
#define CHECK_CUDA(call)                                                                   \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      fprintf(stderr, "%s -> %s\n", #call, cudaGetErrorString(e_));                        \
      return 1;                                                                            \
    }                                                                                      \
  } while (0)

/* fp32 -> bf16 bits, round to nearest even (inputs are bf16-representable: exact) */
static uint16_t f2bf(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

static uint16_t* load_bf16(const char* dir, const char* name, size_t n) {
  char path[1024];
  snprintf(path, sizeof(path), "%s/%s.f32", dir, name);
  FILE* fp = fopen(path, "rb");
  if (!fp) return NULL;
  float* tmp = (float*)malloc(n * sizeof(float));
  uint16_t* out = (uint16_t*)malloc(n * sizeof(uint16_t));
  size_t got = fread(tmp, sizeof(float), n, fp);
  fclose(fp);
  if (got != n) { free(tmp); free(out); return NULL; }
  for (size_t i = 0; i < n; ++i) out[i] = f2bf(tmp[i]);
  free(tmp);
  return out;
}

static void* to_device(const void* host, size_t bytes) {
  void* d = NULL;
  if (cudaMalloc(&d, bytes) != cudaSuccess) return NULL;
  if (cudaMemcpy(d, host, bytes, cudaMemcpyHostToDevice) != cudaSuccess) return NULL;
  return d;
}

int main(int argc, char** argv) {
  if (argc != 9) {
    fprintf(stderr, "usage: %s <dir> d f m K way T ratio\n", argv[0]);
    return 2;
  }
  const char* dir = argv[1];
  const int d = atoi(argv[2]), f = atoi(argv[3]), m = atoi(argv[4]), K = atoi(argv[5]), way = atoi(argv[6]);
  const int64_t T = atoll(argv[7]);
  const double ratio = atof(argv[8]);
  const int G = (m + way - 1) / way;

  bo_config cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.hidden = d; cfg.ffn = f; cfg.num_experts = m; cfg.top_k = K; cfg.way = way;
  cfg.dtype = BO_BF16; cfg.add_residual = 0; cfg.max_tokens = T;
  bo_handle* h = NULL;
  CHECK_BO(bo_create(&cfg, &h));

  /* the error contract: a bad ratio is rejected, the handle stays usable */
  if (bo_set_brownout(h, 1.5, BO_PARTIAL) != BO_ERR_INVALID_ARG) {
    fprintf(stderr, "ratio 1.5 was not rejected\n");
    return 1;
  }

  const size_t nx = (size_t)T * d, nr = (size_t)m * d, ne = (size_t)m * f * d;
  uint16_t* hx = load_bf16(dir, "x", nx);
  uint16_t* hwr = load_bf16(dir, "Wr", nr);
  uint16_t* hwg = load_bf16(dir, "Wg", ne);
  uint16_t* hwu = load_bf16(dir, "Wu", ne);
  uint16_t* hwd = load_bf16(dir, "Wd", ne);
  if (!hx || !hwr || !hwg || !hwu || !hwd) {
    fprintf(stderr, "cannot read inputs from %s\n", dir);
    return 1;
  }
  void *x = to_device(hx, nx * 2), *Wr = to_device(hwr, nr * 2), *Wg = to_device(hwg, ne * 2),
       *Wu = to_device(hwu, ne * 2), *Wd = to_device(hwd, ne * 2);
  void *UWg = NULL, *UWu = NULL, *UWd = NULL, *y = NULL, *ws = NULL;
  const size_t nu = (size_t)G * f * d;
  CHECK_CUDA(cudaMalloc(&UWg, nu * 2));
  CHECK_CUDA(cudaMalloc(&UWu, nu * 2));
  CHECK_CUDA(cudaMalloc(&UWd, nu * 2));
  CHECK_CUDA(cudaMalloc(&y, nx * 2));
  size_t ws_bytes = 0;
  CHECK_BO(bo_workspace_size(h, T, &ws_bytes));
  CHECK_CUDA(cudaMalloc(&ws, ws_bytes));
  if (!x || !Wr || !Wg || !Wu || !Wd) {
    fprintf(stderr, "device allocation failed\n");
    return 1;
  }
  cudaStream_t s;
  CHECK_CUDA(cudaStreamCreate(&s));

  /* the three calls of the problem statement (B:5) */
  CHECK_BO(bo_build_united(h, Wg, Wu, Wd, BO_UNITED_MEAN, UWg, UWu, UWd, (void*)s));
  CHECK_BO(bo_set_brownout(h, ratio, BO_PARTIAL));
  CHECK_BO(bo_moe_forward(h, x, T, Wr, Wg, Wu, Wd, UWg, UWu, UWd, y, ws, ws_bytes, (void*)s));
  CHECK_CUDA(cudaStreamSynchronize(s));
  const int32_t n_launch = bo_last_launch_count(h);
  char kernels[256];
  snprintf(kernels, sizeof(kernels), "%s", bo_last_kernels(h));

  /* too small a workspace is a status, not a crash */
  if (bo_moe_forward(h, x, T, Wr, Wg, Wu, Wd, UWg, UWu, UWd, y, ws, 16, (void*)s) != BO_ERR_WORKSPACE) {
    fprintf(stderr, "short workspace was not rejected\n");
    return 1;
  }

  uint16_t* hy = (uint16_t*)malloc(nx * 2);
  CHECK_CUDA(cudaMemcpy(hy, y, nx * 2, cudaMemcpyDeviceToHost));
  bo_ws_layout L;
  CHECK_BO(bo_workspace_layout(h, T, &L));
  bo_plan_stats st;
  CHECK_CUDA(cudaMemcpy(&st, (char*)ws + L.stats, sizeof(st), cudaMemcpyDeviceToHost));

  char path[1024];
  snprintf(path, sizeof(path), "%s/y_c.bf16", dir);
  FILE* fp = fopen(path, "wb");
  if (!fp || fwrite(hy, 2, nx, fp) != nx) {
    fprintf(stderr, "cannot write %s\n", path);
    return 1;
  }
  fclose(fp);
  printf("stats %lld %lld %lld %lld %lld %lld %lld %lld\n", (long long)st.executors_accessed, (long long)st.n_s1,
         (long long)st.n_united, (long long)st.n_singleton, (long long)st.rows_original, (long long)st.rows_united,
         (long long)st.rows_dropped, (long long)st.rows_total);
  printf("kernels %d %s\n", n_launch, kernels);
  printf("version %s\n", bo_version());
  CHECK_BO(bo_destroy(h));
  return 0;
}
