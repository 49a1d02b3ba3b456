// bo_internal.h - state and stage functions shared by the C-ABI translation units
// (bo_api.cu: single-GPU forward, distillation; bo_ep_api.cu: expert parallelism).
// Internal to libbrownout; not part of the C ABI.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <string>

#include "../../include/brownout.h"
#include "bo_kernels.h"

// Engine options (bo_engine_option, include/brownout.h): per handle, defaults set by
// bo_create (overridable from the environment, BO_<NAME>, for A/B runs and tests).
struct EngineOptions {
  int32_t cta_pairs = 1;       // prefill FFN GEMMs on cta_group::2 CTA pairs
  int32_t pair_rows1 = 2048;   // GEMM1 uses pairs from this many rows
  int32_t pair_rows2 = 2048;   // GEMM2 likewise
  int32_t tile_alt = 1;        // GEMM1 may pick a narrower SwiGLU tile on the device
  int32_t swap_tail = 1;       // CTA-pair GEMM1 runs each executor's ragged last m-tile with swapped operands
  int32_t decode_pair2 = 1;    // decode steps with >= 256 rows per executor: GEMM2 pairs + split-K
  int32_t gemm2_splitk = 0;    // 1: GEMM2 split-K for every decode-sized step
  int32_t fused_combine = 2;   // a8 in GEMM2's epilogue: 0 never, 1 always, 2 auto
  int32_t tma_store = 1;       // GEMM2 full 32-row Yp slabs leave through TMA bulk stores
  int32_t store_hint = 1;      // FFN epilogue stores hint L2 evict_first (prefill)
  int32_t b_policy = -1;       // weight loads: 0 evict_normal, 1 evict_first, -1 auto (evict_first for decode)
  int32_t router_mma = 1;      // prefill-sized bf16 m <= 32 batches: mma.sync router
  int32_t router_split = 1;    // decode-sized m <= 32 batches: split-warp router
  int32_t pdl = 1;             // programmatic dependent launch of the GEMMs
  int32_t route_fused = 1;     // decode-sized m <= 32: routing, Alg. 1, permute + gather in one launch
  int32_t tail_split = 1;      // GEMM2 on pairs: a partial last wave shared out by k-blocks over every pair
};

struct bo_handle {
  bo_config cfg;
  double ratio;
  int32_t mode;
  int num_sms;
  int device;
  int32_t last_launches;
  void** prof_events;
  int32_t prof_n;
  int64_t route_T;     // token count / tile of the last route stage (bo_route, forward)
  int32_t route_tile;
  EngineOptions opt;
  std::string last_kernels;   // comma-separated names of the kernels the last forward launched
  const void* SWg;       // shared experts (Eq. 5 second term): [N_s, f, d], [N_s, f, d], [N_s, d, f]
  const void* SWu;
  const void* SWd;
};

namespace bo_impl {

constexpr int64_t kSplitRows = 1024;   // GEMM2 split-K (decode) only for R <= this
constexpr int kSplitMax = 8;
constexpr int64_t kTailSplitRows = 2048;   // workspace carries GEMM2's last-wave-split partials from here

bo_status fail(bo_status s, const char* fmt, ...);
bo_status cuda_fail(cudaError_t e, const char* what);
#define BO_CUDA(call, what)                                        \
  do {                                                             \
    cudaError_t e_ = (call);                                       \
    if (e_ != cudaSuccess) return bo_impl::cuda_fail(e_, what);    \
  } while (0)

size_t align256(size_t v);
int elem_bytes(int32_t dtype);
bool aligned16(const void* p);
int gemm2_bn(int d);

template <typename P>
P* at(void* ws, size_t off) {
  return reinterpret_cast<P*>(static_cast<char*>(ws) + off);
}

// Per-kernel profiling events (bo_set_profile_events); graph-capture aware.  Also NVTX
// ranges (header-only NVTX3; no-ops unless a tool such as Nsight Systems is attached):
// one "bo" range per entry-point call, one nested range per kernel launch named as in
// bo_last_kernels.
struct Prof {
  bo_handle* h;
  cudaStream_t s;
  bool on = false;
  unsigned flags = 0;
  cudaError_t err = cudaSuccess;
  bool nvtx_open = false;
  Prof(const Prof&) = delete;
  Prof& operator=(const Prof&) = delete;
  ~Prof() {
    if (nvtx_open) nvtxRangePop();
    nvtxRangePop();
  }
  Prof(bo_handle* h_, cudaStream_t s_, int max_launches) : h(h_), s(s_) {
    nvtxRangePushA("bo");
    on = h->prof_events && h->prof_n >= max_launches + 1;
    if (on) {
      cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
      err = cudaStreamIsCapturing(s, &cap);
      // under stream capture the events must become graph event-record nodes (external)
      flags = cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0u;
    }
  }
  // event i precedes launch i; `name` (forward path) is appended to the handle's kernel list
  void mark(int i, const char* name = nullptr) {
    if (name) {
      if (nvtx_open) nvtxRangePop();
      nvtxRangePushA(name);
      nvtx_open = true;
      if (!h->last_kernels.empty()) h->last_kernels += ",";
      h->last_kernels += name;
    }
    if (on && err == cudaSuccess && h->prof_events[i])   // NULL entries: no event at that boundary
      err = cudaEventRecordWithFlags(static_cast<cudaEvent_t>(h->prof_events[i]), s, flags);
  }
};

// Weights of one executor class: stacked [n, f, d] gate / up and [n, d, f] down.
struct FfnClass {
  const void* Wg = nullptr;
  const void* Wu = nullptr;
  const void* Wd = nullptr;
  int n = 0;        // executors of this class in the row layout
  int f = 0;        // width (united: f-slice under expert parallelism)
  int64_t stack = 0;  // experts in the weight stacks (>= n; tensor-map extent)
};

// The combine (a8) fused into GEMM2's epilogue (bo::GemmParams::comb_cnt).
struct CombFuse {
  int32_t* cnt;            // [T, d / BN2] arrival counters (workspace)
  const int32_t* row_of;   // [T, KR]
  int KR;
  int64_t T;
  const void* x;
  void* y;
  int add_residual;
};

// Workspace layout of a forward over T tokens (bo_ws_layout) and its check.
bo_status compute_layout(const bo_handle* h, int64_t T, bo_ws_layout* L, bool route_only = false);
bo_status check_ws(const bo_handle* h, int64_t T, void* ws, size_t ws_bytes, bo_ws_layout* L);
// a1-a4 (router, top-K, histogram, Alg. 1 on the local counts); `tile` = token tile used.
bo_status route_stage(bo_handle* h, const void* x, int64_t T, const void* Wr, const float* logits_in, void* ws,
                      const bo_ws_layout& L, cudaStream_t s, Prof& prof, int& launches, int& tile,
                      int32_t* ep_row = nullptr);
// a6-a7 over rows grouped by executor (exec_off / mtile_off device arrays); R an upper bound
// of the rows (the kernels read the exact counts from exec_off on the device).
bo_status ffn_stage(bo_handle* h, const void* X, int64_t R, const float* row_w, const int32_t* exec_off,
                    const int32_t* mtile_off, const FfnClass& orig, const FfnClass& uni, const FfnClass& shr,
                    void* Hbuf, void* Y, cudaStream_t s, Prof& prof, int& launches, float* partial = nullptr,
                    int* ks_dev = nullptr, const CombFuse* comb = nullptr, const int32_t* comb_row_tok = nullptr,
                    bool force_pair2 = false, float* sk_part = nullptr, int* sk_flag = nullptr);

}  // namespace bo_impl
