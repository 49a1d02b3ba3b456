// bo_kernels.h - internal launch interface between the C-ABI layer and the kernels.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace bo {

constexpr int kTileTok = 128;   // token tile of the tcgen05 router (= GEMM BM)
constexpr int kBM = 128;        // rows per GEMM tile (TMEM lanes)
constexpr int kMaxExperts = 256;
constexpr int kMaxExec = 512;   // m + G

enum Epi : int { EPI_SWIGLU = 0, EPI_WEIGHTED = 1, EPI_ROUTER = 2,
                 EPI_SWIGLU_PAIR = 3, EPI_WEIGHTED_PAIR = 4 };   // *_PAIR: cta_group::2, grid even

struct GemmParams {
  int Kdim;              // reduction length (executors < m_orig)
  int n_tiles;           // output tiles per executor along N (executors < m_orig)
  int Kdim_u;            // reduction length of executors >= m_orig
  int n_tiles_u;         // output tiles of executors >= m_orig
  int b_rows_u;          // rows of B per executor >= m_orig in its stacked view
  int ldo;               // leading dimension of the output (elements)
  int n_valid;           // valid output columns (router: m)
  int m_orig;            // executors < m_orig read B maps 0/1 (originals)
  int m_united;          // next m_united executors read maps 2/3 (united); the rest maps 4/5 (shared)
  int b_rows_per_exec;   // rows of B per executor in the stacked [E*rows, K] view
  int num_exec;          // executors (1 for the router)
  int single_rows;       // >= 0: one executor with this many rows (no device schedule)
  const int* exec_off;   // [num_exec+1] first row of each executor (device)
  const int* mtile_off;  // [num_exec+1] prefix of ceil(rows/128) (device)
  void* out;             // output base
  const float* row_w;    // EPI_WEIGHTED: per-row gate weight (Eq. 6)
  int topk_k;            // EPI_ROUTER: K of Eq. 7
  int32_t* topk_id;      // EPI_ROUTER: [T, K]
  float* topk_w;         // EPI_ROUTER: [T, K]
  int32_t* tile_cnt;     // EPI_ROUTER: [ceil(T/128), m] histogram per 128-token tile
  const int32_t* row_tok;  // fused combine: token of each row
  int rows_total;          // split-K partial rows (R)
  int ksplit_max;          // EPI_WEIGHTED: > 1 enables split-K (fp32 partials [ks, R, ldo] into `partial`)
  float* partial;          // EPI_WEIGHTED split-K output
  int* ks_out;             // EPI_WEIGHTED split-K: the kernel publishes the split count it chose
  int a_shared;            // 1: every executor reads A rows from 0 (one shared A, e.g. distillation tokens)
  int f32_mode;            // EPI_WEIGHTED: 1 = fp32 output to `partial`; 2 = fp32 accumulate (+=) into `partial`
  float alpha;             // EPI_WEIGHTED: row scale when row_w == nullptr
  int bh_alt;              // EPI_SWIGLU: > 0 enables an alternative half-width (gate / up columns per tile)
  int store_hint;          // 1: epilogue stores carry an L2 evict_first hint (streaming H / Yp)
  int nt_alt, nt_alt_u;    // its n-tile counts (originals & shared / united); the kernel picks the width
                           // with the fewer estimated tile-column waves over the device-side plan
  // Combine (a8, Eq. 5 sum over a token's rows) fused into GEMM2's epilogue:
  // every GEMM2 epilogue warp that has stored its rows' Yp segment of n-tile n
  // counts them in comb_cnt[t, n]; the warp whose arrival completes token t's
  // rows sums them in slot order (fp32, same order as k_combine) and writes
  // y[t, n-tile].  GEMM1 (always launched first) zeroes the counters in its
  // prologue and writes y of tokens that have no row (full brownout).
  int32_t* comb_cnt;        // [comb_T, comb_nt] arrival counters; nullptr: separate combine kernel
  const int32_t* row_of;    // [comb_T, comb_KR] row of (token, slot), -1: none
  int comb_KR;
  int comb_T;
  int comb_nt;              // GEMM2 n-tiles (counters per token)
  int comb_d;               // hidden size (y / x leading dimension)
  int add_residual;         // y = x + ... (Eq. 5 residual term)
  const void* comb_x;       // [T, d]
  void* comb_y;             // [T, d]
  int b_policy;             // L2 policy of the B (weight) tile loads: 0 evict_normal, 1 evict_first
  // Swapped-operand tail tiles (CG = 2 SwiGLU, BN = 256): an executor's last m-tile with
  // fewer than 256 rows runs as D^T = W X^T, the 256 gate / up weight rows on the MMA's
  // M side and its rows (rounded up to 32) on N, so a ragged tile costs its rows, not 256.
  // Maps [6..11] then hold 64-row gate / up boxes and [12..14] 16 / 32 / 64-row boxes of A (Xp).
  int swap_tail;
  int tma_store;            // EPI_WEIGHTED: full 32-row slabs leave through TMA bulk stores (map B[6], 32 x 32 box, 64B swizzle)
  // EPI_WEIGHTED on CTA pairs: a partial last wave's tiles shared out by k-blocks over every
  // pair (see the kernel); sk_part [units * 2][kSkPartElems] fp32 partials, sk_flag [units * 2]
  // arrival counts (4 epilogue warps), zeroed before every launch.
  int tail_split;
  float* sk_part;
  int* sk_flag;
};
constexpr int kSkPartElems = 256 * 128;   // one CTA's fp32 accumulator: 256 columns x 128 rows

// Combine of split-K fp32 partials: y[t] = [x_t] + sum_slots sum_splits P[sp][row].
cudaError_t launch_combine_partials(int dtype, const float* partial, const int* ks, int64_t R, const void* x, int T,
                                    int d, int KR, const int32_t* row_of, int add_residual, void* y, int num_sms,
                                    cudaStream_t s);

// Grouped tcgen05 GEMM: for each executor x and each 128-row tile of its rows,
// D = A[rows] * B_x^T with an epilogue selected by `epi`.
// dtype: 0 bf16, 1 fp32 (tf32 MMA).  bn: MMA N (SwiGLU: gate+up columns).
// B operand maps by executor class: [0]/[1] originals (gate or the only B / up),
// [2]/[3] united experts, [4]/[5] shared experts (Eq. 5 second term).
// [6..11]: the same three classes encoded for the alternative SwiGLU tile
// width (GemmParams::bh_alt rows per gate / up half), when it is enabled, or the
// 64-row gate / up boxes of the swapped tail tiles (GemmParams::swap_tail; [12..14] = A).
struct BMaps {
  CUtensorMap m[15];
};
// pdl: programmatic dependent launch (the GEMM's prologue may overlap the previous kernel's tail).
cudaError_t launch_grouped_gemm(int dtype, int epi, int bn, const CUtensorMap& A, const BMaps& B,
                                const GemmParams& p, int grid, cudaStream_t s, bool pdl);
int gemm_smem_bytes(int dtype, int epi, int bn);

constexpr int kTileMin = 8;     // smallest token tile (workspace histograms are sized for it)
constexpr int kTileSmall = 32;  // token tile of the injected-logits top-k
constexpr int kPermRowsSmem = 1024;   // (token, slot) rows of a permute tile kept in shared memory for its gather

cudaError_t launch_topk_hist(const float* logits, int T, int m, int K, int tile, int32_t* topk_id, float* topk_w,
                             int32_t* tile_cnt, cudaStream_t s);

bool router_small_ok(int dtype, int m, int d);
int router_small_tile(int T, int num_sms);   // 8..32 tokens per CTA
// Prefill-sized batches, bf16, m <= 32, d % 128 == 0: mma.sync router over 16-token tiles.
bool router_mma_ok(int dtype, int m, int d, int T, int num_sms);
cudaError_t launch_router_mma(const void* x, const void* Wr, int T, int d, int m, int K, float* logits,
                              int32_t* topk_id, float* topk_w, int32_t* tile_cnt, cudaStream_t s);
// Decode-sized batches: tpc tokens per CTA (0: use k_router_small), hidden dim split over 8/tpc warps.
int router_split_tpc(int T, int num_sms);
cudaError_t launch_router_split(int dtype, const void* x, const void* Wr, int T, int d, int m, int K, int tpc,
                                float* logits, int32_t* topk_id, float* topk_w, int32_t* tile_cnt, cudaStream_t s);
cudaError_t launch_router_small(int dtype, const void* x, const void* Wr, int T, int d, int m, int K, int tile,
                                float* logits, int32_t* topk_id, float* topk_w, int32_t* tile_cnt, cudaStream_t s);

// Expert-parallel extensions of the plan kernel: ld = row stride of the count rows (0: m);
// knob_in (nullable, device int32[4] = [T, mode, ratio lo, ratio hi]) overrides ratio / mode;
// row_tail (nullable, device int32[4]) receives [row_T, mode, ratio lo, ratio hi] of the knob used.
struct PlanExt {
  int ld = 0;
  const int32_t* knob_in = nullptr;
  int32_t* row_tail = nullptr;
  int row_T = 0;
};
// n_shared shared experts (Eq. 5) are appended after the m + G routed executors with shared_rows rows each.
cudaError_t launch_plan(const int32_t* tile_cnt, int ntiles, int m, int way, double ratio, int mode,
                        int32_t* tile_base, int32_t* counts, int32_t* exec_of_expert, int32_t* expert_row_off,
                        int32_t* exec_off, int32_t* mtile_off, int64_t* stats, cudaStream_t s, int n_shared = 0,
                        int shared_rows = 0, PlanExt ext = PlanExt());

// xp != nullptr: the permute also copies each token's x row to its rows (fused gather).
cudaError_t launch_permute(const int32_t* topk_id, const float* topk_w, int T, int K, int m, int tile,
                           const int32_t* tile_base, const int32_t* row_base, int nrep, int32_t* row_of,
                           int32_t* row_tok, float* row_w, cudaStream_t s, int dtype = 0, const void* x = nullptr,
                           void* xp = nullptr, int d = 0, int n_shared = 0, const int32_t* shared_off = nullptr);

// Decode-sized steps on one GPU: router (split-warp, m <= 32) + Eq. 7 + histogram, Alg. 1
// and the permutation (+ the gather when xp != nullptr) in one cooperative launch, every
// plan output written as by launch_plan / launch_permute (the per-tile prefixes stay in
// shared memory).  route_fused_ok: the shapes fit and the grid is co-resident.
constexpr int kRouteFusedMaxExec = 64;   // m + G + N_s executors (two per lane of the planning warp)
constexpr int kRouteFusedStage = 4096;   // tile histograms staged per CTA (ntiles * m)
int route_fused_tpc(int T, int num_sms);   // tokens per CTA (1/2/4/8) keeping the grid within #SM; 0: none
bool route_fused_ok(int dtype, int m, int way, int T, int tpc, int n_shared, int num_sms);
cudaError_t launch_route_fused(int dtype, const void* x, const void* Wr, int T, int d, int m, int K, int tpc,
                               float* logits, int32_t* topk_id, float* topk_w, int32_t* tile_cnt, int way,
                               double ratio, int mode, int32_t* counts, int32_t* exec_of_expert,
                               int32_t* expert_row_off, int32_t* exec_off, int32_t* mtile_off, int64_t* stats,
                               int n_shared, int32_t* row_of, int32_t* row_tok, float* row_w, void* xp,
                               cudaStream_t s);

cudaError_t launch_gather(int dtype, const void* x, int T, int d, int KR, const int32_t* row_of, void* xp,
                          int num_sms, cudaStream_t s);

cudaError_t launch_combine(int dtype, const void* yp, const void* x, int T, int d, int KR,
                           const int32_t* row_of, int add_residual, void* y, int num_sms, cudaStream_t s);

// ---- expert parallelism (bo_ep.cu)
constexpr int kEpMaxRanks = 8;     // one node
constexpr int kEpMaxV = 512;       // virtual executors (originals + united f-slices, all ranks)
// Static placement of one rank (kernel parameter image).  vexec[v] packs rank (bits
// 24-31), kind (bit 23: 1 = united slice), idx (bits 0-15: expert or group); virtual
// executors are rank-major, vfirst[q] the first of rank q.
struct EpStatic {
  int R, rank, m, way, nrep, nslices, V, nl, padded;
  int64_t cap;                      // rows per (source, destination) message in padded mode
  int32_t vexec[kEpMaxV];
  int32_t vfirst[kEpMaxRanks + 1];
  int32_t v_of_orig[kMaxExperts];
  int32_t v_of_slice[kEpMaxV];      // [group * nrep + slice]
  int32_t local_v[kEpMaxV];         // this rank's executors in GEMM order (originals, then slices)
};
// Per-forward tables (device int32 arrays in the EP workspace).
struct EpTables {
  int32_t* row_base;    // [m * nrep]   send position of expert e's first row (replica rep), -1 none
  int32_t* send_rows;   // [R]          rows this rank sends to each rank
  int32_t* recv_rows;   // [R]          rows this rank receives from each rank
  int32_t* fwd_dst;     // [nl*R + 1]   receive -> grouped blocks, (executor, source) order
  int32_t* fwd_len;     // [nl*R]
  int32_t* fwd_src;     // [nl*R]
  int32_t* inv_dst;     // [R*nl + 1]   grouped -> receive layout, (source, executor) order
  int32_t* inv_len;     // [R*nl]
  int32_t* inv_src;     // [R*nl]
  int32_t* exec_off;    // [nl + 1]     grouped rows per local executor
  int32_t* mtile_off;   // [nl + 1]
  int32_t* totals;      // [2]          grouped rows, receive-layout extent
  int64_t* splits;      // [2R]         send_rows, recv_rows (for the host in exact-size mode)
};
cudaError_t launch_ep_tables(const EpStatic& st, const int32_t* gathered, int ld, const int32_t* exec_of,
                             const EpTables& tb, cudaStream_t s);
// Row-block permutation: block b moves len[b] rows src_off[b] + k -> dst_start[b] + k
// (dst_start ascending, n_blocks + 1 entries); destination extent read from `extent`
// (device, nullable) capped at extent_max.
cudaError_t launch_block_copy(const void* src, void* dst, int row_bytes, const float* w_src, float* w_dst,
                              int n_blocks, const int32_t* dst_start, const int32_t* len, const int32_t* src_off,
                              const int32_t* extent, int64_t extent_max, int num_sms, cudaStream_t s);

// United-row de-duplication, stage 0: count, 1: per-executor prefix, 2: permute.
cudaError_t launch_dedup(int stage, const int32_t* topk_id, const float* topk_w, int T, int K, int tile, int m, int E,
                         const int32_t* exec_of, int32_t* tile_xcnt, int32_t* tile_xbase, int32_t* exec_off,
                         int32_t* mtile_off, int64_t* stats, int32_t* row_of, int32_t* row_tok, float* row_w,
                         cudaStream_t s);

cudaError_t launch_build_united(int dtype, const void* W, int m, int way, int64_t per_expert, void* U,
                                cudaStream_t s);

// ---- united-expert distillation (bo_distill.cu; Eq. 4)
cudaError_t launch_fill_offsets(int32_t* off, int n, int stride, cudaStream_t s);
int group_mean_blocks(int64_t N, int d, int num_sms);
int mse_grad_blocks(int64_t N, int64_t d);
cudaError_t launch_group_mean(const float* Yo, int m, int way, int64_t N, int d, float* Hbar, double* part,
                              double* floor_out, int num_sms, cudaStream_t s);
cudaError_t launch_swiglu_fwd(const void* P, const void* Q, void* Hs, void* HsT, int64_t G, int64_t N, int64_t f,
                              cudaStream_t s);
cudaError_t launch_mse_grad(const float* Y, const float* Hbar, void* dY, void* dYT, int64_t G, int64_t N, int64_t d,
                            double* part, const double* floor_in, int m, int way, double* loss_out, cudaStream_t s);
cudaError_t launch_swiglu_bwd(const void* dHs, const void* P, const void* Q, void* dPT, void* dQT, int64_t G,
                              int64_t N, int64_t f, cudaStream_t s);
cudaError_t launch_cast_master(const float* W, void* Wb, void* WbT, int64_t G, int64_t R, int64_t C, cudaStream_t s);
cudaError_t launch_widen(const void* Wb, float* W, int64_t n, int num_sms, cudaStream_t s);

}  // namespace bo
