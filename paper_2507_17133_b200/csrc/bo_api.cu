// bo_api.cu - the C ABI (include/brownout.h): validation, workspace carving,
// TMA descriptor encoding and the stream-ordered launch sequence of the
// brownout MoE-layer forward.  No device memory is allocated here.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cstdarg>
#include <mutex>
#include <string>

#include "../../include/brownout.h"
#include "bo_internal.h"
#include "bo_kernels.h"



namespace bo_impl {

thread_local std::string g_last_error;

bo_status fail(bo_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return s;
}

bo_status cuda_fail(cudaError_t e, const char* what) {
  return fail(BO_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}


size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

int elem_bytes(int32_t dtype) { return dtype == BO_BF16 ? 2 : 4; }

// ---- TMA descriptor encoding through the driver entry point (no -lcuda)
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  });
  return fn;
}

// 2-D K-major tile map over a row-major [rows, k] matrix: box [box_rows, 128 B], SWIZZLE_128B.
bo_status make_map(CUtensorMap* m, const void* base, int32_t dtype, uint64_t rows, uint64_t k, uint32_t box_rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return fail(BO_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int eb = elem_bytes(dtype);
  cuuint64_t dims[2] = {k, rows};
  cuuint64_t strides[1] = {k * static_cast<cuuint64_t>(eb)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / eb), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, dtype == BO_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(BO_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) rows=%llu k=%llu box_rows=%u", static_cast<int>(r),
                static_cast<unsigned long long>(rows), static_cast<unsigned long long>(k), box_rows);
  return BO_OK;
}

// Output box map for TMA bulk stores: [rows, cols] bf16 row-major, box 32 x 32, SWIZZLE_64B.
bo_status make_map_store32(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return fail(BO_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(BO_ERR_CUDA, "cuTensorMapEncodeTiled (store box) failed (%d)", static_cast<int>(r));
  return BO_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int router_bn(int m) {
  int bn = 16;
  while (bn < m) bn <<= 1;
  return bn;
}


int gemm2_bn(int d) { return d % 256 == 0 ? 256 : d % 128 == 0 ? 128 : 64; }
int gemm1_bn(int f) { return f % 128 == 0 ? 256 : 128; }   // gate + up columns

bo_status compute_layout(const bo_handle* h, int64_t T, bo_ws_layout* L, bool route_only) {
  const bo_config& c = h->cfg;
  const int64_t m = c.num_experts, K = c.top_k, d = c.hidden, f = c.ffn;
  const int64_t G = (m + c.way - 1) / c.way, Ns = c.num_shared, E = m + G + Ns;
  // upper bound over every token tile the route stage may pick (the decode router: 1 token per tile)
  const int64_t ntiles = T < 8 * h->num_sms ? T : (T + bo::kTileMin - 1) / bo::kTileMin;
  const int64_t Rk = T * K;          // routed (token, slot) pairs
  const int64_t R = Rk + Ns * T;     // expert rows incl. the shared experts' (every token)
  const int eb = elem_bytes(c.dtype);
  memset(L, 0, sizeof(*L));
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align256(off + (bytes ? bytes : 1));
    return o;
  };
  L->logits = take(sizeof(float) * T * m);
  L->topk_id = take(sizeof(int32_t) * Rk);
  L->topk_w = take(sizeof(float) * Rk);
  L->tile_cnt = take(sizeof(int32_t) * ntiles * m);
  L->tile_base = take(sizeof(int32_t) * ntiles * m);
  L->counts = take(sizeof(int32_t) * m);
  L->exec_of_expert = take(sizeof(int32_t) * m);
  L->expert_row_off = take(sizeof(int32_t) * m);
  L->exec_off = take(sizeof(int32_t) * (E + 1));
  L->mtile_off = take(sizeof(int32_t) * (E + 1));
  L->stats = take(sizeof(bo_plan_stats));
  L->row_of = take(sizeof(int32_t) * R);
  L->row_tok = take(sizeof(int32_t) * R);
  L->row_w = take(sizeof(float) * R);
  const int64_t Rf = route_only ? 0 : R;   // route-only (expert parallelism): no FFN buffers
  L->xp = take(static_cast<size_t>(eb) * Rf * d);
  L->h = take(static_cast<size_t>(eb) * Rf * f);
  L->yp = take(static_cast<size_t>(eb) * Rf * d);
  L->partial = take(Rf > 0 && Rf <= kSplitRows ? sizeof(float) * kSplitMax * Rf * d : 0);
  L->tile_xcnt = take(c.dedup_united && !route_only ? sizeof(int32_t) * ntiles * (m + G) : 0);
  L->tile_xbase = take(c.dedup_united && !route_only ? sizeof(int32_t) * ntiles * (m + G) : 0);
  L->ksplit = take(sizeof(int32_t));
  L->comb_cnt = take(route_only ? 0 : sizeof(int32_t) * T * (d / gemm2_bn(static_cast<int>(d))));
  // GEMM2's last-wave split (CTA pairs, prefill-sized): one fp32 accumulator and one flag per SM
  const bool ts = Rf >= kTailSplitRows;
  L->sk_part = take(ts ? sizeof(float) * h->num_sms * bo::kSkPartElems : 0);
  L->sk_flag = take(ts ? sizeof(int32_t) * h->num_sms : 0);
  L->total_bytes = off;
  L->T = T;
  L->ntiles = ntiles;
  L->num_executors = E;
  return BO_OK;
}



// Steps a1-a3: router logits (Eq. 8), top-K softmax (Eq. 7), per-tile expert
// histogram; then the local counts / per-tile prefix (and Alg. 1 on the local
// counts) via the plan kernel.  Returns the token tile used.
bo_status route_stage(bo_handle* h, const void* x, int64_t T, const void* Wr, const float* logits_in, void* ws,
                      const bo_ws_layout& L, cudaStream_t s, Prof& prof, int& launches, int& tile, int32_t* ep_row) {
  const bo_config& c = h->cfg;
  const int dt = c.dtype == BO_BF16 ? 0 : 1;
  const int m = c.num_experts, K = c.top_k, d = c.hidden;
  float* logits = at<float>(ws, L.logits);
  int32_t* topk_id = at<int32_t>(ws, L.topk_id);
  float* topk_w = at<float>(ws, L.topk_w);
  int32_t* tile_cnt = at<int32_t>(ws, L.tile_cnt);
  bo_status st;
  if (logits_in) {
    tile = bo::kTileSmall;
    prof.mark(launches, "router_topk");
    BO_CUDA(bo::launch_topk_hist(logits_in, static_cast<int>(T), m, K, tile, topk_id, topk_w, tile_cnt, s), "topk");
    ++launches;
  } else if (bo::router_small_ok(dt, m, d)) {
    // m <= 32: CUDA-core router (HBM-bound); decode-sized batches split each token over several warps
    const int tpc = h->opt.router_split ? bo::router_split_tpc(static_cast<int>(T), h->num_sms) : 0;
    prof.mark(launches, "router_topk");
    if (h->opt.router_mma && bo::router_mma_ok(dt, m, d, static_cast<int>(T), h->num_sms)) {
      tile = 16;
      BO_CUDA(bo::launch_router_mma(x, Wr, static_cast<int>(T), d, m, K, logits, topk_id, topk_w, tile_cnt, s),
              "router");
    } else if (tpc > 0) {
      tile = tpc;
      BO_CUDA(bo::launch_router_split(dt, x, Wr, static_cast<int>(T), d, m, K, tpc, logits, topk_id, topk_w,
                                      tile_cnt, s),
              "router");
    } else {
      tile = bo::router_small_tile(static_cast<int>(T), h->num_sms);
      BO_CUDA(bo::launch_router_small(dt, x, Wr, static_cast<int>(T), d, m, K, tile, logits, topk_id, topk_w,
                                      tile_cnt, s),
              "router");
    }
    ++launches;
  } else {
    tile = bo::kTileTok;     // tcgen05 router, top-K fused into the epilogue
    CUtensorMap mA, mB;
    const int bn = router_bn(m);
    if ((st = make_map(&mA, x, c.dtype, T, d, bo::kBM)) != BO_OK) return st;
    if ((st = make_map(&mB, Wr, c.dtype, m, d, bn)) != BO_OK) return st;
    bo::GemmParams p{};
    p.Kdim = d;
    p.n_tiles = 1;
    p.Kdim_u = d;
    p.n_tiles_u = 1;
    p.b_rows_u = 0;
    p.ldo = m;
    p.n_valid = m;
    p.m_orig = 1;
    p.b_rows_per_exec = 0;
    p.num_exec = 1;
    p.single_rows = static_cast<int>(T);
    p.out = logits;
    p.topk_k = K;
    p.topk_id = topk_id;
    p.topk_w = topk_w;
    p.tile_cnt = tile_cnt;
    const int work = static_cast<int>((T + bo::kBM - 1) / bo::kBM);
    const int grid = work < h->num_sms ? work : h->num_sms;
    prof.mark(launches, "router_topk");
    bo::BMaps mbs;
    for (int i = 0; i < 12; ++i) mbs.m[i] = mB;
    BO_CUDA(bo::launch_grouped_gemm(dt, bo::EPI_ROUTER, bn, mA, mbs, p, grid, s, h->opt.pdl), "router gemm");
    ++launches;
  }
  const int ntiles = static_cast<int>((T + tile - 1) / tile);
  // Alg. 1 over this batch (snapshot of the knob at enqueue time); also yields
  // cnt_i and the per-tile prefix the permutation needs.
  prof.mark(launches, "plan");
  bo::PlanExt ext;
  if (ep_row) {   // expert parallelism: this rank's counts row [m] + knob tail [4] (the all-gather input)
    ext.row_tail = ep_row + m;
    ext.row_T = static_cast<int>(T);
  }
  BO_CUDA(bo::launch_plan(tile_cnt, ntiles, m, c.way, h->ratio, h->mode, at<int32_t>(ws, L.tile_base),
                          ep_row ? ep_row : at<int32_t>(ws, L.counts), at<int32_t>(ws, L.exec_of_expert),
                          at<int32_t>(ws, L.expert_row_off), at<int32_t>(ws, L.exec_off),
                          at<int32_t>(ws, L.mtile_off), at<int64_t>(ws, L.stats), s, c.num_shared,
                          static_cast<int>(T), ext),
          "plan");
  ++launches;
  h->route_T = T;
  h->route_tile = tile;
  return BO_OK;
}

// Steps a6-a7 over rows already grouped by executor: GEMM1 + SwiGLU, GEMM2 x
// row gate weight.  Executors [0, n_orig) read Wg/Wu/Wd stacks of width f,
// executors [n_orig, n_orig + n_united) read UWg/UWu/UWd stacks of width f_u
// (f_u < f: expert-parallel f-slices of united experts).

// L2 policy of the weight (B) tile loads: decode-sized steps stream every weight tile
// once per concurrent m-tile pair, so evict_first keeps the re-read activations in L2.
int b_policy_for(const bo_handle* h, int64_t R) {
  if (h->opt.b_policy >= 0) return h->opt.b_policy;
  return R <= kSplitRows ? 1 : 0;
}


void set_comb(bo::GemmParams& p, const CombFuse* cf, int d, int nt2) {
  if (!cf) return;
  p.comb_cnt = cf->cnt;
  p.row_of = cf->row_of;
  p.comb_KR = cf->KR;
  p.comb_T = static_cast<int>(cf->T);
  p.comb_nt = nt2;
  p.comb_d = d;
  p.add_residual = cf->add_residual;
  p.comb_x = cf->x;
  p.comb_y = cf->y;
}

// Steps a6-a7 over rows already grouped by executor: GEMM1 + SwiGLU, GEMM2 x
// row gate weight.  Executors are laid out originals, united, shared (Eq. 5
// second term: every token, weight 1); the united class may have its own width.
bo_status ffn_stage(bo_handle* h, const void* X, int64_t R, const float* row_w, const int32_t* exec_off,
                    const int32_t* mtile_off, const FfnClass& orig, const FfnClass& uni, const FfnClass& shr,
                    void* Hbuf, void* Y, cudaStream_t s, Prof& prof, int& launches, float* partial,
                    int* ks_dev, const CombFuse* comb, const int32_t* comb_row_tok, bool force_pair2,
                    float* sk_part, int* sk_flag) {
  // partial != nullptr: GEMM2 runs split-K into fp32 partials [<=8, R, d] (the
  // caller combines them with launch_combine_partials); Y is then unused.
  const bo_config& c = h->cfg;
  const EngineOptions& o = h->opt;
  const int dt = c.dtype == BO_BF16 ? 0 : 1;
  const int d = c.hidden, f = c.ffn;
  const int f_u = uni.n > 0 ? uni.f : f;
  const int n_exec = orig.n + uni.n + shr.n;
  bo_status st;
  if (R == 0 || n_exec == 0) return BO_OK;
  // Any present class's pointers stand in for an empty class (its map is never used).
  const FfnClass& any = orig.n ? orig : (uni.n ? uni : shr);
  auto ptr = [&](const FfnClass& k, int which) {
    const FfnClass& q = k.Wg ? k : any;
    return which == 0 ? q.Wg : (which == 1 ? q.Wu : q.Wd);
  };
  auto rows_of = [&](const FfnClass& k, int width) {
    const FfnClass& q = k.Wg ? k : any;
    return static_cast<uint64_t>(q.stack > 0 ? q.stack : 1) * width;
  };
  const FfnClass* cls[3] = {&orig, &uni, &shr};
  {
    // Widest tile everywhere (narrower decode tiles, tried to cut the wave quantisation
    // of few-row steps, measured slower: r01 profiles); the device may still pick the
    // alternative width below.
    int bn = 256;                                                   // gate + up columns per tile
    while (bn > 64 && (f % (bn / 2) || f_u % (bn / 2))) bn >>= 1;
    CUtensorMap mA;
    bo::BMaps mb;
    if ((st = make_map(&mA, X, c.dtype, R, d, bo::kBM)) != BO_OK) return st;
    for (int k = 0; k < 3; ++k) {
      const int width = k == 1 ? f_u : f;
      if ((st = make_map(&mb.m[2 * k], ptr(*cls[k], 0), c.dtype, rows_of(*cls[k], width), d, bn / 2)) != BO_OK)
        return st;
      if ((st = make_map(&mb.m[2 * k + 1], ptr(*cls[k], 1), c.dtype, rows_of(*cls[k], width), d, bn / 2)) != BO_OK)
        return st;
    }
    bo::GemmParams p{};
    // 256 x 256 tiles on CTA pairs when rows are plentiful (prefill); few-row
    // (decode) steps keep 128-row tiles so that more tiles share the SMs.
    const bool pair = o.cta_pairs && dt == 0 && bn == 256 && R >= o.pair_rows1;
    // swapped-operand tail tiles (pairs): maps [6..11] = 64-row gate / up boxes,
    // [12..14] = Xp in 16 / 32 / 64-row boxes
    const bool swap = pair && o.swap_tail;
    if (swap) {
      for (int k = 0; k < 3; ++k) {
        const int width = k == 1 ? f_u : f;
        if ((st = make_map(&mb.m[6 + 2 * k], ptr(*cls[k], 0), c.dtype, rows_of(*cls[k], width), d, 64)) != BO_OK)
          return st;
        if ((st = make_map(&mb.m[7 + 2 * k], ptr(*cls[k], 1), c.dtype, rows_of(*cls[k], width), d, 64)) != BO_OK)
          return st;
      }
      for (int i = 0; i < 3; ++i)
        if ((st = make_map(&mb.m[12 + i], X, c.dtype, R, d, 16u << i)) != BO_OK) return st;
      p.swap_tail = 1;
    }
    // alternative tile width for the device-side wave choice: the widest gate/up half
    // below bn/2 (multiple of 16, >= 64) that divides both widths
    int bh_alt = 0;
    if (o.tile_alt && !swap)
      for (int bh = bn / 2 - 16; bh >= 64 && !bh_alt; bh -= 16)
        if (f % bh == 0 && f_u % bh == 0) bh_alt = bh;
    if (bh_alt) {
      for (int k = 0; k < 3; ++k) {
        const int width = k == 1 ? f_u : f;
        if ((st = make_map(&mb.m[6 + 2 * k], ptr(*cls[k], 0), c.dtype, rows_of(*cls[k], width), d, bh_alt)) != BO_OK)
          return st;
        if ((st = make_map(&mb.m[7 + 2 * k], ptr(*cls[k], 1), c.dtype, rows_of(*cls[k], width), d, bh_alt)) != BO_OK)
          return st;
      }
      p.bh_alt = bh_alt;
      p.nt_alt = f / bh_alt;
      p.nt_alt_u = f_u / bh_alt;
    }
    p.Kdim = d;
    p.n_tiles = f / (bn / 2);
    p.Kdim_u = d;
    p.n_tiles_u = f_u / (bn / 2);
    p.b_rows_u = f_u;
    p.ldo = f;
    p.n_valid = f;
    p.m_orig = orig.n;
    p.m_united = uni.n;
    p.store_hint = o.store_hint && R > kSplitRows;   // decode: H / Yp (a few MB) stay in L2 for the next kernel
    p.b_policy = b_policy_for(h, R);
    p.b_rows_per_exec = f;
    p.num_exec = n_exec;
    p.single_rows = -1;
    p.exec_off = exec_off;
    p.mtile_off = mtile_off;
    p.out = Hbuf;
    p.rows_total = static_cast<int>(R);
    set_comb(p, comb, d, d / gemm2_bn(d));   // GEMM1's prologue zeroes GEMM2's arrival counters
    const int tile_m = pair ? 2 * bo::kBM : bo::kBM;
    const int64_t max_work = ((R + tile_m - 1) / tile_m + n_exec) * p.n_tiles;
    const int units = pair ? h->num_sms / 2 : h->num_sms;
    const int grid = static_cast<int>(max_work < units ? max_work : units) * (pair ? 2 : 1);
    prof.mark(launches, "gemm1_swiglu");
    BO_CUDA(bo::launch_grouped_gemm(dt, pair ? bo::EPI_SWIGLU_PAIR : bo::EPI_SWIGLU, bn, mA, mb, p, grid, s, o.pdl),
            "gemm1");
    ++launches;
  }
  {
    const int bn = gemm2_bn(d);
    const bool pair = o.cta_pairs && dt == 0 && bn == 256 && (R >= o.pair_rows2 || force_pair2);   // each CTA of a pair stages BN/2 of B
    const uint32_t box_b = pair ? bn / 2 : bn;
    CUtensorMap mA;
    bo::BMaps mb;
    if ((st = make_map(&mA, Hbuf, c.dtype, R, f, bo::kBM)) != BO_OK) return st;
    for (int k = 0; k < 3; ++k) {
      const FfnClass& q = cls[k]->Wg ? *cls[k] : any;
      const int kdim = k == 1 ? f_u : f;
      const uint64_t rows = static_cast<uint64_t>(q.stack > 0 ? q.stack : 1) * d;
      if ((st = make_map(&mb.m[2 * k], ptr(*cls[k], 2), c.dtype, rows, kdim, box_b)) != BO_OK) return st;
      mb.m[2 * k + 1] = mb.m[2 * k];
    }
    bo::GemmParams p{};
    p.Kdim = f;
    p.n_tiles = d / bn;
    p.Kdim_u = f_u;
    p.n_tiles_u = p.n_tiles;
    p.b_rows_u = d;
    p.ldo = d;
    p.n_valid = d;
    p.m_orig = orig.n;
    p.m_united = uni.n;
    p.store_hint = o.store_hint && R > kSplitRows;   // decode: H / Yp (a few MB) stay in L2 for the next kernel
    p.b_policy = b_policy_for(h, R);
    p.b_rows_per_exec = d;
    p.num_exec = n_exec;
    p.single_rows = -1;
    p.exec_off = exec_off;
    p.mtile_off = mtile_off;
    p.out = Y;
    if (o.tma_store && dt == 0 && !partial) {
      if ((st = make_map_store32(&mb.m[6], Y, static_cast<uint64_t>(R), static_cast<uint64_t>(d))) != BO_OK) return st;
      p.tma_store = 1;
    }
    p.row_w = row_w;
    p.rows_total = static_cast<int>(R);
    if (pair && o.tail_split && sk_part && sk_flag && !partial) {   // the kernel decides on the device
      p.tail_split = 1;
      p.sk_part = sk_part;
      p.sk_flag = sk_flag;
      BO_CUDA(cudaMemsetAsync(sk_flag, 0, sizeof(int) * h->num_sms, s), "tail-split flags");
    }
    if (comb) {
      set_comb(p, comb, d, d / bn);
      p.row_tok = comb_row_tok;
      p.store_hint = 0;   // the completing warp re-reads the token's other Yp rows: keep them in L2
    }
    if (partial) {
      p.ksplit_max = kSplitMax;
      p.partial = partial;
      p.ks_out = ks_dev;
    }
    const int tile_m = pair ? 2 * bo::kBM : bo::kBM;
    const int64_t max_work = ((R + tile_m - 1) / tile_m + n_exec) * p.n_tiles;
    const int units = pair ? h->num_sms / 2 : h->num_sms;
    const int grid = static_cast<int>(max_work < units ? max_work : units) * (pair ? 2 : 1);
    prof.mark(launches, comb ? "gemm2_weighted_combine" : "gemm2_weighted");
    BO_CUDA(bo::launch_grouped_gemm(dt, pair ? bo::EPI_WEIGHTED_PAIR : bo::EPI_WEIGHTED, bn, mA, mb, p, grid, s,
                                    o.pdl),
            "gemm2");
    ++launches;
  }
  return BO_OK;
}

// Engine options by bo_engine_option id (include/brownout.h): field, environment name,
// allowed range.
struct OptionSpec {
  int32_t EngineOptions::*field;
  const char* env;
  int32_t lo, hi;
};
const OptionSpec kOptions[BO_OPT_COUNT] = {
    {&EngineOptions::cta_pairs, "BO_CTA_PAIRS", 0, 1},
    {&EngineOptions::pair_rows1, "BO_PAIR_ROWS1", 1, 1 << 30},
    {&EngineOptions::pair_rows2, "BO_PAIR_ROWS2", 1, 1 << 30},
    {&EngineOptions::tile_alt, "BO_TILE_ALT", 0, 1},
    {&EngineOptions::swap_tail, "BO_SWAP_TAIL", 0, 1},
    {&EngineOptions::decode_pair2, "BO_DECODE_PAIR2", 0, 1},
    {&EngineOptions::gemm2_splitk, "BO_GEMM2_SPLITK", 0, 1},
    {&EngineOptions::fused_combine, "BO_FUSED_COMBINE", 0, 2},
    {&EngineOptions::tma_store, "BO_TMA_STORE", 0, 1},
    {&EngineOptions::store_hint, "BO_STORE_HINT", 0, 1},
    {&EngineOptions::b_policy, "BO_B_POLICY", -1, 1},
    {&EngineOptions::router_mma, "BO_ROUTER_MMA", 0, 1},
    {&EngineOptions::router_split, "BO_ROUTER_SPLIT", 0, 1},
    {&EngineOptions::pdl, "BO_PDL", 0, 1},
    {&EngineOptions::route_fused, "BO_ROUTE_FUSED", 0, 1},
    {&EngineOptions::tail_split, "BO_TAIL_SPLIT", 0, 1},
};

void options_from_env(EngineOptions* o) {
  for (const OptionSpec& sp : kOptions) {
    const char* v = getenv(sp.env);
    if (!v || !*v) continue;
    char* end = nullptr;
    const long x = strtol(v, &end, 10);
    if (end && *end == 0 && x >= sp.lo && x <= sp.hi) o->*sp.field = static_cast<int32_t>(x);
  }
}

bo_status check_ws(const bo_handle* h, int64_t T, void* ws, size_t ws_bytes, bo_ws_layout* L) {
  compute_layout(h, T, L);
  if (!ws || ws_bytes < L->total_bytes)
    return fail(BO_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, L->total_bytes);
  if (!aligned16(ws)) return fail(BO_ERR_SHAPE, "workspace must be 16-byte aligned");
  return BO_OK;
}

const char* const kDedupNames[3] = {"dedup_count", "dedup_plan", "dedup_permute"};

bo_status forward_impl(bo_handle* h, const void* x, int64_t T, const void* Wr, const void* Wg, const void* Wu,
                       const void* Wd, const void* UWg, const void* UWu, const void* UWd, void* y, void* ws,
                       size_t ws_bytes, const float* logits_in, void* stream) {
  if (!h) return fail(BO_ERR_INVALID_ARG, "null handle");
  h->last_launches = 0;
  h->last_kernels.clear();
  const bo_config& c = h->cfg;
  if (T < 0 || T > c.max_tokens) return fail(BO_ERR_INVALID_ARG, "T=%lld outside [0, max_tokens=%lld]",
                                             static_cast<long long>(T), static_cast<long long>(c.max_tokens));
  if (T == 0) return BO_OK;
  if (!x || !Wg || !Wu || !Wd || !y || (!Wr && !logits_in))
    return fail(BO_ERR_INVALID_ARG, "null tensor pointer");
  const bool may_use_united = h->mode == BO_PARTIAL && h->ratio > 0.0;
  if (may_use_united && (!UWg || !UWu || !UWd))
    return fail(BO_ERR_INVALID_ARG, "united weights are required when ratio > 0 in partial mode");
  const bool have_united = UWg != nullptr;
  if (!have_united) { UWg = Wg; UWu = Wu; UWd = Wd; }   // never selected by the plan (ratio 0 or full mode)
  const void* ptrs[] = {x, Wr ? Wr : x, Wg, Wu, Wd, UWg, UWu, UWd, y};
  for (const void* p : ptrs)
    if (!aligned16(p)) return fail(BO_ERR_SHAPE, "tensor pointers must be 16-byte aligned");
  bo_ws_layout L;
  bo_status st;
  if ((st = check_ws(h, T, ws, ws_bytes, &L)) != BO_OK) return st;

  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int dt = c.dtype == BO_BF16 ? 0 : 1;
  const int m = c.num_experts, K = c.top_k, d = c.hidden, f = c.ffn;
  const int G = (m + c.way - 1) / c.way, E = m + G;
  const int Ns = c.num_shared;
  const int KR = K + Ns;               // row_of slots per token: K routed, then the N_s shared experts
  const int64_t R = T * K;
  const int64_t Rt = R + static_cast<int64_t>(Ns) * T;
  if (Ns > 0 && (!h->SWg || !h->SWu || !h->SWd))
    return fail(BO_ERR_INVALID_ARG, "num_shared=%d but bo_set_shared_experts was not called", Ns);
  int launches = 0;
  Prof prof(h, s, 10);
  int tile = 0;
  int32_t* row_of = at<int32_t>(ws, L.row_of);
  float* row_w = at<float>(ws, L.row_w);
  // Small batches: the permute CTAs also copy the rows (one launch less).  Large
  // batches: a separate grid-wide gather (the permute has too few CTAs to move
  // R*d*2 bytes at HBM speed; measured r01).
  const bool gather_in_permute = Rt <= kSplitRows * 2 && !c.dedup_united;
  // Decode-sized steps on the split-warp router: a1-a5 in one cooperative launch
  const int tpc = h->opt.router_split && bo::router_split_tpc(static_cast<int>(T), h->num_sms) > 0
                      ? bo::route_fused_tpc(static_cast<int>(T), h->num_sms) : 0;
  const bool route_fused = h->opt.route_fused && !logits_in && !c.dedup_united && Wr != nullptr &&
                           bo::router_small_ok(dt, m, d) && tpc > 0 &&
                           !(h->opt.router_mma && bo::router_mma_ok(dt, m, d, static_cast<int>(T), h->num_sms)) &&
                           bo::route_fused_ok(dt, m, c.way, static_cast<int>(T), tpc, Ns, h->num_sms);
  if (route_fused) {
    tile = tpc;
    prof.mark(launches, "route_fused");
    BO_CUDA(bo::launch_route_fused(dt, x, Wr, static_cast<int>(T), d, m, K, tpc, at<float>(ws, L.logits),
                                   at<int32_t>(ws, L.topk_id), at<float>(ws, L.topk_w), at<int32_t>(ws, L.tile_cnt),
                                   c.way, h->ratio, h->mode, at<int32_t>(ws, L.counts),
                                   at<int32_t>(ws, L.exec_of_expert), at<int32_t>(ws, L.expert_row_off),
                                   at<int32_t>(ws, L.exec_off), at<int32_t>(ws, L.mtile_off),
                                   at<int64_t>(ws, L.stats), Ns, row_of, at<int32_t>(ws, L.row_tok), row_w,
                                   gather_in_permute ? at<char>(ws, L.xp) : nullptr, s),
            "route_fused");
    ++launches;
    h->route_T = T;
    h->route_tile = tile;
  } else {
    // a1-a4: router, top-K, histogram, Alg. 1 plan
    if ((st = route_stage(h, x, T, Wr, logits_in, ws, L, s, prof, launches, tile)) != BO_OK) return st;
  }
  // a5: permutation (rows in executor / expert / token order) and gather of Xp
  if (route_fused) {
  } else if (c.dedup_united) {
    // f3: one row per (token, united executor); Alg. 1 above is unchanged
    for (int stage = 0; stage < 3; ++stage) {
      prof.mark(launches, kDedupNames[stage]);
      BO_CUDA(bo::launch_dedup(stage, at<int32_t>(ws, L.topk_id), at<float>(ws, L.topk_w), static_cast<int>(T), K,
                               tile, m, E, at<int32_t>(ws, L.exec_of_expert), at<int32_t>(ws, L.tile_xcnt),
                               at<int32_t>(ws, L.tile_xbase), at<int32_t>(ws, L.exec_off),
                               at<int32_t>(ws, L.mtile_off), at<int64_t>(ws, L.stats), row_of,
                               at<int32_t>(ws, L.row_tok), row_w, s),
              "dedup");
      ++launches;
    }
  } else {
    prof.mark(launches, gather_in_permute ? "permute_gather" : "permute");
    BO_CUDA(bo::launch_permute(at<int32_t>(ws, L.topk_id), at<float>(ws, L.topk_w), static_cast<int>(T), K, m, tile,
                               at<int32_t>(ws, L.tile_base), at<int32_t>(ws, L.expert_row_off), 1, row_of,
                               at<int32_t>(ws, L.row_tok), row_w, s, dt, x,
                               gather_in_permute ? at<char>(ws, L.xp) : nullptr, d, Ns,
                               at<int32_t>(ws, L.exec_off) + E),
            "permute");
    ++launches;
  }
  if (!gather_in_permute) {
    prof.mark(launches, "gather");
    BO_CUDA(bo::launch_gather(dt, x, static_cast<int>(T), d, KR, row_of, at<char>(ws, L.xp), h->num_sms, s), "gather");
    ++launches;
  }
  // a6-a7: grouped SwiGLU FFN over the m original + G united (+ N_s shared) executors
  // on the materialised Xp (concat_tokens).
  void* yp = at<char>(ws, L.yp);
  const int32_t* row_tok = at<int32_t>(ws, L.row_tok);
  // Decode-sized steps whose executors hold >= 256 rows each (brownout ratio near 1: the
  // G united experts take almost every row; estimate (1 - ratio) m + ratio G executors):
  // GEMM2 on CTA pairs (one 256-row tile per executor instead of two 128-row tiles reading
  // the same weights) with split-K partials to fill the SMs.  C3 ratio 1: GEMM2
  // 0.101 -> 0.071 ms (profiles/r01_ab_decode_pairs_splitk.json); a loss at ratios 0 / 0.5.
  const EngineOptions& o = h->opt;
  const double est_exec = (1.0 - h->ratio) * m + h->ratio * G;
  const bool decode_pair2 = o.decode_pair2 && o.cta_pairs && dt == 0 && Rt <= kSplitRows &&
                            h->mode == BO_PARTIAL && Ns == 0 &&
                            static_cast<double>(Rt) >= 256.0 * (est_exec < 1.0 ? 1.0 : est_exec);
  const bool split = (o.gemm2_splitk || decode_pair2) && Rt <= kSplitRows;
  // a8 fused into GEMM2's epilogue unless split-K partials need their own combine
  // Auto: fused only where it measured faster (interleaved A/B, profiles/r01_ab_fused_combine.json):
  // prefill-sized steps with <= 2 rows per token (C2: GEMM2 + combine -5 %); with K = 8 (C4) the
  // completing warps' memory round trips (fence, count, 8 row loads) outrun GEMM2's short
  // per-tile mainloop, and decode steps (< 1 wave of GEMM2 tiles) expose them at the end.
  const bool fuse_comb = !split && KR <= 16 &&   // 16 = kCombSlots (bo_gemm.cu)
                         (o.fused_combine == 1 || (o.fused_combine == 2 && KR <= 2 && Rt >= 2048));
  CombFuse cf;
  cf.cnt = at<int32_t>(ws, L.comb_cnt);
  cf.row_of = row_of;
  cf.KR = KR;
  cf.T = T;
  cf.x = x;
  cf.y = y;
  cf.add_residual = c.add_residual;
  const CombFuse* cfp = fuse_comb ? &cf : nullptr;
  FfnClass orig, uni, shr;
  orig.Wg = Wg; orig.Wu = Wu; orig.Wd = Wd; orig.n = m; orig.f = f; orig.stack = m;
  uni.Wg = UWg; uni.Wu = UWu; uni.Wd = UWd; uni.n = G; uni.f = f; uni.stack = have_united ? G : m;
  if (Ns > 0) { shr.Wg = h->SWg; shr.Wu = h->SWu; shr.Wd = h->SWd; shr.n = Ns; shr.f = f; shr.stack = Ns; }
  void* xp = at<char>(ws, L.xp);   // filled by the permute (small batches) or the gather kernel
  if ((st = ffn_stage(h, xp, Rt, row_w, at<int32_t>(ws, L.exec_off), at<int32_t>(ws, L.mtile_off), orig, uni, shr,
                      at<char>(ws, L.h), yp, s, prof, launches, split ? at<float>(ws, L.partial) : nullptr,
                      split ? at<int>(ws, L.ksplit) : nullptr, cfp, row_tok, decode_pair2,
                      Rt >= kTailSplitRows ? at<float>(ws, L.sk_part) : nullptr,
                      Rt >= kTailSplitRows ? at<int>(ws, L.sk_flag) : nullptr)) != BO_OK)
    return st;
  // a8: combine (Eq. 5 sum over the token's K slots; split-K partials summed first)
  if (!fuse_comb) {
    prof.mark(launches, "combine");
    if (split)
      BO_CUDA(bo::launch_combine_partials(dt, at<float>(ws, L.partial), at<int>(ws, L.ksplit), Rt, x,
                                          static_cast<int>(T), d, KR, row_of, c.add_residual, y, h->num_sms, s),
              "combine");
    else
      BO_CUDA(bo::launch_combine(dt, yp, x, static_cast<int>(T), d, KR, row_of, c.add_residual, y, h->num_sms, s),
              "combine");
    ++launches;
  }
  prof.mark(launches);
  if (prof.err != cudaSuccess) return cuda_fail(prof.err, "profile event record");
  h->last_launches = launches;
  return BO_OK;
}

// ---------------------------------------------------------------- distillation
// One ungrouped-epilogue GEMM on the grouped engine: for executor x,
// out[rows of x] = alpha * A[rows of x (or 0.. when a_shared)] B_x^T, with
// B_x = rows [x * b_rows_per_exec, +n_cols) of B.  f32_mode 0: bf16 out;
// 1: fp32 out; 2: fp32 out += (the fused gradient-descent update).
struct PlainGemm {
  const void* A = nullptr;
  int64_t a_rows = 0;
  int Kdim = 0;
  int a_shared = 0;
  const void* B = nullptr;
  int64_t b_rows = 0;
  int b_rows_per_exec = 0;
  const int32_t* exec_off = nullptr;
  int num_exec = 0;
  int64_t rows_total = 0;
  int n_cols = 0;
  void* out = nullptr;
  void* out_bf16 = nullptr;   // f32_mode 2: also write the updated values rounded to bf16 here
  int ldo = 0;
  int f32_mode = 0;
  float alpha = 1.0f;
};

bo_status plain_gemm(bo_handle* h, const PlainGemm& g, cudaStream_t s, Prof& prof, int& launches) {
  if (g.rows_total == 0) return BO_OK;
  bo_status st;
  int bn = gemm2_bn(g.n_cols);
  const bool pair = h->opt.cta_pairs && bn == 256 && g.rows_total >= 2048;
  CUtensorMap mA, mB;
  if ((st = make_map(&mA, g.A, BO_BF16, g.a_rows, g.Kdim, bo::kBM)) != BO_OK) return st;
  if ((st = make_map(&mB, g.B, BO_BF16, g.b_rows, g.Kdim, pair ? bn / 2 : bn)) != BO_OK) return st;
  bo::BMaps mb;
  for (int i = 0; i < 6; ++i) mb.m[i] = mB;
  bo::GemmParams p{};
  p.Kdim = g.Kdim;
  p.n_tiles = g.n_cols / bn;
  p.Kdim_u = g.Kdim;
  p.n_tiles_u = p.n_tiles;
  p.b_rows_u = g.b_rows_per_exec;
  p.ldo = g.ldo;
  p.n_valid = g.n_cols;
  p.m_orig = g.num_exec;
  p.m_united = 0;
  p.b_rows_per_exec = g.b_rows_per_exec;
  p.num_exec = g.num_exec;
  p.single_rows = -1;
  p.exec_off = g.exec_off;
  p.rows_total = static_cast<int>(g.rows_total);
  p.a_shared = g.a_shared;
  p.alpha = g.alpha;
  p.f32_mode = g.f32_mode;
  if (g.f32_mode) {
    p.partial = static_cast<float*>(g.out);
    p.out = g.out_bf16;
  } else {
    p.out = g.out;
  }
  const int tile_m = pair ? 2 * bo::kBM : bo::kBM;
  const int64_t max_work = ((g.rows_total + tile_m - 1) / tile_m + g.num_exec) * p.n_tiles;
  const int units = pair ? h->num_sms / 2 : h->num_sms;
  const int grid = static_cast<int>(max_work < units ? max_work : units) * (pair ? 2 : 1);
  prof.mark(launches);
  BO_CUDA(bo::launch_grouped_gemm(0, pair ? bo::EPI_WEIGHTED_PAIR : bo::EPI_WEIGHTED, bn, mA, mb, p, grid, s,
                                  h->opt.pdl),
          "distill gemm");
  ++launches;
  return BO_OK;
}

void distill_layout(const bo_handle* h, int64_t N, bo_distill_layout* L) {
  const bo_config& c = h->cfg;
  const int64_t m = c.num_experts, d = c.hidden, f = c.ffn, G = (m + c.way - 1) / c.way;
  memset(L, 0, sizeof(*L));
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align256(off + (bytes ? bytes : 1));
    return o;
  };
  const int nb_mean = bo::group_mean_blocks(N, static_cast<int>(d), h->num_sms);
  const int64_t nb_mse = bo::mse_grad_blocks(N, d);
  L->hbar = take(4 * G * N * d);
  L->floor_ = take(8 * G);
  L->loss = take(8 * G);
  L->xt = take(2 * d * N);
  L->teach_h = take(2 * m * N * f);
  L->teach_y = take(4 * m * N * d);
  L->p = take(2 * G * N * f);
  L->q = take(2 * G * N * f);
  L->hs = take(2 * G * N * f);
  L->hst = take(2 * G * f * N);
  L->y = take(4 * G * N * d);
  L->dy = take(2 * G * N * d);
  L->dyt = take(2 * G * d * N);
  L->dhs = take(2 * G * N * f);
  L->dpt = take(2 * G * f * N);
  L->dqt = take(2 * G * f * N);
  L->uwdt = take(2 * G * f * d);
  L->part = take(8 * G * (nb_mean > nb_mse ? nb_mean : nb_mse));
  L->off_tok = take(4 * (G + 1));
  L->off_teach = take(4 * (m + 1));
  L->off_f = take(4 * (G + 1));
  L->off_d = take(4 * (G + 1));
  L->total_bytes = off;
  L->N = N;
}

bo_status distill_check(const bo_handle* h, int64_t N, void* ws, size_t ws_bytes, bo_distill_layout* L) {
  if (!h) return fail(BO_ERR_INVALID_ARG, "null handle");
  if (h->cfg.dtype != BO_BF16) return fail(BO_ERR_UNSUPPORTED, "distillation is built for bf16 handles");
  if (N <= 0 || N % 64 || N > (int64_t(1) << 24))
    return fail(BO_ERR_SHAPE, "N=%lld must be a positive multiple of 64", static_cast<long long>(N));
  const int64_t rows = N * h->cfg.num_experts;
  if (rows > (int64_t(1) << 31) - 1) return fail(BO_ERR_SHAPE, "m * N too large");
  distill_layout(h, N, L);
  if (!ws || ws_bytes < L->total_bytes)
    return fail(BO_ERR_WORKSPACE, "distill workspace %zu bytes < required %zu", ws_bytes, L->total_bytes);
  if (!aligned16(ws)) return fail(BO_ERR_SHAPE, "workspace must be 16-byte aligned");
  return BO_OK;
}

}  // namespace bo_impl

using namespace bo_impl;

extern "C" {

bo_status bo_distill_workspace_layout(const bo_handle* h, int64_t N, bo_distill_layout* out) {
  if (!h || !out) return fail(BO_ERR_INVALID_ARG, "null argument");
  if (N < 0) return fail(BO_ERR_INVALID_ARG, "N < 0");
  distill_layout(h, N, out);
  return BO_OK;
}

bo_status bo_distill_prepare(bo_handle* h, const void* X, int64_t N, const void* Wg, const void* Wu, const void* Wd,
                             void* ws, size_t ws_bytes, void* stream) {
  bo_distill_layout L;
  bo_status st;
  if ((st = distill_check(h, N, ws, ws_bytes, &L)) != BO_OK) return st;
  if (!X || !Wg || !Wu || !Wd) return fail(BO_ERR_INVALID_ARG, "null tensor pointer");
  const void* ptrs[] = {X, Wg, Wu, Wd};
  for (const void* q : ptrs)
    if (!aligned16(q)) return fail(BO_ERR_SHAPE, "tensor pointers must be 16-byte aligned");
  const bo_config& c = h->cfg;
  const int m = c.num_experts, d = c.hidden, f = c.ffn, G = (m + c.way - 1) / c.way;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Prof prof(h, s, 1 << 30);
  int launches = 0;
  int32_t* off_teach = at<int32_t>(ws, L.off_teach);
  BO_CUDA(bo::launch_fill_offsets(off_teach, m, static_cast<int>(N), s), "offsets");
  BO_CUDA(bo::launch_fill_offsets(at<int32_t>(ws, L.off_tok), G, static_cast<int>(N), s), "offsets");
  BO_CUDA(bo::launch_fill_offsets(at<int32_t>(ws, L.off_f), G, f, s), "offsets");
  BO_CUDA(bo::launch_fill_offsets(at<int32_t>(ws, L.off_d), G, d, s), "offsets");
  // teacher: every original expert on every token, H_o = Wd (silu(Wg x) * Wu x)
  {
    // GEMM1 + SwiGLU with the shared token matrix as A
    const int64_t R = N * m;
    int bn = 256;
    while (bn > 64 && f % (bn / 2)) bn >>= 1;
    const bool pair = h->opt.cta_pairs && bn == 256 && R >= 2048;
    CUtensorMap mA;
    bo::BMaps mb;
    if ((st = make_map(&mA, X, BO_BF16, N, d, bo::kBM)) != BO_OK) return st;
    if ((st = make_map(&mb.m[0], Wg, BO_BF16, static_cast<uint64_t>(m) * f, d, bn / 2)) != BO_OK) return st;
    if ((st = make_map(&mb.m[1], Wu, BO_BF16, static_cast<uint64_t>(m) * f, d, bn / 2)) != BO_OK) return st;
    for (int i = 2; i < 6; ++i) mb.m[i] = mb.m[i & 1];
    bo::GemmParams p{};
    p.Kdim = d;
    p.n_tiles = f / (bn / 2);
    p.Kdim_u = d;
    p.n_tiles_u = p.n_tiles;
    p.b_rows_u = f;
    p.ldo = f;
    p.n_valid = f;
    p.m_orig = m;
    p.b_rows_per_exec = f;
    p.num_exec = m;
    p.single_rows = -1;
    p.exec_off = off_teach;
    p.out = at<char>(ws, L.teach_h);
    p.rows_total = static_cast<int>(R);
    p.a_shared = 1;
    const int tile_m = pair ? 2 * bo::kBM : bo::kBM;
    const int64_t max_work = ((R + tile_m - 1) / tile_m + m) * p.n_tiles;
    const int units = pair ? h->num_sms / 2 : h->num_sms;
    const int grid = static_cast<int>(max_work < units ? max_work : units) * (pair ? 2 : 1);
    BO_CUDA(bo::launch_grouped_gemm(0, pair ? bo::EPI_SWIGLU_PAIR : bo::EPI_SWIGLU, bn, mA, mb, p, grid, s,
                                    h->opt.pdl),
            "teacher gemm1");
  }
  PlainGemm g2;   // H_o = H Wd^T in fp32
  g2.A = at<char>(ws, L.teach_h);
  g2.a_rows = N * m;
  g2.Kdim = f;
  g2.B = Wd;
  g2.b_rows = static_cast<int64_t>(m) * d;
  g2.b_rows_per_exec = d;
  g2.exec_off = off_teach;
  g2.num_exec = m;
  g2.rows_total = N * m;
  g2.n_cols = d;
  g2.out = at<char>(ws, L.teach_y);
  g2.ldo = d;
  g2.f32_mode = 1;
  if ((st = plain_gemm(h, g2, s, prof, launches)) != BO_OK) return st;
  BO_CUDA(bo::launch_group_mean(at<float>(ws, L.teach_y), m, c.way, N, d, at<float>(ws, L.hbar),
                                at<double>(ws, L.part), at<double>(ws, L.floor_), h->num_sms, s),
          "group mean");
  // X^T for the weight gradients (a cast of bf16 through fp32 is exact)
  BO_CUDA(bo::launch_widen(X, at<float>(ws, L.teach_y), N * d, h->num_sms, s), "widen X");
  BO_CUDA(bo::launch_cast_master(at<float>(ws, L.teach_y), nullptr, at<char>(ws, L.xt), 1, N, d, s), "X^T");
  return BO_OK;
}

bo_status bo_distill_load_united(bo_handle* h, int64_t N, const void* UWg, const void* UWu, const void* UWd,
                                 float* UWg_m, float* UWu_m, float* UWd_m, void* ws, size_t ws_bytes, void* stream) {
  bo_distill_layout L;
  bo_status st;
  if ((st = distill_check(h, N, ws, ws_bytes, &L)) != BO_OK) return st;
  if (!UWg || !UWu || !UWd || !UWg_m || !UWu_m || !UWd_m) return fail(BO_ERR_INVALID_ARG, "null tensor pointer");
  const bo_config& c = h->cfg;
  const int64_t m = c.num_experts, d = c.hidden, f = c.ffn, G = (m + c.way - 1) / c.way;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  BO_CUDA(bo::launch_widen(UWg, UWg_m, G * f * d, h->num_sms, s), "widen");
  BO_CUDA(bo::launch_widen(UWu, UWu_m, G * f * d, h->num_sms, s), "widen");
  BO_CUDA(bo::launch_widen(UWd, UWd_m, G * d * f, h->num_sms, s), "widen");
  BO_CUDA(bo::launch_cast_master(UWd_m, nullptr, at<char>(ws, L.uwdt), G, d, f, s), "UWd^T");
  return BO_OK;
}

bo_status bo_distill_step(bo_handle* h, const void* X, int64_t N, float lr, float* UWg_m, float* UWu_m,
                          float* UWd_m, void* UWg, void* UWu, void* UWd, void* ws, size_t ws_bytes, void* stream) {
  bo_distill_layout L;
  bo_status st;
  if ((st = distill_check(h, N, ws, ws_bytes, &L)) != BO_OK) return st;
  if (!X || !UWg_m || !UWu_m || !UWd_m || !UWg || !UWu || !UWd) return fail(BO_ERR_INVALID_ARG, "null tensor pointer");
  const void* ptrs[] = {X, UWg_m, UWu_m, UWd_m, UWg, UWu, UWd};
  for (const void* q : ptrs)
    if (!aligned16(q)) return fail(BO_ERR_SHAPE, "tensor pointers must be 16-byte aligned");
  if (!(lr >= 0.0f)) return fail(BO_ERR_INVALID_ARG, "lr must be >= 0");
  const bo_config& c = h->cfg;
  const int m = c.num_experts, d = c.hidden, f = c.ffn, G = (m + c.way - 1) / c.way;
  const int64_t R = static_cast<int64_t>(G) * N;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Prof prof(h, s, 11);   // 11 marked launch regions (the loss region is 2 kernels)
  int launches = 0;
  const int32_t* off_tok = at<int32_t>(ws, L.off_tok);
  // student forward: P = X UWg^T, Q = X UWu^T (shared A = X)
  PlainGemm g;
  g.A = X;
  g.a_rows = N;
  g.Kdim = d;
  g.a_shared = 1;
  g.b_rows = static_cast<int64_t>(G) * f;
  g.b_rows_per_exec = f;
  g.exec_off = off_tok;
  g.num_exec = G;
  g.rows_total = R;
  g.n_cols = f;
  g.ldo = f;
  g.B = UWg;
  g.out = at<char>(ws, L.p);
  if ((st = plain_gemm(h, g, s, prof, launches)) != BO_OK) return st;
  g.B = UWu;
  g.out = at<char>(ws, L.q);
  if ((st = plain_gemm(h, g, s, prof, launches)) != BO_OK) return st;
  prof.mark(launches);
  BO_CUDA(bo::launch_swiglu_fwd(at<char>(ws, L.p), at<char>(ws, L.q), at<char>(ws, L.hs), at<char>(ws, L.hst), G,
                                N, f, s),
          "swiglu fwd");
  ++launches;
  // H_u = Hs UWd^T (fp32)
  PlainGemm gy;
  gy.A = at<char>(ws, L.hs);
  gy.a_rows = R;
  gy.Kdim = f;
  gy.B = UWd;
  gy.b_rows = static_cast<int64_t>(G) * d;
  gy.b_rows_per_exec = d;
  gy.exec_off = off_tok;
  gy.num_exec = G;
  gy.rows_total = R;
  gy.n_cols = d;
  gy.out = at<char>(ws, L.y);
  gy.ldo = d;
  gy.f32_mode = 1;
  if ((st = plain_gemm(h, gy, s, prof, launches)) != BO_OK) return st;
  // Eq. 4 loss and dL/dH_u
  prof.mark(launches);
  BO_CUDA(bo::launch_mse_grad(at<float>(ws, L.y), at<float>(ws, L.hbar), at<char>(ws, L.dy), at<char>(ws, L.dyt), G,
                              N, d, at<double>(ws, L.part), at<double>(ws, L.floor_), m, c.way,
                              at<double>(ws, L.loss), s),
          "mse grad");
  ++launches;
  // dHs = dY UWd  (B = UWd^T [G, f, d])
  PlainGemm gh;
  gh.A = at<char>(ws, L.dy);
  gh.a_rows = R;
  gh.Kdim = d;
  gh.B = at<char>(ws, L.uwdt);
  gh.b_rows = static_cast<int64_t>(G) * f;
  gh.b_rows_per_exec = f;
  gh.exec_off = off_tok;
  gh.num_exec = G;
  gh.rows_total = R;
  gh.n_cols = f;
  gh.out = at<char>(ws, L.dhs);
  gh.ldo = f;
  if ((st = plain_gemm(h, gh, s, prof, launches)) != BO_OK) return st;
  prof.mark(launches);
  BO_CUDA(bo::launch_swiglu_bwd(at<char>(ws, L.dhs), at<char>(ws, L.p), at<char>(ws, L.q), at<char>(ws, L.dpt),
                                at<char>(ws, L.dqt), G, N, f, s),
          "swiglu bwd");
  ++launches;
  // weight gradients with the fused update W_m += (-lr) dL/dW_m (reduction over tokens)
  PlainGemm gw;
  gw.Kdim = static_cast<int>(N);
  gw.a_rows = static_cast<int64_t>(G) * f;
  gw.B = at<char>(ws, L.xt);
  gw.b_rows = d;
  gw.b_rows_per_exec = 0;   // X^T shared by every group
  gw.exec_off = at<int32_t>(ws, L.off_f);
  gw.num_exec = G;
  gw.rows_total = static_cast<int64_t>(G) * f;
  gw.n_cols = d;
  gw.ldo = d;
  gw.f32_mode = 2;
  gw.alpha = -lr;
  gw.A = at<char>(ws, L.dpt);
  gw.out = UWg_m;
  gw.out_bf16 = UWg;      // the bf16 copy is written by the same epilogue
  if ((st = plain_gemm(h, gw, s, prof, launches)) != BO_OK) return st;
  gw.A = at<char>(ws, L.dqt);
  gw.out = UWu_m;
  gw.out_bf16 = UWu;
  if ((st = plain_gemm(h, gw, s, prof, launches)) != BO_OK) return st;
  PlainGemm gd;   // dL/dUWd = dY^T Hs: A = dY^T [G, d, N], B = Hs^T [G, f, N]
  gd.A = at<char>(ws, L.dyt);
  gd.a_rows = static_cast<int64_t>(G) * d;
  gd.Kdim = static_cast<int>(N);
  gd.B = at<char>(ws, L.hst);
  gd.b_rows = static_cast<int64_t>(G) * f;
  gd.b_rows_per_exec = f;
  gd.exec_off = at<int32_t>(ws, L.off_d);
  gd.num_exec = G;
  gd.rows_total = static_cast<int64_t>(G) * d;
  gd.n_cols = f;
  gd.out = UWd_m;
  gd.ldo = f;
  gd.f32_mode = 2;
  gd.alpha = -lr;
  if ((st = plain_gemm(h, gd, s, prof, launches)) != BO_OK) return st;
  // refresh the bf16 UWd and UWd^T from the master (UWg / UWu: in the GEMM epilogues)
  prof.mark(launches);
  BO_CUDA(bo::launch_cast_master(UWd_m, UWd, at<char>(ws, L.uwdt), G, d, f, s), "cast");
  ++launches;
  prof.mark(launches);
  if (prof.err != cudaSuccess) return cuda_fail(prof.err, "profile event record");
  h->last_launches = launches + 1;   // + the loss reduction kernel
  return BO_OK;
}


const char* bo_version(void) { return "brownout-b200 0.1 (sm_100a)"; }

const char* bo_status_string(bo_status s) {
  switch (s) {
    case BO_OK: return "BO_OK";
    case BO_ERR_INVALID_ARG: return "BO_ERR_INVALID_ARG";
    case BO_ERR_SHAPE: return "BO_ERR_SHAPE";
    case BO_ERR_UNSUPPORTED: return "BO_ERR_UNSUPPORTED";
    case BO_ERR_CUDA: return "BO_ERR_CUDA";
    case BO_ERR_NCCL: return "BO_ERR_NCCL";
    case BO_ERR_WORKSPACE: return "BO_ERR_WORKSPACE";
  }
  return "BO_ERR_UNKNOWN";
}

const char* bo_last_error(void) { return g_last_error.c_str(); }

bo_status bo_create(const bo_config* cfg, bo_handle** out) {
  if (!cfg || !out) return fail(BO_ERR_INVALID_ARG, "null argument");
  *out = nullptr;
  const bo_config& c = *cfg;
  if (c.dtype != BO_BF16 && c.dtype != BO_FP32) return fail(BO_ERR_UNSUPPORTED, "dtype %d not built", c.dtype);
  if (c.num_experts < 1 || c.num_experts > bo::kMaxExperts)
    return fail(BO_ERR_SHAPE, "num_experts=%d outside [1, %d]", c.num_experts, bo::kMaxExperts);
  const int kmax = c.num_experts < 16 ? c.num_experts : 16;
  if (c.top_k < 1 || c.top_k > kmax) return fail(BO_ERR_INVALID_ARG, "top_k=%d outside [1, %d]", c.top_k, kmax);
  if (c.way < 1) return fail(BO_ERR_INVALID_ARG, "way=%d < 1", c.way);
  const int mult = c.dtype == BO_BF16 ? 64 : 32;
  if (c.hidden <= 0 || c.hidden % mult || c.ffn <= 0 || c.ffn % mult)
    return fail(BO_ERR_SHAPE, "hidden=%d / ffn=%d must be positive multiples of %d", c.hidden, c.ffn, mult);
  if (c.ffn % 64) return fail(BO_ERR_SHAPE, "ffn=%d must be a multiple of 64", c.ffn);
  const int G = (c.num_experts + c.way - 1) / c.way;
  if (c.num_shared < 0 || c.num_experts + G + c.num_shared > bo::kMaxExec)
    return fail(BO_ERR_INVALID_ARG, "num_shared=%d: m + G + N_s must be <= %d", c.num_shared, bo::kMaxExec);
  if (c.num_shared > 0 && c.dedup_united)
    return fail(BO_ERR_UNSUPPORTED, "dedup_united with shared experts is not built");
  if (c.max_tokens < 0 || c.max_tokens * (c.top_k + c.num_shared) > (int64_t(1) << 31) - 1)
    return fail(BO_ERR_INVALID_ARG, "max_tokens=%lld out of range", static_cast<long long>(c.max_tokens));
  int dev = 0, sms = 0;
  BO_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
  BO_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "cudaDeviceGetAttribute");
  bo_handle* h = new bo_handle();
  h->cfg = c;
  h->ratio = 0.0;
  h->mode = BO_PARTIAL;
  h->num_sms = sms;
  h->device = dev;
  h->last_launches = 0;
  h->prof_events = nullptr;
  h->prof_n = 0;
  h->route_T = -1;
  h->route_tile = 0;
  h->SWg = h->SWu = h->SWd = nullptr;
  options_from_env(&h->opt);
  *out = h;
  return BO_OK;
}

bo_status bo_set_engine_option(bo_handle* h, int32_t option, int32_t value) {
  if (!h) return fail(BO_ERR_INVALID_ARG, "null handle");
  if (option < 0 || option >= BO_OPT_COUNT) return fail(BO_ERR_INVALID_ARG, "engine option %d unknown", option);
  const OptionSpec& sp = kOptions[option];
  if (value < sp.lo || value > sp.hi)
    return fail(BO_ERR_INVALID_ARG, "%s=%d outside [%d, %d]", sp.env, value, sp.lo, sp.hi);
  h->opt.*sp.field = value;
  return BO_OK;
}

bo_status bo_get_engine_option(const bo_handle* h, int32_t option, int32_t* value) {
  if (!h || !value) return fail(BO_ERR_INVALID_ARG, "null argument");
  if (option < 0 || option >= BO_OPT_COUNT) return fail(BO_ERR_INVALID_ARG, "engine option %d unknown", option);
  *value = h->opt.*kOptions[option].field;
  return BO_OK;
}

bo_status bo_destroy(bo_handle* h) {
  delete h;
  return BO_OK;
}

bo_status bo_workspace_layout(const bo_handle* h, int64_t T, bo_ws_layout* out) {
  if (!h || !out) return fail(BO_ERR_INVALID_ARG, "null argument");
  if (T < 0 || T > h->cfg.max_tokens) return fail(BO_ERR_INVALID_ARG, "T out of range");
  return compute_layout(h, T, out);
}

bo_status bo_workspace_size(const bo_handle* h, int64_t T, size_t* bytes) {
  if (!bytes) return fail(BO_ERR_INVALID_ARG, "null argument");
  bo_ws_layout L;
  bo_status s = bo_workspace_layout(h, T, &L);
  if (s == BO_OK) *bytes = L.total_bytes;
  return s;
}

bo_status bo_set_brownout(bo_handle* h, double ratio, int32_t mode) {
  if (!h) return fail(BO_ERR_INVALID_ARG, "null handle");
  if (!(ratio >= 0.0 && ratio <= 1.0)) return fail(BO_ERR_INVALID_ARG, "ratio %g outside [0, 1]", ratio);
  if (mode != BO_PARTIAL && mode != BO_FULL) return fail(BO_ERR_INVALID_ARG, "mode %d invalid", mode);
  h->ratio = ratio;
  h->mode = mode;
  return BO_OK;
}

bo_status bo_get_brownout(const bo_handle* h, double* ratio, int32_t* mode) {
  if (!h || !ratio || !mode) return fail(BO_ERR_INVALID_ARG, "null argument");
  *ratio = h->ratio;
  *mode = h->mode;
  return BO_OK;
}

bo_status bo_build_united(bo_handle* h, const void* Wg, const void* Wu, const void* Wd, int32_t init, void* UWg,
                          void* UWu, void* UWd, void* stream) {
  if (!h || !Wg || !Wu || !Wd || !UWg || !UWu || !UWd) return fail(BO_ERR_INVALID_ARG, "null argument");
  if (init != BO_UNITED_MEAN) return fail(BO_ERR_UNSUPPORTED, "united init %d not built", init);
  const bo_config& c = h->cfg;
  const int dt = c.dtype == BO_BF16 ? 0 : 1;
  const int64_t per = static_cast<int64_t>(c.ffn) * c.hidden;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  BO_CUDA(bo::launch_build_united(dt, Wg, c.num_experts, c.way, per, UWg, s), "build_united Wg");
  BO_CUDA(bo::launch_build_united(dt, Wu, c.num_experts, c.way, per, UWu, s), "build_united Wu");
  BO_CUDA(bo::launch_build_united(dt, Wd, c.num_experts, c.way, per, UWd, s), "build_united Wd");
  return BO_OK;
}

bo_status bo_set_shared_experts(bo_handle* h, const void* SWg, const void* SWu, const void* SWd) {
  if (!h) return fail(BO_ERR_INVALID_ARG, "null handle");
  if (h->cfg.num_shared == 0) return fail(BO_ERR_INVALID_ARG, "handle was created with num_shared = 0");
  if (!SWg || !SWu || !SWd) return fail(BO_ERR_INVALID_ARG, "null shared-expert weights");
  if (!aligned16(SWg) || !aligned16(SWu) || !aligned16(SWd))
    return fail(BO_ERR_SHAPE, "tensor pointers must be 16-byte aligned");
  h->SWg = SWg;
  h->SWu = SWu;
  h->SWd = SWd;
  return BO_OK;
}

bo_status bo_moe_forward(bo_handle* h, const void* x, int64_t T, const void* Wr, const void* Wg, const void* Wu,
                         const void* Wd, const void* UWg, const void* UWu, const void* UWd, void* y,
                         void* workspace, size_t ws_bytes, void* stream) {
  if (!Wr) return fail(BO_ERR_INVALID_ARG, "null router");
  return forward_impl(h, x, T, Wr, Wg, Wu, Wd, UWg, UWu, UWd, y, workspace, ws_bytes, nullptr, stream);
}

bo_status bo_moe_forward_ex(bo_handle* h, const void* x, int64_t T, const void* Wr, const void* Wg,
                            const void* Wu, const void* Wd, const void* UWg, const void* UWu, const void* UWd,
                            void* y, void* workspace, size_t ws_bytes, const float* logits_in, void* stream) {
  return forward_impl(h, x, T, Wr, Wg, Wu, Wd, UWg, UWu, UWd, y, workspace, ws_bytes, logits_in, stream);
}

bo_status bo_plan_from_counts(bo_handle* h, const int32_t* counts, int32_t* exec_of_expert,
                              int32_t* expert_row_off, int32_t* exec_off, void* stats, void* stream) {
  if (!h || !counts || !exec_of_expert || !expert_row_off || !exec_off || !stats)
    return fail(BO_ERR_INVALID_ARG, "null argument");
  const bo_config& c = h->cfg;
  const int m = c.num_experts;
  const int E = m + (m + c.way - 1) / c.way;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int32_t* mtile_scratch = exec_off + (E + 1);   // exec_off holds 2*(E+1) + m ints (brownout.h)
  int32_t* counts_out = mtile_scratch + (E + 1);
  BO_CUDA(bo::launch_plan(counts, 1, m, c.way, h->ratio, h->mode, nullptr, counts_out, exec_of_expert,
                          expert_row_off, exec_off, mtile_scratch, static_cast<int64_t*>(stats), s),
          "plan_from_counts");
  return BO_OK;
}

bo_status bo_route(bo_handle* h, const void* x, int64_t T, const void* Wr, const float* logits_in, void* workspace,
                   size_t ws_bytes, void* stream) {
  if (!h) return fail(BO_ERR_INVALID_ARG, "null handle");
  h->last_kernels.clear();
  if (T < 0 || T > h->cfg.max_tokens) return fail(BO_ERR_INVALID_ARG, "T out of range");
  if (!x || (!Wr && !logits_in)) return fail(BO_ERR_INVALID_ARG, "null tensor pointer");
  bo_ws_layout L;
  bo_status st;
  if ((st = check_ws(h, T, workspace, ws_bytes, &L)) != BO_OK) return st;
  h->route_T = T;
  if (T == 0) return BO_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Prof prof(h, s, 1 << 30);
  int launches = 0, tile = 0;
  return route_stage(h, x, T, Wr, logits_in, workspace, L, s, prof, launches, tile);
}

bo_status bo_expert_ffn(bo_handle* h, const void* rows, int64_t R, const float* row_w, const int32_t* exec_off,
                        const int32_t* mtile_off, int32_t n_orig, int32_t n_united, int32_t f_united, const void* Wg,
                        const void* Wu, const void* Wd, const void* UWg, const void* UWu, const void* UWd,
                        void* h_buf, void* out, void* stream) {
  if (!h) return fail(BO_ERR_INVALID_ARG, "null handle");
  h->last_kernels.clear();
  if (R == 0) return BO_OK;
  const bo_config& c = h->cfg;
  if (n_orig < 0 || n_united < 0 || n_orig + n_united > bo::kMaxExec)
    return fail(BO_ERR_INVALID_ARG, "executor counts out of range");
  if (n_united > 0 && (f_united <= 0 || f_united > c.ffn || f_united % 128))
    return fail(BO_ERR_SHAPE, "f_united=%d must be a positive multiple of 128 and <= ffn", f_united);
  if (!rows || !row_w || !exec_off || !mtile_off || !h_buf || !out) return fail(BO_ERR_INVALID_ARG, "null argument");
  if ((n_orig > 0 && (!Wg || !Wu || !Wd)) || (n_united > 0 && (!UWg || !UWu || !UWd)))
    return fail(BO_ERR_INVALID_ARG, "null weights");
  const void* ptrs[] = {rows, h_buf, out, Wg ? Wg : rows, Wu ? Wu : rows, Wd ? Wd : rows,
                        UWg ? UWg : rows, UWu ? UWu : rows, UWd ? UWd : rows};
  for (const void* p : ptrs)
    if (!aligned16(p)) return fail(BO_ERR_SHAPE, "tensor pointers must be 16-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Prof prof(h, s, 1 << 30);
  int launches = 0;
  FfnClass orig, uni, shr;
  if (n_orig > 0) { orig.Wg = Wg; orig.Wu = Wu; orig.Wd = Wd; orig.n = n_orig; orig.f = c.ffn; orig.stack = n_orig; }
  if (n_united > 0) { uni.Wg = UWg; uni.Wu = UWu; uni.Wd = UWd; uni.n = n_united; uni.f = f_united; uni.stack = n_united; }
  return ffn_stage(h, rows, R, row_w, exec_off, mtile_off, orig, uni, shr, h_buf, out, s, prof, launches);
}

bo_status bo_combine(bo_handle* h, int64_t T, const void* rows, const int32_t* row_of, int32_t nrep, const void* x,
                     void* y, void* stream) {
  if (!h) return fail(BO_ERR_INVALID_ARG, "null handle");
  if (T == 0) return BO_OK;
  if (!rows || !row_of || !y || (h->cfg.add_residual && !x) || nrep < 1)
    return fail(BO_ERR_INVALID_ARG, "null argument");
  const bo_config& c = h->cfg;
  BO_CUDA(bo::launch_combine(c.dtype == BO_BF16 ? 0 : 1, rows, x, static_cast<int>(T), c.hidden, c.top_k * nrep,
                             row_of, c.add_residual, y, h->num_sms, static_cast<cudaStream_t>(stream)),
          "combine");
  return BO_OK;
}

bo_status bo_set_profile_events(bo_handle* h, void** events, int32_t n) {
  if (!h) return fail(BO_ERR_INVALID_ARG, "null handle");
  h->prof_events = events;
  h->prof_n = events ? n : 0;
  return BO_OK;
}

int32_t bo_last_launch_count(const bo_handle* h) { return h ? h->last_launches : 0; }
const char* bo_last_kernels(const bo_handle* h) { return h ? h->last_kernels.c_str() : ""; }

}  // extern "C"
