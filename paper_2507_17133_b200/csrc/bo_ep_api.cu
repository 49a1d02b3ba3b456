// bo_ep_api.cu - expert-parallel forward (include/brownout.h "Expert parallelism";
// SURVEY §8(e)): static placement, workspace carving, the stage entry
// points and the forward over a library-owned NCCL communicator.  The exchange
// tables are computed on the device from the all-gathered count rows
// (bo::launch_ep_tables); nothing of the method's arithmetic runs on the host.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <type_traits>
#include <vector>

#include "../../include/brownout.h"
#include "bo_internal.h"
#include "bo_kernels.h"

using namespace bo_impl;

namespace {

// ------------------------------------------------------------------ placement
// Original expert e on rank floor(e R / m); united expert j f-sliced over the
// distinct owner ranks of its members when every group has the same number n of
// them and f / n is a multiple of 128 (else whole on its first member's rank).
// Virtual executors are rank-major: a rank's originals ascending, then its slices.
struct Placement {
  int m = 0, way = 0, f = 0, R = 0, rank = 0, G = 0;
  bool sliced = false;
  int nslices = 1, f_u = 0, nrep = 1;
  std::vector<int> owner;                    // [m]
  std::vector<std::vector<int>> gowners;     // [G] owner ranks of group j
  struct V { int rank, kind, idx, slice; };  // kind 0 original (idx = e), 1 united slice (idx = j)
  std::vector<V> vexec;
  std::vector<int> vfirst;                   // [R + 1]
  std::vector<int> local_v;
  int e0 = 0, e1 = 0, n_united_local = 0;
};

bo_status make_placement(int m, int way, int f, int R, int rank, Placement* P) {
  if (R < 1 || R > bo::kEpMaxRanks) return fail(BO_ERR_INVALID_ARG, "world=%d outside [1, %d]", R, bo::kEpMaxRanks);
  if (rank < 0 || rank >= R) return fail(BO_ERR_INVALID_ARG, "rank=%d outside [0, %d)", rank, R);
  if (m < 1 || m > bo::kMaxExperts || way < 1 || f < 1) return fail(BO_ERR_SHAPE, "m=%d way=%d f=%d", m, way, f);
  Placement& p = *P;
  p.m = m; p.way = way; p.f = f; p.R = R; p.rank = rank;
  p.G = (m + way - 1) / way;
  p.owner.resize(m);
  for (int e = 0; e < m; ++e) p.owner[e] = static_cast<int>((static_cast<int64_t>(e) * R) / m);
  p.gowners.assign(p.G, {});
  for (int j = 0; j < p.G; ++j) {
    for (int e = j * way; e < std::min((j + 1) * way, m); ++e)
      if (std::find(p.gowners[j].begin(), p.gowners[j].end(), p.owner[e]) == p.gowners[j].end())
        p.gowners[j].push_back(p.owner[e]);
    std::sort(p.gowners[j].begin(), p.gowners[j].end());
  }
  const size_t n0 = p.gowners[0].size();
  bool same = true;
  for (const auto& g : p.gowners) same &= g.size() == n0;
  p.sliced = same && f % static_cast<int>(n0 * 128) == 0;
  if (!p.sliced)
    for (int j = 0; j < p.G; ++j) p.gowners[j] = {p.owner[j * way]};
  p.nslices = static_cast<int>(p.gowners[0].size());
  p.f_u = f / p.nslices;
  p.nrep = p.nslices;
  p.vexec.clear();
  p.vfirst.assign(R + 1, 0);
  for (int q = 0; q < R; ++q) {
    p.vfirst[q] = static_cast<int>(p.vexec.size());
    for (int e = 0; e < m; ++e)
      if (p.owner[e] == q) p.vexec.push_back({q, 0, e, 0});
    for (int j = 0; j < p.G; ++j)
      for (int s = 0; s < static_cast<int>(p.gowners[j].size()); ++s)
        if (p.gowners[j][s] == q) p.vexec.push_back({q, 1, j, s});
  }
  p.vfirst[R] = static_cast<int>(p.vexec.size());
  if (static_cast<int>(p.vexec.size()) > bo::kEpMaxV)
    return fail(BO_ERR_SHAPE, "%zu virtual executors exceed %d", p.vexec.size(), bo::kEpMaxV);
  p.local_v.clear();
  p.e0 = m; p.e1 = 0; p.n_united_local = 0;
  for (int v = p.vfirst[rank]; v < p.vfirst[rank + 1]; ++v) {
    p.local_v.push_back(v);
    if (p.vexec[v].kind == 0) { p.e0 = std::min(p.e0, p.vexec[v].idx); p.e1 = std::max(p.e1, p.vexec[v].idx + 1); }
    else ++p.n_united_local;
  }
  if (p.e1 <= p.e0) p.e0 = p.e1 = 0;
  return BO_OK;
}

void fill_info(const Placement& p, bo_ep_info* o) {
  memset(o, 0, sizeof(*o));
  o->world = p.R;
  o->rank = p.rank;
  o->e0 = p.e0;
  o->e1 = p.e1;
  o->n_united_local = p.n_united_local;
  o->f_united = p.f_u;
  o->nrep = p.nrep;
  o->sliced = p.sliced ? 1 : 0;
  o->n_exec = static_cast<int32_t>(p.vexec.size());
  o->n_local = static_cast<int32_t>(p.local_v.size());
}

// ----------------------------------------------------------------------- NCCL
// Loaded at run time so that the library has no link-time NCCL dependency (torch
// already maps its bundled libnccl.so.2 into the process; dlopen returns that one).
struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) return;
    auto sym = [&](auto& fn, const char* name) { fn = reinterpret_cast<std::decay_t<decltype(fn)>>(dlsym(lib, name)); };
    sym(api.getUniqueId, "ncclGetUniqueId");
    sym(api.commInitRank, "ncclCommInitRank");
    sym(api.commDestroy, "ncclCommDestroy");
    sym(api.allGather, "ncclAllGather");
    sym(api.send, "ncclSend");
    sym(api.recv, "ncclRecv");
    sym(api.groupStart, "ncclGroupStart");
    sym(api.groupEnd, "ncclGroupEnd");
    sym(api.errorString, "ncclGetErrorString");
    api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.allGather && api.send && api.recv &&
             api.groupStart && api.groupEnd && api.errorString;
  });
  return api;
}

#define BO_NCCL(call, what)                                                                            \
  do {                                                                                                 \
    ncclResult_t r_ = (call);                                                                          \
    if (r_ != ncclSuccess) return fail(BO_ERR_NCCL, "%s: %s", what, nccl().errorString(r_));          \
  } while (0)

}  // namespace

struct bo_ep {
  bo_handle* h = nullptr;
  bo_ep_config cfg{};
  Placement pl;
  bo::EpStatic st{};
  int padded = 0;
  int64_t cap = 0, rows_max = 0;
  int64_t T = -1;                 // tokens of the last bo_ep_route
  int tile = 0;                   // its token tile (the per-tile prefix the permutation reads)
  int64_t splits[2 * bo::kEpMaxRanks] = {};
  bool have_splits = false;       // exact mode: splits of this forward read by the host
  int launches = 0;               // kernels of this forward so far (bo_last_launch_count of the handle)
  ncclComm_t comm = nullptr;
};

namespace {

bo_status ep_layout(const bo_ep* ep, bo_ep_ws_layout* L) {
  const bo_handle* h = ep->h;
  const bo_config& c = h->cfg;
  const int64_t m = c.num_experts, d = c.hidden, f = c.ffn, R = ep->pl.R;
  const int64_t E = m + (m + c.way - 1) / c.way;
  const int nl = static_cast<int>(ep->pl.local_v.size());
  const int eb = elem_bytes(c.dtype);
  memset(L, 0, sizeof(*L));
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align256(off + (bytes ? bytes : 1));
    return o;
  };
  bo_ws_layout rl;
  compute_layout(h, ep->cfg.max_tokens, &rl, true);
  L->route = take(rl.total_bytes);
  L->count_row = take(sizeof(int32_t) * (m + 4));
  L->gathered = take(sizeof(int32_t) * R * (m + 4));
  L->exec_of_expert = take(sizeof(int32_t) * m);
  L->expert_row_off = take(sizeof(int32_t) * m);
  L->plan_scratch = take(sizeof(int32_t) * (2 * (E + 1) + m));
  L->stats = take(sizeof(bo_plan_stats));
  L->counts = take(sizeof(int32_t) * m);
  const int64_t nb = static_cast<int64_t>(nl) * R;
  L->tables = take(sizeof(int32_t) * (m * ep->pl.nrep + 2 * R + 6 * nb + 2 + 2 * (nl + 1) + 2));
  L->splits = take(sizeof(int64_t) * 2 * R);
  L->send = take(static_cast<size_t>(eb) * ep->rows_max * d);
  L->send_w = take(sizeof(float) * ep->rows_max);
  L->recv = take(static_cast<size_t>(eb) * ep->rows_max * d);
  L->recv_w = take(sizeof(float) * ep->rows_max);
  L->grouped = take(static_cast<size_t>(eb) * ep->rows_max * d);
  L->grouped_w = take(sizeof(float) * ep->rows_max);
  L->h = take(static_cast<size_t>(eb) * ep->rows_max * f);
  L->row_of = take(sizeof(int32_t) * ep->cfg.max_tokens * c.top_k * ep->pl.nrep);
  L->total_bytes = off;
  L->rows_max = ep->rows_max;
  return BO_OK;
}

bo::EpTables tables_at(const bo_ep* ep, void* ws, const bo_ep_ws_layout& L) {
  const int m = ep->h->cfg.num_experts, R = ep->pl.R;
  const int nl = static_cast<int>(ep->pl.local_v.size());
  const int nb = nl * R;
  int32_t* t = at<int32_t>(ws, L.tables);
  bo::EpTables tb;
  tb.row_base = t; t += m * ep->pl.nrep;
  tb.send_rows = t; t += R;
  tb.recv_rows = t; t += R;
  tb.fwd_dst = t; t += nb + 1;
  tb.fwd_len = t; t += nb;
  tb.fwd_src = t; t += nb;
  tb.inv_dst = t; t += nb + 1;
  tb.inv_len = t; t += nb;
  tb.inv_src = t; t += nb;
  tb.exec_off = t; t += nl + 1;
  tb.mtile_off = t; t += nl + 1;
  tb.totals = t;
  tb.splits = at<int64_t>(ws, L.splits);
  return tb;
}

bo_status ep_check_ws(const bo_ep* ep, void* ws, size_t ws_bytes, bo_ep_ws_layout* L) {
  ep_layout(ep, L);
  if (!ws || ws_bytes < L->total_bytes)
    return fail(BO_ERR_WORKSPACE, "EP workspace %zu bytes < required %zu", ws_bytes, L->total_bytes);
  if (!aligned16(ws)) return fail(BO_ERR_SHAPE, "workspace must be 16-byte aligned");
  return BO_OK;
}

// message offset / size (rows) of peer q: send side (out = true) or receive side
void peer_rows(const bo_ep* ep, int q, bool send_side, int64_t* off, int64_t* n) {
  if (ep->padded) {
    *off = q * ep->cap;
    *n = ep->cap;
    return;
  }
  const int R = ep->pl.R;
  const int64_t* sp = ep->splits + (send_side ? 0 : R);
  int64_t o = 0;
  for (int r = 0; r < q; ++r) o += sp[r];
  *off = o;
  *n = sp[q];
}

bo_status ep_splits_host(bo_ep* ep, void* ws, const bo_ep_ws_layout& L, cudaStream_t s) {
  const int R = ep->pl.R;
  if (ep->padded) {
    for (int i = 0; i < 2 * R; ++i) ep->splits[i] = ep->cap;
  } else {
    BO_CUDA(cudaMemcpyAsync(ep->splits, at<int64_t>(ws, L.splits), sizeof(int64_t) * 2 * R, cudaMemcpyDeviceToHost,
                            s),
            "EP splits");
    BO_CUDA(cudaStreamSynchronize(s), "EP splits sync");
  }
  ep->have_splits = true;
  return BO_OK;
}

bo_status ep_route_impl(bo_ep* ep, const void* x, int64_t T, const void* Wr, const float* logits_in, void* ws,
                        const bo_ep_ws_layout& L, cudaStream_t s) {
  bo_handle* h = ep->h;
  if (T < 0 || T > ep->cfg.max_tokens)
    return fail(BO_ERR_INVALID_ARG, "T=%lld outside [0, max_tokens=%lld]", static_cast<long long>(T),
                static_cast<long long>(ep->cfg.max_tokens));
  if (!x || (!Wr && !logits_in)) return fail(BO_ERR_INVALID_ARG, "null tensor pointer");
  if (!aligned16(x) || (Wr && !aligned16(Wr))) return fail(BO_ERR_SHAPE, "tensor pointers must be 16-byte aligned");
  void* rws = at<char>(ws, L.route);
  bo_ws_layout rl;
  compute_layout(h, ep->cfg.max_tokens, &rl, true);
  ep->T = T;
  ep->have_splits = false;
  ep->launches = 0;
  h->last_kernels.clear();
  int32_t* row = at<int32_t>(ws, L.count_row);
  const int m = h->cfg.num_experts;
  if (T == 0) {   // an empty batch still takes part in the exchange: zero counts + the knob
    BO_CUDA(cudaMemsetAsync(row, 0, sizeof(int32_t) * m, s), "EP empty row");
    // the plan kernel writes the knob tail; run it on zero counts
    bo::PlanExt ext;
    ext.row_tail = row + m;
    ext.row_T = 0;
    BO_CUDA(bo::launch_plan(row, 1, m, h->cfg.way, h->ratio, h->mode, nullptr, row, at<int32_t>(rws, rl.exec_of_expert),
                            at<int32_t>(rws, rl.expert_row_off), at<int32_t>(rws, rl.exec_off),
                            at<int32_t>(rws, rl.mtile_off), at<int64_t>(rws, rl.stats), s, 0, 0, ext),
            "EP empty plan");
    ep->launches = 1;
    return BO_OK;
  }
  Prof prof(h, s, 1 << 30);
  int launches = 0, tile = 0;
  // local route; the plan kernel writes this rank's counts + knob tail into count_row
  const bo_status st = route_stage(h, x, T, Wr, logits_in, rws, rl, s, prof, launches, tile, row);
  ep->tile = tile;
  ep->launches = launches;
  return st;
}

bo_status ep_dispatch_impl(bo_ep* ep, const void* x, void* ws, const bo_ep_ws_layout& L, cudaStream_t s) {
  bo_handle* h = ep->h;
  const bo_config& c = h->cfg;
  const int m = c.num_experts, R = ep->pl.R;
  if (ep->T < 0) return fail(BO_ERR_INVALID_ARG, "bo_ep_dispatch before bo_ep_route");
  const int E = m + (m + c.way - 1) / c.way;
  int32_t* scratch = at<int32_t>(ws, L.plan_scratch);
  // Alg. 1 on the column sums of the gathered rows, with rank 0's knob (its row tail)
  bo::PlanExt ext;
  ext.ld = m + 4;
  ext.knob_in = at<int32_t>(ws, L.gathered) + m;
  BO_CUDA(bo::launch_plan(at<int32_t>(ws, L.gathered), R, m, c.way, h->ratio, h->mode, nullptr,
                          at<int32_t>(ws, L.counts), at<int32_t>(ws, L.exec_of_expert),
                          at<int32_t>(ws, L.expert_row_off), scratch, scratch + (E + 1),
                          at<int64_t>(ws, L.stats), s, 0, 0, ext),
          "EP plan");
  const bo::EpTables tb = tables_at(ep, ws, L);
  BO_CUDA(bo::launch_ep_tables(ep->st, at<int32_t>(ws, L.gathered), m + 4, at<int32_t>(ws, L.exec_of_expert), tb, s),
          "EP tables");
  ep->launches += 2;
  h->last_kernels += ",ep_plan,ep_tables";
  if (ep->T == 0) return BO_OK;
  if (!x || !aligned16(x)) return fail(BO_ERR_INVALID_ARG, "x null or not 16-byte aligned");
  // a5: each (token, slot, replica) -> its send row (row_base + stable local rank), x copied there
  void* rws = at<char>(ws, L.route);
  bo_ws_layout rl;
  compute_layout(h, ep->cfg.max_tokens, &rl, true);
  BO_CUDA(bo::launch_permute(at<int32_t>(rws, rl.topk_id), at<float>(rws, rl.topk_w), static_cast<int>(ep->T),
                             c.top_k, m, ep->tile, at<int32_t>(rws, rl.tile_base), tb.row_base, ep->pl.nrep,
                             at<int32_t>(ws, L.row_of), nullptr, at<float>(ws, L.send_w), s,
                             c.dtype == BO_BF16 ? 0 : 1, x, at<char>(ws, L.send), c.hidden),
          "EP dispatch");
  ++ep->launches;
  h->last_kernels += ",ep_dispatch";
  return BO_OK;
}

bo_status ep_compute_impl(bo_ep* ep, const void* Wg, const void* Wu, const void* Wd, const void* UWg, const void* UWu,
                          const void* UWd, void* ws, const bo_ep_ws_layout& L, cudaStream_t s) {
  bo_handle* h = ep->h;
  const bo_config& c = h->cfg;
  const int R = ep->pl.R;
  const int nl = static_cast<int>(ep->pl.local_v.size());
  const int n_orig = ep->pl.e1 - ep->pl.e0, n_uni = ep->pl.n_united_local;
  if ((n_orig > 0 && (!Wg || !Wu || !Wd)) || (n_uni > 0 && (!UWg || !UWu || !UWd)))
    return fail(BO_ERR_INVALID_ARG, "null local weights");
  const void* ptrs[] = {Wg, Wu, Wd, UWg, UWu, UWd};
  for (const void* p : ptrs)
    if (p && !aligned16(p)) return fail(BO_ERR_SHAPE, "weight pointers must be 16-byte aligned");
  const bo::EpTables tb = tables_at(ep, ws, L);
  const int row_bytes = c.hidden * elem_bytes(c.dtype);
  // rows grouped by local executor (upper bound: exact mode knows the received rows)
  int64_t Rb = ep->rows_max;
  if (!ep->padded && ep->have_splits) {
    Rb = 0;
    for (int r = 0; r < R; ++r) Rb += ep->splits[R + r];
  }
  if (nl == 0 || Rb == 0) return BO_OK;
  h->last_kernels += ",ep_regroup";
  BO_CUDA(bo::launch_block_copy(at<char>(ws, L.recv), at<char>(ws, L.grouped), row_bytes, at<float>(ws, L.recv_w),
                                at<float>(ws, L.grouped_w), nl * R, tb.fwd_dst, tb.fwd_len, tb.fwd_src, tb.totals,
                                Rb, h->num_sms, s),
          "EP regroup");
  FfnClass orig, uni, shr;
  if (n_orig > 0) { orig.Wg = Wg; orig.Wu = Wu; orig.Wd = Wd; orig.n = n_orig; orig.f = c.ffn; orig.stack = n_orig; }
  if (n_uni > 0) {
    uni.Wg = UWg; uni.Wu = UWu; uni.Wd = UWd; uni.n = n_uni; uni.f = ep->pl.f_u; uni.stack = n_uni;
  }
  // bo_set_profile_events with >= 3 events: events[0] / [1] / [2] around GEMM1 and GEMM2
  Prof prof(h, s, 2);
  int launches = 0;
  // GEMM2 writes its weighted outputs over the grouped rows (Xp is dead after GEMM1)
  bo_status st = ffn_stage(h, at<char>(ws, L.grouped), Rb, at<float>(ws, L.grouped_w), tb.exec_off, tb.mtile_off,
                           orig, uni, shr, at<char>(ws, L.h), at<char>(ws, L.grouped), s, prof, launches);
  if (st != BO_OK) return st;
  prof.mark(launches);
  if (prof.err != cudaSuccess) return cuda_fail(prof.err, "profile event record");
  ep->launches += launches + 2;
  // back to the receive layout (ret aliases recv)
  BO_CUDA(bo::launch_block_copy(at<char>(ws, L.grouped), at<char>(ws, L.recv), row_bytes, nullptr, nullptr, nl * R,
                                tb.inv_dst, tb.inv_len, tb.inv_src, tb.totals + 1, ep->rows_max, h->num_sms, s),
          "EP inverse regroup");
  h->last_kernels += ",ep_unregroup";
  return BO_OK;
}

bo_status ep_combine_impl(bo_ep* ep, const void* x, void* y, void* ws, const bo_ep_ws_layout& L, cudaStream_t s) {
  bo_handle* h = ep->h;
  const bo_config& c = h->cfg;
  if (ep->T <= 0) return BO_OK;
  if (!y || (c.add_residual && !x)) return fail(BO_ERR_INVALID_ARG, "null argument");
  BO_CUDA(bo::launch_combine(c.dtype == BO_BF16 ? 0 : 1, at<char>(ws, L.send), x, static_cast<int>(ep->T), c.hidden,
                             c.top_k * ep->pl.nrep, at<int32_t>(ws, L.row_of), c.add_residual, y, h->num_sms, s),
          "EP combine");
  ++ep->launches;
  h->last_kernels += ",combine";
  h->last_launches = ep->launches;
  return BO_OK;
}

// grouped point-to-point exchange of `rows` rows (row_bytes each) + optional float weights
bo_status ep_exchange(bo_ep* ep, const char* src, char* dst, size_t row_bytes, const float* w_src, float* w_dst,
                      bool forward, cudaStream_t s) {
  const NcclApi& api = nccl();
  const int R = ep->pl.R;
  BO_NCCL(api.groupStart(), "ncclGroupStart");
  for (int q = 0; q < R; ++q) {
    int64_t so, sn, ro, rn;
    // forward: send side = send layout, receive side = recv layout; backward the reverse
    peer_rows(ep, q, forward, &so, &sn);
    peer_rows(ep, q, !forward, &ro, &rn);
    BO_NCCL(api.send(src + so * row_bytes, sn * row_bytes, ncclUint8, q, ep->comm, s), "ncclSend");
    BO_NCCL(api.recv(dst + ro * row_bytes, rn * row_bytes, ncclUint8, q, ep->comm, s), "ncclRecv");
    if (w_src) {
      BO_NCCL(api.send(w_src + so, sn, ncclFloat32, q, ep->comm, s), "ncclSend (weights)");
      BO_NCCL(api.recv(w_dst + ro, rn, ncclFloat32, q, ep->comm, s), "ncclRecv (weights)");
    }
  }
  BO_NCCL(api.groupEnd(), "ncclGroupEnd");
  return BO_OK;
}

}  // namespace

extern "C" {

bo_status bo_ep_placement(int32_t num_experts, int32_t way, int32_t ffn, int32_t world, int32_t rank,
                          bo_ep_info* out) {
  if (!out) return fail(BO_ERR_INVALID_ARG, "null argument");
  Placement p;
  bo_status st = make_placement(num_experts, way, ffn, world, rank, &p);
  if (st != BO_OK) return st;
  fill_info(p, out);
  return BO_OK;
}

bo_status bo_ep_placement_slices(int32_t num_experts, int32_t way, int32_t ffn, int32_t world, int32_t rank,
                                 int32_t* group, int32_t* slice, int32_t n) {
  Placement p;
  bo_status st = make_placement(num_experts, way, ffn, world, rank, &p);
  if (st != BO_OK) return st;
  if (n < p.n_united_local || (p.n_united_local > 0 && (!group || !slice)))
    return fail(BO_ERR_INVALID_ARG, "need room for %d slices", p.n_united_local);
  int k = 0;
  for (int v : p.local_v)
    if (p.vexec[v].kind == 1) {
      group[k] = p.vexec[v].idx;
      slice[k] = p.vexec[v].slice;
      ++k;
    }
  return BO_OK;
}

bo_status bo_ep_create(bo_handle* h, const bo_ep_config* cfg, bo_ep** out) {
  if (!h || !cfg || !out) return fail(BO_ERR_INVALID_ARG, "null argument");
  *out = nullptr;
  const bo_config& c = h->cfg;
  if (c.dedup_united || c.num_shared) return fail(BO_ERR_UNSUPPORTED, "dedup_united / shared experts are single-GPU only");
  if (cfg->max_tokens < 1 || cfg->max_tokens > c.max_tokens)
    return fail(BO_ERR_INVALID_ARG, "EP max_tokens=%lld outside [1, %lld]", static_cast<long long>(cfg->max_tokens),
                static_cast<long long>(c.max_tokens));
  bo_ep* ep = new bo_ep();
  ep->h = h;
  ep->cfg = *cfg;
  bo_status st = make_placement(c.num_experts, c.way, c.ffn, cfg->world, cfg->rank, &ep->pl);
  if (st != BO_OK) {
    delete ep;
    return st;
  }
  const Placement& p = ep->pl;
  ep->cap = cfg->max_tokens * c.top_k;   // rows one source can send one destination (replicas go to distinct ranks)
  ep->padded = cfg->padded >= 0 ? (cfg->padded ? 1 : 0) : (ep->cap <= 4096 ? 1 : 0);
  ep->rows_max = p.R * ep->cap;
  if (ep->rows_max > (int64_t(1) << 31) - 1) {
    delete ep;
    return fail(BO_ERR_INVALID_ARG, "exchange buffers too large");
  }
  bo::EpStatic& s = ep->st;
  s.R = p.R;
  s.rank = p.rank;
  s.m = p.m;
  s.way = p.way;
  s.nrep = p.nrep;
  s.nslices = p.nslices;
  s.V = static_cast<int>(p.vexec.size());
  s.nl = static_cast<int>(p.local_v.size());
  s.padded = ep->padded;
  s.cap = ep->cap;
  for (int v = 0; v < s.V; ++v) {
    const auto& e = p.vexec[v];
    s.vexec[v] = (e.rank << 24) | (e.kind << 23) | e.idx;
    if (e.kind == 0) s.v_of_orig[e.idx] = v;
    else s.v_of_slice[e.idx * p.nrep + e.slice] = v;
  }
  for (int q = 0; q <= p.R; ++q) s.vfirst[q] = p.vfirst[q];
  for (int i = 0; i < s.nl; ++i) s.local_v[i] = p.local_v[i];
  *out = ep;
  return BO_OK;
}

bo_status bo_ep_destroy(bo_ep* ep) {
  if (!ep) return BO_OK;
  if (ep->comm && nccl().ok) nccl().commDestroy(ep->comm);
  delete ep;
  return BO_OK;
}

bo_status bo_ep_get_info(const bo_ep* ep, bo_ep_info* out) {
  if (!ep || !out) return fail(BO_ERR_INVALID_ARG, "null argument");
  fill_info(ep->pl, out);
  out->padded = ep->padded;
  out->cap = ep->cap;
  out->rows_max = ep->rows_max;
  return BO_OK;
}

bo_status bo_ep_workspace_layout(const bo_ep* ep, bo_ep_ws_layout* out) {
  if (!ep || !out) return fail(BO_ERR_INVALID_ARG, "null argument");
  return ep_layout(ep, out);
}

bo_status bo_ep_nccl_unique_id(unsigned char id[128]) {
  if (!id) return fail(BO_ERR_INVALID_ARG, "null argument");
  const NcclApi& api = nccl();
  if (!api.ok) return fail(BO_ERR_NCCL, "libnccl.so.2 not found or incomplete");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId u;
  BO_NCCL(api.getUniqueId(&u), "ncclGetUniqueId");
  memcpy(id, &u, 128);
  return BO_OK;
}

bo_status bo_ep_init(bo_ep* ep, const unsigned char nccl_unique_id[128]) {
  if (!ep || !nccl_unique_id) return fail(BO_ERR_INVALID_ARG, "null argument");
  const NcclApi& api = nccl();
  if (!api.ok) return fail(BO_ERR_NCCL, "libnccl.so.2 not found or incomplete");
  if (ep->comm) return fail(BO_ERR_INVALID_ARG, "communicator already initialised");
  ncclUniqueId u;
  memcpy(&u, nccl_unique_id, 128);
  BO_CUDA(cudaSetDevice(ep->h->device), "cudaSetDevice");
  BO_NCCL(api.commInitRank(&ep->comm, ep->pl.R, u, ep->pl.rank), "ncclCommInitRank");
  return BO_OK;
}

bo_status bo_ep_route(bo_ep* ep, const void* x, int64_t T, const void* Wr, const float* logits_in, void* ws,
                      size_t ws_bytes, void* stream) {
  if (!ep) return fail(BO_ERR_INVALID_ARG, "null EP context");
  bo_ep_ws_layout L;
  bo_status st;
  if ((st = ep_check_ws(ep, ws, ws_bytes, &L)) != BO_OK) return st;
  return ep_route_impl(ep, x, T, Wr, logits_in, ws, L, static_cast<cudaStream_t>(stream));
}

bo_status bo_ep_dispatch(bo_ep* ep, const void* x, void* ws, size_t ws_bytes, void* stream) {
  if (!ep) return fail(BO_ERR_INVALID_ARG, "null EP context");
  bo_ep_ws_layout L;
  bo_status st;
  if ((st = ep_check_ws(ep, ws, ws_bytes, &L)) != BO_OK) return st;
  return ep_dispatch_impl(ep, x, ws, L, static_cast<cudaStream_t>(stream));
}

bo_status bo_ep_splits(bo_ep* ep, void* ws, size_t ws_bytes, int64_t* send_rows, int64_t* recv_rows, void* stream) {
  if (!ep || !send_rows || !recv_rows) return fail(BO_ERR_INVALID_ARG, "null argument");
  bo_ep_ws_layout L;
  bo_status st;
  if ((st = ep_check_ws(ep, ws, ws_bytes, &L)) != BO_OK) return st;
  if ((st = ep_splits_host(ep, ws, L, static_cast<cudaStream_t>(stream))) != BO_OK) return st;
  const int R = ep->pl.R;
  for (int q = 0; q < R; ++q) {
    send_rows[q] = ep->splits[q];
    recv_rows[q] = ep->splits[R + q];
  }
  return BO_OK;
}

bo_status bo_ep_compute(bo_ep* ep, const void* Wg, const void* Wu, const void* Wd, const void* UWg, const void* UWu,
                        const void* UWd, void* ws, size_t ws_bytes, void* stream) {
  if (!ep) return fail(BO_ERR_INVALID_ARG, "null EP context");
  bo_ep_ws_layout L;
  bo_status st;
  if ((st = ep_check_ws(ep, ws, ws_bytes, &L)) != BO_OK) return st;
  return ep_compute_impl(ep, Wg, Wu, Wd, UWg, UWu, UWd, ws, L, static_cast<cudaStream_t>(stream));
}

bo_status bo_ep_combine(bo_ep* ep, const void* x, void* y, void* ws, size_t ws_bytes, void* stream) {
  if (!ep) return fail(BO_ERR_INVALID_ARG, "null EP context");
  bo_ep_ws_layout L;
  bo_status st;
  if ((st = ep_check_ws(ep, ws, ws_bytes, &L)) != BO_OK) return st;
  return ep_combine_impl(ep, x, y, ws, L, static_cast<cudaStream_t>(stream));
}

bo_status bo_ep_forward(bo_ep* ep, const void* x, int64_t T, const void* Wr, const void* Wg, const void* Wu,
                        const void* Wd, const void* UWg, const void* UWu, const void* UWd, void* y, void* ws,
                        size_t ws_bytes, void* stream) {
  if (!ep) return fail(BO_ERR_INVALID_ARG, "null EP context");
  if (!ep->comm) return fail(BO_ERR_INVALID_ARG, "bo_ep_forward needs bo_ep_init (library-owned communicator)");
  bo_ep_ws_layout L;
  bo_status st;
  if ((st = ep_check_ws(ep, ws, ws_bytes, &L)) != BO_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bo_config& c = ep->h->cfg;
  const NcclApi& api = nccl();
  if ((st = ep_route_impl(ep, x, T, Wr, nullptr, ws, L, s)) != BO_OK) return st;
  // count all-gather (fixed size: m + 4 int32 per rank)
  BO_NCCL(api.allGather(at<int32_t>(ws, L.count_row), at<int32_t>(ws, L.gathered), c.num_experts + 4, ncclInt32,
                        ep->comm, s),
          "ncclAllGather (counts)");
  if ((st = ep_dispatch_impl(ep, x, ws, L, s)) != BO_OK) return st;
  if ((st = ep_splits_host(ep, ws, L, s)) != BO_OK) return st;   // padded: no synchronisation
  const size_t row_bytes = static_cast<size_t>(c.hidden) * elem_bytes(c.dtype);
  if ((st = ep_exchange(ep, at<char>(ws, L.send), at<char>(ws, L.recv), row_bytes, at<float>(ws, L.send_w),
                        at<float>(ws, L.recv_w), true, s)) != BO_OK)
    return st;
  if ((st = ep_compute_impl(ep, Wg, Wu, Wd, UWg, UWu, UWd, ws, L, s)) != BO_OK) return st;
  if ((st = ep_exchange(ep, at<char>(ws, L.recv), at<char>(ws, L.send), row_bytes, nullptr, nullptr, false, s)) !=
      BO_OK)
    return st;
  return ep_combine_impl(ep, x, y, ws, L, s);
}

}  // extern "C"
