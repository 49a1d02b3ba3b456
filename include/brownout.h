/*
 * brownout.h - C ABI of the B200-native brownout MoE-layer forward.
 *
 * The method is BrownoutServe's BrownoutMoE layer (arXiv 2507.17133):
 *   router logits     Eq. 8       s_{i,t} = x_t^T e_i
 *   top-K gate        Eq. 7            g = softmax over the K largest s
 *   brownout plan     Alg. 1            S1 / S2 / united groups / special case
 *   expert FFNs       Eq. 5, SwiGLU        process_tokens (Alg. 1)
 *   gate weighting    Eq. 6            p = g for S1, q = g for S2
 *   combine           Eq. 5                h_t = [x_t] + sum of weighted outputs
 * "United experts" (one per group of `way` experts) are passed in
 * by the caller; bo_build_united() makes a deterministic initialisation.
 *
 * Conventions for every call:
 *  - All tensor arguments are DEVICE pointers owned by the caller (PyTorch).
 *    The library never allocates or frees device memory; bo_moe_forward uses
 *    only the caller's workspace.  Layouts are dense row-major (C order).
 *  - `stream` is a cudaStream_t passed as void*; every call that launches work
 *    enqueues it on that stream and returns without synchronising (except where
 *    noted).  The single-GPU forward has no host<->device synchronisation and is
 *    CUDA-graph capturable.
 *  - Every call returns a bo_status.  Nothing throws or aborts across the ABI.
 *    bo_last_error() returns a thread-local message for the last failure.
 *    Asynchronous CUDA errors surface as BO_ERR_CUDA on a later call.
 *  - A handle is not thread-safe: use one host thread per handle.
 *  - Element dtype of x, y, Wr, experts and united is the handle's dtype:
 *    BO_BF16 (bf16 storage, tcgen05 kind::f16 MMAs with fp32 accumulation) or
 *    BO_FP32 (fp32 storage, tcgen05 kind::tf32 MMAs with fp32 accumulation).
 */
#ifndef BROWNOUT_H_
#define BROWNOUT_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define BO_API __attribute__((visibility("default")))
#else
#define BO_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BO_OK = 0,
  BO_ERR_INVALID_ARG = 1,  /* null pointer, ratio outside [0,1], way < 1, K outside [1, min(m,16)], T > max_tokens */
  BO_ERR_SHAPE = 2,        /* hidden or ffn not a multiple of 64 (bf16) / 32 (fp32), m > 256, misaligned pointer */
  BO_ERR_UNSUPPORTED = 3,  /* dtype / mode / init not built */
  BO_ERR_CUDA = 4,         /* a CUDA runtime / driver call failed (message in bo_last_error) */
  BO_ERR_NCCL = 5,         /* NCCL missing or a NCCL call failed (expert-parallel forward) */
  BO_ERR_WORKSPACE = 6     /* workspace null or smaller than bo_workspace_size() */
} bo_status;

typedef enum { BO_BF16 = 0, BO_FP32 = 1 } bo_dtype;

/* Alg. 1 `use_full_brownout`: PARTIAL delegates S2 experts'
 * tokens to united experts; FULL ignores them.  Ratio 0 is
 * zero-brownout in either mode. */
typedef enum { BO_PARTIAL = 0, BO_FULL = 1 } bo_mode;

/* United-expert initialisation (reading D14): element-wise mean of
 * the group's member weights, computed in fp64 and rounded once (RNE). */
typedef enum { BO_UNITED_MEAN = 0 } bo_united_init;

/* Engine options (bo_set_engine_option): how the kernels of the forward are
 * scheduled, never what they compute — every setting gives the same routing,
 * plan and permutation and outputs within the parity tolerance (the tests run
 * each).  bo_create sets the defaults (the measured-best configuration,
 * DESIGN.md §5), overridable from the environment as BO_<NAME>=<int> (e.g.
 * BO_CTA_PAIRS=0) for A/B runs. */
typedef enum {
  BO_OPT_CTA_PAIRS = 0,      /* 1: prefill-sized FFN GEMMs on cta_group::2 CTA pairs (256-row tiles)   [1]    */
  BO_OPT_PAIR_ROWS1 = 1,     /* GEMM1 uses CTA pairs from this many rows                            [2048] */
  BO_OPT_PAIR_ROWS2 = 2,     /* GEMM2 likewise                                                      [2048] */
  BO_OPT_TILE_ALT = 3,       /* 1: GEMM1 may pick a narrower SwiGLU tile on the device (fewer waves)  [1]    */
  BO_OPT_SWAP_TAIL = 4,      /* 1: CTA-pair GEMM1 runs ragged last m-tiles with swapped operands     [1]    */
  BO_OPT_DECODE_PAIR2 = 5,   /* 1: decode GEMM2 on pairs + split-K when executors hold >= 256 rows   [1]    */
  BO_OPT_GEMM2_SPLITK = 6,   /* 1: GEMM2 split-K (fp32 partials) for every decode-sized step         [0]    */
  BO_OPT_FUSED_COMBINE = 7,  /* a8 in GEMM2's epilogue: 0 never, 1 always, 2 auto                    [2]    */
  BO_OPT_TMA_STORE = 8,      /* 1: GEMM2 writes full Yp slabs with TMA bulk stores                   [1]    */
  BO_OPT_STORE_HINT = 9,     /* 1: prefill H / Yp stores carry an L2 evict_first hint                [1]    */
  BO_OPT_B_POLICY = 10,      /* weight loads: 0 evict_normal, 1 evict_first, -1 auto (decode: first) [-1]   */
  BO_OPT_ROUTER_MMA = 11,    /* 1: prefill-sized bf16 batches with m <= 32 use the mma.sync router    [1]    */
  BO_OPT_ROUTER_SPLIT = 12,  /* 1: decode-sized batches with m <= 32 use the split-warp router        [1]    */
  BO_OPT_PDL = 13,           /* 1: GEMMs launch with programmatic dependent launch                   [1]    */
  BO_OPT_ROUTE_FUSED = 14,   /* 1: decode-sized m <= 32 steps run router + top-K + Alg. 1 + permute +
                                   gather as one cooperative launch                                   [1]    */
  BO_OPT_TAIL_SPLIT = 15,    /* 1: prefill GEMM2 on pairs shares a partial last wave out by k-blocks    [1]    */
  BO_OPT_COUNT = 16
} bo_engine_option;

typedef struct {
  int32_t hidden;        /* d   */
  int32_t ffn;           /* f   */
  int32_t num_experts;   /* m   (<= 256) */
  int32_t top_k;         /* K   (1 <= K <= min(m, 16)) */
  int32_t way;           /* k of the paper: experts per united group, G = ceil(m / way) */
  int32_t dtype;         /* bo_dtype */
  int32_t add_residual;  /* 1: h_t = x_t + ... (Eq. 5 first term); 0: omit x_t (parity, reading D12) */
  int32_t dedup_united;  /* 1: a token's slots delegated to the same united expert share ONE row carrying
                            the summed weight (Eq. 5-6 algebra; single-GPU forward only) */
  int32_t num_shared;    /* N_s of Eq. 5: shared experts applied to every token with weight 1, shape
                            of an original expert; weights via bo_set_shared_experts (single-GPU forward only) */
  int64_t max_tokens;    /* largest T a forward will be called with */
} bo_config;

/* Plan statistics (int64 each, written by the device into the workspace). */
typedef struct {
  int64_t executors_accessed;  /* executors with >= 1 row ("access 5 experts") */
  int64_t n_s1;                /* |S1| */
  int64_t n_united;            /* united executors used (groups with >= 2 S2 members) */
  int64_t n_singleton;         /* S2 experts kept original by the special case */
  int64_t rows_original;       /* rows processed by original experts */
  int64_t rows_united;         /* rows processed by united experts */
  int64_t rows_dropped;        /* rows ignored (BO_FULL only) */
  int64_t rows_total;          /* S = T*K */
} bo_plan_stats;

/* Byte offsets of the arrays inside a workspace sized for T tokens.  Every
 * array is 256-byte aligned.  Index arrays are exported for parity tests. */
typedef struct {
  size_t total_bytes;
  size_t logits;          /* float [T, m]       router logits (Eq. 8)                    */
  size_t topk_id;         /* int32 [T, K]       selected experts, logit desc / id asc   */
  size_t topk_w;          /* float [T, K]       gate weights g (Eq. 7)                  */
  size_t tile_cnt;        /* int32 [ntiles, m]  per-tile expert histogram              */
  size_t tile_base;       /* int32 [ntiles, m]  exclusive prefix of tile_cnt over tiles */
  size_t counts;          /* int32 [m]          cnt_i of Alg. 1                          */
  size_t exec_of_expert;  /* int32 [m]          executor of expert (-1 inactive, -2 dropped) */
  size_t expert_row_off;  /* int32 [m]          first row of expert's tokens (-1 if none) */
  size_t exec_off;        /* int32 [E+N_s+1]    first row of each executor (shared last) */
  size_t mtile_off;       /* int32 [E+N_s+1]    prefix of ceil(rows/128) per executor    */
  size_t stats;           /* bo_plan_stats                                              */
  size_t row_of;          /* int32 [T, K + N_s] row of (t, slot); slots K.. are the shared rows; -1: no row */
  size_t row_tok;         /* int32 [R]          token of each row, R = T*K + N_s*T        */
  size_t row_w;           /* float [R]          weight carried by each row (Eq. 6 p / q; 1 for shared) */
  size_t xp;              /* dtype [R, d]       gathered rows (concat_tokens)     */
  size_t h;               /* dtype [R, f]       SwiGLU activations                      */
  size_t yp;              /* dtype [R, d]       weighted executor outputs               */
  size_t partial;         /* float [8, T*K, d]  split-K partials of GEMM2 (T*K <= 1024 only, else 0 bytes) */
  size_t tile_xcnt;       /* int32 [ntiles, E]  rows per executor per tile (dedup_united)   */
  size_t tile_xbase;      /* int32 [ntiles, E]  their exclusive prefix over tiles            */
  size_t ksplit;          /* int32 [1]          split count GEMM2 chose                 */
  size_t comb_cnt;        /* int32 [T, d/BN2]   arrival counters of the combine fused into GEMM2 (a8; BN2 = 256/128/64, GEMM2 tile width) */
  size_t sk_part;         /* float [#SM, 256, 128] GEMM2 last-wave-split partials (T*K+N_s*T >= 2048 only)  */
  size_t sk_flag;         /* int32 [#SM]        their arrival counts (zeroed before each GEMM2)           */
  int64_t T;              /* tokens the layout was computed for                          */
  int64_t ntiles;         /* histogram tiles the workspace is sized for (8 tokens each)  */
  int64_t num_executors;  /* E = m + G                                                   */
} bo_ws_layout;

typedef struct bo_handle bo_handle;

/* Create / destroy a layer handle.  bo_create validates the config (errors as
 * listed in bo_status) and queries the current device; no device memory. */
BO_API bo_status bo_create(const bo_config* cfg, bo_handle** out);
BO_API bo_status bo_destroy(bo_handle* h);

/* Workspace needed for a forward over T tokens (T <= max_tokens). */
BO_API bo_status bo_workspace_size(const bo_handle* h, int64_t T, size_t* bytes);
BO_API bo_status bo_workspace_layout(const bo_handle* h, int64_t T, bo_ws_layout* out);

/* United experts from the original experts (D14, grouping P:149/P:154-155):
 *   Wg, Wu [m, f, d], Wd [m, d, f]  ->  UWg, UWu [G, f, d], UWd [G, d, f],
 * UW*[j] = mean over experts e in [j*way, min((j+1)*way, m)) of W*[e]
 * (fp64 sum in ascending member order, divide, round once to the dtype, RNE).
 * Runs once per layer; not part of the timed forward. */
BO_API bo_status bo_build_united(bo_handle* h, const void* Wg, const void* Wu, const void* Wd,
                          int32_t init, void* UWg, void* UWu, void* UWd, void* stream);

/* Shared experts of Eq. 5 (second term): SWg, SWu [N_s, f, d], SWd [N_s, d, f]
 * device pointers (caller-owned) used by every following forward; N_s is fixed
 * by bo_config.num_shared.  A wider shared FFN (e.g. one of width 4f) is exactly
 * N_s = 4 experts of width f holding its column slices (SwiGLU is elementwise in f). */
BO_API bo_status bo_set_shared_experts(bo_handle* h, const void* SWg, const void* SWu, const void* SWd);

/* Engine options (bo_engine_option): BO_ERR_INVALID_ARG for an unknown option or a
 * value outside its range.  Host state, read by the next forward. */
BO_API bo_status bo_set_engine_option(bo_handle* h, int32_t option, int32_t value);
BO_API bo_status bo_get_engine_option(const bo_handle* h, int32_t option, int32_t* value);

/* The brownout knob: ratio = 1 - threshold, in [0, 1].
 * Host state only; snapshotted by the next forward (may change every
 * iteration).  mode is a bo_mode. */
BO_API bo_status bo_set_brownout(bo_handle* h, double ratio, int32_t mode);
BO_API bo_status bo_get_brownout(const bo_handle* h, double* ratio, int32_t* mode);

/* moe_forward(tokens, router, experts, united) (B:5):
 *   x   [T, d]       tokens
 *   Wr  [m, d]       router centroids e_i (Eq. 8)
 *   Wg, Wu [m, f, d], Wd [m, d, f]   original experts (nn.Linear [out, in])
 *   UWg, UWu [G, f, d], UWd [G, d, f] united experts (may be NULL only if the
 *                    plan never selects a united executor, e.g. ratio 0)
 *   y   [T, d]       output h_t of Eq. 5 (written, never read)
 *   workspace        >= bo_workspace_size(T) bytes, 256-byte aligned
 * T = 0 is a no-op.  T > max_tokens -> BO_ERR_INVALID_ARG. */
BO_API bo_status bo_moe_forward(bo_handle* h, const void* x, int64_t T, const void* Wr,
                         const void* Wg, const void* Wu, const void* Wd,
                         const void* UWg, const void* UWu, const void* UWd,
                         void* y, void* workspace, size_t ws_bytes, void* stream);

/* Parity / debug variant.  If logits_in (device, fp32 [T, m]) is non-NULL the
 * router GEMM is skipped and these logits are routed instead ("given
 * identical fp32 logits", B:5).  All intermediate arrays stay readable in the
 * workspace at the offsets of bo_workspace_layout(T). */
BO_API bo_status bo_moe_forward_ex(bo_handle* h, const void* x, int64_t T, const void* Wr,
                            const void* Wg, const void* Wu, const void* Wd,
                            const void* UWg, const void* UWu, const void* UWd,
                            void* y, void* workspace, size_t ws_bytes,
                            const float* logits_in, void* stream);

/* Alg. 1 alone on given per-expert counts (device int32 [m], any 4-byte-aligned
 * pointer) with the
 * handle's ratio/mode/way (parity entry for the plan).  Outputs (device):
 * exec_of_expert [m], expert_row_off [m], stats (bo_plan_stats, device) and
 * exec_off, a buffer of at least 2*(E+1) + m int32 whose first E+1 entries
 * receive the executor row offsets (the rest is scratch). */
BO_API bo_status bo_plan_from_counts(bo_handle* h, const int32_t* counts, int32_t* exec_of_expert,
                              int32_t* expert_row_off, int32_t* exec_off, void* stats,
                              void* stream);

/* ---------------------------------------------------------------------------
 * Stage entry points of the forward (used by the expert-parallel forward below
 * and available to callers that run the layer in pieces).  Device pointers,
 * stream-ordered.
 * ------------------------------------------------------------------------- */

/* a1-a4 on a local batch: router (Eq. 8), top-K (Eq. 7), per-tile histogram,
 * cnt_i and the per-tile prefix, and Alg. 1 over this batch alone.  Results stay
 * in the workspace at the offsets of bo_workspace_layout(T) (counts, tile_base,
 * topk_id/topk_w, ...).  logits_in as in bo_moe_forward_ex. */
BO_API bo_status bo_route(bo_handle* h, const void* x, int64_t T, const void* Wr, const float* logits_in,
                          void* workspace, size_t ws_bytes, void* stream);

/* a6-a7 on rows already grouped by executor: rows [R, d], row_w [R];
 * exec_off / mtile_off [n_orig + n_united + 1] (row offsets and prefix of
 * ceil(rows/128)); executors [0, n_orig) use Wg/Wu [n_orig, f, d], Wd [n_orig, d, f];
 * executors [n_orig, n_orig + n_united) use UWg/UWu [n_united, f_united, d],
 * UWd [n_united, d, f_united] (f_united <= f, a multiple of 128: expert-parallel
 * f-slices of united experts; SwiGLU is elementwise in f so slice outputs add).
 * h_buf [R, f] scratch; out [R, d] = row_w * FFN(rows). */
BO_API bo_status bo_expert_ffn(bo_handle* h, const void* rows, int64_t R, const float* row_w, const int32_t* exec_off,
                               const int32_t* mtile_off, int32_t n_orig, int32_t n_united, int32_t f_united,
                               const void* Wg, const void* Wu, const void* Wd, const void* UWg, const void* UWu,
                               const void* UWd, void* h_buf, void* out, void* stream);

/* a8: y[t] = [x_t] + sum over (slot, replica) of rows[row_of[(t*K + s)*nrep + r]]
 * in fp32, slot order then replica order (Eq. 5). */
BO_API bo_status bo_combine(bo_handle* h, int64_t T, const void* rows, const int32_t* row_of, int32_t nrep,
                            const void* x, void* y, void* stream);

/* ---------------------------------------------------------------------------
 * Expert parallelism (the paper is silent on
 * communication, its testbed is 4 x A100-PCIe).  One process per GPU,
 * R ranks (1 <= R <= 8, one node).  Tokens are data-parallel: rank r holds its
 * own batch of T_r <= max_tokens tokens (uneven, bursty sizes allowed).  Experts
 * are sharded: original expert e lives on rank floor(e R / m); united expert j
 * (group j) is f-sliced over the distinct owner ranks of its members when
 * every group has the same number of them (SwiGLU is elementwise in f, so the
 * slices' partial outputs add in the combine), else it lives whole on its first
 * member's rank.
 *
 * The brownout plan is global (reading D18): every rank all-gathers the count
 * rows [m + 4] of all ranks (cnt_i of its batch, then T_r, mode and the fp64
 * ratio as two int32 halves), runs Alg. 1 on their sum with RANK 0's knob (so a
 * per-rank SALC loop cannot make ranks disagree), and derives every exchange
 * table on the device.  EP over R ranks therefore computes the single-GPU forward
 * of the rank-order concatenated batch, bit for bit in routing and plan.
 *
 * Exchange buffers (rows of d elements, dtype of the handle, plus one float gate
 * weight per row), all inside the caller's EP workspace:
 *   send    this rank's rows ordered (destination rank, executor, expert, token)
 *   recv    rows of every source, source-major
 *   ret     (aliases recv) weighted FFN outputs in recv's layout, going back
 *   back    (aliases send) outputs returned to this rank, in send's layout
 * Padded mode: the message between every (source, destination) pair is `cap` =
 * max_tokens * K rows at offset q * cap, whatever the plan - no host
 * synchronisation and CUDA-graph capturable (the SURVEY's small-T mode).  Exact
 * mode: messages carry only their rows, contiguous in rank order; the row counts
 * (2R int64) are read by the host once per forward.
 * ------------------------------------------------------------------------- */
typedef struct bo_ep bo_ep;

typedef struct {
  int32_t world;         /* R, 1..8 */
  int32_t rank;          /* this process's rank */
  int32_t padded;        /* 1 padded, 0 exact, -1 auto: padded iff max_tokens * K <= 4096 */
  int64_t max_tokens;    /* largest local batch (<= the handle's max_tokens) */
} bo_ep_config;

typedef struct {
  int32_t world, rank, padded;
  int32_t e0, e1;            /* local original experts [e0, e1) */
  int32_t n_united_local;    /* united f-slices executed here (bo_ep_local_slices) */
  int32_t f_united;          /* their width: ffn / slices per group */
  int32_t nrep;              /* rows per delegated assignment (= slices per united expert) */
  int32_t sliced;            /* 1: united experts f-sliced over their owner ranks */
  int32_t n_exec;            /* virtual executors over all ranks (originals + united slices) */
  int32_t n_local;           /* this rank's executors: (e1 - e0) originals, then n_united_local slices */
  int64_t cap;               /* rows per (source, destination) message in padded mode: max_tokens * K */
  int64_t rows_max;          /* rows of each exchange buffer: R * cap */
} bo_ep_info;

typedef struct {
  size_t total_bytes;
  size_t route;        /* the local route stage's bo_ws_layout workspace (its offsets are relative to here) */
  size_t count_row;    /* int32 [m + 4]     this rank's all-gather input */
  size_t gathered;     /* int32 [R, m + 4]  the all-gather output (every rank's row, rank order) */
  size_t exec_of_expert, expert_row_off, plan_scratch, stats, counts;   /* global plan (Alg. 1) */
  size_t tables;       /* int32 exchange tables (row_base, splits, block tables, exec_off, mtile_off) */
  size_t splits;       /* int64 [2R]        rows sent to / received from each rank */
  size_t send, send_w; /* [rows_max, d], float [rows_max]   (back aliases send) */
  size_t recv, recv_w; /* [rows_max, d], float [rows_max]   (ret aliases recv) */
  size_t grouped, grouped_w;   /* executor-major rows; the GEMM2 output overwrites grouped */
  size_t h;            /* [rows_max, ffn] SwiGLU activations */
  size_t row_of;       /* int32 [max_tokens, K, nrep] send / back row of (token, slot, replica), -1 none */
  int64_t rows_max;
} bo_ep_ws_layout;

/* Static placement alone (host only, no GPU needed): the bo_ep_info fields of
 * rank `rank` (cap / rows_max / padded zero).  BO_ERR_INVALID_ARG for world
 * outside [1, 8] or rank outside [0, world); BO_ERR_SHAPE when the executors
 * exceed the table limits (m <= 256, 512 virtual executors). */
BO_API bo_status bo_ep_placement(int32_t num_experts, int32_t way, int32_t ffn, int32_t world, int32_t rank,
                                 bo_ep_info* out);
/* The (group, slice) of each local united slice, in executor order (n >= n_united_local). */
BO_API bo_status bo_ep_placement_slices(int32_t num_experts, int32_t way, int32_t ffn, int32_t world, int32_t rank,
                                        int32_t* group, int32_t* slice, int32_t n);

/* An EP context on a layer handle (host state only; no device memory). */
BO_API bo_status bo_ep_create(bo_handle* h, const bo_ep_config* cfg, bo_ep** out);
/* Also destroys the NCCL communicator of bo_ep_init.  Destroy every CUDA graph that captured
   bo_ep_forward on this context first: such a graph holds the communicator's persistent NCCL
   resources, and ncclCommDestroy under a live graph blocks (observed on the B200 box). */
BO_API bo_status bo_ep_destroy(bo_ep* ep);
BO_API bo_status bo_ep_get_info(const bo_ep* ep, bo_ep_info* out);
BO_API bo_status bo_ep_workspace_layout(const bo_ep* ep, bo_ep_ws_layout* out);

/* Library-owned communicator: rank 0 calls bo_ep_nccl_unique_id and shares the
 * 128 bytes with every rank (any side channel), then every rank calls bo_ep_init
 * (collective, blocking until all R ranks have joined).  NCCL is loaded at run
 * time (libnccl.so.2); BO_ERR_NCCL if it is missing or a call fails. */
BO_API bo_status bo_ep_nccl_unique_id(unsigned char id[128]);
BO_API bo_status bo_ep_init(bo_ep* ep, const unsigned char nccl_unique_id[128]);

/* The whole EP forward over the library's communicator (after bo_ep_init):
 * x [T, d] local tokens (T <= max_tokens), Wr [m, d]; local weights: originals
 * Wg/Wu [e1-e0, f, d], Wd [e1-e0, d, f]; united slices (bo_ep_placement_slices
 * order) UWg/UWu [n_united_local, f_united, d], UWd [n_united_local, d, f_united]
 * (NULL when n_united_local == 0); y [T, d].  Padded mode: no host
 * synchronisation, graph capturable.  Exact mode: one stream synchronisation. */
BO_API bo_status bo_ep_forward(bo_ep* ep, const void* x, int64_t T, const void* Wr, const void* Wg, const void* Wu,
                               const void* Wd, const void* UWg, const void* UWu, const void* UWd, void* y,
                               void* workspace, size_t ws_bytes, void* stream);

/* The same forward in stages, for callers that run the three exchanges
 * themselves (e.g. torch.distributed):
 *   bo_ep_route     a1-a3 on the local batch -> count_row
 *   (all-gather count_row of every rank into gathered)
 *   bo_ep_dispatch  global Alg. 1, exchange tables, permutation + gather of the
 *                   local rows into send / send_w (a5)
 *   bo_ep_splits    rows per (this rank -> q) and (r -> this rank): exact mode
 *                   reads them (stream synchronisation), padded mode returns cap
 *   (all-to-all send -> recv, send_w -> recv_w with those splits)
 *   bo_ep_compute   regroup, grouped SwiGLU GEMMs x gate weight (a6-a7), back to
 *                   recv's layout in ret
 *   (all-to-all ret -> back, splits swapped)
 *   bo_ep_combine   y_t = [x_t] + sum over slots and slices (a8, Eq. 5) */
BO_API bo_status bo_ep_route(bo_ep* ep, const void* x, int64_t T, const void* Wr, const float* logits_in,
                             void* workspace, size_t ws_bytes, void* stream);
BO_API bo_status bo_ep_dispatch(bo_ep* ep, const void* x, void* workspace, size_t ws_bytes, void* stream);
BO_API bo_status bo_ep_splits(bo_ep* ep, void* workspace, size_t ws_bytes, int64_t* send_rows, int64_t* recv_rows,
                              void* stream);
BO_API bo_status bo_ep_compute(bo_ep* ep, const void* Wg, const void* Wu, const void* Wd, const void* UWg,
                               const void* UWu, const void* UWd, void* workspace, size_t ws_bytes, void* stream);
BO_API bo_status bo_ep_combine(bo_ep* ep, const void* x, void* y, void* workspace, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * United-expert distillation (paper §4.2, Eq. 4 at P:152; SURVEY
 * §8(f) row f4).  For every group j (experts [j*way, min((j+1)*way, m)))
 * the united expert UE_j (student) is trained so that its hidden states match
 * the group's original experts (teacher) under
 *     L^j = (1/k) sum_i || H_u^j - H_o^{j*k+i} ||^2                  (Eq. 4)
 * averaged over the N training tokens (reading D21; k = the group's size),
 * with plain gradient descent on fp32 master weights (D22).  Every group
 * trains on the same token matrix X [N, d] (D23).  Operands are bf16
 * (fp32 accumulation); handles must be BO_BF16.  N must be a positive
 * multiple of 64 (the weight-gradient GEMMs reduce over tokens in 64-token
 * blocks).  Shapes and layouts: X [N, d]; originals Wg/Wu [m, f, d], Wd
 * [m, d, f]; masters UWg_m/UWu_m [G, f, d] and UWd_m [G, d, f] fp32 (caller-
 * owned, updated in place); bf16 copies UWg/UWu [G, f, d], UWd [G, d, f]
 * (caller-owned; these are the united experts bo_moe_forward consumes).
 * ------------------------------------------------------------------------- */
typedef struct {
  size_t total_bytes;
  size_t hbar;     /* f32 [G, N, d]: mean of the group's teacher outputs (the minimiser of Eq. 4) */
  size_t floor_;   /* f64 [G]: variance floor (1/N)(1/k) sum_t sum_i ||Hbar - H_o^i||^2 */
  size_t loss;     /* f64 [G]: Eq. 4 of the weights entering the last bo_distill_step */
  size_t xt;       /* bf16 [d, N]: X^T (weight-gradient operand) */
  size_t teach_h;  /* bf16 [m, N, f]: teacher SwiGLU activations */
  size_t teach_y;  /* f32 [m, N, d]: teacher outputs H_o */
  size_t p, q;     /* bf16 [G, N, f]: student pre-activations X UWg^T, X UWu^T */
  size_t hs;       /* bf16 [G, N, f]: silu(P) * Q */
  size_t hst;      /* bf16 [G, f, N] */
  size_t y;        /* f32 [G, N, d]: student output H_u */
  size_t dy;       /* bf16 [G, N, d]: dL/dH_u = (2/N)(H_u - Hbar) */
  size_t dyt;      /* bf16 [G, d, N] */
  size_t dhs;      /* bf16 [G, N, f] */
  size_t dpt, dqt; /* bf16 [G, f, N]: dL/dP^T, dL/dQ^T */
  size_t uwdt;     /* bf16 [G, f, d]: UWd^T (backward operand), refreshed with the bf16 copies */
  size_t part;     /* f64 partial sums of the reductions */
  size_t off_tok, off_teach, off_f, off_d; /* int32 executor row offsets of the four GEMM schedules */
  int64_t N;
} bo_distill_layout;

BO_API bo_status bo_distill_workspace_layout(const bo_handle* h, int64_t N, bo_distill_layout* out);

/* Once per token set: teacher outputs of all m originals on X (grouped tcgen05
 * GEMMs), their per-group mean Hbar and variance floor, X^T. */
BO_API bo_status bo_distill_prepare(bo_handle* h, const void* X, int64_t N, const void* Wg, const void* Wu,
                                    const void* Wd, void* workspace, size_t ws_bytes, void* stream);

/* Masters <- widen(bf16 united UWg/UWu/UWd) (e.g. the bo_build_united mean
 * initialisation) and UWd^T into the workspace. */
BO_API bo_status bo_distill_load_united(bo_handle* h, int64_t N, const void* UWg, const void* UWu, const void* UWd,
                                        float* UWg_m, float* UWu_m, float* UWd_m, void* workspace, size_t ws_bytes,
                                        void* stream);

/* One gradient-descent step on every group: student forward, Eq. 4 loss
 * (written to layout.loss, before the update), backward, W_m -= lr dL/dW_m
 * (fused into the weight-gradient GEMM epilogue), then the bf16 copies and
 * UWd^T are refreshed from the masters.  X must be the matrix given to
 * bo_distill_prepare.  Requires bo_distill_prepare and bo_distill_load_united
 * (or a previous step) on the same workspace.  No host synchronisation. */
BO_API bo_status bo_distill_step(bo_handle* h, const void* X, int64_t N, float lr, float* UWg_m, float* UWu_m,
                                 float* UWd_m, void* UWg, void* UWu, void* UWd, void* workspace, size_t ws_bytes,
                                 void* stream);

/* Optional per-kernel timing: when `events` (an array of n cudaEvent_t cast
 * to void*) is non-NULL, each following forward records events[i] on its
 * stream immediately before its i-th kernel launch and events[L] after the
 * last one (L = launch count; requires n >= L + 1, else the events are not
 * recorded); a NULL entry skips that boundary (e.g. only the two events around
 * one kernel).  Pass NULL to disable.  The events stay owned by the caller. */
BO_API bo_status bo_set_profile_events(bo_handle* h, void** events, int32_t n);

/* Number of GPU kernels the last forward on this handle enqueued. */
BO_API int32_t bo_last_launch_count(const bo_handle* h);
/* Names of those kernels in launch order, comma-separated (e.g.
 * "router_topk,plan,permute,gather,gemm1_swiglu,gemm2_weighted_combine"; a
 * "_combine" suffix marks GEMM2 with the combine, a8, fused into its epilogue).
 * Owned by the handle, valid until its next forward / bo_route / bo_expert_ffn. */
BO_API const char* bo_last_kernels(const bo_handle* h);

BO_API const char* bo_status_string(bo_status s);
BO_API const char* bo_last_error(void);
BO_API const char* bo_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BROWNOUT_H_ */
