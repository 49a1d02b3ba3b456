// bo_gemm.cu - persistent, warp-specialised grouped GEMM on tcgen05 / TMEM / TMA.
//
// One engine serves the three dense contractions of the brownout MoE forward:
//   router   (Eq. 8):  logits[T, m]  = x  Wr^T                (EPI_ROUTER, top-K fused)
//   GEMM1    (Eq. 5 FFN, SwiGLU, D13): H[r] = silu(Xp[r] Wg_x^T) * (Xp[r] Wu_x^T)  (EPI_SWIGLU)
//   GEMM2    (Eq. 5-6):       Yp[r] = row_w[r] * (H[r] Wd_x^T)          (EPI_WEIGHTED)
// where x is the executor (original expert or united expert, Alg. 1)
// that owns row r.  Executor row ranges come from the device-side plan
// (exec_off / mtile_off), so no host synchronisation is needed.
//
// CTA layout (192 threads, 1 CTA per SM, persistent over a static round-robin
// work list; split-K for decode-sized GEMM2 steps):
//   warp 0      TMA producer: A tile [128 x BK] + B tile [BN x BK] per stage
//   warp 1      MMA issuer: tcgen05.mma.cta_group::1 M=128 N=BN K=16(bf16)/8(tf32)
//               into a double-buffered TMEM accumulator (2 x BN fp32 columns)
//   warps 2-5   epilogue: tcgen05.ld 32x32b -> registers -> fused op -> global
// Work item w -> (executor x, n-tile, m-tile) with the m-tile fastest, so
// concurrently running CTAs share the same weight tile (B) through L2.
#include <atomic>

#include "bo_kernels.h"
#include "bo_ptx.cuh"

namespace bo {

template <int BN, int EPI>
struct GemmShape {
  static constexpr int kTmemCols = (2 * BN + (BN < 32 ? 32 : 0)) <= 32    ? 32
                                   : (2 * BN + (BN < 32 ? 32 : 0)) <= 64  ? 64
                                   : (2 * BN + (BN < 32 ? 32 : 0)) <= 128 ? 128
                                   : (2 * BN + (BN < 32 ? 32 : 0)) <= 256 ? 256
                                                                          : 512;
};

// Work items per unit whose (executor, m-tile, n-tile, split) is decoded once in the prologue
// (later items, if any, are decoded when reached).
constexpr int kSchedItems = 256;

template <typename T, int BN, int CG = 1>
struct GemmCfg {
  static constexpr int BM = kBM;                         // rows per CTA (the pair covers CG * 128)
  static constexpr int BK = 128 / (int)sizeof(T);       // one 128-byte swizzle row
  static constexpr int UK = 32 / (int)sizeof(T);        // MMA K per instruction
  static constexpr int A_BYTES = BM * 128;
  static constexpr int B_BYTES = (BN / CG) * 128;       // each CTA of a pair holds half of B
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_BYTES = 1024;                 // mbarriers + TMEM slot
  // executor offsets + m-tile prefix, then this unit's packed work list (keeps the staging 16B-aligned)
  static constexpr int SCHED_BYTES = ((2 * (kMaxExec + 1) + kSchedItems) * 4 + 127) / 128 * 128;
  static constexpr int EPI_ROW = 32 * (int)sizeof(T) + 16;   // staged 32-column row chunk + bank pad
  static constexpr int EPI_BYTES = 4 * 32 * EPI_ROW          // one staging tile per epilogue warp
                                   + 1024 + 4 * 4096;          // + two dense 2 KB TMA-store boxes per warp (1 KB aligned)
  static constexpr int OTHER = 1024 /*align slack*/ + BAR_BYTES + SCHED_BYTES + EPI_BYTES;
  static constexpr int STAGES_RAW = (227 * 1024 - OTHER) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int SMEM = OTHER + STAGES * STAGE_BYTES;
};

// silu(g) = g / (1 + e^-g).  __fdividef, not the IEEE division: the latter's
// out-of-line slow-path code made a single-tile SwiGLU epilogue take ~12 us
// (in-kernel globaltimer probe, tiny layer); __fdividef is within 2 ulp and returns
// 0 for the huge denominators of g < -87, where silu(g) underflows anyway.
__device__ __forceinline__ float silu_f(float g) { return __fdividef(g, 1.0f + __expf(-g)); }

// Coalesced epilogue store of a 32-row x 32-column chunk owned by one warp
// (thread = row, as tcgen05.ld 32x32b delivers it): rows are staged in the
// warp's shared-memory tile (16-byte pad -> conflict-free), then written back
// as whole 64/128-byte row segments, several rows per store instruction.
template <typename T>
__device__ __forceinline__ void stage_row32(uint8_t* stage, int lane, const float (&v)[32]) {
  constexpr int ROW = 32 * (int)sizeof(T) + 16;
  uint4* d = reinterpret_cast<uint4*>(stage + lane * ROW);
  if constexpr (sizeof(T) == 2) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 u;
      u.x = pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
      u.y = pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
      u.z = pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
      u.w = pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
      d[q] = u;
    }
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      d[q] = make_uint4(__float_as_uint(v[4 * q]), __float_as_uint(v[4 * q + 1]), __float_as_uint(v[4 * q + 2]),
                        __float_as_uint(v[4 * q + 3]));
  }
}
// rows of the warp: global row index = row0 + r (r < nrows valid), column offset col0.
// The lane's first row address is formed once; later rows add a uniform stride, and
// every store carries the L2 policy `pol` (evict_normal when no hint is wanted), so
// the loop holds no 64-bit row multiply and no per-store policy branch (the C4 GEMM2
// epilogue, 12 k-blocks per tile, was bound by these instructions: ncu source page).
template <typename T>
__device__ __forceinline__ void flush_rows32(const uint8_t* stage, int lane, T* out, int64_t row0, int nrows,
                                             int64_t ldo, int vmax, uint64_t pol) {
  constexpr int V16 = 32 * (int)sizeof(T) / 16;   // 16-byte pieces per row chunk
  constexpr int ROW = 32 * (int)sizeof(T) + 16;
  constexpr int RPI = 32 / V16;                    // rows per store instruction
  const int piece = lane % V16;
  const int rf = lane / V16;
  T* base = out + (row0 + rf) * ldo + piece * (16 / (int)sizeof(T));
  const int64_t step = static_cast<int64_t>(RPI) * ldo;
#pragma unroll
  for (int i = 0; i < V16; ++i) {
    const int r = i * RPI + rf;
    if (r < nrows && piece < vmax) {
      const uint4 v = *reinterpret_cast<const uint4*>(stage + r * ROW + piece * 16);
      st_global_hint(base + i * step, v, pol);
    }
  }
}

template <typename T>
__device__ __forceinline__ void store_row32(T* dst, const float (&v)[32]);

template <>
__device__ __forceinline__ void store_row32<__nv_bfloat16>(__nv_bfloat16* dst, const float (&v)[32]) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 u;
    u.x = pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
    u.y = pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
    u.z = pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
    u.w = pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
    d[q] = u;
  }
}
template <>
__device__ __forceinline__ void store_row32<float>(float* dst, const float (&v)[32]) {
  float4* d = reinterpret_cast<float4*>(dst);
#pragma unroll
  for (int q = 0; q < 8; ++q) d[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
}

// dst += v; v <- the updated values
__device__ __forceinline__ void add_row32(float* dst, float (&v)[32]) {
  float4* d = reinterpret_cast<float4*>(dst);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 o = d[q];
    v[4 * q] += o.x;
    v[4 * q + 1] += o.y;
    v[4 * q + 2] += o.z;
    v[4 * q + 3] += o.w;
    d[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  }
}

// Running top-K list, (value desc, id asc); ids arrive in ascending order so a
// new element only overtakes strictly smaller values (reading D8).  (A select-only
// variant that kept all KMAX slots from -inf returned duplicated ids on the m = 32
// tcgen05 router of tests/test_gpu_router_exact.py although the same function is
// exact in isolation on the device (scripts/topk_check.cu); this form stays.)
template <int KMAX>
__device__ __forceinline__ void topk_insert(float (&tv)[KMAX], int (&ti)[KMAX], int K, float v, int e) {
#pragma unroll
  for (int j = KMAX - 1; j >= 0; --j) {
    if (j < K) {
      const bool b_j = ti[j] < 0 || v > tv[j];
      const bool b_jm1 = j > 0 && (ti[j - 1] < 0 || v > tv[j - 1]);
      if (b_j) {
        if (b_jm1) { tv[j] = tv[j - 1]; ti[j] = ti[j - 1]; }
        else { tv[j] = v; ti[j] = e; }
      }
    }
  }
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
// two epilogue warps (swapped tail tiles: the gate warp and the up warp of the same columns)
__device__ __forceinline__ void pair_bar(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }

// 16-byte vector <-> fp32 (8 bf16 or 4 fp32 elements); loads bypass L1 (rows
// written by other CTAs of the same kernel).
template <typename T>
__device__ __forceinline__ void unpack16(const uint4& u, float (&f)[16 / sizeof(T)]) {
  if constexpr (sizeof(T) == 2) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 t = __bfloat1622float2(h[i]);
      f[2 * i] = t.x;
      f[2 * i + 1] = t.y;
    }
  } else {
    f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
  }
}
template <typename T>
__device__ __forceinline__ void ld16_cg(const T* p, float (&f)[16 / sizeof(T)]) {
  unpack16<T>(__ldcg(reinterpret_cast<const uint4*>(p)), f);
}
template <typename T>
__device__ __forceinline__ void st16(T* p, const float (&f)[16 / sizeof(T)]) {
  uint4 u;
  if constexpr (sizeof(T) == 2) {
    u.x = pack_bf16x2(f[0], f[1]); u.y = pack_bf16x2(f[2], f[3]);
    u.z = pack_bf16x2(f[4], f[5]); u.w = pack_bf16x2(f[6], f[7]);
  } else {
    u = make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
  }
  *reinterpret_cast<uint4*>(p) = u;
}

// Eq. 5 sum for token t over columns [c0, c0 + ncols) by one warp:
// y[t] = [x[t]] + sum over the token's rows in slot order (rows < 0 skipped),
// fp32 accumulation of the stored (rounded) Yp values - the order and
// arithmetic of k_combine, so fused and separate combines agree bitwise.
// The same Eq. 5 sum for every token of the warp's `done` mask over columns
// [c0, c0 + ncols).  Lane i holds token t_lane and its row indices rr[] (slot
// order) when bit i is set.  The warp's (token, 16-byte vector) items are
// spread over the lanes, U items per lane at a time, the row indices arrive by
// shuffle and all KRB row loads of the U items are issued before the in-order
// accumulation, so a warp keeps U * KRB loads in flight (one round trip per
// batch instead of one per token and slot).
constexpr int kCombSlots = 16;   // max row slots per token on the fused path (host falls back above)
template <typename T, int KRB, int U>
__device__ __forceinline__ void combine_tokens_batched(const GemmParams& p, const T* yp, int64_t ldy, uint32_t done,
                                                       int t_lane, const int (&rr)[kCombSlots], int c0, int ncols,
                                                       int lane) {
  constexpr int EV = 16 / (int)sizeof(T);
  const int nv = ncols / EV;
  const int nitems = __popc(done) * nv;
  for (int base = 0; base < nitems; base += 32 * U) {
    int src[U], vec[U], tok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int it = base + u * 32 + lane;
      const int k = it < nitems ? it / nv : 0;
      vec[u] = it < nitems ? it - k * nv : -1;
      src[u] = __fns(done, 0, k + 1);
      tok[u] = __shfl_sync(0xffffffffu, t_lane, src[u]);
    }
    float acc[U][EV];
    uint4 xr[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (vec[u] >= 0 && p.add_residual)
        xr[u] = __ldcg(reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(p.comb_x) +
                                                      static_cast<int64_t>(tok[u]) * p.comb_d + c0 + vec[u] * EV));
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (vec[u] >= 0 && p.add_residual) {
        unpack16<T>(xr[u], acc[u]);
      } else {
#pragma unroll
        for (int k = 0; k < EV; ++k) acc[u][k] = 0.0f;
      }
    }
#pragma unroll
    for (int s0 = 0; s0 < kCombSlots; s0 += KRB) {
      if (s0 >= p.comb_KR) break;   // warp-uniform
      int r[U][KRB];
      uint4 raw[U][KRB];
#pragma unroll
      for (int j = 0; j < KRB; ++j)
#pragma unroll
        for (int u = 0; u < U; ++u) r[u][j] = __shfl_sync(0xffffffffu, rr[s0 + j], src[u]);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < KRB; ++j)
          if (vec[u] >= 0 && r[u][j] >= 0)
            raw[u][j] = __ldcg(reinterpret_cast<const uint4*>(yp + static_cast<int64_t>(r[u][j]) * ldy + c0 +
                                                              vec[u] * EV));
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < KRB; ++j)
          if (vec[u] >= 0 && r[u][j] >= 0) {   // slot order (Eq. 5 sum), as k_combine
            float f[EV];
            unpack16<T>(raw[u][j], f);
#pragma unroll
            for (int k = 0; k < EV; ++k) acc[u][k] += f[k];
          }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (vec[u] >= 0)
        st16<T>(reinterpret_cast<T*>(p.comb_y) + static_cast<int64_t>(tok[u]) * p.comb_d + c0 + vec[u] * EV, acc[u]);
  }
}

template <typename T>
__device__ __forceinline__ void combine_token_cols(const GemmParams& p, const T* yp, int64_t ldy, int t, int c0,
                                                   int ncols, int lane) {
  constexpr int EV = 16 / (int)sizeof(T);
  const int nv = ncols / EV;
  const int32_t* ro = p.row_of + static_cast<int64_t>(t) * p.comb_KR;
  const T* xr = reinterpret_cast<const T*>(p.comb_x) + static_cast<int64_t>(t) * p.comb_d + c0;
  T* yr = reinterpret_cast<T*>(p.comb_y) + static_cast<int64_t>(t) * p.comb_d + c0;
  for (int v = lane; v < nv; v += 32) {
    float acc[EV];
    if (p.add_residual) {
      ld16_cg<T>(xr + v * EV, acc);
    } else {
#pragma unroll
      for (int k = 0; k < EV; ++k) acc[k] = 0.0f;
    }
    for (int sl = 0; sl < p.comb_KR; ++sl) {
      const int r = __ldg(ro + sl);
      if (r >= 0) {
        float u[EV];
        ld16_cg<T>(yp + static_cast<int64_t>(r) * ldy + c0 + v * EV, u);
#pragma unroll
        for (int k = 0; k < EV; ++k) acc[k] += u[k];
      }
    }
    st16<T>(yr + v * EV, acc);
  }
}

#ifdef BO_PROBE
// Instrumentation build only (build.py --variant probe): per (launch class, CTA, work item)
// globaltimer stamps [producer starts the tile, MMA has its first stage, MMA committed the
// last k-block, epilogue done, MMA has the accumulator (tempty), producer issued the first
// k-block (empty slot)] and the tile id (x | mi << 10 | n << 16).
constexpr int kProbeCtas = 160, kProbeItems = 48;
__device__ unsigned long long g_probe[2][kProbeCtas][kProbeItems][6];
__device__ int g_probe_id[2][kProbeCtas][kProbeItems];
#define BO_STAMP(j, k)                                                                      \
  do {                                                                                      \
    if (blockIdx.x < kProbeCtas && (j) < kProbeItems)                                       \
      g_probe[EPI == EPI_SWIGLU ? 0 : 1][blockIdx.x][(j)][(k)] = globaltimer_ns();          \
  } while (0)
#else
#define BO_STAMP(j, k) \
  do {                 \
  } while (0)
#endif

template <typename T, int BN, int EPI, int KMAX, int CG>
__global__ void __launch_bounds__(192, 1)
    k_grouped_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ BMaps tmB, const GemmParams p) {
  // CG = 1: one CTA computes a 128 x BN tile with tcgen05.mma.cta_group::1.
  // CG = 2: a CTA pair (cluster of 2) computes a 256 x BN tile with
  //         tcgen05.mma.cta_group::2 issued by the leader: each CTA stages its
  //         128 rows of A and half of B (BN/2 rows), halving the shared-memory
  //         and L2 traffic per MMA; each CTA's TMEM holds its 128 rows.
  static_assert(CG == 1 || (CG == 2 && EPI != EPI_ROUTER && sizeof(T) == 2), "pair mode: bf16 FFN GEMMs");
  using C = GemmCfg<T, BN, CG>;
  constexpr int STAGES = C::STAGES;
  constexpr int TMEM_COLS = GemmShape<BN, EPI>::kTmemCols;
  constexpr uint32_t IDESC = idesc_f32acc<T>(128 * CG, BN);
  constexpr int TILE_M = kBM * CG;

  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned (SWIZZLE_128B atoms); offset arithmetic on the __shared__
  // array keeps the shared address space visible to the compiler (LDS/STS for the
  // epilogue staging instead of generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  uint64_t* fix_bar = tempty_bar + 3;   // last-wave split: a contributor's partial landed in the (idle) ring
  int* s_mtile = reinterpret_cast<int*>(smem + STAGES * C::STAGE_BYTES + C::BAR_BYTES);
  int* s_eoff = s_mtile + (kMaxExec + 1);
  int* s_sched = s_eoff + (kMaxExec + 1);   // [kSchedItems] this unit's decoded work list
  uint8_t* s_epi = smem + STAGES * C::STAGE_BYTES + C::BAR_BYTES + C::SCHED_BYTES;
  // per-warp 4 KB region (1 KB aligned): TMA-store boxes (GEMM2), swizzled logits staging (router)
  uint8_t* s_box = smem + ((STAGES * C::STAGE_BYTES + C::BAR_BYTES + C::SCHED_BYTES + 4 * 32 * C::EPI_ROW + 1023) & ~1023);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = CG == 2 ? cluster_ctarank() : 0u;
  const bool leader = crank == 0;
  const int unit = CG == 2 ? (blockIdx.x >> 1) : blockIdx.x;       // work-unit (CTA or CTA pair) index
  const int n_units = CG == 2 ? (gridDim.x >> 1) : gridDim.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], CG);         // pair: both producers arrive on the leader's barrier
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 4 * CG);   // pair: epilogue warps of both CTAs arrive on the leader's
    }
    mbar_init(fix_bar, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    for (int i = 0; i < 6; ++i) tma_prefetch_desc(&tmB.m[i]);
    if (p.bh_alt > 0 || p.swap_tail)
      for (int i = 6; i < (p.swap_tail ? 15 : 12); ++i) tma_prefetch_desc(&tmB.m[i]);
  }
  if constexpr (CG == 2) cluster_sync();   // peer barriers initialised before any remote arrive / alloc
  if (warp == 1) {
    if constexpr (CG == 2) {
      tmem_alloc_pair(tmem_slot, TMEM_COLS);
      tmem_relinquish_pair();
    } else {
      tmem_alloc(tmem_slot, TMEM_COLS);
      tmem_relinquish();
    }
  }
  // Programmatic dependent launch: everything above (barriers, TMEM, descriptor
  // prefetch) may overlap the previous kernel's tail; no global memory is touched
  // before the previous kernel has completed and flushed.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // ... and let the next kernel (if launched programmatically) start its own prologue
  // on the SMs this grid frees in its tail; it still waits for this grid to finish.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // executor row offsets and the prefix of TILE_M-row m-tiles (warp 2, shuffle scan)
  const int nexec = p.single_rows >= 0 ? 1 : p.num_exec;
  if (p.single_rows >= 0) {
    if (threadIdx.x == 0) {
      s_eoff[0] = 0;
      s_eoff[1] = p.single_rows;
    }
  } else {
    for (int i = threadIdx.x; i <= nexec; i += blockDim.x) s_eoff[i] = p.exec_off[i];
  }
  __syncthreads();
  if (warp == 2) {
    int carry = 0;
    for (int i0 = 0; i0 < nexec; i0 += 32) {
      const int i = i0 + lane;
      const int v = i < nexec ? (s_eoff[i + 1] - s_eoff[i] + TILE_M - 1) / TILE_M : 0;
      int incl = v;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
      }
      if (i < nexec) s_mtile[i] = carry + incl - v;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) s_mtile[nexec] = carry;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // Executor classes: originals [0, mo), united [mo, mu), shared [mu, nexec).
  // United experts may differ in n-tiles, reduction length and B rows
  // (expert-parallel f-slices); shared experts have the originals' shape.
  const int mo = p.m_orig < nexec ? p.m_orig : nexec;
  const int mu = mo + p.m_united < nexec ? mo + p.m_united : nexec;
  int nt_o = p.n_tiles, nt_u = p.n_tiles_u;
  auto start_of = [&](int x) {
    const int a = x < mo ? x : mo;                      // min(x, mo)
    const int b = x < mo ? mo : (x < mu ? x : mu);      // clamp(x, mo, mu)
    const int c = x < mu ? mu : x;                      // max(x, mu)
    return nt_o * s_mtile[a] + nt_u * (s_mtile[b] - s_mtile[mo]) + nt_o * (s_mtile[c] - s_mtile[mu]);
  };
  // SwiGLU tile width: BN (gate + up columns) or the alternative 2 * bh_alt, whichever
  // needs fewer tile-column waves over the persistent grid: decode-sized steps have
  // few m-tiles, and the last partial wave of BN-wide tiles can idle most SMs.
  int bh = BN / 2;
  bool alt = false;
  if constexpr (EPI == EPI_SWIGLU) {
    if (p.bh_alt > 0) {
      const int items_p = start_of(nexec);
      nt_o = p.nt_alt;
      nt_u = p.nt_alt_u;
      const int items_a = start_of(nexec);
      auto waves = [&](int items) -> long long { return (items + n_units - 1) / n_units; };
      alt = waves(items_a) * (2 * p.bh_alt + 32) < waves(items_p) * (BN + 32);
      if (alt) {
        bh = p.bh_alt;
      } else {
        nt_o = p.n_tiles;
        nt_u = p.n_tiles_u;
      }
    }
  }
  const uint32_t idesc = alt ? idesc_f32acc<T>(128 * CG, 2 * bh) : IDESC;
  // Swapped-operand tail tile (CTA pairs, SwiGLU): an executor's last m-tile holding
  // rin < 256 rows computes D^T = [Wg; Wu] Xp^T instead, with this CTA's 64 gate and
  // 64 up weight rows on the MMA's M side (TMEM lanes 0-63 gate, 64-127 up of the same
  // columns) and the tile's rows, rounded up to 32, on N (each CTA stages half of
  // them).  The MMA and the shared-memory traffic then scale with rin instead of a
  // full 256-row tile.  Three TMA boxes per k-block (gate, up, rows): the TMA issue
  // cost of 16-row boxes (8-12 per k-block) made such a tile slower than a full one.
  constexpr bool kSwap = CG == 2 && EPI == EPI_SWIGLU;
  const bool swap_ok = kSwap && p.swap_tail && !alt && !p.a_shared;
  auto tile_rows = [&](int x, int mi) {   // rows of executor x in m-tile mi
    const int r = s_eoff[x + 1] - s_eoff[x] - mi * TILE_M;
    return r < TILE_M ? r : TILE_M;
  };
  auto swapped_tile = [&](int x, int mi) { return swap_ok && tile_rows(x, mi) < TILE_M; };
  const int stage_tx = C::A_BYTES + (EPI == EPI_SWIGLU ? 2 * bh : BN) * 128 / CG;   // bytes per CTA per stage
  const int base_work = start_of(nexec);
  auto kblocks = [&](int x) { return (x < mo || x >= mu ? p.Kdim : p.Kdim_u) / C::BK; };
  // Split-K (GEMM2, few rows): when the tiles would leave SMs idle, each tile's
  // reduction is cut into ks contiguous k-block ranges written as fp32 partials
  // (summed, in split order, by the combine).  ks is a function of the plan only.
  int ks = 1;
  if constexpr (EPI == EPI_WEIGHTED) {
    if (p.ksplit_max > 1 && base_work > 0) {
      // the split count with the least time per unit of work, ceil(items * ks / units) / ks
      // (fewest splits on ties: each split adds an fp32 partial of the tile)
      const int kmin = (p.Kdim < p.Kdim_u ? p.Kdim : p.Kdim_u) / C::BK;
      const int kmax = p.ksplit_max < kmin ? p.ksplit_max : kmin;
      long long best_num = (base_work + n_units - 1) / n_units, best_den = 1;
      for (int k = 2; k <= kmax; ++k) {
        const long long w = (static_cast<long long>(base_work) * k + n_units - 1) / n_units;
        if (w * best_den < best_num * k) { best_num = w; best_den = k; ks = k; }
      }
    }
    if (p.ksplit_max > 1 && blockIdx.x == 0 && threadIdx.x == 0) *p.ks_out = ks;
  }
  const int total_work = base_work * ks;
  // Last-wave split (GEMM2 on CTA pairs, GemmParams::tail_split): the X = tiles mod units
  // tiles of a partial last wave are not handed out whole; their X * nkb k-blocks are shared
  // out evenly over ALL units after each unit's whole tiles (units u take [U u / n, U (u+1) / n)).
  // A share (>= 8 k-blocks, < nkb) covers at most two tiles, so a unit holds at most one
  // contributor piece (a tile's later k-blocks: fp32 partial to sk_part[blockIdx], counted in
  // sk_flag[blockIdx]) and one finishing piece (from k-block 0: it adds the partials of the
  // following units holding the tile's other pieces, in unit order, then runs the epilogue).
  // Only for long reductions (>= 64 k-blocks per tile, e.g. C2's 224), where a piece's
  // 128 KB partial is small against its work.
  int tsx = 0;          // tiles of the split last wave
  int nkb_t = 0;
  int64_t tsU = 0;      // their k-blocks
  if constexpr (EPI == EPI_WEIGHTED && CG == 2) {
    if (p.tail_split && p.sk_part && ks == 1 && p.Kdim == p.Kdim_u && !p.f32_mode) {
      nkb_t = p.Kdim / C::BK;
      const int X = base_work % n_units;
      if (nkb_t >= 64 && X > 0 && static_cast<int64_t>(X) * nkb_t >= 8LL * n_units) {
        tsx = X;
        tsU = static_cast<int64_t>(X) * nkb_t;
      }
    }
  }
  const int n_whole = base_work - tsx;   // tiles handed out whole, round robin
  const int n_my_whole = n_whole > unit ? (n_whole - unit + n_units - 1) / n_units : 0;
  auto ts_lo = [&](int u) { return tsU * u / n_units; };   // first split k-block of unit u
  enum { SEG_FULL = 0, SEG_FINISH = 1, SEG_CONTRIB = 2 };
  // s-th segment of this unit: work item w, k-block override [s0, s1) (tail pieces) and kind
  auto segment = [&](int s, int& w, int& s0, int& s1, int& kind) -> bool {
    kind = SEG_FULL;
    if (!tsx) {
      w = unit + s * n_units;
      return w < total_work;
    }
    if (s < n_my_whole) {
      w = unit + s * n_units;
      return true;
    }
    const int64_t lo = ts_lo(unit), hi = ts_lo(unit + 1);
    const int64_t i = lo / nkb_t + (s - n_my_whole);
    if (i * nkb_t >= hi) return false;
    w = n_whole + static_cast<int>(i);
    const int64_t a = lo - i * nkb_t, b = hi - i * nkb_t;
    s0 = a > 0 ? static_cast<int>(a) : 0;
    s1 = b < nkb_t ? static_cast<int>(b) : nkb_t;
    kind = s0 > 0 ? SEG_CONTRIB : (s1 < nkb_t ? SEG_FINISH : SEG_FULL);
    return true;
  };

  // work item -> tile (executor x, m-tile mi fastest, n-tile n) + k-block range
  // [kb0, kb1) of split sp; units take items unit, unit + n_units, ... (the
  // concurrently running CTAs share each weight tile through L2)
  auto decode = [&](int w, int& x, int& mi, int& n, int& sp, int& kb0, int& kb1) {
    const int tw = w / ks;
    sp = w - tw * ks;
    int lo = 0, hi = nexec;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (start_of(mid) <= tw) lo = mid; else hi = mid;
    }
    x = lo;
    const int mt = s_mtile[x + 1] - s_mtile[x];
    const int local = tw - start_of(x);
    n = local / mt;
    mi = local - n * mt;
    const int nkb = kblocks(x);
    const int per = (nkb + ks - 1) / ks;
    kb0 = sp * per < nkb ? sp * per : nkb;
    kb1 = kb0 + per < nkb ? kb0 + per : nkb;
  };
  // This unit's work list, decoded by all threads at once: the binary search over the
  // executors sat on the MMA warp's critical path between tiles (0.5-0.9 us per tile with
  // 5-57 executors, probe build), ~10 % of a 12-k-block C4 GEMM2 tile.  Packed as
  // x | mi << 10 | n << 20 | sp << 29; -1 = decode when reached (a field does not fit).
  // (with the last-wave split only the whole tiles are listed; the pieces decode when reached)
  const int n_my = tsx ? n_my_whole : (total_work > unit ? (total_work - unit + n_units - 1) / n_units : 0);
  const int n_tab = n_my < kSchedItems ? n_my : kSchedItems;
  {
    for (int j = threadIdx.x; j < n_tab; j += blockDim.x) {
      int x, mi, n, sp, a, b;
      decode(unit + j * n_units, x, mi, n, sp, a, b);
      s_sched[j] = (x < 1024 && mi < 1024 && n < 512 && sp < 4) ? (x | (mi << 10) | (n << 20) | (sp << 29)) : -1;
    }
    __syncthreads();
  }
  auto item_at = [&](int j, int w, int& x, int& mi, int& n, int& sp, int& kb0, int& kb1) {
    const int e = j < n_tab ? s_sched[j] : -1;
    if (e < 0) {
      decode(w, x, mi, n, sp, kb0, kb1);
      return;
    }
    x = e & 1023;
    mi = (e >> 10) & 1023;
    n = (e >> 20) & 511;
    sp = e >> 29;
    const int nkb = kblocks(x);
    if (ks == 1) {
      kb0 = 0;
      kb1 = nkb;
    } else {
      const int per = (nkb + ks - 1) / ks;
      kb0 = sp * per < nkb ? sp * per : nkb;
      kb1 = kb0 + per < nkb ? kb0 + per : nkb;
    }
  };

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      // activations are re-read per n-tile (evict_last); the weight tile is re-read by the
      // executor's other m-tiles running alongside (b_policy 1: evict_first for decode-sized
      // steps, where the streamed weights should make way for the re-read activations)
      const uint64_t pol_a = policy_evict_last();
      const uint64_t pol_b = p.b_policy == 1 ? policy_evict_first() : policy_evict_normal();
      int stage = 0;
      uint32_t phase = 0;
      int x, mi, n, sp, kb0, kb1;
      int w, s0 = 0, s1 = 0, kind;
      for (int item = 0; segment(item, w, s0, s1, kind); ++item) {
        item_at(item, w, x, mi, n, sp, kb0, kb1);
        if (item >= n_my_whole && tsx) { kb0 = s0; kb1 = s1; }
        BO_STAMP(item, 0);
#ifdef BO_PROBE
        if (blockIdx.x < kProbeCtas && item < kProbeItems)
          g_probe_id[EPI == EPI_SWIGLU ? 0 : 1][blockIdx.x][item] = x | (mi << 10) | (n << 16);
#endif
        const int arow = (p.a_shared ? 0 : s_eoff[x]) + mi * TILE_M + static_cast<int>(crank) * kBM;
        const int cls = x < mo ? 0 : (x < mu ? 1 : 2);      // original / united / shared
        const CUtensorMap* mb0 = &tmB.m[(alt ? 6 : 0) + 2 * cls];
        const CUtensorMap* mb1 = &tmB.m[(alt ? 6 : 0) + 2 * cls + 1];
        const int brow = cls == 0 ? x * p.b_rows_per_exec
                                  : (cls == 1 ? (x - mo) * p.b_rows_u : (x - mu) * p.b_rows_per_exec);
        if constexpr (kSwap) {
          if (swapped_tile(x, mi)) {
            const int rin = tile_rows(x, mi);
            const int nsh = ((rin + 31) & ~31) / 2;   // token rows staged by this CTA (N / 2)
            const int wrow = brow + n * 128 + static_cast<int>(crank) * 64;
            const int trow = s_eoff[x] + mi * TILE_M + static_cast<int>(crank) * nsh;
            // one box of >= nsh rows (16 / 32 / 64 / 128; rows past nsh land unused)
            const int tbox = nsh <= 16 ? 16 : (nsh <= 32 ? 32 : (nsh <= 64 ? 64 : 128));
            const CUtensorMap* mt = tbox == 128 ? &tmA : &tmB.m[tbox == 16 ? 12 : (tbox == 32 ? 13 : 14)];
            for (int kb = kb0; kb < kb1; ++kb) {
              mbar_wait(&empty_bar[stage], phase ^ 1);
              uint8_t* sa = smem + stage * C::STAGE_BYTES;
              if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * (C::A_BYTES + tbox * 128));
              else mbar_arrive_remote(&full_bar[stage], 0);
              tma_load_2d_pair(sa, &tmB.m[6 + 2 * cls], &full_bar[stage], kb * C::BK, wrow, pol_b);
              tma_load_2d_pair(sa + 64 * 128, &tmB.m[7 + 2 * cls], &full_bar[stage], kb * C::BK, wrow, pol_b);
              tma_load_2d_pair(sa + C::A_BYTES, mt, &full_bar[stage], kb * C::BK, trow, pol_a);
              if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
            continue;
          }
        }
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          if (kb == kb0) BO_STAMP(item, 5);
          uint8_t* sa = smem + stage * C::STAGE_BYTES;
          uint8_t* sb = sa + C::A_BYTES;
          if constexpr (CG == 1) {
            mbar_arrive_expect_tx(&full_bar[stage], stage_tx);
            tma_load_2d(sa, &tmA, &full_bar[stage], kb * C::BK, arow, pol_a);
            if constexpr (EPI == EPI_SWIGLU) {
              tma_load_2d(sb, mb0, &full_bar[stage], kb * C::BK, brow + n * bh, pol_b);
              tma_load_2d(sb + bh * 128, mb1, &full_bar[stage], kb * C::BK, brow + n * bh, pol_b);
            } else {
              tma_load_2d(sb, mb0, &full_bar[stage], kb * C::BK, brow + n * BN, pol_b);
            }
          } else {
            // Both CTAs load their halves; completion is counted on the leader's barrier.
            if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * stage_tx);
            else mbar_arrive_remote(&full_bar[stage], 0);
            tma_load_2d_pair(sa, &tmA, &full_bar[stage], kb * C::BK, arow, pol_a);
            if constexpr (EPI == EPI_SWIGLU) {
              // leader: gate rows, peer: up rows of the same f-columns -> D[:, 0:BN/2] = gate, D[:, BN/2:] = up
              tma_load_2d_pair(sb, leader ? mb0 : mb1, &full_bar[stage], kb * C::BK, brow + n * bh, pol_b);
            } else {
              tma_load_2d_pair(sb, mb0, &full_bar[stage], kb * C::BK,
                               brow + n * BN + static_cast<int>(crank) * (BN / 2), pol_b);
            }
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // --------------------------------------------------------- MMA issuer
    if (lane == 0 && leader) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int x, mi, n, sp, kb0, kb1;
      int w, s0 = 0, s1 = 0, kind;
      int item = 0;
      for (; segment(item, w, s0, s1, kind); ++item) {
        item_at(item, w, x, mi, n, sp, kb0, kb1);
        if (item >= n_my_whole && tsx) { kb0 = s0; kb1 = s1; }
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        BO_STAMP(item, 4);
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
        uint32_t idesc_t = idesc;
        if constexpr (kSwap) {
          if (swapped_tile(x, mi)) idesc_t = idesc_f32acc<T>(256, (tile_rows(x, mi) + 31) & ~31);
        }
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          if (kb == kb0) BO_STAMP(item, 1);
          const uint32_t a_addr = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t b_addr = a_addr + C::A_BYTES;
#pragma unroll
          for (int k = 0; k < C::BK / C::UK; ++k) {
            const uint32_t accum = (kb != kb0 || k != 0) ? 1u : 0u;
            if constexpr (CG == 1)
              mma_ss<T>(sdesc_k_sw128(a_addr + k * 32), sdesc_k_sw128(b_addr + k * 32), d_tmem, idesc, accum);
            else
              mma_ss_pair_bf16(sdesc_k_sw128(a_addr + k * 32), sdesc_k_sw128(b_addr + k * 32), d_tmem, idesc_t, accum);
          }
          if constexpr (CG == 1) tc_commit(&empty_bar[stage]);
          else tc_commit_pair(&empty_bar[stage]);   // frees the stage in both CTAs
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if constexpr (CG == 1) tc_commit(&tfull_bar[acc]);
        else tc_commit_pair(&tfull_bar[acc]);       // both CTAs' epilogues
        BO_STAMP(item, 2);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      if constexpr (CG == 2) {
        // drain: the peer's last remote arrivals must land before the CTAs exit
        const int iters = item;   // segments this unit ran
        if (iters > 0) {
          const int last = iters - 1;
          mbar_wait(&tempty_bar[last & 1], (last >> 1) & 1);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    if constexpr (EPI == EPI_SWIGLU) {
      // Fused-combine bookkeeping for the GEMM2 that follows (while the first
      // accumulator fills): zero the arrival counters; a token with no row
      // (every slot dropped, full brownout) gets y = [x] here.
      if (p.comb_cnt) {
        const int et = threadIdx.x - 64;
        const int64_t ncnt = static_cast<int64_t>(p.comb_T) * p.comb_nt;
        for (int64_t i = static_cast<int64_t>(blockIdx.x) * 128 + et; i < ncnt;
             i += static_cast<int64_t>(gridDim.x) * 128)
          p.comb_cnt[i] = 0;
        for (int t = blockIdx.x * 4 + (warp - 2); t < p.comb_T; t += gridDim.x * 4) {
          bool mine = false;
          for (int sl = lane; sl < p.comb_KR; sl += 32)
            mine |= __ldg(p.row_of + static_cast<int64_t>(t) * p.comb_KR + sl) >= 0;
          const bool has = __any_sync(0xffffffffu, mine);
          if (!has) combine_token_cols<T>(p, reinterpret_cast<const T*>(p.out), 0, t, 0, p.comb_d, lane);
        }
      }
    }
    const int q = warp & 3;   // TMEM lane quarter this warp may access
    const uint64_t pol_out = p.store_hint ? policy_evict_first() : policy_evict_normal();
    uint8_t* stage = s_epi + (warp - 2) * 32 * C::EPI_ROW;
    uint8_t* box = s_box + (warp - 2) * 4096;   // 1 KB aligned (smem is): swizzles follow address bits 4-9
    int acc = 0;
    uint32_t acc_phase = 0;
    int x, mi, n, sp, kb0, kb1;
    int w, s0 = 0, s1 = 0, kind;
    int item = 0;
    for (; segment(item, w, s0, s1, kind); ++item) {
      if (item > 0 && warp == 2 && lane == 0) BO_STAMP(item - 1, 3);   // the previous tile's epilogue is done
      item_at(item, w, x, mi, n, sp, kb0, kb1);
      if (item >= n_my_whole && tsx) { kb0 = s0; kb1 = s1; }
      const int rows_x = s_eoff[x + 1] - s_eoff[x];
      const int r_local = mi * TILE_M + static_cast<int>(crank) * kBM + q * 32 + lane;
      const bool valid = r_local < rows_x;
      const int64_t grow = static_cast<int64_t>(s_eoff[x]) + r_local;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t t0 = tmem_base + static_cast<uint32_t>(acc * BN) + (static_cast<uint32_t>(q * 32) << 16);
      // rows of this warp's 32-row slab that belong to the executor
      const int slab = mi * TILE_M + static_cast<int>(crank) * kBM + q * 32;
      const int nrows = rows_x - slab < 0 ? 0 : (rows_x - slab > 32 ? 32 : rows_x - slab);
      const int64_t row0 = static_cast<int64_t>(s_eoff[x]) + slab;
      bool swapped = false;
      if constexpr (kSwap) {
        if (swapped_tile(x, mi)) {
          // D^T tile: lane = weight row, TMEM column = the tile's row.  Warp q < 2 holds
          // the gate rows of columns colb..colb+31, warp q + 2 their up rows: the up warp
          // hands its values over through its staging tile, 16 rows at a time; the gate
          // warp computes H, stages [32 rows][32 columns] and writes it back.
          swapped = true;
          const int rin = tile_rows(x, mi);
          const int ns = (rin + 31) & ~31;
          const bool up_w = q >= 2;
          const int bid = 2 + (q & 1);
          float* xch = reinterpret_cast<float*>(s_epi + (q & 1) * 32 * C::EPI_ROW);   // the up warp's tile
          T* out = reinterpret_cast<T*>(p.out) + n * 128 + static_cast<int>(crank) * 64 + (q & 1) * 32;
          const int64_t tok0 = static_cast<int64_t>(s_eoff[x]) + mi * TILE_M;
#pragma unroll 1
          for (int c = 0; c < ns; c += 32) {
            uint32_t v[32];
            tmem_ld32(t0 + c, v);
            tmem_ld_wait();
            float hv[32];
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              pair_bar(bid);   // the previous half has been read
              if (up_w) {
#pragma unroll
                for (int j = 0; j < 16; ++j) xch[j * 32 + lane] = __uint_as_float(v[hf * 16 + j]);
              }
              pair_bar(bid);
              if (!up_w) {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                  hv[hf * 16 + j] = silu_f(__uint_as_float(v[hf * 16 + j])) * xch[j * 32 + lane];
              }
            }
            if (!up_w) {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                *reinterpret_cast<T*>(stage + j * C::EPI_ROW + lane * (int)sizeof(T)) = static_cast<T>(hv[j]);
              __syncwarp();
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int pc = i * 32 + lane, tk = pc >> 2, part = pc & 3;
                if (c + tk < rin) {
                  const uint4 val = *reinterpret_cast<const uint4*>(stage + tk * C::EPI_ROW + part * 16);
                  T* dst = out + (tok0 + c + tk) * p.ldo + part * (16 / (int)sizeof(T));
                  st_global_hint(dst, val, pol_out);
                }
              }
              __syncwarp();
            }
          }
          // the gate warp has read the last half before the up warp reuses its staging tile
          // (the next tile's stage_row32); racecheck flagged the write-after-read without it
          pair_bar(bid);
        }
      }
      if constexpr (EPI == EPI_SWIGLU) {
        T* out = reinterpret_cast<T*>(p.out) + n * bh;
#pragma unroll 1
        for (int c = 0; c < (swapped ? 0 : bh); c += 32) {
          // a 16-column tail (bh % 32 == 16) reads 16 columns past each half (inside
          // this accumulator's BN-column slot) and stores only the valid ones
          uint32_t g[32], u[32];
          tmem_ld32(t0 + c, g);
          tmem_ld32(t0 + bh + c, u);
          tmem_ld_wait();
          float h[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) h[i] = silu_f(__uint_as_float(g[i])) * __uint_as_float(u[i]);
          stage_row32<T>(stage, lane, h);
          __syncwarp();
          const int cols = bh - c < 32 ? bh - c : 32;
          flush_rows32<T>(stage, lane, out + c, row0, nrows, p.ldo, cols * (int)sizeof(T) / 16, pol_out);
          __syncwarp();
        }
      } else if constexpr (EPI == EPI_WEIGHTED) {
        // last-wave split (tail_split): a contributor piece hands its fp32 accumulator to the
        // tile's finishing unit; a finishing piece waits for and adds the later pieces' partials
        if constexpr (CG == 2) {
          const int lrow = q * 32 + lane;   // TMEM lane of this thread
          if (kind == SEG_CONTRIB) {
            float* part = p.sk_part + static_cast<int64_t>(blockIdx.x) * kSkPartElems;
#pragma unroll 1
            for (int c = 0; c < BN; c += 32) {
              uint32_t v[32];
              tmem_ld32(t0 + c, v);
              tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 32; ++j) __stcg(part + (c + j) * 128 + lrow, __uint_as_float(v[j]));
            }
            tc_fence_before();
            __threadfence();   // release: the partial precedes the count
            __syncwarp();
            if (lane == 0) {
              atomicAdd(p.sk_flag + blockIdx.x, 1);
              if (leader) mbar_arrive(&tempty_bar[acc]);
              else mbar_arrive_remote(&tempty_bar[acc], 0);
            }
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            continue;
          }
          if (kind == SEG_FINISH) {
            // Add the later pieces' partials into the accumulator, in unit order: each is
            // brought into the stage ring (idle: this is the unit's last piece and its MMAs
            // have completed) by one bulk copy, then every warp adds its lanes' columns and
            // writes them back to TMEM.
            const int64_t tile_end = static_cast<int64_t>(w - n_whole + 1) * nkb_t;
            const int c_first = unit + 1;
            int c_last = unit;
            while (c_last + 1 < n_units && ts_lo(c_last + 1) < tile_end) ++c_last;
            const float* ring = reinterpret_cast<const float*>(smem);
            for (int cu = c_first; cu <= c_last; ++cu) {
              epi_bar();   // every warp has read the previous partial (and the ring is idle)
              if (warp == 2 && lane == 0) {
                const int* flag = p.sk_flag + cu * 2 + static_cast<int>(crank);
                int v;
                do {
                  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
                } while (v < 4);
                fence_proxy_async_global();   // the partial's generic writes before the async-proxy read
                fence_proxy_async_smem();     // our generic reads of the ring before its async overwrite
                mbar_arrive_expect_tx(fix_bar, kSkPartElems * 4);
                bulk_g2s(smem, p.sk_part + static_cast<int64_t>(cu * 2 + static_cast<int>(crank)) * kSkPartElems,
                         kSkPartElems * 4, fix_bar);
              }
              mbar_wait(fix_bar, static_cast<uint32_t>((cu - c_first) & 1));
#pragma unroll 1
              for (int c = 0; c < BN; c += 32) {
                uint32_t a[32];
                tmem_ld32(t0 + c, a);
                tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  a[j] = __float_as_uint(__uint_as_float(a[j]) + ring[(c + j) * 128 + lrow]);
                tmem_st32(t0 + c, a);
              }
              tmem_st_wait();
            }
            tc_fence_before();
            tc_fence_after();
          }
        }
        const float wr = valid ? (p.row_w ? p.row_w[grow] : p.alpha) : 0.0f;
        if (p.ksplit_max > 1 || p.f32_mode) {   // split-K: fp32 partial of split sp, row-scaled (Eq. 6)
          float* outp = p.partial + (static_cast<int64_t>(sp) * p.rows_total + grow) * p.ldo + n * BN;
          const float scale = kb1 > kb0 ? wr : 0.0f;   // an empty k-range contributes 0 (stale TMEM)
#pragma unroll 1
          for (int c = 0; c < BN; c += 32) {
            uint32_t a[32];
            tmem_ld32(t0 + c, a);
            tmem_ld_wait();
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = kb1 > kb0 ? __uint_as_float(a[i]) * scale : 0.0f;
            if (valid) {
              if (p.f32_mode == 2) {   // W += alpha * acc (distillation update), optional bf16 copy in p.out
                add_row32(outp + c, v);
                if (p.out) store_row32<T>(reinterpret_cast<T*>(p.out) + grow * p.ldo + n * BN + c, v);
              } else {
                store_row32<float>(outp + c, v);
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (CG == 1 || leader) mbar_arrive(&tempty_bar[acc]);
            else mbar_arrive_remote(&tempty_bar[acc], 0);
          }
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
          continue;
        }
        T* out = reinterpret_cast<T*>(p.out) + n * BN;
        // TMA bulk stores for full slabs (no fused combine, which re-reads the rows at once):
        // thread = row writes its 64 bytes into a dense 32 x 32 box (64B swizzle: 16-byte
        // chunk q of row r at q ^ ((r >> 1) & 3), conflict-free), one elected lane stores
        // the box; two boxes per warp alternate.
        const bool tma_out = sizeof(T) == 2 && p.tma_store && nrows == 32 && !p.comb_cnt;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          uint32_t a[32];
          tmem_ld32(t0 + c, a);
          tmem_ld_wait();
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(a[i]) * wr;
          if (tma_out) {
            uint8_t* tb = box + ((c >> 5) & 1) * 2048;
            if (lane == 0) bulk_wait_read<1>();   // this box's store from two chunks ago has read it
            __syncwarp();
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              uint4 u;
              u.x = pack_bf16x2(v[8 * q4 + 0], v[8 * q4 + 1]);
              u.y = pack_bf16x2(v[8 * q4 + 2], v[8 * q4 + 3]);
              u.z = pack_bf16x2(v[8 * q4 + 4], v[8 * q4 + 5]);
              u.w = pack_bf16x2(v[8 * q4 + 6], v[8 * q4 + 7]);
              *reinterpret_cast<uint4*>(tb + lane * 64 + ((q4 ^ ((lane >> 1) & 3)) << 4)) = u;
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tmB.m[6], tb, n * BN + c, static_cast<int>(row0));
              bulk_commit();
            }
            continue;
          }
          stage_row32<T>(stage, lane, v);
          __syncwarp();
          flush_rows32<T>(stage, lane, out + c, row0, nrows, p.ldo, 32 * (int)sizeof(T) / 16, pol_out);
          __syncwarp();
        }
        if (p.comb_cnt) {
          // Fused combine (a8).  The accumulator is no longer needed: hand it back
          // to the MMA warp first, so the count / combine below overlaps the next
          // tile's mainloop.
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (CG == 1 || leader) mbar_arrive(&tempty_bar[acc]);
            else mbar_arrive_remote(&tempty_bar[acc], 0);
          }
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
          // Release this warp's Yp rows (every lane fences its own stores, then the
          // warp barrier), count each row's BN columns against its token; the warp
          // whose arrival completes a token (all BN columns of every slot landed)
          // sums its rows for this n-tile.
          __threadfence();
          __syncwarp();
          int t = -1;
          int need = 0;
          int rr[kCombSlots];
          if (valid) t = __ldg(p.row_tok + grow);
#pragma unroll
          for (int sl = 0; sl < kCombSlots; ++sl) {
            rr[sl] = (valid && sl < p.comb_KR) ? __ldg(p.row_of + static_cast<int64_t>(t) * p.comb_KR + sl) : -1;
            need += rr[sl] >= 0 ? 1 : 0;
          }
          const bool last =
              valid && atomicAdd(p.comb_cnt + static_cast<int64_t>(t) * p.comb_nt + n, BN) == need * BN - BN;
          const uint32_t done = __ballot_sync(0xffffffffu, last);
          if (done) {
            __threadfence();   // acquire: the other rows' stores precede their counts
            const T* yb = reinterpret_cast<const T*>(p.out);
            if (p.comb_KR <= 2) combine_tokens_batched<T, 2, 4>(p, yb, p.ldo, done, t, rr, n * BN, BN, lane);
            else if (p.comb_KR <= 4) combine_tokens_batched<T, 4, 2>(p, yb, p.ldo, done, t, rr, n * BN, BN, lane);
            else combine_tokens_batched<T, 8, 2>(p, yb, p.ldo, done, t, rr, n * BN, BN, lane);
          }
          continue;
        }
      } else {
        // Router (Eq. 8) with Eq. 7 fused: this thread owns token `grow`'s m logits.
        // The logits leave through a swizzled 32 x 32 fp32 staging box per warp
        // (16-byte chunk c of row r at c ^ (r & 7): conflict-free both ways) as whole
        // 128-byte row segments, not as 32 scattered 4-byte stores per instruction.
        float tv[KMAX];
        int ti[KMAX];
#pragma unroll
        for (int j = 0; j < KMAX; ++j) { tv[j] = 0.0f; ti[j] = -1; }
        float* lbase = reinterpret_cast<float*>(p.out) + row0 * p.ldo;
        const bool vec_ok = (p.ldo & 3) == 0;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          uint32_t a[32];
          tmem_ld32(t0 + c, a);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int col = c + i;
            if (col < p.n_valid) topk_insert<KMAX>(tv, ti, p.topk_k, __uint_as_float(a[i]), col);
          }
          const int ncol = p.n_valid - c < 32 ? p.n_valid - c : 32;
          if (ncol <= 0) continue;
#pragma unroll
          for (int c4 = 0; c4 < 8; ++c4)
            *reinterpret_cast<uint4*>(box + lane * 128 + ((c4 ^ (lane & 7)) << 4)) =
                make_uint4(a[4 * c4], a[4 * c4 + 1], a[4 * c4 + 2], a[4 * c4 + 3]);
          __syncwarp();
          if (vec_ok && ncol == 32) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {   // 4 rows x 8 chunks per instruction
              const int r = i * 4 + (lane >> 3), c4 = lane & 7;
              if (r < nrows)
                *reinterpret_cast<uint4*>(lbase + r * p.ldo + c + 4 * c4) =
                    *reinterpret_cast<const uint4*>(box + r * 128 + ((c4 ^ (r & 7)) << 4));
            }
          } else {
            for (int i = lane; i < nrows * ncol; i += 32) {   // row-major element order: coalesced
              const int r = i / ncol, cc = i - r * ncol;
              lbase[r * p.ldo + c + cc] =
                  *reinterpret_cast<const float*>(box + r * 128 + (((cc >> 2) ^ (r & 7)) << 4) + (cc & 3) * 4);
            }
          }
          __syncwarp();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[acc]);   // TMEM free: the rest is register work
        const float vmax = tv[0];
        float ex[KMAX];
        float sum = 0.0f;
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
          ex[j] = j < p.topk_k ? expf(tv[j] - vmax) : 0.0f;
          sum += ex[j];
        }
        if (valid) {
          int32_t* idr = p.topk_id + grow * p.topk_k;
          float* wr = p.topk_w + grow * p.topk_k;
          if ((p.topk_k & 3) == 0) {   // 16-byte rows pieces
#pragma unroll
            for (int j = 0; j < KMAX; j += 4)
              if (j < p.topk_k) {
                *reinterpret_cast<int4*>(idr + j) = make_int4(ti[j], ti[j + 1], ti[j + 2], ti[j + 3]);
                *reinterpret_cast<float4*>(wr + j) =
                    make_float4(__fdividef(ex[j], sum), __fdividef(ex[j + 1], sum), __fdividef(ex[j + 2], sum),
                                __fdividef(ex[j + 3], sum));
              }
          } else {
#pragma unroll
            for (int j = 0; j < KMAX; ++j)
              if (j < p.topk_k) {
                idr[j] = ti[j];
                wr[j] = __fdividef(ex[j], sum);   // sum >= 1 (see silu_f)
              }
          }
        }
        // Per-tile expert histogram (Alg. 1 cnt_i input, tile = this 128-token m-tile),
        // atomics-free: each warp counts its 32 tokens' choices per expert with
        // __match_any_sync (the lowest lane of each equal-id group adds the group's
        // size to the warp's own row), then the 4 warp rows are summed in order.
        int* whist = reinterpret_cast<int*>(stage);   // this warp's row (m <= 256 ints <= its staging tile)
        for (int e = lane; e < p.n_valid; e += 32) whist[e] = 0;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
          if (j < p.topk_k) {
            const int e = valid ? ti[j] : -1;
            const uint32_t peers = __match_any_sync(0xffffffffu, e);
            if (e >= 0 && lane == __ffs(peers) - 1) whist[e] += __popc(peers);
            __syncwarp();
          }
        }
        epi_bar();
        for (int e = threadIdx.x - 64; e < p.n_valid; e += 128) {
          int cnt = 0;
#pragma unroll
          for (int w4 = 0; w4 < 4; ++w4) cnt += reinterpret_cast<const int*>(s_epi + w4 * 32 * C::EPI_ROW)[e];
          p.tile_cnt[static_cast<int64_t>(mi) * p.n_valid + e] = cnt;
        }
        epi_bar();   // the staging rows are reused by the next tile
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        continue;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 1 || leader) mbar_arrive(&tempty_bar[acc]);
        else mbar_arrive_remote(&tempty_bar[acc], 0);
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

#ifdef BO_PROBE
  if (warp == 2 && lane == 0) {
    int last = -1, w_, a_, b_, k_;
    while (segment(last + 1, w_, a_, b_, k_)) ++last;
    if (last >= 0) BO_STAMP(last, 3);
  }
#endif
  if constexpr (EPI == EPI_WEIGHTED) {
    if (warp >= 2 && lane == 0) bulk_wait_all();   // TMA-stored Yp boxes complete before exit
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    if constexpr (CG == 2) tmem_dealloc_pair(tmem_base, TMEM_COLS);
    else tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

// cudaFuncSetAttribute applies to the current device's context: remember it per
// device (bit per device ordinal; a process driving several GPUs sets it on each).
template <typename K>
static cudaError_t ensure_smem_attr(K kern, int bytes, std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = dev < 64 ? (uint64_t(1) << dev) : 0;
  if (bit && (done.load(std::memory_order_acquire) & bit)) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && bit) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

template <typename T, int BN, int EPI, int KMAX = 0, int CG = 1>
static cudaError_t launch_t(const CUtensorMap& A, const BMaps& B, const GemmParams& p, int grid, cudaStream_t s,
                            bool pdl) {
  using C = GemmCfg<T, BN, CG>;
  static std::atomic<uint64_t> attr_done{0};
  auto kern = k_grouped_gemm<T, BN, EPI, KMAX, CG>;
  cudaError_t e = ensure_smem_attr(kern, C::SMEM, attr_done);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(CG == 2 ? (grid & ~1) : grid));
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if constexpr (CG == 2) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl) {   // may launch while the previous kernel drains; waits in-kernel (griddepcontrol.wait)
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  e = cudaLaunchKernelEx(&cfg, kern, A, B, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <typename T>
static cudaError_t dispatch(int epi, int bn, const CUtensorMap& A, const BMaps& B, const GemmParams& p, int grid,
                            cudaStream_t s, bool pdl) {
  if (epi == EPI_SWIGLU_PAIR) {
    if constexpr (sizeof(T) == 2)
      if (bn == 256) return launch_t<T, 256, EPI_SWIGLU, 0, 2>(A, B, p, grid, s, pdl);
  } else if (epi == EPI_WEIGHTED_PAIR) {
    if constexpr (sizeof(T) == 2)
      if (bn == 256) return launch_t<T, 256, EPI_WEIGHTED, 0, 2>(A, B, p, grid, s, pdl);
  } else if (epi == EPI_SWIGLU) {
    if (bn == 256) return launch_t<T, 256, EPI_SWIGLU>(A, B, p, grid, s, pdl);
    if (bn == 128) return launch_t<T, 128, EPI_SWIGLU>(A, B, p, grid, s, pdl);
    if (bn == 64) return launch_t<T, 64, EPI_SWIGLU>(A, B, p, grid, s, pdl);
  } else if (epi == EPI_WEIGHTED) {
    if (bn == 256) return launch_t<T, 256, EPI_WEIGHTED>(A, B, p, grid, s, pdl);
    if (bn == 128) return launch_t<T, 128, EPI_WEIGHTED>(A, B, p, grid, s, pdl);
    if (bn == 64) return launch_t<T, 64, EPI_WEIGHTED>(A, B, p, grid, s, pdl);
  } else if (epi == EPI_ROUTER) {
    const bool k8 = p.topk_k <= 8;
#define BO_R(BNV)                                                                        \
  if (bn == BNV) return k8 ? launch_t<T, BNV, EPI_ROUTER, 8>(A, B, p, grid, s, pdl) \
                           : launch_t<T, BNV, EPI_ROUTER, 16>(A, B, p, grid, s, pdl);
    BO_R(256) BO_R(128) BO_R(64) BO_R(32) BO_R(16)
#undef BO_R
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_grouped_gemm(int dtype, int epi, int bn, const CUtensorMap& A, const BMaps& B,
                                const GemmParams& p, int grid, cudaStream_t s, bool pdl) {
  if (grid <= 0) return cudaSuccess;
  if (dtype == 0) return dispatch<__nv_bfloat16>(epi, bn, A, B, p, grid, s, pdl);
  return dispatch<float>(epi, bn, A, B, p, grid, s, pdl);
}

#ifdef BO_PROBE
extern "C" __attribute__((visibility("default"))) int bo_probe_copy(void* stamps, void* ids) {
  if (cudaMemcpyFromSymbol(stamps, g_probe, sizeof(g_probe)) != cudaSuccess) return 1;
  if (cudaMemcpyFromSymbol(ids, g_probe_id, sizeof(g_probe_id)) != cudaSuccess) return 1;
  return 0;
}
#endif

int gemm_smem_bytes(int dtype, int epi, int bn) {
  (void)epi;
  // STAGE_BYTES depends only on BN (128-byte rows for both dtypes)
  switch (bn) {
    case 256: return dtype == 0 ? GemmCfg<__nv_bfloat16, 256>::SMEM : GemmCfg<float, 256>::SMEM;
    case 128: return dtype == 0 ? GemmCfg<__nv_bfloat16, 128>::SMEM : GemmCfg<float, 128>::SMEM;
    case 64: return dtype == 0 ? GemmCfg<__nv_bfloat16, 64>::SMEM : GemmCfg<float, 64>::SMEM;
    case 32: return dtype == 0 ? GemmCfg<__nv_bfloat16, 32>::SMEM : GemmCfg<float, 32>::SMEM;
    case 16: return dtype == 0 ? GemmCfg<__nv_bfloat16, 16>::SMEM : GemmCfg<float, 16>::SMEM;
  }
  return -1;
}

}  // namespace bo
