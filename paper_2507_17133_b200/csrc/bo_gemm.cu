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
// work list):
//   warp 0      TMA producer: A tile [128 x BK] + B tile [BN x BK] per stage
//   warp 1      MMA issuer: tcgen05.mma.cta_group::1 M=128 N=BN K=16(bf16)/8(tf32)
//               into a double-buffered TMEM accumulator (2 x BN fp32 columns)
//   warps 2-5   epilogue: tcgen05.ld 32x32b -> registers -> fused op -> global
// Work item w -> (executor x, n-tile, m-tile) with the m-tile fastest, so
// concurrently running CTAs share the same weight tile (B) through L2.
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

template <typename T, int BN, int CG = 1>
struct GemmCfg {
  static constexpr int BM = kBM;                         // rows per CTA (the pair covers CG * 128)
  static constexpr int BK = 128 / (int)sizeof(T);       // one 128-byte swizzle row
  static constexpr int UK = 32 / (int)sizeof(T);        // MMA K per instruction
  static constexpr int A_BYTES = BM * 128;
  static constexpr int B_BYTES = (BN / CG) * 128;       // each CTA of a pair holds half of B
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_BYTES = 2048;                 // barriers + tmem slot (1 KB) + router histogram (1 KB)
  static constexpr int SCHED_BYTES = ((2 * (kMaxExec + 1) * 4) + 127) / 128 * 128;   // keeps the staging 16B-aligned
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
// new element only overtakes strictly smaller values (reading D8).
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

__device__ __forceinline__ void st_release_gpu(int* ptr, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(ptr), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_gpu(const int* ptr) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(ptr) : "memory");
  return v;
}

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

template <typename T, int BN, int EPI, int KMAX, int CG, bool GATHER>
__global__ void __launch_bounds__(192, 1)
    k_grouped_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ BMaps tmB, const GemmParams p) {
  // CG = 1: one CTA computes a 128 x BN tile with tcgen05.mma.cta_group::1.
  // CG = 2: a CTA pair (cluster of 2) computes a 256 x BN tile with
  //         tcgen05.mma.cta_group::2 issued by the leader: each CTA stages its
  //         128 rows of A and half of B (BN/2 rows), halving the shared-memory
  //         and L2 traffic per MMA; each CTA's TMEM holds its 128 rows.
  static_assert(CG == 1 || (CG == 2 && EPI != EPI_ROUTER && sizeof(T) == 2), "pair mode: bf16 FFN GEMMs");
  // GATHER: the A rows are not read from a packed Xp but gathered from the token
  // matrix x by TMA tile::gather4 (4 rows per instruction, row index = row_tok),
  // i.e. concat_tokens fused into GEMM1's operand load.
  static_assert(!GATHER || EPI == EPI_SWIGLU, "gather feeds GEMM1 only");
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
  uint64_t* fix_bar = tempty_bar + 2;   // split-tile fix-up: contributor partial landed in shared memory
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 3);
  int* s_hist = reinterpret_cast<int*>(smem + STAGES * C::STAGE_BYTES + 1024);
  int* s_mtile = reinterpret_cast<int*>(smem + STAGES * C::STAGE_BYTES + C::BAR_BYTES);
  int* s_eoff = s_mtile + (kMaxExec + 1);
  uint8_t* s_epi = smem + STAGES * C::STAGE_BYTES + C::BAR_BYTES + C::SCHED_BYTES;

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
  if constexpr (EPI == EPI_SWIGLU && !GATHER) {
    if (p.bh_alt > 0) {
      const int items_p = start_of(nexec);
      nt_o = p.nt_alt;
      nt_u = p.nt_alt_u;
      const int items_a = start_of(nexec);
      // waves x width; stream-K spreads the k-blocks evenly (no wave rounding), the
      // lockstep tail split shortens the last partial wave by its split count
      auto wave_cost = [&](int items) -> long long {
        if (p.stream_k == 1) return 8LL * items;
        const int full = items / n_units, r = items - full * n_units;
        if (r == 0) return 8LL * full;
        if (p.stream_k != 2) return 8LL * (full + 1);
        int k = n_units / r;
        k = k > 4 ? 4 : k;
        const int kbm = p.Kdim / C::BK;
        k = k > kbm ? kbm : k;
        return 8LL * full + 8 / (k < 1 ? 1 : k);
      };
      const long long cost_p = wave_cost(items_p) * (BN + 32);
      const long long cost_a = wave_cost(items_a) * (2 * p.bh_alt + 32);
      alt = cost_a < cost_p;
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
  // GEMM2 (EPI_WEIGHTED) likewise: this CTA's 128 Wd rows (output columns) on M, the
  // tile's H rows on N; the epilogue writes Yp column-sliced and counts columns for
  // the fused combine.
  constexpr bool kSwap = CG == 2 && (EPI == EPI_SWIGLU || EPI == EPI_WEIGHTED) && !GATHER;
  const bool swap_ok = kSwap && p.swap_tail && !alt && !p.a_shared && !p.b_packed &&
                       (EPI != EPI_WEIGHTED || (p.ksplit_max <= 1 && !p.f32_mode));
  // largest tail swapped: a tail near 256 rows gains no MMA work and loses pipelining
  // (swap_max >= TILE_M swaps full tiles too: an experiment knob)
  const int swap_lim = p.swap_max > 0 ? (p.swap_max < TILE_M ? p.swap_max : TILE_M) : TILE_M - 1;
  auto tile_rows = [&](int x, int mi) {   // rows of executor x in m-tile mi
    const int r = s_eoff[x + 1] - s_eoff[x] - mi * TILE_M;
    return r < TILE_M ? r : TILE_M;
  };
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

  // work item -> (executor, m-tile inside executor, n-tile); m-tile fastest
  auto decode = [&](int w, int& x, int& mi, int& n) {
    int lo = 0, hi = nexec;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (start_of(mid) <= w) lo = mid; else hi = mid;
    }
    x = lo;
    const int mt = s_mtile[x + 1] - s_mtile[x];
    const int local = w - start_of(x);
    n = local / mt;
    mi = local - n * mt;
  };
  // work item -> tile + k-block range [kb0, kb1) of split sp
  auto decode_k = [&](int w, int& x, int& mi, int& n, int& sp, int& kb0, int& kb1) {
    const int tw = w / ks;
    sp = w - tw * ks;
    decode(tw, x, mi, n);
    const int nkb = kblocks(x);
    const int per = (nkb + ks - 1) / ks;
    kb0 = sp * per < nkb ? sp * per : nkb;
    kb1 = kb0 + per < nkb ? kb0 + per : nkb;
  };
  // Segments this CTA (unit) processes, in order.  Classic: work items
  // unit, unit + n_units, ... (whole tiles or split-K ranges).  Stream-K
  // (decode-sized steps, CG = 1, uniform reduction length), the "data-parallel +
  // two-tile stream-K" hybrid: all but the last two waves of tiles run whole
  // (tile w on unit w % n_units, so concurrently running CTAs still share weight
  // and activation tiles in L2); the remaining (<= 2 waves of) tiles are cut into
  // n_units equal contiguous ranges of their (tile, k-block) space, so every SM
  // streams the same number of k-blocks.  A tile cut between CTAs is finished by
  // the CTA holding its k-block 0 (the owner), which adds the fp32 partials the
  // later CTAs left in sk_part (slot = their unit).
  const bool stream = CG == 1 && p.stream_k == 1 && EPI != EPI_ROUTER;
  const int kb_u = kblocks(0);
  // Lockstep tail split-K (p.stream_k == 2): the complete waves of tiles run whole
  // (tile w on unit w % n_units); the r tiles of the last, partial wave have their
  // reduction cut into ks_l equal k-ranges run side by side on units
  // tile * ks_l + sp (every split of every tail tile concurrently, so CTAs reading
  // the same weight / activation tile do it together); split 0 owns the tile and
  // adds the other splits' fp32 partials (slot = their unit: a CTA contributes at
  // most once, in the tail).
  const int full_tiles = (base_work / n_units) * n_units;
  const int tail = base_work - full_tiles;
  int ks_l = 1;
  if (CG == 1 && p.stream_k == 2 && ks == 1 && tail > 0)
    for (int k = 2; k <= 4 && k <= kb_u && tail * k <= n_units; ++k) ks_l = k;
  const bool lock = ks_l > 1;
  const long long dpl = lock ? full_tiles / n_units : 0;   // whole tiles per unit before the tail
  const int waves = (base_work + n_units - 1) / n_units;
  const int dp_tiles = stream ? (waves > 2 ? (waves - 2) * n_units : 0) : 0;
  const long long dp_cnt = stream ? (dp_tiles > unit ? (dp_tiles - unit + n_units - 1) / n_units : 0) : 0;
  const long long tu = stream ? static_cast<long long>(base_work - dp_tiles) * kb_u : 0;   // stream-K units
  const long long su_lo = stream ? tu * unit / n_units : 0;
  const long long su_hi = stream ? tu * (unit + 1) / n_units : 0;
  long long sk_pos = 0;   // stream-K position of the current segment (set by seg_at)
  auto seg_at = [&](long long cur, int& x, int& mi, int& n, int& sp, int& kb0, int& kb1) -> bool {
    if (lock) {
      if (cur < dpl) {   // whole tile of a complete wave
        decode(static_cast<int>(unit + cur * n_units), x, mi, n);
        sp = 0;
        kb0 = 0;
        kb1 = kb_u;
        return true;
      }
      if (cur != dpl || unit >= tail * ks_l) return false;
      decode(full_tiles + unit / ks_l, x, mi, n);
      sp = unit % ks_l;
      kb0 = sp * kb_u / ks_l;
      kb1 = (sp + 1) * kb_u / ks_l;
      return true;
    }
    if (!stream) {
      if (cur >= total_work) return false;
      decode_k(static_cast<int>(cur), x, mi, n, sp, kb0, kb1);
      return true;
    }
    sp = 0;
    if (cur < dp_cnt) {   // whole tile of the data-parallel waves
      decode(static_cast<int>(unit + cur * n_units), x, mi, n);
      kb0 = 0;
      kb1 = kb_u;
      return true;
    }
    sk_pos = su_lo + (cur - dp_cnt);
    if (sk_pos >= su_hi) return false;
    const long long tile = sk_pos / kb_u;
    kb0 = static_cast<int>(sk_pos - tile * kb_u);
    const long long end = su_hi < (tile + 1) * kb_u ? su_hi : (tile + 1) * kb_u;
    kb1 = static_cast<int>(end - tile * kb_u);
    decode(dp_tiles + static_cast<int>(tile), x, mi, n);
    return true;
  };
  auto seg_next = [&](long long cur, int kb0, int kb1) -> long long {
    return lock ? cur + 1 : (stream ? (cur < dp_cnt ? cur + 1 : cur + (kb1 - kb0)) : cur + n_units);
  };
  const long long seg0 = (stream || lock) ? 0 : unit;
  // stream-K: the unit whose range holds stream-K position u, and whether unit c
  // holds any position (empty ranges when the stream-K tiles * k-blocks < grid)
  auto unit_of = [&](long long u) -> int { return static_cast<int>(((u + 1) * n_units - 1) / tu); };
  auto unit_busy = [&](int c) -> bool { return lock || tu * c / n_units != tu * (c + 1) / n_units; };

  // L2 prefetch of k-block kq of the B tile(s) the producer will load (CTA-pair
  // mode: this CTA's half)
  auto prefetch_b = [&](const CUtensorMap* mb0, const CUtensorMap* mb1, int kq, int brow, int n) {
    if constexpr (EPI == EPI_SWIGLU) {
      if constexpr (CG == 1) {
        tma_prefetch_l2_2d(mb0, kq * C::BK, brow + n * bh);
        tma_prefetch_l2_2d(mb1, kq * C::BK, brow + n * bh);
      } else {
        tma_prefetch_l2_2d(crank == 0 ? mb0 : mb1, kq * C::BK, brow + n * bh);
      }
    } else {
      tma_prefetch_l2_2d(mb0, kq * C::BK, brow + n * BN + (CG == 2 ? static_cast<int>(crank) * (BN / 2) : 0));
    }
  };

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (GATHER || lane == 0) {
      // activations are re-read per n-tile: evict_last (a_policy 0), or normal / first (1 / 2)
      const uint64_t pol_a =
          p.a_policy == 1 ? policy_evict_normal() : (p.a_policy == 2 ? policy_evict_first() : policy_evict_last());
      // weight tile is re-read by the executor's other m-tiles (running alongside);
      // b_policy 1: evict_first (streamed weights make way for the re-read activations)
      const uint64_t pol_b = p.b_policy == 1 ? policy_evict_first() : policy_evict_normal();
      int stage = 0;
      uint32_t phase = 0;
      int x, mi, n, sp, kb0, kb1;
      for (long long cur = seg0; seg_at(cur, x, mi, n, sp, kb0, kb1); cur = seg_next(cur, kb0, kb1)) {
        const int arow = (p.a_shared ? 0 : s_eoff[x]) + mi * TILE_M + static_cast<int>(crank) * kBM;
        const int cls = x < mo ? 0 : (x < mu ? 1 : 2);      // original / united / shared
        const CUtensorMap* mb0 = &tmB.m[(alt ? 6 : 0) + 2 * cls];
        const CUtensorMap* mb1 = &tmB.m[(alt ? 6 : 0) + 2 * cls + 1];
        const int brow = cls == 0 ? x * p.b_rows_per_exec
                                  : (cls == 1 ? (x - mo) * p.b_rows_u : (x - mu) * p.b_rows_per_exec);
        int4 tok = make_int4(0, 0, 0, 0);
        if constexpr (GATHER) {   // this lane gathers rows arow + 4*lane .. +3 (their tokens)
          const int r = arow + 4 * lane;
          tok.x = r + 0 < p.rows_total ? __ldg(p.row_tok + r + 0) : 0;
          tok.y = r + 1 < p.rows_total ? __ldg(p.row_tok + r + 1) : 0;
          tok.z = r + 2 < p.rows_total ? __ldg(p.row_tok + r + 2) : 0;
          tok.w = r + 3 < p.rows_total ? __ldg(p.row_tok + r + 3) : 0;
        }
        if constexpr (kSwap) {
          const int rin = tile_rows(x, mi);
          if (swap_ok && rin <= swap_lim) {
            const int nsh = ((rin + 31) & ~31) / 2;   // token rows staged by this CTA (N / 2)
            const int wrow = brow + n * 128 + static_cast<int>(crank) * 64;
            const int trow = s_eoff[x] + mi * TILE_M + static_cast<int>(crank) * nsh;
            // one box of >= nsh rows (16 / 32 / 64 / 128; rows past nsh land unused)
            const int tbox = nsh <= 16 ? 16 : (nsh <= 32 ? 32 : (nsh <= 64 ? 64 : 128));
            const CUtensorMap* mt = tbox == 128 ? &tmA : &tmB.m[tbox == 16 ? 12 : (tbox == 32 ? 13 : 14)];
            for (int kb = kb0; kb < kb1; ++kb) {
              mbar_wait(&empty_bar[stage], phase ^ 1);
              uint8_t* sa = smem + stage * C::STAGE_BYTES;
              if (lane == 0) {
                if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * (C::A_BYTES + tbox * 128));
                else mbar_arrive_remote(&full_bar[stage], 0);
                if constexpr (EPI == EPI_SWIGLU) {
                  tma_load_2d_pair(sa, &tmB.m[6 + 2 * cls], &full_bar[stage], kb * C::BK, wrow, pol_b);
                  tma_load_2d_pair(sa + 64 * 128, &tmB.m[7 + 2 * cls], &full_bar[stage], kb * C::BK, wrow, pol_b);
                } else {   // Wd rows n * BN + crank * 128 .. + 127 (the pair's usual B half box)
                  tma_load_2d_pair(sa, &tmB.m[2 * cls], &full_bar[stage], kb * C::BK,
                                   brow + n * BN + static_cast<int>(crank) * 128, pol_b);
                }
                tma_load_2d_pair(sa + C::A_BYTES, mt, &full_bar[stage], kb * C::BK, trow, pol_a);
              }
              if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
            continue;
          }
        }
        // L2 prefetch of the first pf_dist k-blocks' B tiles of this segment (weight
        // streaming: more DRAM requests in flight than the stage ring holds)
        if (p.pf_dist > 0 && !p.b_packed && lane == 0) {
          const int kpf = kb0 + p.pf_dist < kb1 ? kb0 + p.pf_dist : kb1;
          for (int kq = kb0; kq < kpf; ++kq) prefetch_b(mb0, mb1, kq, brow, n);
        }
        for (int kb = kb0; kb < kb1; ++kb) {
          if (p.pf_dist > 0 && !p.b_packed && lane == 0 && kb + p.pf_dist < kb1)
            prefetch_b(mb0, mb1, kb + p.pf_dist, brow, n);
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::STAGE_BYTES;
          uint8_t* sb = sa + C::A_BYTES;
          if (lane == 0) {
            // B rows [grow, grow + nr) of k-block kb: one 2-D box, or (tile-packed weights)
            // one 3-D box per 128-row band, each a contiguous block in memory
            const int kbs = kblocks(x);
            auto load_b = [&](uint8_t* dst, const CUtensorMap* mb, int grow, int nr) {
              if (!p.b_packed) {
                if constexpr (CG == 1) tma_load_2d(dst, mb, &full_bar[stage], kb * C::BK, grow, pol_b);
                else tma_load_2d_pair(dst, mb, &full_bar[stage], kb * C::BK, grow, pol_b);
                return;
              }
              for (int r0 = 0; r0 < nr; r0 += kPackRows) {
                const int gr = grow + r0;
                const int c2 = (gr / kPackRows) * kbs + kb;
                if constexpr (CG == 1)
                  tma_load_3d(dst + r0 * 128, mb, &full_bar[stage], 0, gr % kPackRows, c2, pol_b);
                else
                  tma_load_3d_pair(dst + r0 * 128, mb, &full_bar[stage], 0, gr % kPackRows, c2, pol_b);
              }
            };
            if constexpr (CG == 1) {
              mbar_arrive_expect_tx(&full_bar[stage], stage_tx);
              if constexpr (!GATHER) tma_load_2d(sa, &tmA, &full_bar[stage], kb * C::BK, arow, pol_a);
              if constexpr (EPI == EPI_SWIGLU) {
                load_b(sb, mb0, brow + n * bh, bh);
                load_b(sb + bh * 128, mb1, brow + n * bh, bh);
              } else {
                load_b(sb, mb0, brow + n * BN, BN);
              }
            } else {
              // Both CTAs load their halves; completion is counted on the leader's barrier.
              if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * stage_tx);
              else mbar_arrive_remote(&full_bar[stage], 0);
              if constexpr (!GATHER) tma_load_2d_pair(sa, &tmA, &full_bar[stage], kb * C::BK, arow, pol_a);
              if constexpr (EPI == EPI_SWIGLU) {
                // leader: gate rows, peer: up rows of the same f-columns -> D[:, 0:BN/2] = gate, D[:, BN/2:] = up
                load_b(sb, leader ? mb0 : mb1, brow + n * bh, bh);
              } else {
                load_b(sb, mb0, brow + n * BN + static_cast<int>(crank) * (BN / 2), BN / 2);
              }
            }
          }
          if constexpr (GATHER) {
            if constexpr (CG == 1) tma_gather4(sa + lane * 512, &tmA, &full_bar[stage], kb * C::BK, tok, pol_a);
            else tma_gather4_pair(sa + lane * 512, &tmA, &full_bar[stage], kb * C::BK, tok, pol_a);
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
      for (long long cur = seg0; seg_at(cur, x, mi, n, sp, kb0, kb1); cur = seg_next(cur, kb0, kb1)) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
        uint32_t idesc_t = idesc;
        if constexpr (kSwap) {
          const int rin = tile_rows(x, mi);
          if (swap_ok && rin <= swap_lim) idesc_t = idesc_f32acc<T>(256, (rin + 31) & ~31);
        }
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
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
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      if constexpr (CG == 2) {
        // drain: the peer's last remote arrivals must land before the CTAs exit
        const int iters = total_work > unit ? (total_work - unit + n_units - 1) / n_units : 0;
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
    int acc = 0;
    uint32_t acc_phase = 0;
    int x, mi, n, sp, kb0, kb1;
    uint32_t fix_phase = 0;
    for (long long cur = seg0; seg_at(cur, x, mi, n, sp, kb0, kb1); cur = seg_next(cur, kb0, kb1)) {
      const int rows_x = s_eoff[x + 1] - s_eoff[x];
      const int r_local = mi * TILE_M + static_cast<int>(crank) * kBM + q * 32 + lane;
      const bool valid = r_local < rows_x;
      const int64_t grow = static_cast<int64_t>(s_eoff[x]) + r_local;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t t0 = tmem_base + static_cast<uint32_t>(acc * BN) + (static_cast<uint32_t>(q * 32) << 16);
      if ((stream || lock) && kb0 > 0) {
        // stream-K contributor: this tile's k-blocks [kb0, kb1) as an fp32 partial in
        // slot `unit` (TMEM column order), then publish it (every thread fences its
        // stores, the epilogue barrier, one release store of the flag)
        // layout [column quad][128 rows] of float4: a warp's stores are 512 contiguous
        // bytes, and the owner's fix-up reads it back from shared memory conflict-free
        float4* dst = reinterpret_cast<float4*>(p.sk_part + static_cast<int64_t>(unit) * kBM * kSkCols) +
                      (q * 32 + lane);
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          uint32_t a[32];
          tmem_ld32(t0 + c, a);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            __stcg(dst + (c / 4 + j) * kBM,
                   make_float4(__uint_as_float(a[4 * j]), __uint_as_float(a[4 * j + 1]),
                               __uint_as_float(a[4 * j + 2]), __uint_as_float(a[4 * j + 3])));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        __threadfence();
        epi_bar();
        if (threadIdx.x == 64) st_release_gpu(p.sk_flag + unit, 1);
        continue;
      }
      // Owner of a tile cut between CTAs (stream-K / lockstep split): this is the CTA's
      // last segment, so its MMAs are done and the stage ring is free.  For each
      // contributing unit in order: wait for its flag, bulk-copy its partial tile into
      // the ring (one TMA transfer), TMEM accumulator += partial, then the epilogue
      // below reads the finished sum.
      if ((stream || lock) && kb1 < kb_u) {   // (only stream-K segments are cut: sk_pos is this segment's)
        const int c_first = unit + 1;
        const int c_last = lock ? unit + ks_l - 1 : unit_of((sk_pos / kb_u + 1) * kb_u - 1);
        const uint32_t bytes = static_cast<uint32_t>(kBM) * BN * 4;
        const float4* fbuf = reinterpret_cast<const float4*>(smem) + (q * 32 + lane);
        for (int cc = c_first; cc <= c_last; ++cc) {
          if (!unit_busy(cc)) continue;
          if (threadIdx.x == 64) {
            while (ld_acquire_gpu(p.sk_flag + cc) == 0) {
            }
            p.sk_flag[cc] = 0;   // consumed (the next launch starts from zero)
            fence_proxy_async_global();   // generic-proxy partial -> async-proxy bulk read
            fence_proxy_async_smem();     // earlier generic reads of the ring -> async-proxy write
            mbar_arrive_expect_tx(fix_bar, bytes);
            bulk_g2s(smem, p.sk_part + static_cast<int64_t>(cc) * kBM * kSkCols, bytes, fix_bar);
          }
          mbar_wait(fix_bar, fix_phase);
          fix_phase ^= 1;
#pragma unroll 1
          for (int c = 0; c < BN; c += 32) {
            uint32_t a[32];
            tmem_ld32(t0 + c, a);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 f = fbuf[(c / 4 + j) * kBM];
              a[4 * j] = __float_as_uint(__uint_as_float(a[4 * j]) + f.x);
              a[4 * j + 1] = __float_as_uint(__uint_as_float(a[4 * j + 1]) + f.y);
              a[4 * j + 2] = __float_as_uint(__uint_as_float(a[4 * j + 2]) + f.z);
              a[4 * j + 3] = __float_as_uint(__uint_as_float(a[4 * j + 3]) + f.w);
            }
            tmem_st32(t0 + c, a);
          }
          tmem_st_wait();
          epi_bar();   // the ring is read by every epilogue thread before the next copy lands
        }
      }
      // rows of this warp's 32-row slab that belong to the executor
      const int slab = mi * TILE_M + static_cast<int>(crank) * kBM + q * 32;
      const int nrows = rows_x - slab < 0 ? 0 : (rows_x - slab > 32 ? 32 : rows_x - slab);
      const int64_t row0 = static_cast<int64_t>(s_eoff[x]) + slab;
      uint8_t* stage = s_epi + (warp - 2) * 32 * C::EPI_ROW;
      bool swapped = false;
      // swapped GEMM2 tail tile: Yp stores here, the shared release / count / combine below
      int sw_rin = 0;
      if constexpr (kSwap && EPI == EPI_WEIGHTED) {
        const int rin = tile_rows(x, mi);
        if (swap_ok && rin <= swap_lim) {
          // D^T tile: lane = output column col0 + lane, TMEM column = the tile's row:
          // Yp[row, cols] = row_w[row] * acc, staged [32 rows][32 columns] per warp.
          sw_rin = rin;
          const int ns = (rin + 31) & ~31;
          T* out = reinterpret_cast<T*>(p.out) + n * BN + static_cast<int>(crank) * 128 + q * 32;
          const int64_t tok0 = static_cast<int64_t>(s_eoff[x]) + mi * TILE_M;
#pragma unroll 1
          for (int c = 0; c < ns; c += 32) {
            uint32_t v[32];
            tmem_ld32(t0 + c, v);
            tmem_ld_wait();
            const float wl = c + lane < rin ? (p.row_w ? p.row_w[tok0 + c + lane] : p.alpha) : 0.0f;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              *reinterpret_cast<T*>(stage + j * C::EPI_ROW + lane * (int)sizeof(T)) =
                  static_cast<T>(__uint_as_float(v[j]) * __shfl_sync(0xffffffffu, wl, j));
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
      }
      if constexpr (kSwap && EPI == EPI_SWIGLU) {
        const int rin = tile_rows(x, mi);
        if (swap_ok && rin <= swap_lim) {
          // D^T tile: lane = weight row, TMEM column = the tile's row.  Warp q < 2 holds
          // the gate rows of columns colb..colb+31, warp q + 2 their up rows: the up warp
          // hands its values over through its staging tile, 16 rows at a time; the gate
          // warp computes H, stages [32 rows][32 columns] and writes it back.
          swapped = true;
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
        const bool tma_out = sizeof(T) == 2 && p.tma_store && nrows == 32 && !p.comb_cnt && !sw_rin;
        uint8_t* tbox0 = smem +
                         ((STAGES * C::STAGE_BYTES + C::BAR_BYTES + C::SCHED_BYTES + 4 * 32 * C::EPI_ROW + 1023) & ~1023) +
                         (warp - 2) * 4096;   // 1 KB aligned (smem is): the swizzle follows address bits 7-8
#pragma unroll 1
        for (int c = 0; c < (sw_rin ? 0 : BN); c += 32) {
          uint32_t a[32];
          tmem_ld32(t0 + c, a);
          tmem_ld_wait();
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(a[i]) * wr;
          if (tma_out) {
            uint8_t* tb = tbox0 + ((c >> 5) & 1) * 2048;
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
          // warp barrier), count each row against its token; the warp whose arrival
          // completes a token sums its rows for this n-tile.  Arrivals are counted in
          // columns: a row is complete when all BN columns of every slot have landed (a
          // swapped tail tile's CTAs each deliver BN / 2 columns of its rows).
          // A swapped tile's four warps first meet at the epilogue barrier (each lane's
          // stores fenced before it), so each row is counted once per CTA with the CTA's
          // BN / 2 columns; the warps split the row chunks.  (One arrival per warp and
          // row made 8 atomics per row on the same counter and cost ~30 us per wave.)
          __threadfence();
          if (sw_rin) epi_bar();
          else __syncwarp();
          const int iters = sw_rin ? (sw_rin + 31) >> 5 : 1;
          const int add = sw_rin ? BN / 2 : BN;
          const int64_t tok0 = static_cast<int64_t>(s_eoff[x]) + mi * TILE_M;
#pragma unroll 1
          for (int it = sw_rin ? q : 0; it < iters; it += sw_rin ? 4 : 1) {
            const bool rv = sw_rin ? it * 32 + lane < sw_rin : valid;
            const int64_t gr = sw_rin ? tok0 + it * 32 + lane : grow;
            int t = -1;
            int need = 0;
            int rr[kCombSlots];
            if (rv) t = __ldg(p.row_tok + gr);
#pragma unroll
            for (int sl = 0; sl < kCombSlots; ++sl) {
              rr[sl] = (rv && sl < p.comb_KR) ? __ldg(p.row_of + static_cast<int64_t>(t) * p.comb_KR + sl) : -1;
              need += rr[sl] >= 0 ? 1 : 0;
            }
            const bool last =
                rv && atomicAdd(p.comb_cnt + static_cast<int64_t>(t) * p.comb_nt + n, add) == need * BN - add;
            const uint32_t done = __ballot_sync(0xffffffffu, last);
            if (done) {
              __threadfence();   // acquire: the other rows' stores precede their counts
              const T* yb = reinterpret_cast<const T*>(p.out);
              if (p.comb_KR <= 2) combine_tokens_batched<T, 2, 4>(p, yb, p.ldo, done, t, rr, n * BN, BN, lane);
              else if (p.comb_KR <= 4) combine_tokens_batched<T, 4, 2>(p, yb, p.ldo, done, t, rr, n * BN, BN, lane);
              else combine_tokens_batched<T, 8, 2>(p, yb, p.ldo, done, t, rr, n * BN, BN, lane);
            }
          }
          continue;
        }
      } else {
        // Router (Eq. 8) with Eq. 7 fused: this thread owns token `grow`'s m logits.
        float tv[KMAX];
        int ti[KMAX];
#pragma unroll
        for (int j = 0; j < KMAX; ++j) { tv[j] = 0.0f; ti[j] = -1; }
        float* lrow = reinterpret_cast<float*>(p.out) + grow * p.ldo;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          uint32_t a[32];
          tmem_ld32(t0 + c, a);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int col = c + i;
            if (col < p.n_valid) {
              const float v = __uint_as_float(a[i]);
              if (valid) lrow[col] = v;
              topk_insert<KMAX>(tv, ti, p.topk_k, v, col);
            }
          }
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
#pragma unroll
          for (int j = 0; j < KMAX; ++j) {
            if (j < p.topk_k) {
              p.topk_id[grow * p.topk_k + j] = ti[j];
              p.topk_w[grow * p.topk_k + j] = __fdividef(ex[j], sum);   // sum >= 1 (see silu_f)
            }
          }
        }
        // per-tile expert histogram (tile = this 128-token m-tile)
        const int et = threadIdx.x - 64;
        epi_bar();
        for (int e = et; e < p.n_valid; e += 128) s_hist[e] = 0;
        epi_bar();
        if (valid) {
#pragma unroll
          for (int j = 0; j < KMAX; ++j)
            if (j < p.topk_k) atomicAdd(&s_hist[ti[j]], 1);
        }
        epi_bar();
        for (int e = et; e < p.n_valid; e += 128) p.tile_cnt[static_cast<int64_t>(mi) * p.n_valid + e] = s_hist[e];
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

static bool g_pdl = true;   // programmatic dependent launch of the GEMMs (set_gemm_pdl)

template <typename T, int BN, int EPI, int KMAX = 0, int CG = 1, bool GATHER = false>
static cudaError_t launch_t(const CUtensorMap& A, const BMaps& B, const GemmParams& p, int grid, cudaStream_t s) {
  using C = GemmCfg<T, BN, CG>;
  static bool attr_set = false;
  auto kern = k_grouped_gemm<T, BN, EPI, KMAX, CG, GATHER>;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
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
  if (g_pdl) {   // may launch while the previous kernel drains; waits in-kernel (griddepcontrol.wait)
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, A, B, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <typename T>
static cudaError_t dispatch(int epi, int bn, const CUtensorMap& A, const BMaps& B, const GemmParams& p, int grid,
                            cudaStream_t s) {
  if (epi == EPI_SWIGLU_GATHER) {
    if (bn == 256) return launch_t<T, 256, EPI_SWIGLU, 0, 1, true>(A, B, p, grid, s);
    if (bn == 128) return launch_t<T, 128, EPI_SWIGLU, 0, 1, true>(A, B, p, grid, s);
  } else if (epi == EPI_SWIGLU_PAIR_GATHER) {
    if constexpr (sizeof(T) == 2)
      if (bn == 256) return launch_t<T, 256, EPI_SWIGLU, 0, 2, true>(A, B, p, grid, s);
  } else if (epi == EPI_SWIGLU_PAIR) {
    if constexpr (sizeof(T) == 2)
      if (bn == 256) return launch_t<T, 256, EPI_SWIGLU, 0, 2>(A, B, p, grid, s);
  } else if (epi == EPI_WEIGHTED_PAIR) {
    if constexpr (sizeof(T) == 2)
      if (bn == 256) return launch_t<T, 256, EPI_WEIGHTED, 0, 2>(A, B, p, grid, s);
  } else if (epi == EPI_SWIGLU) {
    if (bn == 256) return launch_t<T, 256, EPI_SWIGLU>(A, B, p, grid, s);
    if (bn == 128) return launch_t<T, 128, EPI_SWIGLU>(A, B, p, grid, s);
    if (bn == 64) return launch_t<T, 64, EPI_SWIGLU>(A, B, p, grid, s);
  } else if (epi == EPI_WEIGHTED) {
    if (bn == 256) return launch_t<T, 256, EPI_WEIGHTED>(A, B, p, grid, s);
    if (bn == 128) return launch_t<T, 128, EPI_WEIGHTED>(A, B, p, grid, s);
    if (bn == 64) return launch_t<T, 64, EPI_WEIGHTED>(A, B, p, grid, s);
  } else if (epi == EPI_ROUTER) {
    const bool k8 = p.topk_k <= 8;
#define BO_R(BNV)                                                                        \
  if (bn == BNV) return k8 ? launch_t<T, BNV, EPI_ROUTER, 8>(A, B, p, grid, s) \
                           : launch_t<T, BNV, EPI_ROUTER, 16>(A, B, p, grid, s);
    BO_R(256) BO_R(128) BO_R(64) BO_R(32) BO_R(16)
#undef BO_R
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_grouped_gemm(int dtype, int epi, int bn, const CUtensorMap& A, const BMaps& B,
                                const GemmParams& p, int grid, cudaStream_t s) {
  if (grid <= 0) return cudaSuccess;
  if (dtype == 0) return dispatch<__nv_bfloat16>(epi, bn, A, B, p, grid, s);
  return dispatch<float>(epi, bn, A, B, p, grid, s);
}

void set_gemm_pdl(bool on) { g_pdl = on; }

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
