// gemm_tc.cuh — the tcgen05 GEMM engine every dense contraction of the learner
// and of inference runs on (conv as implicit GEMM, FC, LSTM input projection,
// weight / data gradients).
//
//   D[m][n] = sum_k A(m,k) * B(n,k)          bf16 x bf16 -> fp32 (TMEM)
//
// Persistent, warp-specialized (one CTA per SM, 288 threads):
//   warps 0-3  producers: fill a ring of S shared-memory stages with the
//              128x64 A tile and BNx64 B tile of each k-block through the
//              Problem's loaders (implicit-GEMM gathers, transposed sources):
//              cp.async (LDGSTS) chunks that arrive on the stage's full
//              mbarrier when they land, or register-staged chunks (uint8 ->
//              bf16 conversion) followed by a proxy fence and an arrive;
//   warp 4     MMA issuer: one thread issues tcgen05.mma (cta_group::1,
//              M=128, N=BN, K=16, bf16 -> fp32) into one of two TMEM
//              accumulators and commits each stage back to the producers;
//   warps 5-8  epilogue: tcgen05.ld of the finished accumulator (bias, ReLU,
//              masks, bf16 packing or split-K partials), overlapped with the
//              MMAs of the next tile in the other accumulator.
// Work items (m tile, n tile, K split) are strided over the CTAs.
//
// Problem concept (all __device__):
//   static constexpr bool A_MN, B_MN;   // false: K-major source, true: MN-major
//   int M, N, K, kb_per_split;
//   uint4 load_a(int i, int j) const;   // K-major: A(i, j..j+7); MN-major: A(j..j+7, k=i)
//   uint4 load_b(int i, int j) const;   // same convention for B
//   void store(int m, int n, float v) const;   // final value of D[m][n] (epilogue)
// split-K (grid.z > 1): the engine writes fp32 partials part[z][m][n] and
// splitk_finish() sums them in fixed z order before calling store() —
// deterministic, no atomics.
// Bounds: the engine zero-fills chunks with m >= M / n >= N / k >= K; K-major
// sources need K % 8 == 0, MN-major sources need M (or N) % 8 == 0.
#pragma once
#include <algorithm>
#include <stdio.h>
#include <stdlib.h>
#include <type_traits>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "common.cuh"

namespace seed {

// ---------------------------------------------------------------- TMA tensor maps
// A Problem whose A and B are plain K-major bf16 matrices ([rows][K], row stride
// ld elements) may declare `static constexpr bool TMA = true` with CUtensorMap
// members ta / tb (filled by its host method tmaps()): one producer thread then
// moves each 128x64 / BNx64 tile with one cp.async.bulk.tensor (UTMALDG) into the
// same 128-byte-swizzled layout the cp.async path writes (TileMap K-major), the
// tensor unit zero-filling rows >= M / N and k >= K.
inline PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}
// K-major bf16 [rows][K] (row stride ld elements, 16-byte aligned base and stride)
// with a box of 64 k x box_rows rows, 128-byte swizzle
inline bool tmap_kmajor(CUtensorMap* m, const void* base, int64_t rows, int64_t K, int64_t ld, int box_rows) {
  auto enc = tmap_encoder();
  if (!enc || ((uintptr_t)base & 15) || (ld * 2) % 16) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  const cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* m, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
template <class P, class = void>
struct HasTma : std::false_type {};
template <class P>
struct HasTma<P, std::void_t<decltype(P::TMA)>> : std::integral_constant<bool, P::TMA> {};

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;

// Shared-memory image of one R x 64 (bf16) operand tile in a canonical UMMA
// layout.  Chunks (16 B) are assigned so that consecutive lanes read
// consecutive 16-byte pieces of one source row (coalesced) and the 8 lanes of
// a shared-memory store phase hit distinct bank groups.
//  * K-major (source row = MN index, contiguous along K): 128-byte swizzle —
//    row r at r*128, chunk kc stored at ((kc ^ (r & 7)) * 16); SBO = 1024
//    (8-row atom stride); per-MMA K advance = 32 bytes.
//  * MN-major, R % 64 == 0 (source row = k, contiguous along MN): 128-byte
//    swizzle — atom = 64 MN x 8 k (1024 B), k-row j of an atom at j*128,
//    chunk mc%8 at ((mc%8 ^ k%8) * 16); LBO = 1024 (MN-atom stride),
//    SBO = (R/64)*1024 (8-k-row stride); per-MMA K advance = 2*SBO.
//  * MN-major, R < 64: no swizzle, core matrices (8 k x 16 B), SBO = 144
//    (padded MN-core stride), LBO = 144 R/8 (K-core stride).
template <int R, bool MN>
struct TileMap {
  static constexpr bool SWZ = !MN || (R % 64 == 0);
  static constexpr uint32_t LAYOUT = SWZ ? 2u : 0u;   // SWIZZLE_128B / SWIZZLE_NONE
  static constexpr int LBO = !MN ? 16 : (SWZ ? 1024 : (R / 8) * 144);
  static constexpr int SBO = !MN ? 1024 : (SWZ ? (R / 64) * 1024 : 144);
  static constexpr int KSTEP = !MN ? 32 : (SWZ ? 2 * SBO : 2 * LBO);
  static constexpr int BYTES = !MN ? R * 128 : (SWZ ? 8 * SBO : 8 * LBO);
  static constexpr int CHUNKS = R * GEMM_BK / 8;
  __device__ __forceinline__ static void chunk(int c, int r0, int k0, int& i, int& j, int& off,
                                               bool& in_r, bool& in_k, int Rlim, int Klim) {
    if (!MN) {
      const int kc = c & 7, r = c >> 3;
      i = r0 + r; j = k0 + kc * 8;
      off = r * 128 + ((kc ^ (r & 7)) << 4);
      in_r = i < Rlim; in_k = j < Klim;
    } else if (SWZ) {
      const int mc = c % (R / 8), k = c / (R / 8);
      i = k0 + k; j = r0 + mc * 8;
      off = (k >> 3) * SBO + (mc >> 3) * LBO + (k & 7) * 128 + (((mc & 7) ^ (k & 7)) << 4);
      in_r = j < Rlim; in_k = i < Klim;
    } else {
      const int mc = c % (R / 8), k = c / (R / 8);
      i = k0 + k; j = r0 + mc * 8;
      off = (k >> 3) * LBO + mc * SBO + (k & 7) * 16;
      in_r = j < Rlim; in_k = i < Klim;
    }
  }
  __device__ __forceinline__ static uint64_t desc(uint32_t base, int kk) {
    return umma_desc(base + kk * KSTEP, LBO, SBO, LAYOUT);
  }
};

constexpr int GEMM_PRODUCER_WARPS = 8;
constexpr int GEMM_PRODUCERS = 32 * GEMM_PRODUCER_WARPS;   // warps 0-7
constexpr int GEMM_MMA_WARP = GEMM_PRODUCER_WARPS;           // warp 8
constexpr int GEMM_THREADS = GEMM_PRODUCERS + 32 + 128;     // + MMA warp + 4 epilogue warps

template <int BN, bool A_MN, bool B_MN>
struct GemmCfg {
  using TA = TileMap<GEMM_BM, A_MN>;
  using TB = TileMap<BN, B_MN>;
  static constexpr int A_BYTES = (TA::BYTES + 1023) / 1024 * 1024;   // swizzle atoms 1024-aligned
  static constexpr int B_BYTES = (TB::BYTES + 1023) / 1024 * 1024;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES_FIT = (200 * 1024) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  // + barriers (256 B) + the epilogue's per-warp 32 x 33 fp32 transpose buffers
  static constexpr int EPI_BYTES = 4 * 32 * 33 * 4;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 256 + EPI_BYTES;
  static constexpr uint32_t ACC_COLS = BN;   // two accumulators of BN columns
  static constexpr uint32_t TMEM_COLS =
      2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
  static constexpr int A_CHUNKS = (TA::CHUNKS + GEMM_PRODUCERS - 1) / GEMM_PRODUCERS;
  static constexpr int B_CHUNKS = (TB::CHUNKS + GEMM_PRODUCERS - 1) / GEMM_PRODUCERS;
  static_assert(STAGES >= 2, "stage ring");
};

template <class Prob, class = void>
struct IsAsync : std::false_type {};
template <class Prob>
struct IsAsync<Prob, decltype((void)Prob::ASYNC)> : std::integral_constant<bool, Prob::ASYNC> {};

template <class Prob, class = void>
struct HasStore16 : std::false_type {};
template <class Prob>
struct HasStore16<Prob, decltype((void)Prob::VEC_STORE)> : std::integral_constant<bool, Prob::VEC_STORE> {};

// Problems whose output row m is a contiguous fp32 row (out_row(m)[n] = post(m, n, acc))
template <class Prob, class = void>
struct HasRowOut : std::false_type {};
template <class Prob>
struct HasRowOut<Prob, decltype((void)Prob::ROW_OUT)> : std::integral_constant<bool, Prob::ROW_OUT> {};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void st_shared_zero16(uint32_t dst) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(dst), "r"(0) : "memory");
}
// arrive on `bar` once all of this thread's prior cp.async have landed
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

constexpr int GEMM_COUNTERS = 4096;   // per-tile split-K arrival counters (workspace)

__device__ __forceinline__ void epi_bar_sync() {   // the 4 epilogue warps only
  asm volatile("bar.sync 1, 128;" ::: "memory");
}

template <class Prob>
__device__ __forceinline__ void gemm_store16(const Prob& p, int m, int n, float (&v)[16]) {
  bool done_vec = false;
  if constexpr (HasStore16<Prob>::value) {
    if (n + 16 <= p.N) {
      p.store16(m, n, v);
      done_vec = true;
    }
  }
  if (!done_vec) {
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (n + i < p.N) p.store(m, n + i, v[i]);
  }
}

// Epilogue of one 128 x BN accumulator: epilogue warp `q` (0..3) owns TMEM
// lanes / tile rows [32q, 32q+32).  Split-K (splits > 1): the partial goes to
// part[z]; with `cnt`, the last CTA to finish a tile (integer arrival counter,
// re-armed by that CTA) sums the partials of all splits in z order — the same
// fixed order whichever CTA arrives last — and runs the store epilogue, so no
// separate reduction launch is needed.
template <int BN, class Prob>
__device__ __forceinline__ void gemm_epilogue(const Prob& p, float* __restrict__ part, int splits,
                                              int z, int m0, int n0, bool have, uint32_t tmem,
                                              int q, int lane, unsigned* cnt, int tile,
                                              int* s_last, float* stg) {
  const int m = m0 + q * 32 + lane;
  constexpr bool ROWOUT = HasRowOut<Prob>::value;
  if (splits > 1 || ROWOUT) {
    // Coalesced path: the warp's 32 rows x 32 columns go through a padded shared
    // buffer, then each store instruction covers 4 rows x 128 contiguous bytes
    // (one lane per row would scatter 32 rows per instruction).
    float* out = nullptr;
    size_t ld = 0;
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      float v[32];
      if (have) {
        if (c + 32 <= BN) {
          tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + c, v);
        } else {
          tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + c, v);
#pragma unroll
          for (int i = 16; i < 32; ++i) v[i] = 0.f;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.f;
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) stg[lane * 33 + i] = v[i];
      __syncwarp();
      const int cc = 4 * (lane & 7);
#pragma unroll
      for (int r0 = 0; r0 < 32; r0 += 4) {
        const int r = r0 + (lane >> 3);
        const int mm = m0 + q * 32 + r, nn = n0 + c + cc;
        if (mm < p.M && nn < p.N && c + cc < BN) {
          float4 o = make_float4(stg[r * 33 + cc], stg[r * 33 + cc + 1], stg[r * 33 + cc + 2],
                                 stg[r * 33 + cc + 3]);
          if constexpr (ROWOUT) {
            if (splits == 1) {
              out = p.out_row(mm);
              o.x = p.post(mm, nn, o.x); o.y = p.post(mm, nn + 1, o.y);
              o.z = p.post(mm, nn + 2, o.z); o.w = p.post(mm, nn + 3, o.w);
            }
          }
          if (splits > 1) { out = part + ((size_t)z * p.M + mm) * p.N; ld = 0; }
          (void)ld;
          if (nn + 4 <= p.N && (p.N & 3) == 0) {
            *reinterpret_cast<float4*>(out + nn) = o;
          } else {
            const float t4[4] = {o.x, o.y, o.z, o.w};
            for (int i = 0; i < 4 && nn + i < p.N; ++i) out[nn + i] = t4[i];
          }
        }
      }
      __syncwarp();
    }
  } else {
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
      float v[16];
      if (have) {
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + c, v);
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0.f;
      }
      const int n = n0 + c;
      if (m < p.M && n < p.N) gemm_store16(p, m, n, v);
    }
  }
  if (splits > 1 && cnt) {
    __threadfence();
    epi_bar_sync();
    if (q == 0 && lane == 0) *s_last = atomicAdd(&cnt[tile], 1u) == (unsigned)(splits - 1);
    epi_bar_sync();
    if (*s_last) {
      __threadfence();
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        const int n = n0 + c;
        if (m < p.M && n < p.N) {
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
          const bool vec = n + 16 <= p.N && (p.N & 3) == 0;
#pragma unroll 1
          for (int zz = 0; zz < splits; ++zz) {
            const float* src = part + ((size_t)zz * p.M + m) * p.N + n;
            if (vec) {
#pragma unroll
              for (int i = 0; i < 16; i += 4) {
                const float4 t = __ldcg(reinterpret_cast<const float4*>(src + i));
                v[i] += t.x; v[i + 1] += t.y; v[i + 2] += t.z; v[i + 3] += t.w;
              }
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (n + i < p.N) v[i] += __ldcg(src + i);
            }
          }
          gemm_store16(p, m, n, v);
        }
      }
      if (q == 0 && lane == 0) cnt[tile] = 0u;
    }
  }
}

#ifdef SEED_LSTM_PROF
// diagnostic build only: clock64 stamps of CTA 0 (setup, producer, MMA, epilogue)
__device__ long long g_gemm_prof[8];
#define GEMM_STAMP(I, COND) \
  if (blockIdx.x == 0 && (COND)) g_gemm_prof[I] = clock64();
#else
#define GEMM_STAMP(I, COND)
#endif

template <int BN, class Prob>
__global__ void __launch_bounds__(GEMM_THREADS, 1) gemm_tc_kernel(const __grid_constant__ Prob p,
                                                                  float* __restrict__ part, int splits,
                                                                  unsigned* cnt) {
  GEMM_STAMP(0, threadIdx.x == 0)
  using Cfg = GemmCfg<BN, Prob::A_MN, Prob::B_MN>;
  using TA = typename Cfg::TA;
  using TB = typename Cfg::TB;
  constexpr int BK = GEMM_BK, S = Cfg::STAGES;
  constexpr bool ASYNC = IsAsync<Prob>::value;
  constexpr bool TMA = HasTma<Prob>::value;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * Cfg::STAGE_BYTES);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* s_last = reinterpret_cast<int*>(tmem_slot + 1);
  float* epi_stage = reinterpret_cast<float*>(smem + S * Cfg::STAGE_BYTES + 256);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int mt = (p.M + GEMM_BM - 1) / GEMM_BM, nt = (p.N + BN - 1) / BN;
  const int nitems = mt * nt * splits;
  const int nkb_total = (p.K + BK - 1) / BK;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], TMA ? 1 : GEMM_PRODUCERS);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_mbar_init();
  }
  if (warp == GEMM_MMA_WARP) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait_trig();
  GEMM_STAMP(1, threadIdx.x == 0)
  const uint32_t tmem = *tmem_slot;

  auto decode = [&](int w, int& m0, int& n0, int& kb0, int& nkb, int& z) {
    z = w % splits;
    const int t = w / splits;
    m0 = (t % mt) * GEMM_BM;
    n0 = (t / mt) * BN;
    kb0 = z * p.kb_per_split;
    nkb = max(0, min(nkb_total, kb0 + p.kb_per_split) - kb0);
  };

  if (warp < GEMM_PRODUCER_WARPS) {
    // ------------------------------------------------------------ producers
    const uint32_t smem0 = smem_u32(smem);
    int g = 0;
    for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
      int m0, n0, kb0, nkb, z;
      decode(w, m0, n0, kb0, nkb, z);
      for (int i = 0; i < nkb; ++i, ++g) {
        const int s = g % S;
        if (g >= S) mbar_wait(&empty[s], ((g / S) - 1) & 1);
        const int k0 = (kb0 + i) * BK;
        const uint32_t sa = smem0 + s * Cfg::STAGE_BYTES, sb = sa + Cfg::A_BYTES;
        if constexpr (TMA) {   // one thread: two tensor copies credited to the stage
          if (tid == 0) {
            mbar_expect_tx(&full[s], (uint32_t)(GEMM_BM + BN) * BK * 2);
            tma_load_2d(sa, &p.ta, k0, m0, &full[s]);
            tma_load_2d(sb, &p.tb, k0, n0, &full[s]);
          }
        } else if constexpr (ASYNC) {
          // zero chunks (padding, transposed-conv zero taps) are plain shared
          // stores: a zero-fill cp.async would still send a request to memory
          bool zeroed = false;
#pragma unroll
          for (int j = 0; j < Cfg::A_CHUNKS; ++j) {
            int a, b, off;
            bool ir, ik;
            TA::chunk(j * GEMM_PRODUCERS + tid, m0, k0, a, b, off, ir, ik, p.M, p.K);
            const void* src = (ir && ik) ? p.ptr_a(a, b) : nullptr;
            if (src) cp_async16(sa + off, src, true);
            else { st_shared_zero16(sa + off); zeroed = true; }
          }
#pragma unroll
          for (int j = 0; j < Cfg::B_CHUNKS; ++j) {
            const int cb = j * GEMM_PRODUCERS + tid;
            if (TB::CHUNKS % GEMM_PRODUCERS != 0 && cb >= TB::CHUNKS) continue;
            int a, b, off;
            bool ir, ik;
            TB::chunk(cb, n0, k0, a, b, off, ir, ik, p.N, p.K);
            const void* src = (ir && ik) ? p.ptr_b(a, b) : nullptr;
            if (src) cp_async16(sb + off, src, true);
            else { st_shared_zero16(sb + off); zeroed = true; }
          }
          if (zeroed) fence_proxy_async_smem();
          cp_async_arrive(&full[s]);
          GEMM_STAMP(2, tid == 0 && g == 0)
        } else {
          uint4 ra[Cfg::A_CHUNKS], rb[Cfg::B_CHUNKS];
          int oa[Cfg::A_CHUNKS], ob[Cfg::B_CHUNKS];
          const uint4 zero4 = make_uint4(0, 0, 0, 0);
#pragma unroll
          for (int j = 0; j < Cfg::A_CHUNKS; ++j) {
            int a, b;
            bool ir, ik;
            TA::chunk(j * GEMM_PRODUCERS + tid, m0, k0, a, b, oa[j], ir, ik, p.M, p.K);
            ra[j] = (ir && ik) ? p.load_a(a, b) : zero4;
          }
#pragma unroll
          for (int j = 0; j < Cfg::B_CHUNKS; ++j) {
            const int cb = j * GEMM_PRODUCERS + tid;
            int a, b;
            bool ir, ik;
            TB::chunk(cb < TB::CHUNKS ? cb : 0, n0, k0, a, b, ob[j], ir, ik, p.N, p.K);
            rb[j] = (cb < TB::CHUNKS && ir && ik) ? p.load_b(a, b) : zero4;
            if (cb >= TB::CHUNKS) ob[j] = -1;
          }
          uint8_t* gsa = smem + s * Cfg::STAGE_BYTES;
#pragma unroll
          for (int j = 0; j < Cfg::A_CHUNKS; ++j) *reinterpret_cast<uint4*>(gsa + oa[j]) = ra[j];
#pragma unroll
          for (int j = 0; j < Cfg::B_CHUNKS; ++j)
            if (ob[j] >= 0) *reinterpret_cast<uint4*>(gsa + Cfg::A_BYTES + ob[j]) = rb[j];
          fence_proxy_async_smem();
          mbar_arrive(&full[s]);
        }
      }
    }
  } else if (warp == GEMM_MMA_WARP) {
    // ------------------------------------------------------------ MMA issuer (warp-uniform,
    // one elected lane issues: common.cuh tc_mma_bf16_w)
    {
      constexpr uint32_t idesc = umma_idesc_bf16(GEMM_BM, BN, Prob::A_MN, Prob::B_MN);
      const uint32_t smem0 = smem_u32(smem);
      int g = 0, it = 0;
      for (int w = blockIdx.x; w < nitems; w += gridDim.x, ++it) {
        int m0, n0, kb0, nkb, z;
        decode(w, m0, n0, kb0, nkb, z);
        const int acc = it & 1;
        if (it >= 2) mbar_wait(&tempty[acc], ((it >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * Cfg::ACC_COLS;
        for (int i = 0; i < nkb; ++i, ++g) {
          const int s = g % S;
          mbar_wait(&full[s], (g / S) & 1);
          GEMM_STAMP(3, g == 0)
          tc_fence_after();
          const uint32_t a_base = smem0 + s * Cfg::STAGE_BYTES;
          const uint32_t b_base = a_base + Cfg::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = TA::desc(a_base, kk);
            const uint64_t bd = TB::desc(b_base, kk);
            tc_mma_bf16_w(d, ad, bd, idesc, (i > 0 || kk > 0) ? 1u : 0u);
          }
          tc_commit_w(&empty[s]);
        }
        if (nkb > 0) tc_commit_w(&tfull[acc]);
        else if (lane == 0) mbar_arrive(&tfull[acc]);
        GEMM_STAMP(4, it == 0)
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;   // TMEM lane quarter of this warp (warps 9..12 -> 1,2,3,0)
    int it = 0;
    for (int w = blockIdx.x; w < nitems; w += gridDim.x, ++it) {
      int m0, n0, kb0, nkb, z;
      decode(w, m0, n0, kb0, nkb, z);
      const int acc = it & 1;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      GEMM_STAMP(5, it == 0 && q == 0 && lane == 0)
      tc_fence_after();
      gemm_epilogue<BN>(p, part, splits, z, m0, n0, nkb > 0, tmem + acc * Cfg::ACC_COLS, q, lane, cnt,
                        w / splits, s_last, epi_stage + q * 32 * 33);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      GEMM_STAMP(6, it == 0 && q == 0 && lane == 0)
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == GEMM_MMA_WARP) tmem_dealloc(tmem, Cfg::TMEM_COLS);
  GEMM_STAMP(7, threadIdx.x == 0)
}

// Fixed-order split-K reduction: each thread owns 4 consecutive outputs and
// adds the splits z = 0, 1, ... in order (float4 loads, all in flight) —
// deterministic.  Requires N % 4 == 0 (else the scalar path per output).
template <class Prob>
__global__ void __launch_bounds__(256) splitk_finish(const Prob p, const float* __restrict__ part,
                                                     int splits) {
  pdl_wait_trig();
  const size_t MN = (size_t)p.M * p.N;
  const size_t n4 = (MN + 3) / 4;
  const bool vec = (p.N & 3) == 0;
  for (size_t i4 = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i4 < n4;
       i4 += (size_t)gridDim.x * blockDim.x) {
    const size_t i = i4 * 4;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (vec) {
#pragma unroll 4
      for (int z = 0; z < splits; ++z) {
        const float4 t = __ldcs(reinterpret_cast<const float4*>(part + (size_t)z * MN + i));
        v[0] += t.x; v[1] += t.y; v[2] += t.z; v[3] += t.w;
      }
      const int m = (int)(i / p.N), n = (int)(i % p.N);
#pragma unroll
      for (int q = 0; q < 4; ++q) p.store(m, n + q, v[q]);
    } else {
      for (int q = 0; q < 4 && i + q < MN; ++q) {
        for (int z = 0; z < splits; ++z) v[q] += part[(size_t)z * MN + i + q];
        p.store((int)((i + q) / p.N), (int)((i + q) % p.N), v[q]);
      }
    }
  }
}

// Host launcher.  splits > 1 runs split-K into `part` ([splits][M][N] fp32,
// caller workspace); with `cnt` (GEMM_COUNTERS zeroed unsigned, left zeroed)
// the last CTA of each tile reduces in-kernel, otherwise the fixed-order
// splitk_finish kernel follows.  max_ctas > 0 caps the persistent grid.
// run_finish = false: with splits > 1 the caller reduces `part` itself (e.g. the
// consumer kernel sums the splits in z order while loading)
template <int BN, class Prob>
seed_status launch_gemm(Prob p, int splits, cudaStream_t st, float* part = nullptr,
                        int max_ctas = 0, unsigned* cnt = nullptr, bool run_finish = true) {
  using Cfg = GemmCfg<BN, Prob::A_MN, Prob::B_MN>;
  if (p.M <= 0 || p.N <= 0) return SEED_OK;
  const int nkb = (p.K + GEMM_BK - 1) / GEMM_BK;
  if (splits < 1) splits = 1;
  if (splits > nkb) splits = nkb > 0 ? nkb : 1;
  p.kb_per_split = (nkb + splits - 1) / splits;
  splits = nkb > 0 ? (nkb + p.kb_per_split - 1) / p.kb_per_split : 1;
  if constexpr (HasTma<Prob>::value) {
    if (!p.tmaps(BN)) return SEED_E_ARG;   // base / stride not 16-byte aligned, or no driver entry point
  }
  static PerDevice attr;
  SEED_TRY(smem_optin(attr, gemm_tc_kernel<BN, Prob>, Cfg::SMEM));
  const int sms = sm_count();
  if (splits > 1 && !part) return SEED_E_WORKSPACE;
  const int tiles = ceil_div(p.M, GEMM_BM) * ceil_div(p.N, BN);
  if (tiles > GEMM_COUNTERS) cnt = nullptr;
  const int items = tiles * splits;
  const int grid = std::min(items, max_ctas > 0 ? std::min(max_ctas, sms) : sms);
  SEED_TRY(launch_k(gemm_tc_kernel<BN, Prob>, dim3(grid), dim3(GEMM_THREADS), (size_t)Cfg::SMEM, st, p,
                    part, splits, splits > 1 ? cnt : (unsigned*)nullptr));
  if (splits > 1 && !cnt && run_finish) {
    const size_t MN = (size_t)p.M * p.N;
    const int blocks = (int)std::min<size_t>((MN / 4 + 255) / 256 + 1, 148 * 8);
    SEED_TRY(launch_k(splitk_finish<Prob>, dim3(blocks), dim3(256), 0, st, p, (const float*)part, splits));
  }
  return SEED_OK;
}

// effective number of splits launch_gemm will use
inline int gemm_effective_splits(int K, int splits) {
  const int nkb = (K + GEMM_BK - 1) / GEMM_BK;
  if (splits < 1) splits = 1;
  if (splits > nkb) splits = nkb > 0 ? nkb : 1;
  const int per = (nkb + splits - 1) / splits;
  return nkb > 0 ? (nkb + per - 1) / per : 1;
}

// ---------------------------------------------------------------- common loaders
// A 16-byte bf16 chunk [1, 0, 0, 0, 0, 0, 0, 0]: the all-ones column that turns a
// weight-gradient GEMM's extra output column into the bias gradient; also a
// valid dummy source address for zero-filled cp.async chunks.
__device__ __align__(16) const uint32_t k_ones_chunk[4] = {0x3F80u, 0u, 0u, 0u};

__device__ __forceinline__ uint4 ld16(const void* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}

// 8 uint8 -> 8 bf16 (exact integers 0..255)
__device__ __forceinline__ uint4 u8x8_to_bf16(uint2 v) {
  uint4 o;
  uint32_t w[2] = {v.x, v.y};
  uint32_t* out = &o.x;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t x = w[i >> 1] >> ((i & 1) * 16);
    out[i] = pack_bf16((float)(x & 0xFF), (float)((x >> 8) & 0xFF));
  }
  return o;
}

}  // namespace seed
