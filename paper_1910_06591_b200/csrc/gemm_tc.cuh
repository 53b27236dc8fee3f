// gemm_tc.cuh — the tcgen05 GEMM engine every dense contraction of the learner
// and of inference runs on (conv as implicit GEMM, FC, LSTM input projection,
// weight / data gradients).
//
//   D[m][n] = sum_k A(m,k) * B(n,k)          bf16 x bf16 -> fp32 (TMEM)
//
// One CTA = 128 threads computes a 128 x BN tile (tcgen05.mma.cta_group::1,
// M=128, N=BN, K=16 per instruction) over a K range (split-K over grid.z).
// All four warps act as the operand producer: each 16-byte chunk of the
// 128x64 A tile and BNx64 B tile is fetched through the Problem's loader
// (implicit-GEMM gathers, uint8 -> bf16 conversion, transposed sources) and
// stored into the UMMA no-swizzle core-matrix layout in shared memory; a
// single elected thread issues the MMAs and commits them to a per-stage
// mbarrier that releases the stage; the fp32 accumulator lives in TMEM and
// the epilogue (bias, ReLU, masks, bf16 packing, split-K partials) reads it
// back with tcgen05.ld.  Loads for k-block i+1 are in flight while the MMAs
// of k-block i run.
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
#include "common.cuh"

namespace seed {

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;
constexpr int GEMM_THREADS = 128;

template <int BN>
struct GemmCfg {
  static constexpr int STAGES = (BN >= 128) ? 3 : 4;
  static constexpr int A_BYTES = GEMM_BM * GEMM_BK * 2;
  static constexpr int B_BYTES = BN * GEMM_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 128;
  static constexpr uint32_t TMEM_COLS = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
  static constexpr int B_CHUNKS = BN * GEMM_BK / 8 / GEMM_THREADS;  // per thread (>= 1 for BN>=16)
};

template <int BN, class Prob>
__global__ void __launch_bounds__(GEMM_THREADS) gemm_tc_kernel(const Prob p, float* __restrict__ part) {
  using Cfg = GemmCfg<BN>;
  constexpr int BM = GEMM_BM, BK = GEMM_BK, S = Cfg::STAGES;
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N for M=128");
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem + S * Cfg::STAGE_BYTES);
  uint64_t* done = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int nkb_total = (p.K + BK - 1) / BK;
  const int kb_begin = blockIdx.z * p.kb_per_split;
  const int kb_end = min(nkb_total, kb_begin + p.kb_per_split);
  const int nkb = max(0, kb_end - kb_begin);

  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&empty[s], 1);
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t idesc = umma_idesc_bf16(BM, BN, Prob::A_MN, Prob::B_MN);

  uint4 ra[8];
  uint4 rb[Cfg::B_CHUNKS];
  const uint4 zero4 = make_uint4(0, 0, 0, 0);

  auto load_stage = [&](int kb) {
    const int k0 = kb * BK;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = j * GEMM_THREADS + tid;
      if (!Prob::A_MN) {
        const int m = m0 + (c & 127), k = k0 + (c >> 7) * 8;
        ra[j] = (m < p.M && k < p.K) ? p.load_a(m, k) : zero4;
      } else {
        const int kl = c & 7, mc = (c >> 3) & 15, kh = c >> 7;
        const int k = k0 + kh * 8 + kl, m = m0 + mc * 8;
        ra[j] = (m < p.M && k < p.K) ? p.load_a(k, m) : zero4;
      }
    }
#pragma unroll
    for (int j = 0; j < Cfg::B_CHUNKS; ++j) {
      const int c = j * GEMM_THREADS + tid;
      if (!Prob::B_MN) {
        const int n = n0 + (c % BN), k = k0 + (c / BN) * 8;
        rb[j] = (n < p.N && k < p.K) ? p.load_b(n, k) : zero4;
      } else {
        const int kl = c & 7, rest = c >> 3;
        const int nc = rest % (BN / 8), kh = rest / (BN / 8);
        const int k = k0 + kh * 8 + kl, n = n0 + nc * 8;
        rb[j] = (n < p.N && k < p.K) ? p.load_b(k, n) : zero4;
      }
    }
  };
  auto store_stage = [&](int s) {
    uint8_t* sa = smem + s * Cfg::STAGE_BYTES;
    uint8_t* sb = sa + Cfg::A_BYTES;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = j * GEMM_THREADS + tid;
      int off;
      if (!Prob::A_MN) off = (c >> 7) * (BM * 16) + (c & 127) * 16;
      else off = (c >> 7) * (BM * 16) + ((c >> 3) & 15) * 128 + (c & 7) * 16;
      *reinterpret_cast<uint4*>(sa + off) = ra[j];
    }
#pragma unroll
    for (int j = 0; j < Cfg::B_CHUNKS; ++j) {
      const int c = j * GEMM_THREADS + tid;
      int off;
      if (!Prob::B_MN) off = (c / BN) * (BN * 16) + (c % BN) * 16;
      else {
        const int rest = c >> 3;
        off = (rest / (BN / 8)) * (BN * 16) + (rest % (BN / 8)) * 128 + (c & 7) * 16;
      }
      *reinterpret_cast<uint4*>(sb + off) = rb[j];
    }
  };

  if (nkb > 0) load_stage(kb_begin);
  for (int i = 0; i < nkb; ++i) {
    const int s = i % S;
    if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
    store_stage(s);
    fence_proxy_async_smem();
    if (i + 1 < nkb) load_stage(kb_begin + i + 1);
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t a_base = smem_u32(smem + s * Cfg::STAGE_BYTES);
      const uint32_t b_base = a_base + Cfg::A_BYTES;
#pragma unroll
      for (int kk = 0; kk < BK / 16; ++kk) {
        const uint64_t ad = umma_desc(a_base + kk * 2 * (BM * 16), BM * 16, 128);
        const uint64_t bd = umma_desc(b_base + kk * 2 * (BN * 16), BN * 16, 128);
        tc_mma_bf16(tmem, ad, bd, idesc, (i > 0 || kk > 0) ? 1u : 0u);
      }
      tc_commit(&empty[s]);
    }
  }
  if (nkb > 0) {
    if (tid == 0) tc_commit(done);
    mbar_wait(done, 0);
    tc_fence_after();
  }
  const int m = m0 + warp * 32 + lane;
#pragma unroll 1
  for (int c = 0; c < BN; c += 16) {
    float v[16];
    if (nkb > 0) {
      tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
    } else {
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = 0.f;
    }
    if (m < p.M && n0 + c < p.N) {
      if (gridDim.z > 1) {
        float* dst = part + ((size_t)blockIdx.z * p.M + m) * p.N + n0 + c;
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (n0 + c + q < p.N) dst[q] = v[q];
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (n0 + c + q < p.N) p.store(m, n0 + c + q, v[q]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, Cfg::TMEM_COLS);
}

template <class Prob>
__global__ void splitk_finish(const Prob p, const float* __restrict__ part, int splits) {
  const size_t MN = (size_t)p.M * p.N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < MN;
       i += (size_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += part[z * MN + i];
    p.store((int)(i / p.N), (int)(i % p.N), s);
  }
}

// Host launcher.  splits > 1 runs split-K over grid.z into `part`
// ([splits][M][N] fp32, caller workspace) followed by splitk_finish.
template <int BN, class Prob>
seed_status launch_gemm(Prob p, int splits, cudaStream_t st, float* part = nullptr) {
  using Cfg = GemmCfg<BN>;
  if (p.M <= 0 || p.N <= 0) return SEED_OK;
  const int nkb = (p.K + GEMM_BK - 1) / GEMM_BK;
  if (splits < 1) splits = 1;
  if (splits > nkb) splits = nkb > 0 ? nkb : 1;
  p.kb_per_split = (nkb + splits - 1) / splits;
  splits = nkb > 0 ? (nkb + p.kb_per_split - 1) / p.kb_per_split : 1;
  static bool attr_done = false;
  if (!attr_done) {
    if (cudaFuncSetAttribute(gemm_tc_kernel<BN, Prob>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Cfg::SMEM) != cudaSuccess)
      return SEED_E_CUDA;
    attr_done = true;
  }
  if (splits > 1 && !part) return SEED_E_WORKSPACE;
  dim3 grid(ceil_div(p.M, GEMM_BM), ceil_div(p.N, BN), splits);
  gemm_tc_kernel<BN, Prob><<<grid, GEMM_THREADS, Cfg::SMEM, st>>>(p, part);
  if (splits > 1) {
    const size_t MN = (size_t)p.M * p.N;
    const int blocks = (int)std::min<size_t>((MN + 255) / 256, 148 * 8);
    splitk_finish<Prob><<<blocks, 256, 0, st>>>(p, part, splits);
  }
  return last_launch();
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
