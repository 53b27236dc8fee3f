// conv_s2d.cu — see conv_s2d.cuh.  Atari-shallow torso (C14; P:591 network
// table, SURVEY.md §8(a) H1 forward / H9 backward) on tcgen05 with TMA bulk
// slabs.
#include <algorithm>
#include "conv_s2d.cuh"

namespace seed {

constexpr int WC_THREADS = 192;   // wgrad: warp 0 TMA producer, warp 1 MMA, warps 2-5 epilogue
// forward / dgrad: warp 0 producer, warp 1 MMA, warps 2-9 = two epilogue groups
// taking alternate tiles (4 TMEM accumulators), so two tiles drain at once
constexpr int WCF_THREADS = 320;
constexpr int WCF_ACC = 4;
constexpr int WC_MAX_STAGES = 8;
constexpr int WC_SMEM_BUDGET = 200 * 1024;
constexpr int WG_KS = 256;        // rows per weight-gradient k-stage

__device__ __forceinline__ uint4 pack8(const float* o) {
  uint4 u;
  u.x = pack_bf16(o[0], o[1]); u.y = pack_bf16(o[2], o[3]);
  u.z = pack_bf16(o[4], o[5]); u.w = pack_bf16(o[6], o[7]);
  return u;
}

// zero rows [z0, z1) of a slab (generic-proxy stores, then made visible to the
// tensor core's async proxy)
__device__ __forceinline__ void zero_rows(uint8_t* dst, int rb, int z0, int z1, int lane) {
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (int i = z0 * rb / 16 + lane; i < z1 * rb / 16; i += 32) reinterpret_cast<uint4*>(dst)[i] = z;
}

// Copy global rows [R0, R0 + n) (row bytes rb, pre-swizzled) to `slab` keeping the
// 1024-byte address phase; rows outside [0, lim) are zero.  Called by one warp;
// lane 0 arms `bar` (expect_tx) and issues the TMA bulk copy.  Returns the
// phase offset of row R0 inside the slab.
__device__ __forceinline__ int load_slab(uint8_t* slab, const uint8_t* src, int rb, int64_t R0, int n,
                                         int64_t lim, uint64_t* bar, int lane, uint32_t extra_tx) {
  const int off0 = (int)(((R0 * rb) % 1024 + 1024) % 1024);
  uint8_t* dst = slab + off0;
  const int64_t lo = std::max<int64_t>(R0, 0), hi = std::min<int64_t>(R0 + n, lim);
  const int zlo = (int)std::min<int64_t>(std::max<int64_t>(lo - R0, 0), n);
  const int zhi = hi > lo ? (int)(hi - R0) : zlo;
  if (zlo > 0 || zhi < n) {
    zero_rows(dst, rb, 0, zlo, lane);
    zero_rows(dst, rb, zhi, n, lane);
    fence_proxy_async_smem();
  }
  __syncwarp();
  if (lane == 0) {
    const uint32_t bytes = hi > lo ? (uint32_t)((hi - lo) * rb) : 0u;
    if (bytes + extra_tx) mbar_expect_tx(bar, bytes + extra_tx);
    else mbar_arrive(bar);
    if (bytes) bulk_g2s(smem_u32(dst + (lo - R0) * rb), src + lo * rb, bytes, bar);
  }
  return off0;
}

__device__ __forceinline__ int slab_phase(int64_t R0, int rb) {
  return (int)(((R0 * rb) % 1024 + 1024) % 1024);
}

// ------------------------------------------------------------------ forward / dgrad
template <class Epi, int RB>
__global__ void __launch_bounds__(WCF_THREADS, 1)
    win_conv_kernel(const WinConvArgs a, const Epi e, int stages, int slab_bytes) {
  constexpr int N = Epi::N;
  constexpr uint32_t LAYOUT = swz_layout_code(RB);
  constexpr int WB = 4 * N * RB;
  constexpr uint32_t TCOLS = WCF_ACC * N < 32 ? 32 : WCF_ACC * N;
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~(uintptr_t)1023);
  uint8_t* Ws = sm;
  uint8_t* slabs = sm + ((WB + 1023) & ~1023);
  __shared__ uint64_t full[WC_MAX_STAGES], empty[WC_MAX_STAGES], tfull[WCF_ACC], tempty[WCF_ACC], wbar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int mn = a.off[0], mx = a.off[0];
#pragma unroll
  for (int w = 1; w < 4; ++w) { mn = min(mn, a.off[w]); mx = max(mx, a.off[w]); }
  const int nrows = 128 + mx - mn;
  const int64_t tiles = (a.M + 127) / 128;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int i = 0; i < WCF_ACC; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 4); }
    mbar_init(&wbar, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&tbase, TCOLS);
  __syncthreads();
  tc_fence_after();
  pdl_wait();
  const uint32_t tmem = tbase;
  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(&wbar, WB);
      bulk_g2s(smem_u32(Ws), a.wimg, WB, &wbar);
    }
    int it = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const int s = it % stages;
      mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
      load_slab(slabs + (size_t)s * slab_bytes, a.src, RB, t * 128 + mn, nrows, a.src_rows, &full[s],
                lane, 0);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      mbar_wait(&wbar, 0);
      const uint32_t idesc = umma_idesc_bf16(128, N, false, false);
      const uint32_t wb = smem_u32(Ws);
      int it = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
        const int s = it % stages, acc = it % WCF_ACC;
        mbar_wait(&full[s], (it / stages) & 1);
        mbar_wait(&tempty[acc], ((it / WCF_ACC) & 1) ^ 1);
        tc_fence_after();
        const uint32_t base =
            smem_u32(slabs + (size_t)s * slab_bytes) + slab_phase(t * 128 + mn, RB);
#pragma unroll
        for (int w = 0; w < 4; ++w)
#pragma unroll
          for (int ks = 0; ks < RB / 32; ++ks) {
            const uint64_t ad = umma_desc(base + (a.off[w] - mn) * RB + ks * 32, 16, 8 * RB, LAYOUT);
            const uint64_t bd = umma_desc(wb + w * N * RB + ks * 32, 16, 8 * RB, LAYOUT);
            tc_mma_bf16(tmem + acc * N, ad, bd, idesc, (w | ks) != 0);
          }
        tc_commit(&empty[s]);
        tc_commit(&tfull[acc]);
      }
    }
  } else {
    const int q = warp & 3;            // TMEM lanes [32q, 32q+32) of this warp
    const int grp = (warp - 2) >> 2;   // epilogue group: tiles it with it % 2 == grp
    int it = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      if ((it & 1) != grp) continue;
      const int acc = it % WCF_ACC;
      mbar_wait(&tfull[acc], (it / WCF_ACC) & 1);
      tc_fence_after();
      float v[N];
#pragma unroll
      for (int c = 0; c < N / 16; ++c)
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + acc * N + c * 16, v + 16 * c);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      const int64_t m = t * 128 + q * 32 + lane;
      if (m < a.M) e.store(m, v);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, TCOLS);
  }
}

template <class Epi, int RB>
seed_status launch_win_conv(const WinConvArgs& a, const Epi& e, cudaStream_t st) {
  constexpr int WB = 4 * Epi::N * RB;
  int mn = a.off[0], mx = a.off[0];
  for (int w = 1; w < 4; ++w) { mn = std::min(mn, a.off[w]); mx = std::max(mx, a.off[w]); }
  const int slab = (int)align_up((size_t)(128 + mx - mn) * RB + 1024, 1024);
  const int wbytes = (int)align_up(WB, 1024);
  const int stages = std::min(WC_MAX_STAGES, (WC_SMEM_BUDGET - wbytes) / slab);
  if (stages < 2 || a.M <= 0) return a.M == 0 ? SEED_OK : SEED_E_SHAPE;
  const size_t smem = (size_t)wbytes + (size_t)stages * slab + 1024;
  static bool attr = false;
  if (!attr) {
    SEED_CUDA_TRY(cudaFuncSetAttribute(win_conv_kernel<Epi, RB>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       WC_SMEM_BUDGET + 2048));
    attr = true;
  }
  const int64_t tiles = (a.M + 127) / 128;
  const int grid = (int)std::min<int64_t>(tiles, 148);
  return launch_k(win_conv_kernel<Epi, RB>, dim3(grid), dim3(WCF_THREADS), smem, st, a, e, stages, slab);
}

// ------------------------------------------------------------------ epilogues
__device__ void Conv1S2dEpi::store(int64_t m, float (&v)[N]) const {
  uint32_t f, rem, oy, ox;
  P1.divmod((uint32_t)m, f, rem);
  W1.divmod(rem, oy, ox);
  if ((int)oy >= Ho || (int)ox >= Wo) return;
  float o[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) o[q] = fmaxf(v[q] * (1.f / 255.f) + bias[q], 0.f);
  const int64_t g1 = (int64_t)f * P2 + (oy >> 1) * W2s + (ox >> 1);
  const int j0 = 2 * ((oy & 1) * 2 + (ox & 1));
  uint8_t* row = S1 + g1 * 128;
  *reinterpret_cast<uint4*>(row + (swz_chunk(g1, 128, j0) << 4)) = pack8(o);
  *reinterpret_cast<uint4*>(row + (swz_chunk(g1, 128, j0 + 1) << 4)) = pack8(o + 8);
}

__device__ void Conv2S2dEpi::store(int64_t m, float (&v)[N]) const {
  uint32_t f, rem, y, x;
  P2.divmod((uint32_t)m, f, rem);
  W2.divmod(rem, y, x);
  if ((int)y < Ho && (int)x < Wo) {
    float o[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) o[q] = fmaxf(v[q] + bias[q], 0.f);
    uint4* dst = reinterpret_cast<uint4*>(act2 + (size_t)f * fc_in + (y * Wo + x) * 32);
#pragma unroll
    for (int j = 0; j < 4; ++j) dst[j] = pack8(o + 8 * j);
  } else if (dY2z) {
    uint4* dst = reinterpret_cast<uint4*>(dY2z + m * 64);
#pragma unroll
    for (int j = 0; j < 4; ++j) dst[j] = make_uint4(0, 0, 0, 0);
  }
}

__device__ void Conv2DgradS2dEpi::store(int64_t p, float (&v)[N]) const {
  uint32_t f, rem, Y, X;
  P2.divmod((uint32_t)p, f, rem);
  W2.divmod(rem, Y, X);
  // ReLU mask of act1 (S1 row p, 64 channels = 4 conv1 pixels x 16)
  const uint8_t* srow = S1 + p * 128;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint4 u = *reinterpret_cast<const uint4*>(srow + (swz_chunk(p, 128, j) << 4));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (!(bf16_lo(w[k]) > 0.f)) v[8 * j + 2 * k] = 0.f;
      if (!(bf16_hi(w[k]) > 0.f)) v[8 * j + 2 * k + 1] = 0.f;
    }
  }
  const int64_t fb = (int64_t)f * P1;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int dy = q >> 1, dx = q & 1;
    const int64_t m1 = fb + (2 * Y + dy) * W1s + 2 * X + dx;
    uint8_t* row = dY1 + m1 * 32;
    *reinterpret_cast<uint4*>(row + (swz_chunk(m1, 32, 0) << 4)) = pack8(v + 16 * q);
    *reinterpret_cast<uint4*>(row + (swz_chunk(m1, 32, 1) << 4)) = pack8(v + 16 * q + 8);
  }
  // padding rows of conv1 output space (ox = W1s-1 / oy = H1s-1) get zeros
  const uint4 z = make_uint4(0, 0, 0, 0);
  if ((int)X == W2s - 1)
    for (int dy = 0; dy < 2; ++dy) {
      uint4* r = reinterpret_cast<uint4*>(dY1 + (fb + (2 * Y + dy) * W1s + W1s - 1) * 32);
      r[0] = z; r[1] = z;
    }
  if ((int)Y == H2s - 1) {
    for (int dx = 0; dx < 2; ++dx) {
      uint4* r = reinterpret_cast<uint4*>(dY1 + (fb + (int64_t)(H1s - 1) * W1s + 2 * X + dx) * 32);
      r[0] = z; r[1] = z;
    }
    if ((int)X == W2s - 1) {
      uint4* r = reinterpret_cast<uint4*>(dY1 + (fb + (int64_t)(H1s - 1) * W1s + W1s - 1) * 32);
      r[0] = z; r[1] = z;
    }
  }
}

// ------------------------------------------------------------------ weight gradient
// Per CTA: rows [z*R, min((z+1)*R, M)) in k-stages of 128 rows.  Accumulators
// (TMEM): tile a (a = 0, 1) = windows (a, 0) and (a, 1) as the two 64-row MN
// atoms of one M=128 operand (atom stride LBO = 128 bytes = one row), tile 2 =
// all-ones operand (every row = the column sum of dY = the bias gradient).
template <int N>
__global__ void __launch_bounds__(WC_THREADS, 1)
    win_wgrad_kernel(const WinWgradArgs a, int stages, int a_bytes, int b_bytes) {
  constexpr int RBY = 2 * N;
  constexpr uint32_t LB = swz_layout_code(RBY);
  constexpr uint32_t TCOLS = 4 * N < 32 ? 32 : (4 * N <= 64 ? 64 : 128);
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~(uintptr_t)1023);
  uint8_t* ones = sm;                  // 1 KB of bf16 1.0
  uint8_t* stg = sm + 1024;            // stages x (A slab | B slab)
  __shared__ uint64_t full[WC_MAX_STAGES], empty[WC_MAX_STAGES], tfull;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r_begin = (int64_t)blockIdx.x * a.rows_per_cta;
  const int64_t r_end = std::min<int64_t>(a.M, r_begin + a.rows_per_cta);
  const int nks = r_end > r_begin ? (int)((r_end - r_begin + WG_KS - 1) / WG_KS) : 0;
  const int arows = WG_KS + a.wsp + 1;
  for (int i = threadIdx.x; i < 64; i += blockDim.x)
    reinterpret_cast<uint4*>(ones)[i] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(&tfull, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&tbase, TCOLS);
  __syncthreads();
  tc_fence_after();
  pdl_wait();
  const uint32_t tmem = tbase;
  if (warp == 0) {
    for (int it = 0; it < nks; ++it) {
      const int s = it % stages;
      mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
      const int64_t k0 = r_begin + (int64_t)it * WG_KS;
      uint8_t* sa = stg + (size_t)s * (a_bytes + b_bytes);
      // B first (its bytes are credited through the A call's expect_tx)
      const int64_t blo = k0, bhi = std::min<int64_t>(k0 + WG_KS, r_end);
      const int boff = slab_phase(k0, RBY);
      uint8_t* bd = sa + a_bytes + boff;
      if (bhi - blo < WG_KS) {
        zero_rows(bd, RBY, (int)(bhi - blo), WG_KS, lane);
        fence_proxy_async_smem();
      }
      __syncwarp();
      const uint32_t bbytes = (uint32_t)((bhi - blo) * RBY);
      load_slab(sa, a.src, 128, k0, arows, a.src_rows, &full[s], lane, bbytes);
      if (lane == 0) bulk_g2s(smem_u32(bd), a.dy + blo * RBY, bbytes, &full[s]);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_bf16(128, N, true, true);
      const uint64_t od = umma_desc(smem_u32(ones), 0, 0, 2);
      for (int it = 0; it < nks; ++it) {
        const int s = it % stages;
        mbar_wait(&full[s], (it / stages) & 1);
        tc_fence_after();
        const int64_t k0 = r_begin + (int64_t)it * WG_KS;
        uint8_t* sa = stg + (size_t)s * (a_bytes + b_bytes);
        const uint32_t abase = smem_u32(sa) + slab_phase(k0, 128);
        const uint32_t bbase = smem_u32(sa + a_bytes) + slab_phase(k0, RBY);
#pragma unroll
        for (int ks = 0; ks < WG_KS / 16; ++ks) {
          const uint64_t bdsc = umma_desc(bbase + ks * 16 * RBY, 8 * RBY, 8 * RBY, LB);
          const uint32_t accf = (it | ks) != 0;
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const uint64_t adsc = umma_desc(abase + (t * a.wsp + ks * 16) * 128, 128, 1024, 2);
            tc_mma_bf16(tmem + t * N, adsc, bdsc, idesc, accf);
          }
          tc_mma_bf16(tmem + 2 * N, od, bdsc, idesc, accf);
        }
        tc_commit(&empty[s]);
      }
      tc_commit(&tfull);
    }
  } else {
    const int q = warp & 3;
    float* part = a.part + (size_t)blockIdx.x * 3 * 128 * N;
    if (nks > 0) {
      mbar_wait(&tfull, 0);
      tc_fence_after();
    }
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      float v[N];
      if (nks > 0) {
#pragma unroll
        for (int c = 0; c < N / 16; ++c)
          tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + t * N + c * 16, v + 16 * c);
      } else {
#pragma unroll
        for (int c = 0; c < N; ++c) v[c] = 0.f;
      }
      const int row = q * 32 + lane;
      if (t < 2 || row == 0) {
        float4* dst = reinterpret_cast<float4*>(part + ((size_t)t * 128 + row) * N);
#pragma unroll
        for (int c = 0; c < N / 4; ++c) dst[c] = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, TCOLS);
  }
}

// fixed-order sum of the per-CTA partials; block = 32 outputs x 8 split groups
__global__ void __launch_bounds__(256) win_wgrad_finish(const float* __restrict__ part, int G, int N,
                                                        const WinWgradFinish f) {
  pdl_wait();
  const int tot = 2 * 128 * N + N;
  const int o = blockIdx.x * 32 + (threadIdx.x & 31), g = threadIdx.x >> 5;
  __shared__ float sh[8][33];
  float s = 0.f;
  size_t idx = 0;
  if (o < tot) {
    idx = o < 2 * 128 * N ? (size_t)o : (size_t)2 * 128 * N + (o - 2 * 128 * N);
    for (int z = g; z < G; z += 8) s += part[(size_t)z * 3 * 128 * N + idx];
  }
  sh[g][threadIdx.x & 31] = s;
  __syncthreads();
  if (g == 0 && o < tot) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += sh[k][threadIdx.x & 31];
    if (o >= 2 * 128 * N) {
      f.g_b[o - 2 * 128 * N] = t;
      return;
    }
    const S2dGeo& g2 = f.g;
    const int tile = o / (128 * N), i = (o / N) % 128, n = o % N;
    const int b = i >> 6, ch = i & 63;
    const int ky1 = ch / (g2.s * g2.C), kx1 = (ch / g2.C) % g2.s, c = ch % g2.C;
    const int K = 2 * g2.s, ky = g2.s * tile + ky1, kx = g2.s * b + kx1;
    f.g_w[(((size_t)n * K + ky) * K + kx) * g2.C + c] = t * f.scale;
  }
}

static int wgrad_grid(int64_t M, int64_t* rows_per_cta) {
  const int64_t kst = (M + WG_KS - 1) / WG_KS;
  const int64_t G0 = std::min<int64_t>(148, std::max<int64_t>(kst, 1));
  const int64_t per = (kst + G0 - 1) / G0;
  *rows_per_cta = per * WG_KS;
  return (int)std::max<int64_t>(1, (M + per * WG_KS - 1) / (per * WG_KS));
}

size_t win_wgrad_part_bytes(int64_t M, int N) {
  int64_t r;
  return (size_t)wgrad_grid(M, &r) * 3 * 128 * N * 4;
}

template <int N>
seed_status launch_win_wgrad(const WinWgradArgs& a0, const WinWgradFinish& fin, cudaStream_t st) {
  WinWgradArgs a = a0;
  const int G = wgrad_grid(a.M, &a.rows_per_cta);
  const int a_bytes = (int)align_up((size_t)(WG_KS + a.wsp + 1) * 128 + 1024, 1024);
  const int b_bytes = (int)align_up((size_t)WG_KS * 2 * N + 1024, 1024);
  const int stages = std::min(WC_MAX_STAGES, (WC_SMEM_BUDGET - 1024) / (a_bytes + b_bytes));
  if (stages < 2) return SEED_E_SHAPE;
  const size_t smem = 2048 + (size_t)stages * (a_bytes + b_bytes);
  static bool attr = false;
  if (!attr) {
    SEED_CUDA_TRY(cudaFuncSetAttribute(win_wgrad_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       WC_SMEM_BUDGET + 2048));
    attr = true;
  }
  SEED_TRY(launch_k(win_wgrad_kernel<N>, dim3(G), dim3(WC_THREADS), smem, st, a, stages, a_bytes,
                    b_bytes));
  const int tot = 2 * 128 * N + N;
  return launch_k(win_wgrad_finish, dim3(ceil_div(tot, 32)), dim3(256), 0, st, (const float*)a.part, G,
                  N, fin);
}

// ------------------------------------------------------------------ obs -> S0
// 8 threads per S0 row, one 16-byte output chunk each (chunk j = obs row 4Y + j/2,
// pixels 4X + 2(j%2) .. +1, 4 channels = 8 input bytes): a warp writes 4 whole rows
__global__ void s2d_obs_kernel(int64_t nrows, FastDiv P, FastDiv Wd, int H, int W,
                               const uint8_t* __restrict__ obs, uint8_t* __restrict__ S0) {
  pdl_wait();
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t g = t >> 3;
  if (g >= nrows) return;
  const int j = (int)(t & 7);
  uint32_t f, rem, Y, X;
  P.divmod((uint32_t)g, f, rem);
  Wd.divmod(rem, Y, X);
  const uint2 u = __ldg(reinterpret_cast<const uint2*>(
      obs + (((size_t)f * H + 4 * Y + (j >> 1)) * W + 4 * X + 2 * (j & 1)) * 4));
  const uint32_t w[2] = {u.x, u.y};
  uint32_t o[4];
#pragma unroll
  for (int k = 0; k < 2; ++k) {   // bytes -> bf16 (exact): the float's high half
    const uint32_t b0 = w[k] & 0xFF, b1 = (w[k] >> 8) & 0xFF, b2 = (w[k] >> 16) & 0xFF, b3 = w[k] >> 24;
    o[2 * k] = (__float_as_uint((float)b0) >> 16) | (__float_as_uint((float)b1) & 0xFFFF0000u);
    o[2 * k + 1] = (__float_as_uint((float)b2) >> 16) | (__float_as_uint((float)b3) & 0xFFFF0000u);
  }
  *reinterpret_cast<uint4*>(S0 + g * 128 + (swz_chunk(g, 128, j) << 4)) = make_uint4(o[0], o[1], o[2], o[3]);
}

seed_status s2d_obs(const uint8_t* obs, int64_t F, int H, int W, uint8_t* S0, cudaStream_t st) {
  const int Hs = H / 4, Ws = W / 4;
  const int64_t n = F * Hs * Ws;
  if (n == 0) return SEED_OK;
  return launch_k(s2d_obs_kernel, dim3((unsigned)((n * 8 + 255) / 256)), dim3(256), 0, st, n,
                  FastDiv(Hs * Ws), FastDiv(Ws), H, W, obs, S0);
}

// ------------------------------------------------------------------ torso
bool shallow_s2d_supported(int H, int W, int C) {
  return C == 4 && H % 4 == 0 && W % 4 == 0 && H >= 12 && W >= 12 && (H / 4 - 1) % 2 == 0 &&
         (W / 4 - 1) % 2 == 0;
}

ShallowS2d shallow_s2d_geometry(int H, int W, int C) {
  ShallowS2d sg{};
  S2dGeo& a = sg.g1;
  a.s = 4; a.C = C; a.CO = 16;
  a.Hs = H / 4; a.Ws = W / 4; a.P = a.Hs * a.Ws; a.Ho = a.Hs - 1; a.Wo = a.Ws - 1;
  S2dGeo& b = sg.g2;
  b.s = 2; b.C = 16; b.CO = 32;
  b.Hs = a.Ho / 2; b.Ws = a.Wo / 2; b.P = b.Hs * b.Ws; b.Ho = b.Hs - 1; b.Wo = b.Ws - 1;
  sg.fc_in = b.Ho * b.Wo * 32;
  return sg;
}

size_t s2d_S0_bytes(const ShallowS2d& sg, int64_t F) { return (size_t)sg.rows1(F) * 128; }
size_t s2d_S1_bytes(const ShallowS2d& sg, int64_t F) { return (size_t)sg.rows2(F) * 128; }
size_t s2d_dY2_bytes(const ShallowS2d& sg, int64_t F) { return (size_t)sg.rows2(F) * 64; }
size_t s2d_dY1_bytes(const ShallowS2d& sg, int64_t F) { return (size_t)sg.rows1(F) * 32; }

seed_status shallow_s2d_conv1(const ShallowS2d& sg, int64_t F, const uint8_t* S0, const bf16* w1img,
                              const float* b1, uint8_t* S1, cudaStream_t st) {
  const S2dGeo& g = sg.g1;
  WinConvArgs a{};
  a.src = S0; a.src_rows = sg.rows1(F); a.M = sg.rows1(F);
  a.off[0] = 0; a.off[1] = 1; a.off[2] = g.Ws; a.off[3] = g.Ws + 1;
  a.wimg = reinterpret_cast<const uint8_t*>(w1img);
  Conv1S2dEpi e{};
  e.bias = b1; e.S1 = S1; e.P1 = FastDiv(g.P); e.W1 = FastDiv(g.Ws);
  e.Ho = g.Ho; e.Wo = g.Wo; e.W2s = sg.g2.Ws; e.P2 = sg.g2.P;
  return launch_win_conv<Conv1S2dEpi, 128>(a, e, st);
}

seed_status shallow_s2d_conv2(const ShallowS2d& sg, int64_t F, const uint8_t* S1, const bf16* w2img,
                              const float* b2, bf16* act2, uint8_t* dY2z, cudaStream_t st) {
  const S2dGeo& g = sg.g2;
  WinConvArgs a{};
  a.src = S1; a.src_rows = sg.rows2(F); a.M = sg.rows2(F);
  a.off[0] = 0; a.off[1] = 1; a.off[2] = g.Ws; a.off[3] = g.Ws + 1;
  a.wimg = reinterpret_cast<const uint8_t*>(w2img);
  Conv2S2dEpi e{};
  e.bias = b2; e.act2 = act2; e.dY2z = dY2z; e.P2 = FastDiv(g.P); e.W2 = FastDiv(g.Ws);
  e.Ho = g.Ho; e.Wo = g.Wo; e.fc_in = sg.fc_in;
  return launch_win_conv<Conv2S2dEpi, 128>(a, e, st);
}

seed_status shallow_s2d_forward(const ShallowS2d& sg, int64_t F, const uint8_t* obs,
                                const bf16* w1img, const float* b1, const bf16* w2img,
                                const float* b2, uint8_t* S0, uint8_t* S1, bf16* act2,
                                uint8_t* dY2z, cudaStream_t st) {
  SEED_TRY(s2d_obs(obs, F, sg.g1.Hs * 4, sg.g1.Ws * 4, S0, st));
  SEED_TRY(shallow_s2d_conv1(sg, F, S0, w1img, b1, S1, st));
  return shallow_s2d_conv2(sg, F, S1, w2img, b2, act2, dY2z, st);
}

seed_status shallow_s2d_conv2_wgrad(const ShallowS2d& sg, int64_t F, const uint8_t* S1,
                                    const uint8_t* dY2, float* part, float* g_w2, float* g_b2,
                                    cudaStream_t st) {
  WinWgradArgs a{};
  a.src = S1; a.src_rows = sg.rows2(F); a.dy = dY2; a.M = sg.rows2(F); a.wsp = sg.g2.Ws; a.part = part;
  WinWgradFinish f{};
  f.g = sg.g2; f.scale = 1.f; f.g_w = g_w2; f.g_b = g_b2;
  return launch_win_wgrad<32>(a, f, st);
}

seed_status shallow_s2d_conv2_dgrad(const ShallowS2d& sg, int64_t F, const uint8_t* dY2,
                                    const bf16* w2dg_img, const uint8_t* S1, uint8_t* dY1,
                                    cudaStream_t st) {
  const S2dGeo& g = sg.g2;
  WinConvArgs a{};
  a.src = dY2; a.src_rows = sg.rows2(F); a.M = sg.rows2(F);
  a.off[0] = 0; a.off[1] = -1; a.off[2] = -g.Ws; a.off[3] = -g.Ws - 1;
  a.wimg = reinterpret_cast<const uint8_t*>(w2dg_img);
  Conv2DgradS2dEpi e{};
  e.S1 = S1; e.dY1 = dY1; e.P2 = FastDiv(g.P); e.W2 = FastDiv(g.Ws); e.H2s = g.Hs; e.W2s = g.Ws;
  e.P1 = sg.g1.P; e.W1s = sg.g1.Ws; e.H1s = sg.g1.Hs;
  return launch_win_conv<Conv2DgradS2dEpi, 64>(a, e, st);
}

seed_status shallow_s2d_conv1_wgrad(const ShallowS2d& sg, int64_t F, const uint8_t* S0,
                                    const uint8_t* dY1, float* part, float* g_w1, float* g_b1,
                                    cudaStream_t st) {
  WinWgradArgs a{};
  a.src = S0; a.src_rows = sg.rows1(F); a.dy = dY1; a.M = sg.rows1(F); a.wsp = sg.g1.Ws; a.part = part;
  WinWgradFinish f{};
  f.g = sg.g1; f.scale = 1.f / 255.f; f.g_w = g_w1; f.g_b = g_b1;
  return launch_win_wgrad<16>(a, f, st);
}

}  // namespace seed
