// win_engine.cuh — the shifted-window convolution engine on tcgen05 (templates
// shared by the Atari-shallow space-to-depth convs, conv_s2d.cu, and the
// IMPALA-deep 3x3 convs, conv3w.cu).
//
// A convolution whose taps are row offsets of one row space (a stride-1
// convolution over an image stored as rows g = (f, Y, X) of RB bytes, borders
// included) is a sum of NW GEMMs whose A operands are the SAME rows shifted:
//   out[g][n] = sum_w sum_k S[g + off_w][k] * Wimg[w][n][k].
// Forward / data gradient (win_conv_kernel): each 128-row output tile copies
// one contiguous slab of rows (128 + max off - min off) with a single TMA bulk
// copy and issues NW x RB/32 tcgen05.mma whose A descriptors start at the
// shifted rows.  Rows are stored pre-swizzled (the 32B / 64B / 128B swizzle of
// the row-relative byte address, common.cuh swz_chunk), so a linear copy that
// keeps the address phase mod 1024 lands every row in the canonical K-major
// operand layout; a start that is not atom-aligned reads the absolute-address
// swizzle (verified on hardware: scripts/probe_umma_shift.cu).
// Weight gradient (win3_wgrad_kernel): reduce over rows, all taps in one MMA per
// 16 rows — A = input rows as an MN-major operand whose atoms are column shifts,
// B = dY rows as an MN-major operand whose atoms are row-window shifts; bias from
// column sums of the dY slab; split over rows with a fixed-order finish
// (deterministic, C21).
#pragma once
#include <algorithm>
#include <type_traits>
#include "common.cuh"

namespace seed {

constexpr int WC_THREADS = 192;   // wgrad: warp 0 TMA producer, warp 1 MMA, warps 2-5 epilogue
// forward / dgrad: warp 0 producer, warp 1 MMA, warps 2-9 = two epilogue groups
// taking alternate tiles (4 TMEM accumulators), so two tiles drain at once
constexpr int WCF_THREADS = 320;
constexpr int WCF_ACC = 4;
constexpr int WC_MAX_STAGES = 8;
constexpr int WC_SMEM_BUDGET = 200 * 1024;
constexpr int WG_KS = 256;        // rows per weight-gradient k-stage
constexpr int WIN_MAX = 9;        // windows per convolution
// weight-gradient partial rows per CTA: 128, or 256 when 64-channel rows (128 B:
// 2 atoms per MMA) need two MMAs for 3 column taps
constexpr int wgrad_prows(int rbx, int nb) { return rbx == 128 && nb >= 3 ? 256 : 128; }

// uint8 source of a 16-channel padded row space (XF_U8): obs [F][H][W][16] bytes
// whose padded row g = f*P + Y*Wp + X holds pixel (Y-1, X-1) (zero borders)
struct U8Rows {
  const uint8_t* obs;
  int H, W, Wp, P;
  FastDiv fP, fWp;
  // interior pixels before padded row g (g < 2^31): the obs pixel index of g if
  // g is interior; consecutive rows map to a contiguous obs range
  __device__ __forceinline__ int64_t idx(int64_t g) const {
    uint32_t f, r, Y, X;
    fP.divmod((uint32_t)g, f, r);
    fWp.divmod(r, Y, X);
    const int y = min(max((int)Y - 1, 0), H);
    const int x = ((int)Y >= 1 && (int)Y <= H) ? min(max((int)X - 1, 0), W) : 0;
    return (int64_t)f * H * W + (int64_t)y * W + x;
  }
  __device__ __forceinline__ bool interior(int64_t g) const {
    uint32_t f, r, Y, X;
    fP.divmod((uint32_t)g, f, r);
    fWp.divmod(r, Y, X);
    return Y >= 1 && (int)Y <= H && X >= 1 && (int)X <= W;
  }
};

// slab transforms between the TMA and the MMA (done by two extra converter warps):
//   XF_NONE  the slab is the MMA operand as copied;
//   XF_RELU  relu in place (the input is h, the conv reads relu(h): the relu copy
//            hr of the residual stream is never stored);
//   XF_U8    the TMA brings the raw uint8 pixels (U8Rows) into a staging buffer and
//            the converters expand them into the bf16 row slab (0..255 exact in
//            bf16), zero borders included — no converted copy of the obs in HBM.
enum { XF_NONE = 0, XF_RELU = 1, XF_U8 = 2 };

struct WinConvArgs {
  const uint8_t* src;    // pre-swizzled rows of RB bytes
  int64_t src_rows;      // rows that exist (others read as zero)
  int64_t M;             // output rows
  int off[WIN_MAX];      // window row offsets
  const uint8_t* wimg;   // pre-swizzled weight image [NW][N][RB]
  U8Rows u8;             // XF_U8 source
  int trig;              // 1: explicit PDL trigger after the wait (common.cuh pdl_wait_trig;
                         // set for the space-to-depth convs, measured slower for the 3x3 ones)
};

__device__ __forceinline__ uint4 pack8(const float* o) {
  uint4 u;
  u.x = pack_bf16(o[0], o[1]); u.y = pack_bf16(o[2], o[3]);
  u.z = pack_bf16(o[4], o[5]); u.w = pack_bf16(o[6], o[7]);
  return u;
}
__device__ __forceinline__ void unpack8(const uint4 u, float* o) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    o[2 * k] = bf16_lo(w[k]);
    o[2 * k + 1] = bf16_hi(w[k]);
  }
}

// zero rows [z0, z1) of a slab (generic-proxy stores; the caller fences)
__device__ __forceinline__ void zero_rows(uint8_t* dst, int rb, int z0, int z1, int lane) {
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (int i = z0 * rb / 16 + lane; i < z1 * rb / 16; i += 32) reinterpret_cast<uint4*>(dst)[i] = z;
}

__device__ __forceinline__ int slab_phase(int64_t R0, int rb) {
  return (int)(((R0 * rb) % 1024 + 1024) % 1024);
}

// Copy global rows [R0, R0 + n) (row bytes rb, pre-swizzled) to `slab` keeping the
// 1024-byte address phase; rows outside [0, lim) are zero.  Called by one warp;
// lane 0 arms `bar` (expect_tx) and issues the TMA bulk copy.
__device__ __forceinline__ void load_slab(uint8_t* slab, const uint8_t* src, int rb, int64_t R0,
                                          int n, int64_t lim, uint64_t* bar, int lane,
                                          uint32_t extra_tx) {
  uint8_t* dst = slab + slab_phase(R0, rb);
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
}

// bf16 bits of 8 bytes (values 0..255, exact): the float's high half
__device__ __forceinline__ uint4 u8x8_to_bf16(uint32_t lo, uint32_t hi) {
  const uint32_t w[2] = {lo, hi};
  uint32_t o[4];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    // (0x4B000000 | b) as float = 2^23 + b exactly; minus 2^23 -> b (FADD, no I2F)
    const float b0 = __uint_as_float(0x4B000000u | (w[k] & 0xFF)) - 8388608.f;
    const float b1 = __uint_as_float(0x4B000000u | ((w[k] >> 8) & 0xFF)) - 8388608.f;
    const float b2 = __uint_as_float(0x4B000000u | ((w[k] >> 16) & 0xFF)) - 8388608.f;
    const float b3 = __uint_as_float(0x4B000000u | (w[k] >> 24)) - 8388608.f;
    o[2 * k] = __byte_perm(__float_as_uint(b0), __float_as_uint(b1), 0x7632);
    o[2 * k + 1] = __byte_perm(__float_as_uint(b2), __float_as_uint(b3), 0x7632);
  }
  return make_uint4(o[0], o[1], o[2], o[3]);
}

// Converter warps (XF_CW of them) of a stage: expand / transform slab rows [0, n)
// whose first row is global row R0.  XF_U8 (rows of 32 bytes = 16 bf16 channels):
// warp cw takes the contiguous row block [cw*n/XF_CW, (cw+1)*n/XF_CW) with its
// lanes striding 32 rows, tracking each lane's (frame, Y, X) incrementally (one
// division per stage, not per row).
constexpr int XF_CW = 4;
template <int XF, int RB>
__device__ __forceinline__ void convert_slab(uint8_t* slab, const uint8_t* stg, int64_t R0, int n,
                                             int64_t lim, const U8Rows& u, int64_t p_lo, int cw,
                                             int lane) {
  uint8_t* dst = slab + slab_phase(R0, RB);
  if constexpr (XF == XF_RELU) {
    const __nv_bfloat162 z2 = __floats2bfloat162_rn(0.f, 0.f);
    uint4* p = reinterpret_cast<uint4*>(dst);
    for (int i = cw * 32 + lane; i < n * RB / 16; i += 32 * XF_CW) {
      uint4 v = p[i];
      uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const __nv_bfloat162 r = __hmax2(*reinterpret_cast<const __nv_bfloat162*>(&w[k]), z2);
        w[k] = *reinterpret_cast<const uint32_t*>(&r);
      }
      p[i] = v;
    }
  } else if constexpr (XF == XF_U8) {
    static_assert(RB == 32, "XF_U8: 16-channel rows");
    const int i0 = (int)((int64_t)n * cw / XF_CW), i1 = (int)((int64_t)n * (cw + 1) / XF_CW);
    int i = i0 + lane;
    int64_t g = R0 + i;
    // (frame, Y, X) of row g (rows < 0 clamp to frame 0; they are zeroed below)
    uint32_t f = 0, Y = 0, X = 0;
    {
      uint32_t r;
      u.fP.divmod((uint32_t)max(g, (int64_t)0), f, r);
      u.fWp.divmod(r, Y, X);
    }
    const int Hp = u.H + 2;
    const int64_t HW = (int64_t)u.H * u.W;
    for (; i < i1; i += 32, g += 32) {
      uint4 c0 = make_uint4(0, 0, 0, 0), c1 = c0;
      if (g >= 0 && g < lim && Y >= 1 && (int)Y <= u.H && X >= 1 && (int)X <= u.W) {
        const int64_t pix = (int64_t)f * HW + (int64_t)(Y - 1) * u.W + (X - 1);
        const uint4 b = *reinterpret_cast<const uint4*>(stg + (pix - p_lo) * 16);
        c0 = u8x8_to_bf16(b.x, b.y);
        c1 = u8x8_to_bf16(b.z, b.w);
      }
      uint8_t* row = dst + (size_t)i * 32;
      const int sw = (int)((g >> 2) & 1);   // swz_chunk(g, 32, j) = j ^ ((g >> 2) & 1)
      *reinterpret_cast<uint4*>(row + ((0 ^ sw) << 4)) = c0;
      *reinterpret_cast<uint4*>(row + ((1 ^ sw) << 4)) = c1;
      if (g >= 0) {   // advance 32 rows
        X += 32;
        while ((int)X >= u.Wp) {
          X -= u.Wp;
          if ((int)++Y == Hp) { Y = 0; ++f; }
        }
      } else if (g + 32 >= 0) {
        uint32_t r;
        u.fP.divmod((uint32_t)(g + 32), f, r);
        u.fWp.divmod(r, Y, X);
      }
    }
  }
}

// XF_U8 producer: the contiguous obs pixel range of padded rows [R0, R0 + n) into
// the staging buffer (one bulk copy, credited to `bar`); returns its first pixel
// (*plo_out is written before the barrier arrival, whose release orders it for the
// converters waiting on `bar`)
__device__ __forceinline__ void load_u8_rows(uint8_t* stg, const U8Rows& u, int64_t R0, int n,
                                             int64_t lim, uint64_t* bar, int lane, uint32_t extra_tx,
                                             int64_t* plo_out) {
  const int64_t lo = max(R0, (int64_t)0), hi = min(R0 + n, lim);
  const int64_t p_lo = hi > lo ? u.idx(lo) : 0, p_hi = hi > lo ? u.idx(hi) : 0;
  if (lane == 0) {
    *plo_out = p_lo;
    const uint32_t bytes = (uint32_t)((p_hi - p_lo) * 16);
    if (bytes + extra_tx) mbar_expect_tx(bar, bytes + extra_tx);
    else mbar_arrive(bar);
    if (bytes) bulk_g2s(smem_u32(stg), u.obs + p_lo * 16, bytes, bar);
  }
}


// ------------------------------------------------------------------ forward / dgrad
// Epi: static constexpr int N; __device__ void store(int64_t m, float (&v)[N]) const
// An epilogue that reads other rows of global memory (residual input, ReLU mask)
// declares static constexpr int PRE = uint4 chunks per output row and
//   __device__ void pre(int64_t m, uint4 (&p)[PRE]) const   (issue the loads)
//   __device__ void store(int64_t m, float (&v)[N], const uint4 (&p)[PRE]) const
// The engine issues pre() for all of a tile's rows BEFORE waiting for the tile's
// accumulator, so those loads are in flight during the MMAs instead of being
// dependent loads inside the epilogue (measured: the residual / masked epilogues
// were latency-bound on them, profiles/r02/ncu_c4_deep.md).
// A tile is MT x 128 output rows: one slab of MT*128 + (max off - min off) rows, MT
// accumulators of N columns (bigger tiles re-read fewer halo rows from L2 and pay
// the per-tile barrier / commit latency once per MT blocks).
template <class E, class = void>
struct EpiPre { static constexpr int n = 0; };
template <class E>
struct EpiPre<E, std::void_t<decltype(E::PRE)>> { static constexpr int n = E::PRE; };
template <class E, class P>
__device__ __forceinline__ void epi_store(const E& e, int64_t m, float (&v)[E::N], const P& pre) {
  if constexpr (EpiPre<E>::n > 0) e.store(m, v, pre);
  else e.store(m, v);
}

template <class Epi, int RB, int NW, int MT = 1, int XF = XF_NONE>
__global__ void __launch_bounds__(WCF_THREADS + (XF != XF_NONE ? 32 * XF_CW : 0), 1)
    win_conv_kernel(const WinConvArgs a, const Epi e, int stages, int slab_bytes, int stg_bytes) {
  constexpr int N = Epi::N;
  constexpr int TM = 128 * MT;
  constexpr uint32_t LAYOUT = swz_layout_code(RB);
  constexpr int WB = NW * N * RB;
  constexpr int AC = MT * N;   // TMEM columns per tile accumulator
  constexpr uint32_t TCOLS = WCF_ACC * AC <= 32 ? 32 : WCF_ACC * AC <= 64 ? 64 : WCF_ACC * AC <= 128 ? 128
                             : WCF_ACC * AC <= 256 ? 256 : 512;
  static_assert(WCF_ACC * AC <= 512, "TMEM");
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = smem_align1024(smraw);
  uint8_t* Ws = sm;
  uint8_t* slabs = sm + ((WB + 1023) & ~1023);
  uint8_t* stgs = slabs + (size_t)stages * slab_bytes;   // XF_U8 staging, stg_bytes each
  __shared__ uint64_t full[WC_MAX_STAGES], empty[WC_MAX_STAGES], tfull[WCF_ACC], tempty[WCF_ACC], wbar;
  __shared__ uint64_t ready[WC_MAX_STAGES];   // XF: converters done (count XF_CW)
  __shared__ int64_t plo[WC_MAX_STAGES];      // XF_U8: first pixel of each stage's staging
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int mn = a.off[0], mx = a.off[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) { mn = min(mn, a.off[w]); mx = max(mx, a.off[w]); }
  const int nrows = TM + mx - mn;
  const int64_t tiles = (a.M + TM - 1) / TM;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&ready[s], XF_CW);
    }
    for (int i = 0; i < WCF_ACC; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 4); }
    mbar_init(&wbar, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&tbase, TCOLS);
  __syncthreads();
  tc_fence_after();
  // the weight image was last written by the previous step's Adam / image refresh
  // (many kernels back, each of which waited on its predecessor): fetch it before
  // the PDL wait, overlapping the preceding kernel's tail
  if (warp == 0 && lane == 0) {
    mbar_expect_tx(&wbar, WB);
    bulk_g2s(smem_u32(Ws), a.wimg, WB, &wbar);
  }
  pdl_wait();
  if (a.trig) pdl_trigger();
  const uint32_t tmem = tbase;
  if (warp == 0) {
    int it = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const int s = it % stages;
      mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
      if constexpr (XF == XF_U8) {
        load_u8_rows(stgs + (size_t)s * stg_bytes, a.u8, t * TM + mn, nrows, a.src_rows, &full[s], lane, 0,
                     &plo[s]);
      } else {
        load_slab(slabs + (size_t)s * slab_bytes, a.src, RB, t * TM + mn, nrows, a.src_rows, &full[s],
                  lane, 0);
      }
    }
  } else if (XF != XF_NONE && warp >= 10) {   // slab converters
    const int cw = warp - 10;
    int it = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const int s = it % stages;
      mbar_wait(&full[s], (it / stages) & 1);
      convert_slab<XF, RB>(slabs + (size_t)s * slab_bytes, stgs + (size_t)s * stg_bytes, t * TM + mn, nrows,
                           a.src_rows, a.u8, XF == XF_U8 ? plo[s] : 0, cw, lane);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ready[s]);
    }
  } else if (warp == 1) {   // MMA issue: warp-uniform, one elected lane issues
    mbar_wait(&wbar, 0);
    const uint32_t idesc = umma_idesc_bf16(128, N, false, false);
    const uint64_t bd0 = umma_desc(smem_u32(Ws), 16, 8 * RB, LAYOUT);
    int aoff[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) aoff[w] = ((a.off[w] - mn) * RB) >> 4;
    int it = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const int s = it % stages, acc = it % WCF_ACC;
      mbar_wait(XF != XF_NONE ? &ready[s] : &full[s], (it / stages) & 1);
      mbar_wait(&tempty[acc], ((it / WCF_ACC) & 1) ^ 1);
      tc_fence_after();
      const uint32_t base = smem_u32(slabs + (size_t)s * slab_bytes) + slab_phase(t * TM + mn, RB);
      // descriptors advance linearly with the start address (field = addr >> 4)
      const uint64_t ad0 = umma_desc(base, 16, 8 * RB, LAYOUT);
      // fully unrolled unless that would exceed 36 MMAs (register spills)
      constexpr int MT_UNROLL = MT * NW * (RB / 32) > 36 ? 1 : MT;
#pragma unroll MT_UNROLL
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int w = 0; w < NW; ++w)
#pragma unroll
          for (int ks = 0; ks < RB / 32; ++ks)
            tc_mma_bf16_w(tmem + acc * AC + mt * N,
                          ad0 + (uint64_t)(aoff[w] + ((mt * 128 * RB) >> 4) + ks * 2),
                          bd0 + (uint64_t)((w * N * RB + ks * 32) >> 4), idesc, (w | ks) != 0);
      tc_commit_w(&empty[s]);
      tc_commit_w(&tfull[acc]);
    }
  } else if (warp < 10) {
    const int q = warp & 3;            // TMEM lanes [32q, 32q+32) of this warp
    const int grp = (warp - 2) >> 2;   // epilogue group: tiles it with it % 2 == grp
    int it = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      if ((it & 1) != grp) continue;
      const int acc = it % WCF_ACC;
      constexpr int PN = EpiPre<Epi>::n > 0 ? EpiPre<Epi>::n : 1;
      uint4 pre[MT][PN];
      if constexpr (EpiPre<Epi>::n > 0) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int64_t m = t * TM + mt * 128 + q * 32 + lane;
          if (m < a.M) e.pre(m, pre[mt]);
        }
      }
      mbar_wait(&tfull[acc], (it / WCF_ACC) & 1);
      tc_fence_after();
      uint32_t vr[MT][N];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int c = 0; c < N / 16; ++c)
          tmem_ld16_nw(tmem + ((uint32_t)(q * 32) << 16) + acc * AC + mt * N + c * 16,
                       *reinterpret_cast<uint32_t(*)[16]>(&vr[mt][16 * c]));
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        float v[N];
#pragma unroll
        for (int c = 0; c < N; ++c) v[c] = __uint_as_float(vr[mt][c]);
        const int64_t m = t * TM + mt * 128 + q * 32 + lane;
        if (m < a.M) epi_store(e, m, v, pre[mt]);
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, TCOLS);
  }
}

template <class Epi, int RB, int NW, int MT = 1, int XF = XF_NONE>
seed_status launch_win_conv(const WinConvArgs& a, const Epi& e, cudaStream_t st) {
  constexpr int WB = NW * Epi::N * RB;
  constexpr int TM = 128 * MT;
  int mn = a.off[0], mx = a.off[0];
  for (int w = 1; w < NW; ++w) { mn = std::min(mn, a.off[w]); mx = std::max(mx, a.off[w]); }
  const int slab = (int)align_up((size_t)(TM + mx - mn) * RB + 1024, 1024);
  // XF_U8 staging: the slab's pixels as uint8 (16 bytes each)
  const int stg = XF == XF_U8 ? (int)align_up((size_t)(TM + mx - mn) * 16 + 16, 1024) : 0;
  const int wbytes = (int)align_up(WB, 1024);
  const int stages = std::min(WC_MAX_STAGES, (WC_SMEM_BUDGET - wbytes) / (slab + stg));
  if (a.M <= 0) return a.M == 0 ? SEED_OK : SEED_E_SHAPE;
  if (stages < 2) return SEED_E_SHAPE;
  const size_t smem = (size_t)wbytes + (size_t)stages * (slab + stg) + 1024;
  static PerDevice attr;
  SEED_TRY(smem_optin(attr, win_conv_kernel<Epi, RB, NW, MT, XF>, WC_SMEM_BUDGET + 2048));
  const int64_t tiles = (a.M + TM - 1) / TM;
  const int grid = (int)std::min<int64_t>(tiles, sm_count());
  const int threads = WCF_THREADS + (XF != XF_NONE ? 32 * XF_CW : 0);
  return launch_k(win_conv_kernel<Epi, RB, NW, MT, XF>, dim3(grid), dim3(threads), smem, st, a, e,
                  stages, slab, stg);
}

// ------------------------------------------------------------------ column-tap-stacked 3x3
// A 3x3 conv over the padded row space with the three column taps (kx) stacked on
// N: one MMA per row window ky (N = 3*NO, K = RB/2 channels) computes
//   D[g][j*NO + o] = sum_ky sum_k S[g + off_ky][k] * Wimg[ky][j*NO + o][k]
// and the epilogue combines neighbouring rows:
//   out[g][o] = D[g-1][0*NO + o] + D[g][1*NO + o] + D[g+1][2*NO + o]
// (forward: j = kx, off_ky = (ky-1)*Wp; data gradient: j = 2-kx with the mode-1
// image, off_ky = -(ky-1)*Wp — the same combination).  3 MMAs per 128 rows instead
// of 9, reading the A rows 3 times instead of 9: the 16/32-channel convs are bound
// by the shared-memory operand reads of their small tcgen05.mma
// (profiles/r02/conv_pool_fused.md), not by HBM.
// Tiles of TM = 128*MT MMA rows overlap by 2 rows: tile t computes rows
// [t*TS - 1, t*TS - 1 + TM) and outputs [t*TS, t*TS + TS), TS = TM - 2, so every
// output row's neighbours are in its own tile.  Epilogue: NG groups of 4 warps take
// tiles round robin (one TMEM accumulator each).  A warp drains each 32-row block
// of its TMEM lane quarter once (three 16-column loads per 16 outputs) and takes
// rows r-1 / r+1 from the neighbouring lanes (shuffles); lanes 31 / 0 leave the
// part the neighbouring quarter's edge row needs in a shared-memory exchange
// (double-buffered per group) and, after one named barrier, lanes 0 / 31 add it
// and the whole warp stores (the tile's sums stay in registers across the
// barrier: MT*NO <= 32).  Edge rows sum D[g-1] + (D[g] + D[g+1]) /
// (D[g-1] + D[g]) + D[g+1], interior rows (D[g-1] + D[g]) + D[g+1].
// (A non-finite D of a quarter's edge row times the 0 mask would poison that row
// with NaN; the D here are finite bf16-operand sums.)
template <class Epi, int RB, int MT, int NG>
__global__ void __launch_bounds__(64 + 128 * NG, 1)
    win_conv_kx_kernel(const WinConvArgs a, const Epi e, int stages, int slab_bytes) {
  constexpr int NO = Epi::N;          // output channels
  constexpr int N = 3 * NO;           // MMA N: kx-stacked
  constexpr int TM = 128 * MT, TS = TM - 2;
  constexpr uint32_t LAYOUT = swz_layout_code(RB);
  constexpr int WB = 3 * N * RB;
  constexpr int AC = MT * N;          // TMEM columns per tile accumulator (one per group)
  constexpr uint32_t TCOLS = NG * AC <= 128 ? 128 : NG * AC <= 256 ? 256 : 512;
  static_assert(NG * AC <= 512, "TMEM");
  static_assert(NO % 16 == 0, "NO");
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = smem_align1024(smraw);
  uint8_t* Ws = sm;
  uint8_t* slabs = sm + ((WB + 1023) & ~1023);
  // exchange [group][buffer][slot = mt*4 + quarter][ 0: D0 of lane 31 | 1: D2 of lane 0 ][NO]
  float* xch = reinterpret_cast<float*>(slabs + (size_t)stages * slab_bytes);
  __shared__ uint64_t full[WC_MAX_STAGES], empty[WC_MAX_STAGES], tfull[NG], tempty[NG], wbar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mn = min(a.off[0], min(a.off[1], a.off[2]));
  const int mx = max(a.off[0], max(a.off[1], a.off[2]));
  const int nrows = TM + mx - mn;
  const int64_t tiles = (a.M + TS - 1) / TS;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int i = 0; i < NG; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 4); }
    mbar_init(&wbar, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&tbase, TCOLS);
  __syncthreads();
  tc_fence_after();
  if (warp == 0 && lane == 0) {
    mbar_expect_tx(&wbar, WB);
    bulk_g2s(smem_u32(Ws), a.wimg, WB, &wbar);
  }
  pdl_wait();
  const uint32_t tmem = tbase;
  if (warp == 0) {
    int it = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const int s = it % stages;
      mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
      load_slab(slabs + (size_t)s * slab_bytes, a.src, RB, t * TS - 1 + mn, nrows, a.src_rows,
                &full[s], lane, 0);
    }
  } else if (warp == 1) {   // MMA issue: warp-uniform, one elected lane issues
    mbar_wait(&wbar, 0);
    const uint32_t idesc = umma_idesc_bf16(128, N, false, false);
    const uint64_t bd0 = umma_desc(smem_u32(Ws), 16, 8 * RB, LAYOUT);
    int aoff[3];
#pragma unroll
    for (int w = 0; w < 3; ++w) aoff[w] = ((a.off[w] - mn) * RB) >> 4;
    int it = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const int s = it % stages, acc = it % NG;
      mbar_wait(&full[s], (it / stages) & 1);
      mbar_wait(&tempty[acc], ((it / NG) & 1) ^ 1);
      tc_fence_after();
      const uint32_t base = smem_u32(slabs + (size_t)s * slab_bytes) + slab_phase(t * TS - 1 + mn, RB);
      const uint64_t ad0 = umma_desc(base, 16, 8 * RB, LAYOUT);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int w = 0; w < 3; ++w)
#pragma unroll
          for (int ks = 0; ks < RB / 32; ++ks)
            tc_mma_bf16_w(tmem + acc * AC + mt * N,
                          ad0 + (uint64_t)(aoff[w] + ((mt * 128 * RB) >> 4) + ks * 2),
                          bd0 + (uint64_t)((w * N * RB + ks * 32) >> 4), idesc, (w | ks) != 0);
      tc_commit_w(&empty[s]);
      tc_commit_w(&tfull[acc]);
    }
  } else {
    const int q = warp & 3;            // TMEM lanes [32q, 32q+32) of this warp
    const int grp = (warp - 2) >> 2;   // epilogue group: tiles it with it % NG == grp
    constexpr int PN = EpiPre<Epi>::n > 0 ? EpiPre<Epi>::n : 1;
    const float m_up = lane == 0 ? 0.f : 1.f, m_dn = lane == 31 ? 0.f : 1.f;
    int it = 0, gt = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      if (it % NG != grp) continue;
      const int64_t g0 = t * TS - 1;   // global row of MMA row 0
      uint4 pre[MT][PN];
      if constexpr (EpiPre<Epi>::n > 0) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int r = mt * 128 + q * 32 + lane;
          const int64_t m = g0 + r;
          if (r >= 1 && r <= TM - 2 && m < a.M) e.pre(m, pre[mt]);
        }
      }
      mbar_wait(&tfull[grp], (it / NG) & 1);
      tc_fence_after();
      const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16) + grp * AC;
      float* xb = xch + (size_t)(grp * 2 + (gt & 1)) * MT * 4 * 2 * NO;
      float v[MT][NO];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int slot = mt * 4 + q;
#pragma unroll
        for (int c = 0; c < NO / 16; ++c) {
          uint32_t p0[16], p1[16], p2[16];
          tmem_ld16_nw(tb + mt * N + c * 16, p0);
          tmem_ld16_nw(tb + mt * N + NO + c * 16, p1);
          tmem_ld16_nw(tb + mt * N + 2 * NO + c * 16, p2);
          tmem_wait_ld();
          // (up + D1) + dn with the lane-0 up / lane-31 dn masked out by an exact
          // multiply by 0 (one FFMA each instead of a select and an add)
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const float up = __shfl_up_sync(0xffffffffu, __uint_as_float(p0[k]), 1);     // D[r-1] part 0
            const float dn = __shfl_down_sync(0xffffffffu, __uint_as_float(p2[k]), 1);   // D[r+1] part 2
            v[mt][c * 16 + k] = fmaf(dn, m_dn, fmaf(up, m_up, __uint_as_float(p1[k])));
          }
          // the part the neighbouring quarter's edge row needs
          if (lane == 31) {
            float4* dst = reinterpret_cast<float4*>(xb + (slot * 2 + 0) * NO + c * 16);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              dst[k] = make_float4(__uint_as_float(p0[4 * k]), __uint_as_float(p0[4 * k + 1]),
                                   __uint_as_float(p0[4 * k + 2]), __uint_as_float(p0[4 * k + 3]));
          }
          if (lane == 0) {
            float4* dst = reinterpret_cast<float4*>(xb + (slot * 2 + 1) * NO + c * 16);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              dst[k] = make_float4(__uint_as_float(p2[4 * k]), __uint_as_float(p2[4 * k + 1]),
                                   __uint_as_float(p2[4 * k + 2]), __uint_as_float(p2[4 * k + 3]));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[grp]);
      asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory");   // exchange written
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int r = mt * 128 + q * 32 + lane;
        const int slot = mt * 4 + q;
        const int64_t m = g0 + r;
        if (!(r >= 1 && r <= TM - 2 && m < a.M)) continue;   // also slot 0 lane 0 / last slot lane 31
        if (lane == 0) {   // edge rows: D[g-1] + partial / partial + D[g+1]
          const float4* nb = reinterpret_cast<const float4*>(xb + ((slot - 1) * 2 + 0) * NO);
#pragma unroll
          for (int k = 0; k < NO / 4; ++k) {
            const float4 y = nb[k];
            v[mt][4 * k] = y.x + v[mt][4 * k]; v[mt][4 * k + 1] = y.y + v[mt][4 * k + 1];
            v[mt][4 * k + 2] = y.z + v[mt][4 * k + 2]; v[mt][4 * k + 3] = y.w + v[mt][4 * k + 3];
          }
        }
        if (lane == 31) {
          const float4* nb = reinterpret_cast<const float4*>(xb + ((slot + 1) * 2 + 1) * NO);
#pragma unroll
          for (int k = 0; k < NO / 4; ++k) {
            const float4 y = nb[k];
            v[mt][4 * k] += y.x; v[mt][4 * k + 1] += y.y; v[mt][4 * k + 2] += y.z; v[mt][4 * k + 3] += y.w;
          }
        }
        epi_store(e, m, v[mt], pre[mt]);
      }
      ++gt;
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, TCOLS);
  }
}

template <class Epi, int RB, int MT, int NG>
seed_status launch_win_conv_kx(const WinConvArgs& a, const Epi& e, cudaStream_t st) {
  constexpr int WB = 3 * 3 * Epi::N * RB;
  constexpr int TM = 128 * MT, TS = TM - 2;
  const int mn = std::min(a.off[0], std::min(a.off[1], a.off[2]));
  const int mx = std::max(a.off[0], std::max(a.off[1], a.off[2]));
  const int slab = (int)align_up((size_t)(TM + mx - mn) * RB + 1024, 1024);
  const int wbytes = (int)align_up(WB, 1024);
  const int xbytes = NG * 2 * MT * 4 * 2 * Epi::N * 4;   // exchange
  const int stages = std::min(WC_MAX_STAGES, (WC_SMEM_BUDGET - wbytes - xbytes) / slab);
  if (a.M <= 0) return a.M == 0 ? SEED_OK : SEED_E_SHAPE;
  if (stages < 2) return SEED_E_SHAPE;
  const size_t smem = (size_t)wbytes + (size_t)stages * slab + xbytes + 1024;
  static PerDevice attr;
  SEED_TRY(smem_optin(attr, win_conv_kx_kernel<Epi, RB, MT, NG>, WC_SMEM_BUDGET + 2048));
  const int64_t tiles = (a.M + TS - 1) / TS;
  const int grid = (int)std::min<int64_t>(tiles, sm_count());
  return launch_k(win_conv_kx_kernel<Epi, RB, MT, NG>, dim3(grid), dim3(64 + 128 * NG), smem, st, a, e,
                  stages, slab);
}

inline int wgrad_grid(int64_t M, int64_t* rows_per_cta) {
  const int64_t kst = (M + WG_KS - 1) / WG_KS;
  const int64_t G0 = std::min<int64_t>(148, std::max<int64_t>(kst, 1));
  const int64_t per = (kst + G0 - 1) / G0;
  *rows_per_cta = per * WG_KS;
  return (int)std::max<int64_t>(1, (M + per * WG_KS - 1) / (per * WG_KS));
}

// ------------------------------------------------------------------ 3x3 weight gradient
// All nine taps in ONE tcgen05.mma per 16 rows (M = 128, N = 3*CO):
//   dW[ky][kx][c][co] = sum_h X[h + kx][c] * dY[h + boff + (2-ky)*bstride][co]
// A = X rows as an MN-major operand of 256/RBX atoms (kx = atom, LBO = one row),
// B = dY rows as an MN-major operand of 3 atoms (ky = 2 - atom, LBO = bstride rows);
// the bias gradient (BIAS) is summed from the same B slab by the 4 epilogue warps,
// idle during the main loop: rows h + boff + bstride (dY shifted by at most one
// row, which only moves border / zero rows), fixed order, released to the
// producer through the stage's empty barrier (2 arrivals: MMA commit + epilogue).
struct Win3WgradArgs {
  const uint8_t* X;      // rows of RBX bytes (XF_U8: unused, the rows come from u8)
  const uint8_t* dy;     // rows of 2*CO bytes
  int64_t M;             // rows (X and dY share the row space)
  int boff, bstride;     // B atom j starts at row h + boff + j*bstride
  int64_t rows_per_cta;
  float* part;           // [grid][128][4*CO] (cols [0, 3CO) weights, [3CO, 4CO) bias in row 0)
  U8Rows u8;             // XF_U8 source of the X rows
  int trig;              // as WinConvArgs::trig (also for the finish launch)
};

template <int CO, int RBX, bool BIAS, int NB = 3, int XF = XF_NONE>
__global__ void __launch_bounds__(WC_THREADS + (XF != XF_NONE ? 32 * XF_CW : 0), 1)
    win3_wgrad_kernel(const Win3WgradArgs a, int stages, int a_bytes, int b_bytes, int stg_bytes) {
  constexpr int RBY = 2 * CO;
  // M = 64 when the rows are 16 channels (32 B): 4 atoms (kx = 0..2 used of 4)
  // instead of 8 — half the shared-memory operand reads per MMA for the same
  // ~45-cycle issue (the weight gradients were bound by those reads;
  // profiles/r02/wgrad_m64.md).  TMEM layout of M = 64 (scripts/probe_umma_m64.cu):
  // row m at lane (m / 16) * 32 + m % 16.
  constexpr int MM = RBX == 32 ? 64 : 128;
  constexpr int NA = 2 * MM / RBX;        // A atoms per MMA
  // 64-channel rows (RBX = 128): 2 atoms per M = 128, so the three kx taps take two
  // MMAs per 16 rows (atoms kx 0-1, and kx 2-3 from two rows further), two accumulators
  constexpr int NMMA = NA >= NB ? 1 : 2;   // (NB = the kernel's side: column taps too)
  constexpr int PROWS = wgrad_prows(RBX, NB);   // partial rows per CTA (= NMMA * MM, >= 128)
  static_assert(PROWS >= NMMA * MM, "partial rows");
  constexpr int NW = NB * CO;             // weight columns (NB B atoms)
  constexpr int PC = (NB + 1) * CO;       // partial row: weights | bias
  constexpr uint32_t LA = swz_layout_code(RBX), LB = swz_layout_code(RBY);
  constexpr int ACOL = NW <= 64 ? 64 : NW <= 128 ? 128 : 256;   // columns per accumulator
  constexpr uint32_t TCOLS = NMMA * ACOL <= 64 ? 64 : NMMA * ACOL <= 128 ? 128 : NMMA * ACOL <= 256 ? 256 : 512;
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = smem_align1024(smraw);
  uint8_t* stg = sm + 1024;
  const size_t sst = (size_t)a_bytes + b_bytes + stg_bytes;   // stage stride
  __shared__ uint64_t full[WC_MAX_STAGES], empty[WC_MAX_STAGES], tfull;
  __shared__ uint64_t ready[WC_MAX_STAGES];   // XF: A slab transformed (converter warps 6..)
  __shared__ int64_t plo[WC_MAX_STAGES];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r_begin = (int64_t)blockIdx.x * a.rows_per_cta;
  const int64_t r_end = std::min<int64_t>(a.M, r_begin + a.rows_per_cta);
  const int nks = r_end > r_begin ? (int)((r_end - r_begin + WG_KS - 1) / WG_KS) : 0;
  const int arows = WG_KS + NA * NMMA - 1, brows = WG_KS + (NB - 1) * a.bstride;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], BIAS ? 2 : 1);
      mbar_init(&ready[s], XF_CW);
    }
    mbar_init(&tfull, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&tbase, TCOLS);
  __syncthreads();
  tc_fence_after();
  pdl_wait();
  if (a.trig) pdl_trigger();
  const uint32_t tmem = tbase;
  if (warp == 0) {
    for (int it = 0; it < nks; ++it) {
      const int s = it % stages;
      mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
      const int64_t k0 = r_begin + (int64_t)it * WG_KS;
      uint8_t* sa = stg + (size_t)s * sst;
      // rows_per_cta is a multiple of WG_KS, so only the last CTA has a partial last
      // stage, and there every K index h >= M reads X rows >= M (zero-filled)
      const int64_t lo = std::max<int64_t>(k0 + a.boff, 0),
                    hi = std::min<int64_t>(k0 + a.boff + brows, a.M);
      const uint32_t bbytes = hi > lo ? (uint32_t)((hi - lo) * RBY) : 0u;
      // B: zero the out-of-range rows, then one bulk copy (credited via A's expect_tx)
      uint8_t* bd = sa + a_bytes + slab_phase(k0 + a.boff, RBY);
      const int zlo = (int)std::min<int64_t>(std::max<int64_t>(lo - (k0 + a.boff), 0), brows);
      const int zhi = hi > lo ? (int)(hi - (k0 + a.boff)) : zlo;
      if (zlo > 0 || zhi < brows) {
        zero_rows(bd, RBY, 0, zlo, lane);
        zero_rows(bd, RBY, zhi, brows, lane);
        fence_proxy_async_smem();
      }
      __syncwarp();
      if constexpr (XF == XF_U8)
        load_u8_rows(sa + a_bytes + b_bytes, a.u8, k0, arows, a.M, &full[s], lane, bbytes, &plo[s]);
      else
        load_slab(sa, a.X, RBX, k0, arows, a.M, &full[s], lane, bbytes);
      if (lane == 0 && bbytes) bulk_g2s(smem_u32(bd + zlo * RBY), a.dy + lo * RBY, bbytes, &full[s]);
    }
  } else if (XF != XF_NONE && warp >= 6) {   // A-slab converters
    for (int it = 0; it < nks; ++it) {
      const int s = it % stages;
      mbar_wait(&full[s], (it / stages) & 1);
      const int64_t k0 = r_begin + (int64_t)it * WG_KS;
      uint8_t* sa = stg + (size_t)s * sst;
      convert_slab<XF, RBX>(sa, sa + a_bytes + b_bytes, k0, arows, a.M, a.u8, XF == XF_U8 ? plo[s] : 0,
                            warp - 6, lane);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ready[s]);
    }
  } else if (warp == 1) {   // MMA issue: warp-uniform, one elected lane issues
    const uint32_t idesc = umma_idesc_bf16(MM, NW, true, true);
    const uint32_t blbo = (uint32_t)(a.bstride * RBY);
    for (int it = 0; it < nks; ++it) {
      const int s = it % stages;
      mbar_wait(XF != XF_NONE ? &ready[s] : &full[s], (it / stages) & 1);
      tc_fence_after();
      const int64_t k0 = r_begin + (int64_t)it * WG_KS;
      uint8_t* sa = stg + (size_t)s * sst;
      const uint64_t ad0 = umma_desc(smem_u32(sa) + slab_phase(k0, RBX), RBX, 8 * RBX, LA);
      const uint64_t bd0 =
          umma_desc(smem_u32(sa + a_bytes) + slab_phase(k0 + a.boff, RBY), blbo, 8 * RBY, LB);
      const uint32_t acc0 = it != 0;
#pragma unroll
      for (int ks = 0; ks < WG_KS / 16; ++ks) {
        const uint32_t accf = acc0 | (ks != 0);
#pragma unroll
        for (int mi = 0; mi < NMMA; ++mi)
          tc_mma_bf16_w(tmem + mi * ACOL, ad0 + (uint64_t)((ks * 16 * RBX + mi * NA * RBX) >> 4),
                        bd0 + (uint64_t)((ks * 16 * RBY) >> 4), idesc, accf);
      }
      tc_commit_w(&empty[s]);
    }
    tc_commit_w(&tfull);
  } else if (warp < 6) {
    const int q = warp & 3;
    float* part = a.part + (size_t)blockIdx.x * PROWS * PC;
    // accumulator row of this thread's TMEM lane (M = 64: lanes 0-15 of each quarter)
    const int row = MM == 128 ? q * 32 + lane : q * 16 + lane;
    const bool row_ok = MM == 128 || lane < 16;
    const int et = threadIdx.x - 64;   // 0..127
    if (BIAS) {
      // thread = (chunk j of 8 channels, row phase): rows i = rp, rp + 128/NCH, ...
      constexpr int NCH = CO / 8, RSTEP = 128 / NCH;
      const int j = et % NCH, rp = et / NCH;
      float bs[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int it = 0; it < nks; ++it) {
        const int s = it % stages;
        mbar_wait(&full[s], (it / stages) & 1);
        const int64_t k0 = r_begin + (int64_t)it * WG_KS;
        const uint8_t* bsl = stg + (size_t)s * sst + a_bytes + slab_phase(k0 + a.boff, RBY);
#pragma unroll 4
        for (int i = rp; i < WG_KS; i += RSTEP) {
          const int lr = i + a.bstride;                        // slab row of dY[h + boff + bstride]
          const int64_t g = k0 + a.boff + lr;                  // its global row (swizzle phase)
          float v[8];
          unpack8(*reinterpret_cast<const uint4*>(bsl + lr * RBY + (swz_chunk(g, RBY, j) << 4)), v);
#pragma unroll
          for (int k = 0; k < 8; ++k) bs[k] += v[k];
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (et == 0) mbar_arrive(&empty[s]);
      }
      // fixed-order reduction over the row phases, through shared memory (the
      // operand ring is idle once tfull has fired)
      if (nks > 0) {
        mbar_wait(&tfull, 0);
        tc_fence_after();
      }
      float* red = reinterpret_cast<float*>(stg);
      asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
      for (int k = 0; k < 8; ++k) red[et * 8 + k] = bs[k];
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (et < CO) {
        const int jj = et / 8, kk = et % 8;
        float t = 0.f;
        for (int r = 0; r < RSTEP; ++r) t += red[(r * NCH + jj) * 8 + kk];
        part[NW + et] = t;   // row 0, bias columns
      }
    } else if (nks > 0) {
      mbar_wait(&tfull, 0);
      tc_fence_after();
    }
#pragma unroll
    for (int mi = 0; mi < NMMA; ++mi)
      for (int c0 = 0; c0 < NW; c0 += 16) {
        float v[16];
        if (nks > 0) {
          tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + mi * ACOL + c0, v);
        } else {
#pragma unroll
          for (int c = 0; c < 16; ++c) v[c] = 0.f;
        }
        float4* dst = reinterpret_cast<float4*>(part + (size_t)(mi * MM + row) * PC + c0);
        if (row_ok) {
#pragma unroll
          for (int c = 0; c < 4; ++c) dst[c] = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
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

// fixed-order sum; output o < 128*3CO: (row i, col n) -> Fin::weight3(i, n, v);
// o >= 128*3CO: bias column -> Fin::bias
template <int CO, class Fin, int NB = 3, int PROWS = 128>
__global__ void __launch_bounds__(256) win3_wgrad_finish(const float* __restrict__ part, int G,
                                                         int tot, const Fin f, int trig) {
  pdl_wait();
  if (trig) pdl_trigger();
  constexpr int NW = NB * CO, PC = (NB + 1) * CO;
  const int o = blockIdx.x * 32 + (threadIdx.x & 31), g = threadIdx.x >> 5;
  __shared__ float sh[8][33];
  float s = 0.f;
  size_t idx = 0;
  if (o < tot) {
    idx = o < PROWS * NW ? (size_t)(o / NW) * PC + (o % NW) : (size_t)NW + (o - PROWS * NW);
    // unrolled: the loads issue back to back, the adds stay in z order
#pragma unroll 8
    for (int z = g; z < G; z += 8) s += __ldcg(part + (size_t)z * PROWS * PC + idx);
  }
  sh[g][threadIdx.x & 31] = s;
  __syncthreads();
  if (g == 0 && o < tot) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += sh[k][threadIdx.x & 31];
    if (o >= PROWS * NW) f.bias(o - PROWS * NW, t);
    else f.weight3(o / NW, o % NW, t);
  }
}

inline size_t win3_wgrad_part_bytes(int64_t M, int CO, int NB = 3, int rbx = 128) {
  int64_t r;
  return (size_t)wgrad_grid(M, &r) * wgrad_prows(rbx, NB) * (NB + 1) * CO * 4;
}

// bias = false: no all-ones MMA (the bias gradient is a column of the weight
// accumulator, e.g. from a constant-1 input channel)
template <int CO, int RBX, class Fin, int NB = 3, int XF = XF_NONE>
seed_status launch_win3_wgrad(const Win3WgradArgs& a0, const Fin& fin, bool bias, cudaStream_t st) {
  Win3WgradArgs a = a0;
  const int G = wgrad_grid(a.M, &a.rows_per_cta);
  const int arows = WG_KS + 256 / RBX - 1 + (wgrad_prows(RBX, NB) == 256 ? 2 : 0);   // + the second MMA's rows
  const int a_bytes = (int)align_up((size_t)arows * RBX + 1024, 1024);
  const int b_bytes = (int)align_up((size_t)(WG_KS + (NB - 1) * a.bstride) * 2 * CO + 1024, 1024);
  const int stg_bytes = XF == XF_U8 ? (int)align_up((size_t)arows * 16 + 16, 1024) : 0;
  const int stages = std::min(WC_MAX_STAGES, (WC_SMEM_BUDGET - 1024) / (a_bytes + b_bytes + stg_bytes));
  if (stages < 2) return SEED_E_SHAPE;
  const size_t smem = 2048 + (size_t)stages * (a_bytes + b_bytes + stg_bytes);
  static PerDevice attr0;
  SEED_TRY(smem_optin(attr0, win3_wgrad_kernel<CO, RBX, true, NB, XF>, WC_SMEM_BUDGET + 2048));
  static PerDevice attr1;
  SEED_TRY(smem_optin(attr1, win3_wgrad_kernel<CO, RBX, false, NB, XF>, WC_SMEM_BUDGET + 2048));
  const int threads = WC_THREADS + (XF != XF_NONE ? 32 * XF_CW : 0);
  SEED_TRY(launch_k(bias ? win3_wgrad_kernel<CO, RBX, true, NB, XF> : win3_wgrad_kernel<CO, RBX, false, NB, XF>,
                    dim3(G), dim3(threads), smem, st, a, stages, a_bytes, b_bytes, stg_bytes));
  constexpr int PROWS = wgrad_prows(RBX, NB);
  const int tot = PROWS * NB * CO + (bias ? CO : 0);
  return launch_k(win3_wgrad_finish<CO, Fin, NB, PROWS>, dim3(ceil_div(tot, 32)), dim3(256), 0, st,
                  (const float*)a.part, G, tot, fin, a.trig);
}

}  // namespace seed
