// conv3w_pool.cu — the IMPALA-deep section conv fused with its max-pool
// (conv3w.cuh conv3w_conv_pool, PAPER.md C14: conv 3x3 ->
// maxpool 3x3 / stride 2 'same').
//
// The unfused pair writes the full-resolution conv output (section 0 of the GRF
// net: 4224 frames x 74 x 98 rows x 32 B = 0.98 GB) and the pool kernel reads it
// back — ~0.3 ms of the 6.1 ms c4 step (profiles/r02/phases_c4_m64.json:
// deep_pool_fwd#1 308 us).  Here one persistent warp-specialized kernel takes
// BANDS of the conv output:
//   row bands: pool output rows [oy0, oy1) of one frame need conv image rows
//              [2*oy0 - pt, 2*(oy1-1) - pt + 2] (clipped), a contiguous range of
//              padded rows, so the band is one shifted-window GEMM of those rows
//              (adjacent bands recompute their one shared conv row: 1/(2k));
//   frame bands: G whole frames when a padded frame fits (small sections).
// Warp 0 TMA-loads the band's input slab (win_engine.cuh load_slab), warp 1
// issues the window MMAs into one of two TMEM accumulators (so the next band's
// MMAs overlap this band's epilogue), warps 2-13 drain the accumulator (x scale +
// bias, bf16: the conv epilogue of W3FwdEpi<W3_PLAIN>) into a shared-memory band
// buffer, then pool from it (pool_max9: the same first-maximum / -inf rules as
// conv3w_pool_fwd_kernel) and write h0, hr0 = relu(h0), the argmax bytes and the
// zero borders of h0 / hr0.
// The band covers whole padded rows including the frame's border rows that the
// windows reach (TF 'same' pooling pads at most one row / column per side), and
// the drain stores -inf at border positions, so the pool reads its 9 taps with
// no bounds checks (measured: the checked, division-indexed pool loop made the
// epilogue, not the MMAs, the band's critical path).
#include "conv3w.cuh"

namespace seed {

namespace {

constexpr int CP_EW = 12;                      // epilogue / pool warps (3 per TMEM lane quarter)
constexpr int CP_EPI = 32 * CP_EW;
constexpr int CP_THREADS = 64 + CP_EPI;        // warp 0 producer, warp 1 MMA, warps 2.. epilogue
constexpr int CP_SMEM = 226 * 1024;   // dynamic shared memory cap (227 KB less the static barriers)

struct CpArgs {
  const uint8_t* src;       // input rows (RB bytes)
  int64_t src_rows;
  int off[WIN_MAX];
  const uint8_t* wimg;
  PadGeo gi, go;
  int pt, pl;
  int64_t F;
  int G;                    // frames per band (frame bands), 0 = row bands
  int k, nbpf;              // row bands: pool rows per band, bands per frame
  int64_t nbands;
  FastDiv fP, fWp, fRow, fFrame;   // gi.P, gi.Wp, pool items per output row / per frame
  int bb_rs, bb_h1;         // band buffer: bytes per image row, offset of the odd-column half
  float in_scale;
  const float* bias;
  uint8_t* h0;
  uint8_t* hr0;
  uint8_t* arg;
  uint8_t* conv_dbg;
};

struct Band {
  int64_t f0, row0;   // first frame, first conv row (absolute padded row)
  int nf, oy0, oy1;   // frames, pool rows [oy0, oy1) of each frame
  int R;              // conv rows of the band (from row0)
  int base;           // row0 - f0 * gi.P
  int ybase;          // first padded image row of the band (row bands), 0 (frame bands)
};

__device__ __forceinline__ Band band_of(const CpArgs& a, int64_t bi) {
  Band b;
  if (a.G > 0) {
    b.f0 = bi * a.G;
    b.nf = (int)min((int64_t)a.G, a.F - b.f0);
    b.oy0 = 0; b.oy1 = a.go.H;
    b.base = 0;
    b.ybase = 0;
    b.R = b.nf * a.gi.P;
  } else {
    b.f0 = bi / a.nbpf;
    const int j = (int)(bi - b.f0 * a.nbpf);
    b.nf = 1;
    b.oy0 = j * a.k;
    b.oy1 = min(b.oy0 + a.k, a.go.H);
    // padded rows Y of the taps (pt, pb <= 1: within [0, H + 1])
    const int Ya = 2 * b.oy0 - a.pt + 1, Yb = 2 * (b.oy1 - 1) - a.pt + 3;
    b.base = Ya * a.gi.Wp;
    b.ybase = Ya;
    b.R = (Yb - Ya + 1) * a.gi.Wp;
  }
  b.row0 = b.f0 * a.gi.P + b.base;
  return b;
}

// Band buffer layout: per padded image row of the band, the even columns then the
// odd ones (pixel X at (X & 1) * bb_h1 + (X >> 1) * 2N), rows bb_rs bytes apart.
// The pool's taps of consecutive output columns are consecutive pixels of one half
// (stride 2 in X), so a warp's 16-byte tap loads cover a contiguous range (no bank
// conflicts; with whole rows of 32 / 64 bytes the stride-2 taps hit 4 of the 8
// 16-byte bank groups); bb_h1 = 16 mod 32 puts the drain's even / odd-column stores
// of one chunk on disjoint bank groups.
template <int N>
__device__ __forceinline__ uint32_t bb_off(const CpArgs& a, const Band& b, uint32_t fl, int Y, int X) {
  return (uint32_t)(((int)fl * (a.gi.H + 2) + Y - b.ybase) * a.bb_rs + (X & 1) * a.bb_h1 + (X >> 1) * (2 * N));
}

// The max-pool of one band from the shared-memory band buffer (epilogue thread et
// of CP_EPI): output padded rows Y of each frame (with the top / bottom border row
// in the first / last band of a frame), all columns X, 8-channel chunks j.
template <int N, int EPI = CP_EPI>
__device__ __forceinline__ void pool_band(const CpArgs& a, const Band& b, const uint8_t* bandbuf, int et) {
  constexpr int RBO = 2 * N, NC = N / 8;
  const int Ylo = b.oy0 == 0 ? 0 : b.oy0 + 1;
  const int Yhi = b.oy1 == a.go.H ? a.go.H + 1 : b.oy1;
  const int total = b.nf * (Yhi - Ylo + 1) * (int)a.fRow.d;
  for (int i = et; i < total; i += EPI) {
    uint32_t fl = 0, rem = (uint32_t)i, Yr, c2;
    if (a.G > 0) a.fFrame.divmod((uint32_t)i, fl, rem);
    a.fRow.divmod(rem, Yr, c2);
    const int X = (int)(c2 / NC), j = (int)(c2 % NC);
    const int Y = Ylo + (int)Yr;
    // output row (32-bit: F * go.P < 2^32, checked by the launcher)
    const uint32_t g = ((uint32_t)b.f0 + fl) * (uint32_t)a.go.P + (uint32_t)(Y * a.go.Wp + X);
    const size_t off = (size_t)g * RBO + ((size_t)swz_chunk(g, RBO, j) << 4);
    uint4* ph = reinterpret_cast<uint4*>(a.h0 + off);
    uint4* pr = reinterpret_cast<uint4*>(a.hr0 + off);
    if (Y == 0 || Y == a.go.H + 1 || X == 0 || X == a.go.W + 1) {
      *ph = make_uint4(0, 0, 0, 0);
      *pr = make_uint4(0, 0, 0, 0);
      continue;
    }
    // tap (ky, kx) of output (Y-1, X-1): conv pixel (2(Y-1) - pt + ky, 2(X-1) - pl + kx),
    // padded (2Y - 1 - pt + ky, 2X - 1 - pl + kx)
    const int Xc = 2 * X - 1 - a.pl;
    const uint8_t* t0 = bandbuf + bb_off<N>(a, b, fl, 2 * Y - 1 - a.pt, Xc) + 16 * j;
    const uint8_t* t1 = bandbuf + bb_off<N>(a, b, fl, 2 * Y - 1 - a.pt, Xc + 1) + 16 * j;
    uint4 in[9];
#pragma unroll
    for (int ky = 0; ky < 3; ++ky) {
      in[3 * ky] = *reinterpret_cast<const uint4*>(t0 + ky * a.bb_rs);
      in[3 * ky + 1] = *reinterpret_cast<const uint4*>(t1 + ky * a.bb_rs);
      in[3 * ky + 2] = *reinterpret_cast<const uint4*>(t0 + ky * a.bb_rs + 2 * N);
    }
    uint4 best, rl;
    uint2 am;
    pool_max9(in, best, rl, am);
    *ph = best;
    *pr = rl;
    *reinterpret_cast<uint2*>(a.arg + (size_t)g * N + 8 * j) = am;
  }
}

template <int N, int RB, int NW, int EW = CP_EW>
__global__ void __launch_bounds__(64 + 32 * EW, 1)
    conv_pool_kernel(const CpArgs a, int stages, int slab_bytes, int band_bytes) {
  constexpr int RBO = 2 * N, NC = N / 8;
  constexpr int EPI = 32 * EW;
  constexpr uint32_t LAYOUT = swz_layout_code(RB);
  constexpr int WB = NW * N * RB;
  constexpr int AC = 256;   // TMEM columns per accumulator (2 accumulators)
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = smem_align1024(smraw);
  uint8_t* Ws = sm;
  uint8_t* slabs = sm + ((WB + 1023) & ~1023);
  uint8_t* bandbuf = slabs + (size_t)stages * slab_bytes;
  __shared__ uint64_t full[WC_MAX_STAGES], empty[WC_MAX_STAGES], tfull[2], tempty[2], wbar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int mn = a.off[0], mx = a.off[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) { mn = min(mn, a.off[w]); mx = max(mx, a.off[w]); }
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], EW); }
    mbar_init(&wbar, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&tbase, 2 * AC);
  __syncthreads();
  tc_fence_after();
  if (warp == 0 && lane == 0) {   // weights: before the PDL wait (see win_conv_kernel)
    mbar_expect_tx(&wbar, WB);
    bulk_g2s(smem_u32(Ws), a.wimg, WB, &wbar);
  }
  pdl_wait();
  const uint32_t tmem = tbase;
  if (warp == 0) {
    int it = 0;
    for (int64_t bi = blockIdx.x; bi < a.nbands; bi += gridDim.x, ++it) {
      const int s = it % stages;
      const Band b = band_of(a, bi);
      const int nblk = (b.R + 127) >> 7;
      mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
      load_slab(slabs + (size_t)s * slab_bytes, a.src, RB, b.row0 + mn, nblk * 128 + mx - mn, a.src_rows,
                &full[s], lane, 0);
    }
  } else if (warp == 1) {
    mbar_wait(&wbar, 0);
    const uint32_t idesc = umma_idesc_bf16(128, N, false, false);
    const uint64_t bd0 = umma_desc(smem_u32(Ws), 16, 8 * RB, LAYOUT);
    int aoff[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) aoff[w] = ((a.off[w] - mn) * RB) >> 4;
    int it = 0;
    for (int64_t bi = blockIdx.x; bi < a.nbands; bi += gridDim.x, ++it) {
      const int s = it % stages, acc = it & 1;
      const Band b = band_of(a, bi);
      const int nblk = (b.R + 127) >> 7;
      mbar_wait(&full[s], (it / stages) & 1);
      mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t base = smem_u32(slabs + (size_t)s * slab_bytes) + slab_phase(b.row0 + mn, RB);
      const uint64_t ad0 = umma_desc(base, 16, 8 * RB, LAYOUT);
      for (int mt = 0; mt < nblk; ++mt)
#pragma unroll
        for (int w = 0; w < NW; ++w)
#pragma unroll
          for (int ks = 0; ks < RB / 32; ++ks)
            tc_mma_bf16_w(tmem + acc * AC + mt * N, ad0 + (uint64_t)(aoff[w] + ((mt * 128 * RB) >> 4) + ks * 2),
                          bd0 + (uint64_t)((w * N * RB + ks * 32) >> 4), idesc, (w | ks) != 0);
      tc_commit_w(&empty[s]);
      tc_commit_w(&tfull[acc]);
    }
  } else {
    const int q = warp & 3;                      // TMEM lanes [32q, 32q + 32)
    const int part = (warp - 2) >> 2;            // 128-row blocks mt with mt % (EW / 4) == part
    float bias[N];
#pragma unroll
    for (int c = 0; c < N; ++c) bias[c] = __ldg(a.bias + c);
    const uint4 ninf = make_uint4(BF16X2_NEG_INF, BF16X2_NEG_INF, BF16X2_NEG_INF, BF16X2_NEG_INF);
    int it = 0;
    for (int64_t bi = blockIdx.x; bi < a.nbands; bi += gridDim.x, ++it) {
      const int acc = it & 1;
      const Band b = band_of(a, bi);
      const int nblk = (b.R + 127) >> 7;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      for (int mt = part; mt < nblk; mt += EW / 4) {
        uint32_t vr[N];
#pragma unroll
        for (int c = 0; c < N / 16; ++c)
          tmem_ld16_nw(tmem + ((uint32_t)(q * 32) << 16) + acc * AC + mt * N + c * 16,
                       *reinterpret_cast<uint32_t(*)[16]>(&vr[16 * c]));
        tmem_wait_ld();
        const int r = mt * 128 + q * 32 + lane;
        if (r < b.R) {
          uint32_t fl, rem, Y, X;
          a.fP.divmod((uint32_t)(r + b.base), fl, rem);
          a.fWp.divmod(rem, Y, X);
          const bool border = Y == 0 || (int)Y == a.gi.H + 1 || X == 0 || (int)X == a.gi.W + 1;
          float v[N];
#pragma unroll
          for (int c = 0; c < N; ++c) v[c] = __uint_as_float(vr[c]) * a.in_scale + bias[c];
          uint8_t* row = bandbuf + bb_off<N>(a, b, fl, (int)Y, (int)X);
#pragma unroll
          for (int j = 0; j < NC; ++j) {
            const uint4 u = pack8(v + 8 * j);
            *reinterpret_cast<uint4*>(row + 16 * j) = border ? ninf : u;
            if (a.conv_dbg) {
              const int64_t g = b.row0 + r;
              *reinterpret_cast<uint4*>(a.conv_dbg + g * RBO + (swz_chunk(g, RBO, j) << 4)) = u;
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      asm volatile("bar.sync 1, %0;" ::"n"(EPI) : "memory");   // band buffer complete
      pool_band<N, EPI>(a, b, bandbuf, threadIdx.x - 64);
      asm volatile("bar.sync 1, %0;" ::"n"(EPI) : "memory");   // band buffer free
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 2 * AC);
  }
}

// Column-tap-stacked variant (win_engine.cuh win_conv_kx_kernel's MMA form): per
// 128-row block 3 MMAs (one per kernel row ky, window offset (ky-1)*Wp) of
// N = 3*NO — the three column taps' weights side by side on N (the 9-window weight
// image read as 3 windows of 3*NO rows) — instead of 9 MMAs of N = NO; the small
// tcgen05.mma costs ~45 cycles up to N = 48 (profiles/r01/mma_rate_probe.txt), so
// the tensor side is ~3x cheaper.  The conv output of band row r is
//   D_0[r-1] + D_1[r] + D_2[r+1]
// (D_kx: the kx part of the accumulator; the neighbouring rows are the adjacent
// TMEM lanes).  A band's 128-row blocks stream through a ring of NSLOT TMEM slots
// of 3*NO columns (per-slot full / empty barriers), so bands are as large as in the
// 9-window kernel although one block's accumulator is 3x wider.  Each block is
// drained by one epilogue warp per TMEM lane quarter (blocks round robin over the
// CP_EW / 4 warps of a quarter): three 8-column TMEM loads per 8-channel chunk, the
// r-1 / r+1 parts by warp shuffles, interior rows (lanes 1..30) stored to the band
// buffer at once; the quarter-edge rows (lanes 0 / 31) leave their partial sum and
// the part their neighbour needs in a shared-memory exchange and are finished after
// one barrier.  The band's first / last rows are frame border columns (-inf), so no
// row needs a neighbour outside the band.
template <int NO, int RB>
__global__ void __launch_bounds__(CP_THREADS, 1)
    conv_pool_kx_kernel(const CpArgs a, int stages, int slab_bytes, int band_bytes) {
  constexpr int NN = 3 * NO, RBO = 2 * NO, NC = NO / 8;
  constexpr uint32_t LAYOUT = swz_layout_code(RB);
  constexpr int WB = 3 * NN * RB;
  constexpr int NSLOT = 512 / NN;           // TMEM slots of one 128-row block each
  constexpr int XG = 4 * NO;                // exchange floats per 32-row group
  constexpr int EP = CP_EW / 4;             // epilogue warps per lane quarter
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = smem_align1024(smraw);
  uint8_t* Ws = sm;
  uint8_t* slabs = sm + ((WB + 1023) & ~1023);
  uint8_t* bandbuf = slabs + (size_t)stages * slab_bytes;
  // exchange per 32-row group g: [0, NO) D_0 of lane 31 | [NO, 2NO) D_2 of lane 0 |
  // [2NO, 3NO) partial of lane 0 | [3NO, 4NO) partial of lane 31
  float* xch = reinterpret_cast<float*>(bandbuf + band_bytes);
  __shared__ uint64_t full[WC_MAX_STAGES], empty[WC_MAX_STAGES], tfull[NSLOT], tempty[NSLOT], wbar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mn = min(a.off[0], min(a.off[1], a.off[2]));
  const int mx = max(a.off[0], max(a.off[1], a.off[2]));
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int i = 0; i < NSLOT; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 4); }
    mbar_init(&wbar, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&tbase, 512);
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
    for (int64_t bi = blockIdx.x; bi < a.nbands; bi += gridDim.x, ++it) {
      const int s = it % stages;
      const Band b = band_of(a, bi);
      const int nblk = (b.R + 127) >> 7;
      mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
      load_slab(slabs + (size_t)s * slab_bytes, a.src, RB, b.row0 + mn, nblk * 128 + mx - mn, a.src_rows,
                &full[s], lane, 0);
    }
  } else if (warp == 1) {
    mbar_wait(&wbar, 0);
    const uint32_t idesc = umma_idesc_bf16(128, NN, false, false);
    const uint64_t bd0 = umma_desc(smem_u32(Ws), 16, 8 * RB, LAYOUT);
    int aoff[3];
#pragma unroll
    for (int w = 0; w < 3; ++w) aoff[w] = ((a.off[w] - mn) * RB) >> 4;
    int it = 0;
    uint32_t cb = 0;   // blocks issued before this band
    for (int64_t bi = blockIdx.x; bi < a.nbands; bi += gridDim.x, ++it) {
      const int s = it % stages;
      const Band b = band_of(a, bi);
      const int nblk = (b.R + 127) >> 7;
      mbar_wait(&full[s], (it / stages) & 1);
      const uint32_t base = smem_u32(slabs + (size_t)s * slab_bytes) + slab_phase(b.row0 + mn, RB);
      const uint64_t ad0 = umma_desc(base, 16, 8 * RB, LAYOUT);
      for (int mt = 0; mt < nblk; ++mt) {
        const uint32_t idx = cb + mt, slot = idx % NSLOT;
        mbar_wait(&tempty[slot], ((idx / NSLOT) & 1) ^ 1);
        tc_fence_after();
#pragma unroll
        for (int w = 0; w < 3; ++w)
#pragma unroll
          for (int ks = 0; ks < RB / 32; ++ks)
            tc_mma_bf16_w(tmem + slot * NN, ad0 + (uint64_t)(aoff[w] + ((mt * 128 * RB) >> 4) + ks * 2),
                          bd0 + (uint64_t)((w * NN * RB + ks * 32) >> 4), idesc, (w | ks) != 0);
        tc_commit_w(&tfull[slot]);
      }
      tc_commit_w(&empty[s]);
      cb += nblk;
    }
  } else {
    const int q = warp & 3;                      // TMEM lanes [32q, 32q + 32)
    const int part = (warp - 2) >> 2;            // blocks mt with mt % EP == part
    const int et = threadIdx.x - 64;
    const float m_up = lane == 0 ? 0.f : 1.f, m_dn = lane == 31 ? 0.f : 1.f;
    const uint4 ninf = make_uint4(BF16X2_NEG_INF, BF16X2_NEG_INF, BF16X2_NEG_INF, BF16X2_NEG_INF);
    float bias[NO];
#pragma unroll
    for (int c = 0; c < NO; ++c) bias[c] = __ldg(a.bias + c);
    // band-buffer offset of band row r; border flag
    auto locate = [&](const Band& b, int r, bool& border) {
      uint32_t fl, rem, Y, X;
      a.fP.divmod((uint32_t)(r + b.base), fl, rem);
      a.fWp.divmod(rem, Y, X);
      border = Y == 0 || (int)Y == a.gi.H + 1 || X == 0 || (int)X == a.gi.W + 1;
      return bb_off<NO>(a, b, fl, (int)Y, (int)X);
    };
    // conv row r of the band, chunk j -> band buffer (bf16, -inf at frame borders), debug
    // copy; bias b8 = the chunk's 8 biases
    auto put = [&](const Band& b, int r, uint32_t off, int j, bool border, const float* v, const float* b8) {
      float o[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) o[k] = fmaf(v[k], a.in_scale, b8[k]);
      const uint4 u = pack8(o);
      *reinterpret_cast<uint4*>(bandbuf + off + 16 * j) = border ? ninf : u;
      if (a.conv_dbg) {
        const int64_t g = b.row0 + r;
        *reinterpret_cast<uint4*>(a.conv_dbg + g * RBO + (swz_chunk(g, RBO, j) << 4)) = u;
      }
    };
    uint32_t cb = 0;
    for (int64_t bi = blockIdx.x; bi < a.nbands; bi += gridDim.x) {
      const Band b = band_of(a, bi);
      const int nblk = (b.R + 127) >> 7;
      for (int mt = part; mt < nblk; mt += EP) {
        const uint32_t idx = cb + mt, slot = idx % NSLOT;
        const int grp = mt * 4 + q;
        const int r = grp * 32 + lane;
        bool border = true;
        const uint32_t off = r < b.R ? locate(b, r, border) : 0u;
        mbar_wait(&tfull[slot], (idx / NSLOT) & 1);
        tc_fence_after();
        const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16) + slot * NN;
        uint32_t p0[NO], p1[NO], p2[NO];
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          tmem_ld8_nw(tb + j * 8, *reinterpret_cast<uint32_t(*)[8]>(&p0[8 * j]));
          tmem_ld8_nw(tb + NO + j * 8, *reinterpret_cast<uint32_t(*)[8]>(&p1[8 * j]));
          tmem_ld8_nw(tb + 2 * NO + j * 8, *reinterpret_cast<uint32_t(*)[8]>(&p2[8 * j]));
        }
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[slot]);   // the slot's columns are in registers
        float v[NO];
#pragma unroll
        for (int k = 0; k < NO; ++k) {
          const float up = __shfl_up_sync(0xffffffffu, __uint_as_float(p0[k]), 1);     // D_0[r-1]
          const float dn = __shfl_down_sync(0xffffffffu, __uint_as_float(p2[k]), 1);   // D_2[r+1]
          v[k] = fmaf(dn, m_dn, fmaf(up, m_up, __uint_as_float(p1[k])));
        }
        if (lane == 0 || lane == 31) {
          float4* xg = reinterpret_cast<float4*>(xch + grp * XG);
          const uint32_t* pp = lane == 0 ? p2 : p0;
          const int dp = (lane == 0 ? 2 : 3) * NO / 4, dn = (lane == 0 ? 1 : 0) * NO / 4;
#pragma unroll
          for (int k = 0; k < NO / 4; ++k) {
            xg[dp + k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
            xg[dn + k] = make_float4(__uint_as_float(pp[4 * k]), __uint_as_float(pp[4 * k + 1]),
                                     __uint_as_float(pp[4 * k + 2]), __uint_as_float(pp[4 * k + 3]));
          }
        } else if (r < b.R) {
#pragma unroll
          for (int j = 0; j < NC; ++j) put(b, r, off, j, border, v + 8 * j, bias + 8 * j);
        }
      }
      cb += nblk;
      asm volatile("bar.sync 1, %0;" ::"n"(CP_EPI) : "memory");   // interior rows + exchange written
      // quarter-edge rows: lane-0 row of group g adds D_0 of group g-1's lane 31,
      // lane-31 row adds D_2 of group g+1's lane 0
      const int ng = nblk * 4;
      for (int i = et; i < ng * 2 * NC; i += CP_EPI) {
        const int g = i / (2 * NC), side = (i / NC) & 1, j = i % NC;
        const int r = g * 32 + (side ? 31 : 0);
        if (r >= b.R) continue;
        const float* pv = xch + g * XG + (2 + side) * NO + j * 8;
        const float* nb = side ? (g + 1 < ng ? xch + (g + 1) * XG + NO + j * 8 : nullptr)
                               : (g > 0 ? xch + (g - 1) * XG + j * 8 : nullptr);
        float v[8], b8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          v[k] = nb ? pv[k] + nb[k] : pv[k];
          b8[k] = __ldg(a.bias + j * 8 + k);
        }
        bool border;
        const uint32_t off = locate(b, r, border);
        put(b, r, off, j, border, v, b8);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(CP_EPI) : "memory");   // band buffer complete
      pool_band<NO>(a, b, bandbuf, et);
      asm volatile("bar.sync 1, %0;" ::"n"(CP_EPI) : "memory");   // band buffer / exchange free
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// KX: the column-tap-stacked kernel (NW = 9 only): 3 windows, N = 3*out per block
template <int N, int RB, int NW, bool KX = false, int EW = CP_EW>
seed_status launch_conv_pool(CpArgs a, cudaStream_t st) {
  static_assert(!KX || NW == 9, "KX");
  constexpr int WB = NW * N * RB;
  const int cap = (256 / N) * 128;   // rows per band (9-window: per TMEM accumulator)
  const PadGeo& gi = a.gi;
  int Rmax;
  if (gi.P <= cap) {
    a.G = cap / gi.P;
    a.k = 0; a.nbpf = 1;
    a.nbands = (a.F + a.G - 1) / a.G;
    Rmax = (int)std::min<int64_t>(a.G, a.F) * gi.P;
  } else {
    a.G = 0;
    a.k = (cap / gi.Wp - 1) / 2;
    if (a.k < 1) return SEED_E_UNSUPPORTED;
    a.nbpf = (a.go.H + a.k - 1) / a.k;
    a.nbands = a.F * a.nbpf;
    Rmax = std::min(2 * a.k + 1, gi.H + 2) * gi.Wp;
  }
  // taps within the padded frame: TF 'same' 3x3 / 2 pads at most one row / column per side
  if (a.pt < 0 || a.pt > 1 || a.pl < 0 || a.pl > 1 || 2 * (a.go.H - 1) - a.pt + 2 > gi.H ||
      2 * (a.go.W - 1) - a.pl + 2 > gi.W)
    return SEED_E_UNSUPPORTED;
  if (a.F * a.go.P >= (1ll << 32)) return SEED_E_SHAPE;   // 32-bit output rows (pool_band)
  a.fP = FastDiv((uint32_t)gi.P); a.fWp = FastDiv((uint32_t)gi.Wp);
  a.fRow = FastDiv((uint32_t)(a.go.Wp * (N / 8)));
  a.fFrame = FastDiv((uint32_t)((a.go.H + 2) * a.go.Wp * (N / 8)));
  if (KX)
    for (int k = 0; k < 3; ++k) a.off[k] = (k - 1) * gi.Wp;
  const int nw = KX ? 3 : NW;
  int mn = a.off[0], mx = a.off[0];
  for (int w = 1; w < nw; ++w) { mn = std::min(mn, a.off[w]); mx = std::max(mx, a.off[w]); }
  const int nblk_max = (Rmax + 127) / 128;
  const int slab = (int)align_up((size_t)(nblk_max * 128 + mx - mn) * RB + 1024, 1024);
  const int hw = (gi.Wp + 1) / 2;
  a.bb_h1 = hw * 2 * N + 16;
  a.bb_rs = 2 * hw * 2 * N + 32;
  const int band = (int)align_up((size_t)(Rmax / gi.Wp) * a.bb_rs, 1024);
  const int xbytes = KX ? nblk_max * 4 * 4 * N * 4 : 0;   // edge-row exchange
  const int wbytes = (int)align_up(WB, 1024);
  const int stages = std::min(WC_MAX_STAGES, (CP_SMEM - 1024 - wbytes - band - xbytes) / slab);
  if (stages < 2) return SEED_E_UNSUPPORTED;
  if (a.nbands == 0) return SEED_OK;
  const size_t smem = (size_t)wbytes + (size_t)stages * slab + band + xbytes + 1024;
  const int grid = (int)std::min<int64_t>(a.nbands, sm_count());
  static PerDevice attr;
  if constexpr (KX) {
    SEED_TRY(smem_optin(attr, conv_pool_kx_kernel<N, RB>, CP_SMEM));
    return launch_k(conv_pool_kx_kernel<N, RB>, dim3(grid), dim3(CP_THREADS), smem, st, a, stages, slab,
                    band);
  } else {
    SEED_TRY(smem_optin(attr, conv_pool_kernel<N, RB, NW, EW>, CP_SMEM));
    return launch_k(conv_pool_kernel<N, RB, NW, EW>, dim3(grid), dim3(64 + 32 * EW), smem, st, a, stages,
                    slab, band);
  }
}

// Which 9-window section convs take the column-tap-stacked kernel (A/B
// measurement; profiles/r02/conv_pool_kx.md): SEED_CP_KX=0 none (default), 1 the
// 16 -> 16-channel section-0 conv of the GRF net, 2 every 9-window shape.  Measured
// at c4 s0: 775 us vs 593 us for the 9-window kernel — the tensor side is 3x
// cheaper but the combine (three TMEM loads and two shuffles per output value)
// doubles the epilogue's instructions, and the epilogue, not the MMAs, bounds
// the kernel.  SEED_CP_EW selects 16 / 20 epilogue warps for the 9-window s0
// kernel (measured slower: 617 / 625 us).
static int cp_kx() {
  static const int v = [] {
    const char* e = getenv("SEED_CP_KX");
    return e ? atoi(e) : 0;
  }();
  return v;
}

}  // namespace

seed_status conv3w_conv_pool(const Conv3wFwd& f, const PadGeo& go, int pt, int pl, uint8_t* h0,
                             uint8_t* hr0, uint8_t* arg, uint8_t* conv_dbg, cudaStream_t st) {
  if (f.mode != W3_PLAIN || f.xf != XF_NONE || !h0 || !hr0 || !arg) return SEED_E_UNSUPPORTED;
  if (f.g.P <= 0 || f.rows % f.g.P) return SEED_E_SHAPE;
  CpArgs a{};
  a.src = f.in; a.src_rows = f.rows; a.wimg = reinterpret_cast<const uint8_t*>(f.wimg);
  a.gi = f.g; a.go = go; a.pt = pt; a.pl = pl; a.F = f.rows / f.g.P;
  a.in_scale = f.in_scale; a.bias = f.bias; a.h0 = h0; a.hr0 = hr0; a.arg = arg; a.conv_dbg = conv_dbg;
  const int NW = f.xim ? 3 : 9;
  for (int k = 0; k < NW; ++k)
    a.off[k] = NW == 9 ? ((k / 3) - 1) * f.g.Wp + (k % 3) - 1 : (k - 1) * f.g.Wp;
  if (f.xim) {
    if (f.ch == 16 && f.cin_p == 16) return launch_conv_pool<16, 32, 3>(a, st);
    if (f.ch == 32 && f.cin_p == 16) return launch_conv_pool<32, 32, 3>(a, st);
    return SEED_E_UNSUPPORTED;
  }
  const int kx = cp_kx();
  static const int ew = [] {
    const char* e = getenv("SEED_CP_EW");
    return e ? atoi(e) : 12;
  }();
  if (f.ch == 16 && f.cin_p == 16) {
    if (kx >= 1) return launch_conv_pool<16, 32, 9, true>(a, st);
    if (ew == 16) return launch_conv_pool<16, 32, 9, false, 16>(a, st);
    if (ew == 20) return launch_conv_pool<16, 32, 9, false, 20>(a, st);
    return launch_conv_pool<16, 32, 9>(a, st);
  }
  if (f.ch == 32 && f.cin_p == 16)
    return kx >= 2 ? launch_conv_pool<32, 32, 9, true>(a, st) : launch_conv_pool<32, 32, 9>(a, st);
  if (f.ch == 32 && f.cin_p == 32)
    return kx >= 2 ? launch_conv_pool<32, 64, 9, true>(a, st) : launch_conv_pool<32, 64, 9>(a, st);
  return SEED_E_UNSUPPORTED;
}

}  // namespace seed
