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
// MMAs overlap this band's epilogue), warps 2-9 drain the accumulator (x scale +
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
};

__device__ __forceinline__ Band band_of(const CpArgs& a, int64_t bi) {
  Band b;
  if (a.G > 0) {
    b.f0 = bi * a.G;
    b.nf = (int)min((int64_t)a.G, a.F - b.f0);
    b.oy0 = 0; b.oy1 = a.go.H;
    b.base = 0;
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
    b.R = (Yb - Ya + 1) * a.gi.Wp;
  }
  b.row0 = b.f0 * a.gi.P + b.base;
  return b;
}

template <int N, int RB, int NW>
__global__ void __launch_bounds__(CP_THREADS, 1)
    conv_pool_kernel(const CpArgs a, int stages, int slab_bytes, int band_bytes) {
  constexpr int RBO = 2 * N, NC = N / 8;
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
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], CP_EW); }
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
    const int part = (warp - 2) >> 2;            // 128-row blocks mt with mt % (CP_EW / 4) == part
    const int et = threadIdx.x - 64;
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
      for (int mt = part; mt < nblk; mt += CP_EW / 4) {
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
          uint8_t* row = bandbuf + (size_t)r * RBO;
#pragma unroll
          for (int j = 0; j < NC; ++j) {
            const uint4 u = pack8(v + 8 * j);
            *reinterpret_cast<uint4*>(row + (swz_chunk(r, RBO, j) << 4)) = border ? ninf : u;
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
      asm volatile("bar.sync 1, %0;" ::"n"(CP_EPI) : "memory");   // band buffer complete
      // pool: output padded rows Y of each frame (with the top / bottom border row
      // in the first / last band of a frame), all columns X, chunks j
      const int Ylo = b.oy0 == 0 ? 0 : b.oy0 + 1;
      const int Yhi = b.oy1 == a.go.H ? a.go.H + 1 : b.oy1;
      const int total = b.nf * (Yhi - Ylo + 1) * (int)a.fRow.d;
      for (int i = et; i < total; i += CP_EPI) {
        uint32_t fl = 0, rem = (uint32_t)i, Yr, c2;
        if (a.G > 0) a.fFrame.divmod((uint32_t)i, fl, rem);
        a.fRow.divmod(rem, Yr, c2);
        const int X = (int)(c2 / NC), j = (int)(c2 % NC);
        const int Y = Ylo + (int)Yr;
        const int64_t g = (b.f0 + fl) * a.go.P + (int64_t)Y * a.go.Wp + X;
        uint4* ph = reinterpret_cast<uint4*>(a.h0 + g * RBO + (swz_chunk(g, RBO, j) << 4));
        uint4* pr = reinterpret_cast<uint4*>(a.hr0 + g * RBO + (swz_chunk(g, RBO, j) << 4));
        if (Y == 0 || Y == a.go.H + 1 || X == 0 || X == a.go.W + 1) {
          *ph = make_uint4(0, 0, 0, 0);
          *pr = make_uint4(0, 0, 0, 0);
          continue;
        }
        // tap (ky, kx) of output (Y-1, X-1): conv pixel (2(Y-1) - pt + ky, 2(X-1) - pl + kx),
        // band row fl*P + (y+1)*Wp + (x+1) - base
        const int r0 = (int)fl * a.gi.P + (2 * Y - 1 - a.pt) * a.gi.Wp + 2 * X - 1 - a.pl - b.base;
        uint4 in[9];
#pragma unroll
        for (int t = 0; t < 9; ++t) {
          const int r = r0 + (t / 3) * a.gi.Wp + t % 3;
          in[t] = *reinterpret_cast<const uint4*>(bandbuf + (size_t)r * RBO + (swz_chunk(r, RBO, j) << 4));
        }
        uint4 best, rl;
        uint2 am;
        pool_max9(in, best, rl, am);
        *ph = best;
        *pr = rl;
        *reinterpret_cast<uint2*>(a.arg + g * N + 8 * j) = am;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(CP_EPI) : "memory");   // band buffer free
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 2 * AC);
  }
}

template <int N, int RB, int NW>
seed_status launch_conv_pool(CpArgs a, cudaStream_t st) {
  constexpr int WB = NW * N * RB;
  const int cap = (256 / N) * 128;   // rows per accumulator
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
  a.fP = FastDiv((uint32_t)gi.P); a.fWp = FastDiv((uint32_t)gi.Wp);
  a.fRow = FastDiv((uint32_t)(a.go.Wp * (N / 8)));
  a.fFrame = FastDiv((uint32_t)((a.go.H + 2) * a.go.Wp * (N / 8)));
  int mn = a.off[0], mx = a.off[0];
  for (int w = 1; w < NW; ++w) { mn = std::min(mn, a.off[w]); mx = std::max(mx, a.off[w]); }
  const int nblk_max = (Rmax + 127) / 128;
  const int slab = (int)align_up((size_t)(nblk_max * 128 + mx - mn) * RB + 1024, 1024);
  const int band = (int)align_up((size_t)Rmax * 2 * N, 1024);
  const int wbytes = (int)align_up(WB, 1024);
  const int stages = std::min(WC_MAX_STAGES, (CP_SMEM - 1024 - wbytes - band) / slab);
  if (stages < 2) return SEED_E_UNSUPPORTED;
  if (a.nbands == 0) return SEED_OK;
  const size_t smem = (size_t)wbytes + (size_t)stages * slab + band + 1024;
  static PerDevice attr;
  SEED_TRY(smem_optin(attr, conv_pool_kernel<N, RB, NW>, CP_SMEM));
  const int grid = (int)std::min<int64_t>(a.nbands, sm_count());
  return launch_k(conv_pool_kernel<N, RB, NW>, dim3(grid), dim3(CP_THREADS), smem, st, a, stages, slab,
                  band);
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
  if (f.ch == 16 && f.cin_p == 16) return launch_conv_pool<16, 32, 9>(a, st);
  if (f.ch == 32 && f.cin_p == 16) return launch_conv_pool<32, 32, 9>(a, st);
  if (f.ch == 32 && f.cin_p == 32) return launch_conv_pool<32, 64, 9>(a, st);
  return SEED_E_UNSUPPORTED;
}

}  // namespace seed
