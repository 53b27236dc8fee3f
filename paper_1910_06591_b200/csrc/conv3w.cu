// conv3w.cu — see conv3w.cuh.  IMPALA-deep torso (C14; SURVEY.md §8(a) H1
// forward / H9 backward) as shifted-window tcgen05 GEMMs over the padded row
// space, plus the max-pool and obs-conversion kernels.
#include "conv3w.cuh"

namespace seed {

__device__ __forceinline__ uint4* chunk_at(uint8_t* base, int64_t m, int RB, int j) {
  return reinterpret_cast<uint4*>(base + m * RB + (swz_chunk(m, RB, j) << 4));
}
__device__ __forceinline__ const uint4* chunk_at(const uint8_t* base, int64_t m, int RB, int j) {
  return reinterpret_cast<const uint4*>(base + m * RB + (swz_chunk(m, RB, j) << 4));
}

// Explicit PDL triggers in the 3x3 kernels (common.cuh pdl_wait_trig): SEED_DEEP_TRIG
// bit 0 = weight gradients + finishes, bit 1 = forward / data-gradient convs, bit 2 =
// max-pool backward.  Default 2 (profiles/r02/pdl_trigger.md, c4 over two rounds:
// none 5.649 / 5.652 ms, convs 5.637 / 5.636, weight gradients 5.668 / 5.699, pool
// backward 5.658 / 5.657, all 5.668 / 5.672).
static int deep_trig() {
  static const int v = [] {
    const char* e = getenv("SEED_DEEP_TRIG");
    return e ? atoi(e) : 2;
  }();
  return v;
}

// ------------------------------------------------------------------ epilogues
template <int MODE, int NN>
struct W3FwdEpi {
  static constexpr int N = NN;
  static constexpr int RB = 2 * NN;
  static constexpr int PRE = MODE == W3_RES ? N / 8 : 0;   // the residual row
  PadGeo g;
  float in_scale;
  const float* bias;
  const uint8_t* res;
  uint8_t* out;
  uint8_t* outr;
  bf16* dense;
  int dense_ct, dense_off;
  float* part_out;
  const float* part_in;
  __device__ void pre(int64_t m, uint4 (&p)[PRE > 0 ? PRE : 1]) const {
#pragma unroll
    for (int j = 0; j < PRE; ++j) p[j] = __ldg(chunk_at(res, m, RB, j));
  }
  __device__ void store(int64_t m, float (&v)[N]) const {   // PRE == 0 modes
    const uint4 p[1] = {make_uint4(0, 0, 0, 0)};
    store(m, v, p);
  }
  __device__ void store(int64_t m, float (&v)[N], const uint4 (&p)[PRE > 0 ? PRE : 1]) const {
    if constexpr (MODE == W3_PART) {   // the first input plane's fp32 sum (every row)
      float4* d = reinterpret_cast<float4*>(part_out + m * N);
#pragma unroll
      for (int q = 0; q < N / 4; ++q)
        d[q] = make_float4(v[4 * q] * in_scale, v[4 * q + 1] * in_scale, v[4 * q + 2] * in_scale,
                           v[4 * q + 3] * in_scale);
      return;
    }
    int f, y, x;
    if (!g.split(m, f, y, x)) {
      if (MODE != W3_PLAIN) {
        const uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int j = 0; j < N / 8; ++j) {
          *chunk_at(out, m, RB, j) = z;
          if (MODE == W3_RES && outr) *chunk_at(outr, m, RB, j) = z;
        }
      }
      return;
    }
    if (N == 64 && part_in) {   // the other input plane's fp32 sum (plane pairs: 64-ch only)
      const float4* ps = reinterpret_cast<const float4*>(part_in + m * N);
#pragma unroll
      for (int q = 0; q < N / 4; ++q) {
        const float4 t = __ldg(ps + q);
        v[4 * q] = fmaf(v[4 * q], in_scale, t.x); v[4 * q + 1] = fmaf(v[4 * q + 1], in_scale, t.y);
        v[4 * q + 2] = fmaf(v[4 * q + 2], in_scale, t.z); v[4 * q + 3] = fmaf(v[4 * q + 3], in_scale, t.w);
      }
    }
    const float isc = (N == 64 && part_in) ? 1.f : in_scale;
    if ((reinterpret_cast<uintptr_t>(bias) & 15) == 0) {   // 16-byte bias loads (the torso's
#pragma unroll                                              // parameter offsets are multiples of 4)
      for (int q = 0; q < N / 4; ++q) {
        const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias) + q);
        const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          v[4 * q + k] = v[4 * q + k] * isc + bb[k];
          if (MODE == W3_RELU) v[4 * q + k] = fmaxf(v[4 * q + k], 0.f);
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < N; ++q) {
        v[q] = v[q] * isc + __ldg(bias + q);
        if (MODE == W3_RELU) v[q] = fmaxf(v[q], 0.f);
      }
    }
    if constexpr (MODE == W3_RES && N <= 32) {   // (measured faster than the chunked form at N <= 32)
#pragma unroll
      for (int j = 0; j < N / 8; ++j) {
        float r[8];
        unpack8(p[j], r);
#pragma unroll
        for (int k = 0; k < 8; ++k) v[8 * j + k] += r[k];
      }
#pragma unroll
      for (int j = 0; j < N / 8; ++j) *chunk_at(out, m, RB, j) = pack8(v + 8 * j);
      float r[N];
#pragma unroll
      for (int q = 0; q < N; ++q) r[q] = fmaxf(__bfloat162float(__float2bfloat16_rn(v[q])), 0.f);
      if (outr) {
#pragma unroll
        for (int j = 0; j < N / 8; ++j) *chunk_at(outr, m, RB, j) = pack8(r + 8 * j);
      }
      if (dense) {
        const int ct = dense_ct > 0 ? dense_ct : N;
        uint4* d = reinterpret_cast<uint4*>(dense + ((int64_t)f * g.H * g.W + (int64_t)y * g.W + x) * ct + dense_off);
#pragma unroll
        for (int j = 0; j < N / 8; ++j) d[j] = pack8(r + 8 * j);
      }
    } else if constexpr (MODE == W3_RES) {
      // 64 channels, per 8-channel chunk (no second N-float array: the array form spills):
      // + residual, h, relu(h) (of the rounded h), dense relu(h)
      uint4* d = nullptr;
      if (dense) {
        const int ct = dense_ct > 0 ? dense_ct : N;
        d = reinterpret_cast<uint4*>(dense + ((int64_t)f * g.H * g.W + (int64_t)y * g.W + x) * ct + dense_off);
      }
#pragma unroll
      for (int j = 0; j < N / 8; ++j) {
        float r[8];
        unpack8(p[j], r);
#pragma unroll
        for (int k = 0; k < 8; ++k) v[8 * j + k] += r[k];
        const uint4 hv = pack8(v + 8 * j);
        *chunk_at(out, m, RB, j) = hv;
        float h8[8];
        unpack8(hv, h8);
#pragma unroll
        for (int k = 0; k < 8; ++k) h8[k] = fmaxf(h8[k], 0.f);
        const uint4 rv = pack8(h8);
        if (outr) *chunk_at(outr, m, RB, j) = rv;
        if (d) d[j] = rv;
      }
    } else {
#pragma unroll
      for (int j = 0; j < N / 8; ++j) *chunk_at(out, m, RB, j) = pack8(v + 8 * j);
    }
  }
};

template <int MODE, int NN>
struct W3DgradEpi {
  static constexpr int N = NN;
  static constexpr int RB = 2 * NN;
  // the mask row, then (D3W_RES) the incoming residual-gradient row (at 64 channels
  // the residual row is read in the store instead: prefetching both spills)
  static constexpr bool DRES_PRE = N <= 32;
  static constexpr int PRE = (MODE == D3W_PLAIN || MODE == D3W_PART) ? 0
                             : (MODE == D3W_MASK || !DRES_PRE) ? N / 8 : N / 4;
  PadGeo g;
  const uint8_t* mask;
  const uint8_t* dres;
  uint8_t* dX;
  float* part_out;
  const float* part_in;
  __device__ void pre(int64_t m, uint4 (&p)[PRE > 0 ? PRE : 1]) const {
    if (MODE == D3W_PLAIN || MODE == D3W_PART) return;
#pragma unroll
    for (int j = 0; j < N / 8; ++j) p[j] = __ldg(chunk_at(mask, m, RB, j));
    if constexpr (MODE == D3W_RES && DRES_PRE) {
#pragma unroll
      for (int j = 0; j < N / 8; ++j) p[N / 8 + j] = __ldg(chunk_at(dres, m, RB, j));
    }
  }
  __device__ void store(int64_t m, float (&v)[N]) const {   // PRE == 0 modes
    const uint4 p[1] = {make_uint4(0, 0, 0, 0)};
    store(m, v, p);
  }
  __device__ void store(int64_t m, float (&v)[N], const uint4 (&p)[PRE > 0 ? PRE : 1]) const {
    if constexpr (MODE == D3W_PART) {   // the first dY plane's fp32 sum (every row)
      float4* d = reinterpret_cast<float4*>(part_out + m * N);
#pragma unroll
      for (int q = 0; q < N / 4; ++q) d[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      return;
    }
    int f, y, x;
    if (!g.split(m, f, y, x)) {
      const uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int j = 0; j < N / 8; ++j) *chunk_at(dX, m, RB, j) = z;
      return;
    }
    if (N == 64 && part_in) {   // plane pairs: 64-ch only
      const float4* ps = reinterpret_cast<const float4*>(part_in + m * N);
#pragma unroll
      for (int q = 0; q < N / 4; ++q) {
        const float4 t = __ldg(ps + q);
        v[4 * q] += t.x; v[4 * q + 1] += t.y; v[4 * q + 2] += t.z; v[4 * q + 3] += t.w;
      }
    }
    if (MODE != D3W_PLAIN) {
#pragma unroll
      for (int j = 0; j < N / 8; ++j) {
        float mk[8];
        unpack8(p[j], mk);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (!(mk[k] > 0.f)) v[8 * j + k] = 0.f;
      }
    }
    if (MODE == D3W_RES) {
#pragma unroll
      for (int j = 0; j < N / 8; ++j) {
        float r[8];
        if constexpr (DRES_PRE) unpack8(p[N / 8 + j], r);
        else unpack8(__ldg(chunk_at(dres, m, RB, j)), r);
#pragma unroll
        for (int k = 0; k < 8; ++k) v[8 * j + k] += r[k];
      }
    }
#pragma unroll
    for (int j = 0; j < N / 8; ++j) *chunk_at(dX, m, RB, j) = pack8(v + 8 * j);
  }
};

// weight-gradient finish: accumulator group grp, row i = atom * Cp + c
struct W3Fin {
  int xim, Cp, CI;
  float scale;
  float* g_w;
  float* g_b;
  __device__ void weight(int grp, int i, int n, float t) const {
    const int atom = i / Cp, ch = i % Cp;
    int ky, kx, c;
    if (xim) {
      ky = atom; kx = ch / CI; c = ch % CI;
      if (ky >= 3 || ch >= 3 * CI) return;
    } else {
      ky = grp; kx = atom; c = ch;
      if (kx >= 3 || c >= CI) return;
    }
    g_w[(((size_t)n * 3 + ky) * 3 + kx) * CI + c] = t * scale;
  }
  __device__ void bias(int n, float t) const { g_b[n] = t; }
};

// ------------------------------------------------------------------ forward
// 128-row blocks per window-conv tile (measured per shape, scripts/phases.py
// PER_LAUNCH=1 at MT = 1 / 2 / 4): 16-channel outputs 4; 32-channel 2 (the
// residual forward's second input row is prefetched before the accumulator wait)
template <int MODE, int N, bool FWD>
constexpr int w3_mt() { return N == 16 ? 4 : N == 32 ? 2 : 1; }
// NW = 9: 3 x 3 taps as row windows; NW = 3: x-im2col input, 3 row windows (ky)
// Column-tap-stacked kernels (win_engine.cuh win_conv_kx_kernel: 3 MMAs of
// N = 3*out per 128 rows, neighbour-row combine in the epilogue) vs the 9-window
// kernels (9 MMAs of N = out, no combine).  Measured per launch at c4
// (profiles/r02/kx_vs_9window.md): the combine's shuffles cost more than the six
// saved ~45-cycle MMAs everywhere except when K = 32 input channels feed 16
// outputs (RB = 64, N = 16: 18 -> 6 MMAs per 128 rows; 205 -> 165 us), so that is
// the only shape that takes it.  SEED_KX=1 forces it for every 3x3 conv,
// SEED_KX=0 never (A/B measurement).
template <int N, int RB>
static bool kx_stacked() {
  static const int env = [] {
    const char* e = getenv("SEED_KX");
    return e ? (e[0] == '0' ? 0 : 1) : -1;
  }();
  return env >= 0 ? env == 1 : (RB == 64 && N == 16);
}

static U8Rows u8_rows(const uint8_t* obs, const PadGeo& g) {
  U8Rows u{};
  u.obs = obs; u.H = g.H; u.W = g.W; u.Wp = g.Wp; u.P = g.P;
  u.fP = FastDiv((uint32_t)g.P); u.fWp = FastDiv((uint32_t)g.Wp);
  return u;
}

template <int MODE, int N, int RB, int NW, int XF = XF_NONE>
static seed_status fwd_t(const Conv3wFwd& a, cudaStream_t st) {
  WinConvArgs w{};
  w.trig = (deep_trig() >> 1) & 1;
  w.src = a.in; w.src_rows = a.rows; w.M = a.rows;
  w.wimg = reinterpret_cast<const uint8_t*>(a.wimg);
  if (XF == XF_U8) w.u8 = u8_rows(a.obs_u8, a.g);
  W3FwdEpi<MODE, N> e{};
  e.g = a.g; e.in_scale = a.in_scale; e.bias = a.bias; e.res = a.res; e.out = a.out;
  e.outr = a.outr; e.dense = a.dense; e.dense_ct = a.dense_ct; e.dense_off = a.dense_off;
  e.part_out = a.part_out; e.part_in = a.part_in;
  if constexpr (NW == 9 && XF == XF_NONE && N <= 32) {
    if (kx_stacked<N, RB>()) {   // 3 row windows ky, column taps stacked on N
      for (int k = 0; k < 3; ++k) w.off[k] = (k - 1) * a.g.Wp;
      return launch_win_conv_kx<W3FwdEpi<MODE, N>, RB, N == 16 ? 2 : 1, 3>(w, e, st);
    }
  }
  for (int k = 0; k < NW; ++k)
    w.off[k] = NW == 9 ? ((k / 3) - 1) * a.g.Wp + (k % 3) - 1 : (k - 1) * a.g.Wp;
  return launch_win_conv<W3FwdEpi<MODE, N>, RB, NW, w3_mt<MODE, N, true>(), XF>(w, e, st);
}

template <int MODE>
static seed_status fwd_mode(const Conv3wFwd& a, cudaStream_t st) {
  if (a.xf == XF_U8) {   // section 0 of the GRF net: 16 uint8 planes
    if (MODE == W3_PLAIN && !a.xim && a.ch == 16 && a.cin_p == 16 && a.obs_u8)
      return fwd_t<MODE, 16, 32, 9, XF_U8>(a, st);
    return SEED_E_UNSUPPORTED;
  }
  if (a.xf == XF_RELU) {   // residual conv0: relu of the residual stream in shared memory
    if (MODE == W3_RELU && !a.xim && a.ch == 16 && a.cin_p == 16) return fwd_t<MODE, 16, 32, 9, XF_RELU>(a, st);
    if (MODE == W3_RELU && !a.xim && a.ch == 32 && a.cin_p == 32) return fwd_t<MODE, 32, 64, 9, XF_RELU>(a, st);
    return SEED_E_UNSUPPORTED;
  }
  if (a.xim) {
    if (a.ch == 16 && a.cin_p == 16) return fwd_t<MODE, 16, 32, 3>(a, st);
    if (a.ch == 32 && a.cin_p == 16) return fwd_t<MODE, 32, 32, 3>(a, st);
    if (a.ch == 64 && a.cin_p == 16) return fwd_t<MODE, 64, 32, 3>(a, st);   // DMLab 4x
    return SEED_E_UNSUPPORTED;
  }
  if (a.ch == 16 && a.cin_p == 16) return fwd_t<MODE, 16, 32, 9>(a, st);
  if (a.ch == 32 && a.cin_p == 16) return fwd_t<MODE, 32, 32, 9>(a, st);
  if (a.ch == 16 && a.cin_p == 32) return fwd_t<MODE, 16, 64, 9>(a, st);
  if (a.ch == 32 && a.cin_p == 32) return fwd_t<MODE, 32, 64, 9>(a, st);
  if (a.ch == 64 && a.cin_p == 32) return fwd_t<MODE, 64, 64, 9>(a, st);    // DMLab Medium (2x)
  if (a.ch == 64 && a.cin_p == 64) return fwd_t<MODE, 64, 128, 9>(a, st);
  return SEED_E_UNSUPPORTED;
}

seed_status conv3w_forward(const Conv3wFwd& a, cudaStream_t st) {
  if (a.mode == W3_PLAIN) return fwd_mode<W3_PLAIN>(a, st);
  if (a.mode == W3_RELU && !a.xim) return fwd_mode<W3_RELU>(a, st);
  if (a.mode == W3_RES && !a.xim) return fwd_mode<W3_RES>(a, st);
  if (a.mode == W3_PART && !a.xim && a.xf == XF_NONE && a.ch == 64 && a.cin_p == 64 && a.part_out)
    return fwd_t<W3_PART, 64, 128, 9>(a, st);   // plane pairs of the 4x torso
  return SEED_E_UNSUPPORTED;
}

// ------------------------------------------------------------------ data gradient
template <int MODE, int N, int RB>
static seed_status dgrad_t(const Conv3wDgrad& a, cudaStream_t st) {
  WinConvArgs w{};
  w.trig = (deep_trig() >> 1) & 1;
  w.src = a.dY; w.src_rows = a.rows; w.M = a.rows;
  w.wimg = reinterpret_cast<const uint8_t*>(a.wimg);
  // row windows ky at -(ky-1)*Wp; the image stacks the column taps as groups 2 - kx
  // (win3_img_pos mode 1), so out[g] = D[g-1][grp 0] + D[g][grp 1] + D[g+1][grp 2]
  W3DgradEpi<MODE, N> e{};
  e.g = a.g; e.mask = a.mask; e.dres = a.dres; e.dX = a.dX; e.part_out = a.part_out; e.part_in = a.part_in;
  if constexpr (N <= 32) {
    if (kx_stacked<N, RB>()) {   // 3 row windows at -(ky-1)*Wp, column taps stacked on N
      for (int k = 0; k < 3; ++k) w.off[k] = -(k - 1) * a.g.Wp;
      return launch_win_conv_kx<W3DgradEpi<MODE, N>, RB, N == 16 ? 2 : 1, 3>(w, e, st);
    }
  }
  // 9 windows: tap (ky, kx) at -((ky-1)*Wp + kx-1), image row block ky*3 + 2 - kx
  for (int k = 0; k < 9; ++k) w.off[k] = -(((k / 3) - 1) * a.g.Wp + 1 - (k % 3));
  return launch_win_conv<W3DgradEpi<MODE, N>, RB, 9, w3_mt<MODE, N, false>()>(w, e, st);
}

template <int MODE>
static seed_status dgrad_mode(const Conv3wDgrad& a, cudaStream_t st) {
  if (a.cin == 16 && a.ch == 16) return dgrad_t<MODE, 16, 32>(a, st);
  if (a.cin == 16 && a.ch == 32) return dgrad_t<MODE, 16, 64>(a, st);
  if (a.cin == 32 && a.ch == 16) return dgrad_t<MODE, 32, 32>(a, st);
  if (a.cin == 32 && a.ch == 32) return dgrad_t<MODE, 32, 64>(a, st);
  if (a.cin == 32 && a.ch == 64) return dgrad_t<MODE, 32, 128>(a, st);   // DMLab Medium (2x)
  if (a.cin == 64 && a.ch == 64) return dgrad_t<MODE, 64, 128>(a, st);
  return SEED_E_UNSUPPORTED;
}

seed_status conv3w_dgrad(const Conv3wDgrad& a, cudaStream_t st) {
  if (a.mode == D3W_PLAIN) return dgrad_mode<D3W_PLAIN>(a, st);
  if (a.mode == D3W_MASK) return dgrad_mode<D3W_MASK>(a, st);
  if (a.mode == D3W_RES) return dgrad_mode<D3W_RES>(a, st);
  if (a.mode == D3W_PART && a.cin == 64 && a.ch == 64 && a.part_out) return dgrad_t<D3W_PART, 64, 128>(a, st);
  return SEED_E_UNSUPPORTED;
}

// ------------------------------------------------------------------ weight gradient
// win_engine.cuh win3_wgrad_kernel: D[(kx, c)][(j, co)], tap ky = 2 - j.
//   9-window input: dW[co][ky][kx][c] = sum_h X[h + kx][c] dY[h + 1 - Wp + j*Wp][co]
//   x-im2col input: dW[co][ky][(kx, c)] = sum_h X[h][(kx, c)] dY[h - Wp + j*Wp][co] (atom 0)
struct W3Fin3 {
  int xim, Cp, CI, CO;
  int ci_full, co_off, c_off;   // the [co_off..][3][3][c_off..] block of a [..][3][3][ci_full] tensor
  float scale;
  float* g_w;
  float* g_b;
  __device__ void weight3(int i, int n, float t) const {
    const int atom = i / Cp, ch = i % Cp;
    const int ky = 2 - n / CO, co = n % CO;
    int kx, c;
    if (xim) {
      // channel 3*CI of the x-im2col input is constant 1 (conv3_obs_kernel): its
      // row of the accumulator against tap ky = 1 (dY unshifted) is the bias gradient
      if (atom == 0 && ch == 3 * CI && ky == 1) g_b[co] = t;
      if (atom != 0 || ch >= 3 * CI) return;
      kx = ch / CI; c = ch % CI;
    } else {
      if (atom >= 3 || ch >= CI) return;
      kx = atom; c = ch;
    }
    g_w[(((size_t)(co_off + co) * 3 + ky) * 3 + kx) * ci_full + c_off + c] = t * scale;
  }
  __device__ void bias(int n, float t) const { g_b[n] = t; }
};

size_t conv3w_wgrad_part_bytes(int64_t rows, int ch, bool) {
  return win3_wgrad_part_bytes(rows, ch, 3, ch == 64 ? 128 : 64);   // 64-ch inputs: 256 partial rows
}

seed_status conv3w_wgrad(const Conv3wWgrad& a, cudaStream_t st) {
  Win3WgradArgs w{};
  w.trig = deep_trig() & 1;
  w.X = a.X; w.dy = a.dY; w.M = a.rows; w.part = a.part;
  if (a.xf == XF_U8) w.u8 = u8_rows(a.obs_u8, a.g);
  w.boff = a.xim ? -a.g.Wp : 1 - a.g.Wp;
  w.bstride = a.g.Wp;
  W3Fin3 f{};
  f.xim = a.xim ? 1 : 0; f.Cp = a.cin_p; f.CI = a.cin; f.CO = a.ch; f.scale = a.scale; f.g_w = a.g_w;
  f.g_b = a.g_b;
  f.ci_full = a.ci_full > 0 ? a.ci_full : a.cin; f.co_off = a.co_off; f.c_off = a.c_off;
  const bool bias = !a.xim && a.g_b;
  if (a.xim && !a.g_b) return SEED_E_ARG;   // x-im2col: the bias comes with the weights
  if (a.xf == XF_U8) {
    if (a.ch == 16 && a.cin_p == 16 && !a.xim && a.obs_u8)
      return launch_win3_wgrad<16, 32, W3Fin3, 3, XF_U8>(w, f, true, st);
    return SEED_E_UNSUPPORTED;
  }
  if (a.xf == XF_RELU) {
    if (a.ch == 16 && a.cin_p == 16 && !a.xim) return launch_win3_wgrad<16, 32, W3Fin3, 3, XF_RELU>(w, f, true, st);
    if (a.ch == 32 && a.cin_p == 32 && !a.xim) return launch_win3_wgrad<32, 64, W3Fin3, 3, XF_RELU>(w, f, true, st);
    return SEED_E_UNSUPPORTED;
  }
  if (a.ch == 16 && a.cin_p == 16) return launch_win3_wgrad<16, 32>(w, f, bias, st);
  if (a.ch == 32 && a.cin_p == 16) return launch_win3_wgrad<32, 32>(w, f, bias, st);
  if (a.ch == 64 && a.cin_p == 16) return launch_win3_wgrad<64, 32>(w, f, bias, st);   // DMLab 4x s0
  if (a.ch == 16 && a.cin_p == 32) return launch_win3_wgrad<16, 64>(w, f, bias, st);
  if (a.ch == 32 && a.cin_p == 32) return launch_win3_wgrad<32, 64>(w, f, bias, st);
  if (a.ch == 64 && a.cin_p == 32) return launch_win3_wgrad<64, 64>(w, f, bias, st);
  if (a.ch == 64 && a.cin_p == 64) return launch_win3_wgrad<64, 128>(w, f, bias, st);
  return SEED_E_UNSUPPORTED;
}

// ------------------------------------------------------------------ row-parallel kernels
// grid.x = one padded image row (f, Y) of the output space, grid.y * blockDim.x
// threads over (X, chunk j): no per-thread divisions beyond constant shifts.
constexpr int ROWK_THREADS = 128;
constexpr int ROWK_RPB = 8;   // padded rows per block (grid.x = F * ceil(Hp / RPB))

// obs conversion: thread = (X, chunk of 8 channels)
template <int NC, int CX>   // chunks per row; CX = compile-time C for the x-im2col path (0 = runtime)
__global__ void __launch_bounds__(ROWK_THREADS) conv3_obs_kernel(
    PadGeo g, int C, int xim, const uint8_t* __restrict__ obs, uint8_t* __restrict__ X0) {
  pdl_wait();
  constexpr int RB = NC * 16;
  const int t = blockIdx.y * ROWK_THREADS + threadIdx.x;
  if (t >= g.Wp * NC) return;
  const int X = t / NC, j = t % NC;
  const int Hp = g.H + 2, nb = (Hp + ROWK_RPB - 1) / ROWK_RPB;
  const int f = blockIdx.x / nb, Y0 = (blockIdx.x - f * nb) * ROWK_RPB;
  for (int Y = Y0; Y < min(Y0 + ROWK_RPB, Hp); ++Y) {
  const int64_t m = ((int64_t)f * Hp + Y) * g.Wp + X;
  const int y = Y - 1, x = X - 1;
  float v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = 0.f;
  if (y >= 0 && y < g.H && x >= 0 && x < g.W) {
    const int Cr = CX ? CX : C;
    const uint8_t* px = obs + (((size_t)f * g.H + y) * g.W + x) * Cr;
    if (!xim && Cr % 8 == 0) {
      const uint2 u = __ldg(reinterpret_cast<const uint2*>(px + 8 * j));
      const uint32_t w[2] = {u.x, u.y};
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = (float)((w[k >> 2] >> (8 * (k & 3))) & 0xFF);
    } else if (!xim) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (8 * j + k < Cr) v[k] = (float)__ldg(px + 8 * j + k);
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int ch = 8 * j + k;
        const int kx = ch / Cr, c = ch - kx * Cr, xx = x + kx - 1;
        if (ch < 3 * Cr && xx >= 0 && xx < g.W) v[k] = (float)__ldg(px + (kx - 1) * Cr + c);
      }
    }
  }
  // x-im2col: channel 3C is constant 1 (its weights are zero in the forward image;
  // the weight-gradient accumulator turns it into the bias gradient, W3Fin3)
  if (xim) {
    const int Cr = CX ? CX : C;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (8 * j + k == 3 * Cr) v[k] = 1.f;
  }
  *chunk_at(X0, m, RB, j) = pack8(v);
  }
}

// x-im2col conversion for C = CX <= 5 (16-channel rows): thread = one padded-row
// pixel X; its own pixel's C bytes are loaded coalesced, the x-1 / x+1 neighbours
// come from lanes -+1 (direct loads at warp edges); channel 3C = 1 (see above).
template <int CX>
__global__ void __launch_bounds__(ROWK_THREADS) conv3_obs_xim_kernel(
    PadGeo g, const uint8_t* __restrict__ obs, uint8_t* __restrict__ X0) {
  pdl_wait();
  const int X = blockIdx.y * ROWK_THREADS + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int Hp = g.H + 2, nb = (Hp + ROWK_RPB - 1) / ROWK_RPB;
  const int f = blockIdx.x / nb, Y0 = (blockIdx.x - f * nb) * ROWK_RPB;
  const int x = X - 1;
  for (int Y = Y0; Y < min(Y0 + ROWK_RPB, Hp); ++Y) {
    const int y = Y - 1;
    const bool rowok = y >= 0 && y < g.H;
    const uint8_t* pr = obs + ((size_t)f * g.H + (rowok ? y : 0)) * g.W * CX;
    float me[CX], lf[CX], rt[CX];
#pragma unroll
    for (int c = 0; c < CX; ++c) me[c] = (rowok && x >= 0 && x < g.W) ? (float)__ldg(pr + x * CX + c) : 0.f;
#pragma unroll
    for (int c = 0; c < CX; ++c) {
      lf[c] = __shfl_up_sync(0xffffffffu, me[c], 1);
      rt[c] = __shfl_down_sync(0xffffffffu, me[c], 1);
    }
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < CX; ++c) lf[c] = (rowok && x - 1 >= 0 && x - 1 < g.W) ? (float)__ldg(pr + (x - 1) * CX + c) : 0.f;
    }
    if (lane == 31) {
#pragma unroll
      for (int c = 0; c < CX; ++c) rt[c] = (rowok && x + 1 >= 0 && x + 1 < g.W) ? (float)__ldg(pr + (x + 1) * CX + c) : 0.f;
    }
    if (X < g.Wp) {
      float v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = 0.f;
      const bool in = rowok && x >= 0 && x < g.W;
      if (in) {
#pragma unroll
        for (int c = 0; c < CX; ++c) { v[c] = lf[c]; v[CX + c] = me[c]; v[2 * CX + c] = rt[c]; }
      }
      v[3 * CX] = 1.f;
      const int64_t m = ((int64_t)f * Hp + Y) * g.Wp + X;
      *chunk_at(X0, m, 32, 0) = pack8(v);
      *chunk_at(X0, m, 32, 1) = pack8(v + 8);
    }
  }
}

// direct conversion for C = 16 (GRF SMM planes): thread = one padded-row pixel, one
// 16-byte load of its 16 channel bytes, two 16-byte chunk stores
__global__ void __launch_bounds__(ROWK_THREADS) conv3_obs_c16_kernel(
    PadGeo g, const uint8_t* __restrict__ obs, uint8_t* __restrict__ X0) {
  pdl_wait();
  const int X = blockIdx.y * ROWK_THREADS + threadIdx.x;
  if (X >= g.Wp) return;
  const int Hp = g.H + 2, nb = (Hp + ROWK_RPB - 1) / ROWK_RPB;
  const int f = blockIdx.x / nb, Y0 = (blockIdx.x - f * nb) * ROWK_RPB;
  const int x = X - 1;
  for (int Y = Y0; Y < min(Y0 + ROWK_RPB, Hp); ++Y) {
    const int y = Y - 1;
    uint4 u = make_uint4(0, 0, 0, 0);
    if (y >= 0 && y < g.H && x >= 0 && x < g.W)
      u = __ldg(reinterpret_cast<const uint4*>(obs + (((size_t)f * g.H + y) * g.W + x) * 16));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
    uint32_t o[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {   // bytes -> bf16 (exact): the float's high half
      const uint32_t b0 = w[k] & 0xFF, b1 = (w[k] >> 8) & 0xFF, b2 = (w[k] >> 16) & 0xFF, b3 = w[k] >> 24;
      o[2 * k] = (__float_as_uint((float)b0) >> 16) | (__float_as_uint((float)b1) & 0xFFFF0000u);
      o[2 * k + 1] = (__float_as_uint((float)b2) >> 16) | (__float_as_uint((float)b3) & 0xFFFF0000u);
    }
    const int64_t m = ((int64_t)f * Hp + Y) * g.Wp + X;
    *chunk_at(X0, m, 32, 0) = make_uint4(o[0], o[1], o[2], o[3]);
    *chunk_at(X0, m, 32, 1) = make_uint4(o[4], o[5], o[6], o[7]);
  }
}

seed_status conv3_obs(const uint8_t* obs, int64_t F, const PadGeo& g, int C, int Cp, bool xim,
                      uint8_t* X0, cudaStream_t st) {
  if (F == 0) return SEED_OK;
  const int NC = Cp / 8;
  const dim3 grid((unsigned)(F * ceil_div(g.H + 2, ROWK_RPB)), (unsigned)ceil_div(g.Wp * NC, ROWK_THREADS));
  if (NC == 2) {
    if (xim && C == 3) {
      const dim3 gx((unsigned)(F * ceil_div(g.H + 2, ROWK_RPB)), (unsigned)ceil_div(g.Wp, ROWK_THREADS));
      return launch_k(conv3_obs_xim_kernel<3>, gx, dim3(ROWK_THREADS), 0, st, g, obs, X0);
    }
    if (!xim && C == 16 && (reinterpret_cast<uintptr_t>(obs) & 15) == 0) {
      const dim3 gx((unsigned)(F * ceil_div(g.H + 2, ROWK_RPB)), (unsigned)ceil_div(g.Wp, ROWK_THREADS));
      return launch_k(conv3_obs_c16_kernel, gx, dim3(ROWK_THREADS), 0, st, g, obs, X0);
    }
    return launch_k(conv3_obs_kernel<2, 0>, grid, dim3(ROWK_THREADS), 0, st, g, C, xim ? 1 : 0, obs, X0);
  }
  if (NC == 4 && !xim)
    return launch_k(conv3_obs_kernel<4, 0>, grid, dim3(ROWK_THREADS), 0, st, g, C, 0, obs, X0);
  return SEED_E_UNSUPPORTED;
}

// ------------------------------------------------------------------ max-pool
template <int NC>
__global__ void __launch_bounds__(ROWK_THREADS) conv3w_pool_fwd_kernel(
    PadGeo gi, PadGeo go, int pt, int pl, const uint8_t* __restrict__ conv, uint8_t* __restrict__ h0,
    uint8_t* __restrict__ hr0, uint8_t* __restrict__ arg) {
  pdl_wait();
  constexpr int C = NC * 8, RB = NC * 16;
  const int t = blockIdx.y * ROWK_THREADS + threadIdx.x;
  if (t >= go.Wp * NC) return;
  const int X = t / NC, j = t % NC;
  const int Hp = go.H + 2, nb = (Hp + ROWK_RPB - 1) / ROWK_RPB;
  const int f = blockIdx.x / nb, Y0 = (blockIdx.x - f * nb) * ROWK_RPB;
  for (int Y = Y0; Y < min(Y0 + ROWK_RPB, Hp); ++Y) {
  const int64_t m = ((int64_t)f * Hp + Y) * go.Wp + X;
  const int oy = Y - 1, ox = X - 1;
  if (oy < 0 || oy >= go.H || ox < 0 || ox >= go.W) {
    const uint4 z = make_uint4(0, 0, 0, 0);
    *chunk_at(h0, m, RB, j) = z;
    if (hr0) *chunk_at(hr0, m, RB, j) = z;
    continue;
  }
  uint4 in[9];
  const int64_t fb = (int64_t)f * gi.P;
#pragma unroll
  for (int q = 0; q < 9; ++q) {   // issue all window loads first
    const int y = oy * 2 - pt + q / 3, x = ox * 2 - pl + q % 3;
    const bool ok = y >= 0 && y < gi.H && x >= 0 && x < gi.W;
    in[q] = ok ? __ldg(chunk_at(conv, fb + (int64_t)(y + 1) * gi.Wp + (x + 1), RB, j))
               : make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);   // -inf
  }
  uint4 best, rl;
  uint2 a;
  pool_max9(in, best, rl, a);
  *chunk_at(h0, m, RB, j) = best;
  if (hr0) *chunk_at(hr0, m, RB, j) = rl;
  *reinterpret_cast<uint2*>(arg + m * C + 8 * j) = a;
  }
}

// Backward: thread = (frame, 2x2 block of input pixels (y + pt, x + pl) in
// {2a, 2a+1} x {2b, 2b+1}).  The block's pixels receive gradient only from
// the 2x2 windows (a-1 | a) x (b-1 | b): an even offset is tap 2 of window a-1 and
// tap 0 of window a, an odd offset tap 1 of window a.  The four windows' (argmax,
// dout) are loaded once for the four pixels; sums in ascending window order.
// prmt.b32 with selector nibbles >= 8: the selected byte's top bit replicated over
// the output byte (__byte_perm uses the low 3 bits of each nibble only)
__device__ __forceinline__ uint32_t prmt_sign(uint32_t x, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(x), "r"(sel));
  return r;
}

// 16-byte chunk j of padded row `row` (32-bit row index, 64-bit byte address)
__device__ __forceinline__ uint4* chunk_at32(uint8_t* base, uint32_t row, int RB, int j) {
  return reinterpret_cast<uint4*>(base + (size_t)row * RB + (swz_chunk(row, RB, j) << 4));
}
__device__ __forceinline__ const uint4* chunk_at32(const uint8_t* base, uint32_t row, int RB, int j) {
  return reinterpret_cast<const uint4*>(base + (size_t)row * RB + (swz_chunk(row, RB, j) << 4));
}

// One thread per (2x2 block, 16-byte chunk j): a warp's loads / stores of one
// pixel cover whole 32-byte sectors (one thread per block and all chunks was 1.3-2.6x
// slower).  32-bit index arithmetic (with 64-bit indices the kernel was ALU-bound,
// 85 % of the ALU pipe, c4 s0 309 us).  Threads past `total` zero one border chunk
// each of din (per frame: top / bottom rows, then the left / right pixels of the
// interior rows).
template <int NC>
__global__ void __launch_bounds__(256) conv3w_pool_bwd_kernel(
    PadGeo gi, PadGeo go, int pt, int pl, int total, int nz, FastDiv fnbx, FastDiv fnby, FastDiv fper,
    FastDiv fwp, const uint8_t* __restrict__ dout, const uint8_t* __restrict__ arg, uint8_t* __restrict__ din,
    int trig) {
  pdl_wait();
  if (trig) pdl_trigger();
  constexpr int C = NC * 8, RB = NC * 16;
  const int tt = blockIdx.x * blockDim.x + threadIdx.x;
  if (tt >= total) {
    if (tt >= total + nz) return;
    const uint32_t zi = (uint32_t)(tt - total);
    const int j = (int)(zi % NC);
    uint32_t f, k, Y, X;
    fper.divmod(zi / NC, f, k);
    if (k < 2u * gi.Wp) {
      uint32_t hi;
      fwp.divmod(k, hi, X);
      Y = hi ? gi.H + 1 : 0;
    } else {
      const uint32_t e = k - 2u * gi.Wp;
      Y = 1 + (e >> 1);
      X = (e & 1) ? gi.W + 1 : 0;
    }
    *chunk_at32(din, f * gi.P + Y * gi.Wp + X, RB, j) = make_uint4(0, 0, 0, 0);
    return;
  }
  uint32_t fa, rem, f, a;
  fnbx.divmod((uint32_t)tt, fa, rem);   // fnbx: blocks per row x NC
  fnby.divmod(fa, f, a);
  const uint32_t b = rem / NC;
  const int j = (int)(rem % NC);
  const uint32_t fo = f * go.P, fi = f * gi.P;
  uint32_t orow[4];
  bool ok[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {   // windows (a-1, b-1), (a-1, b), (a, b-1), (a, b)
    const int oy = (int)a - 1 + (q >> 1), ox = (int)b - 1 + (q & 1);
    ok[q] = oy >= 0 && oy < go.H && ox >= 0 && ox < go.W;
    orow[q] = fo + (uint32_t)(oy + 1) * go.Wp + (uint32_t)(ox + 1);
  }
  uint32_t irow[4];
  bool in[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int y = 2 * (int)a + (p >> 1) - pt, x = 2 * (int)b + (p & 1) - pl;
    in[p] = y >= 0 && y < gi.H && x >= 0 && x < gi.W;
    irow[p] = fi + (uint32_t)(y + 1) * gi.Wp + (uint32_t)(x + 1);
  }
  {
    uint2 av[4];
    uint4 dv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      av[q] = ok[q] ? __ldg(reinterpret_cast<const uint2*>(arg + (size_t)orow[q] * C + 8 * j))
                    : make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
      dv[q] = ok[q] ? __ldg(chunk_at32(dout, orow[q], RB, j)) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int dy = p >> 1, dx = p & 1;
      if (!in[p]) continue;
      float s[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) s[k] = 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int wy = q >> 1, wx = q & 1;   // window a-1+wy, b-1+wx
        // tap of this pixel in that window: even offset -> 2 (wy = 0) / 0 (wy = 1); odd -> 1 (wy = 1 only)
        const int ky = dy == 0 ? (wy == 0 ? 2 : 0) : (wy == 1 ? 1 : -1);
        const int kx = dx == 0 ? (wx == 0 ? 2 : 0) : (wx == 1 ? 1 : -1);
        if (ky < 0 || kx < 0) continue;
        // argmax byte == tap: the argmax bytes are 0..8 or 0xFF (no window), so a byte
        // of av ^ w4 is 0 (match), 1..15 or >= 0xF7; byte b of ((av ^ w4) | 0x80) - 1
        // has its top bit clear exactly on a match (no borrow crosses bytes); the top
        // bits are replicated into 16-bit lane masks (byte_perm sign mode)
        const uint32_t w4 = (uint32_t)(ky * 3 + kx) * 0x01010101u;
        const uint32_t nx = ((av[q].x ^ w4) | 0x80808080u) - 0x01010101u;
        const uint32_t ny = ((av[q].y ^ w4) | 0x80808080u) - 0x01010101u;
        const uint32_t nm[4] = {prmt_sign(nx, 0x9988), prmt_sign(nx, 0xBBAA), prmt_sign(ny, 0x9988),
                                prmt_sign(ny, 0xBBAA)};
        const uint32_t dw[4] = {dv[q].x, dv[q].y, dv[q].z, dv[q].w};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const uint32_t d = dw[r] & ~nm[r];
          s[2 * r] += bf16_lo(d);
          s[2 * r + 1] += bf16_hi(d);
        }
      }
      *chunk_at32(din, irow[p], RB, j) = pack8(s);
    }
  }
}


seed_status conv3w_pool_fwd(int64_t F, const PadGeo& gi, const PadGeo& go, int C, int pt, int pl,
                            const uint8_t* conv, uint8_t* h0, uint8_t* hr0, uint8_t* arg,
                            cudaStream_t st) {
  if (F == 0) return SEED_OK;
  const int NC = C / 8;
  const dim3 grid((unsigned)(F * ceil_div(go.H + 2, ROWK_RPB)), (unsigned)ceil_div(go.Wp * NC, ROWK_THREADS));
  if (NC == 2)
    return launch_k(conv3w_pool_fwd_kernel<2>, grid, dim3(ROWK_THREADS), 0, st, gi, go, pt, pl, conv, h0, hr0, arg);
  if (NC == 4)
    return launch_k(conv3w_pool_fwd_kernel<4>, grid, dim3(ROWK_THREADS), 0, st, gi, go, pt, pl, conv, h0, hr0, arg);
  if (NC == 8)
    return launch_k(conv3w_pool_fwd_kernel<8>, grid, dim3(ROWK_THREADS), 0, st, gi, go, pt, pl, conv, h0, hr0, arg);
  return SEED_E_UNSUPPORTED;
}

seed_status conv3w_pool_bwd(int64_t F, const PadGeo& gi, const PadGeo& go, int C, int pt, int pl,
                            const uint8_t* dout, const uint8_t* arg, uint8_t* din,
                            cudaStream_t st) {
  if (F == 0) return SEED_OK;
  const int NC = C / 8;
  const int nby = (gi.H + pt + 1) >> 1, nbx = (gi.W + pl + 1) >> 1;
  const int64_t total = F * nby * nbx * NC;
  const int per = 2 * gi.Wp + 2 * gi.H;
  const int64_t nz = F * per * NC;
  // 32-bit thread and row indices
  if (total + nz >= (1ll << 31) || F * gi.P >= (1ll << 32) || F * go.P >= (1ll << 32)) return SEED_E_SHAPE;
  const FastDiv fnbx((uint32_t)(nbx * NC)), fnby((uint32_t)nby), fper((uint32_t)per), fwp((uint32_t)gi.Wp);
  const dim3 grid((unsigned)((total + nz + 255) / 256));
  const int t32 = (int)total, z32 = (int)nz;
  if (NC == 2)
    return launch_k(conv3w_pool_bwd_kernel<2>, grid, dim3(256), 0, st, gi, go, pt, pl, t32, z32, fnbx, fnby,
                    fper, fwp, dout, arg, din, (deep_trig() >> 2) & 1);
  if (NC == 4)
    return launch_k(conv3w_pool_bwd_kernel<4>, grid, dim3(256), 0, st, gi, go, pt, pl, t32, z32, fnbx, fnby,
                    fper, fwp, dout, arg, din, (deep_trig() >> 2) & 1);
  if (NC == 8)
    return launch_k(conv3w_pool_bwd_kernel<8>, grid, dim3(256), 0, st, gi, go, pt, pl, t32, z32, fnbx, fnby,
                    fper, fwp, dout, arg, din, (deep_trig() >> 2) & 1);
  return SEED_E_UNSUPPORTED;
}

}  // namespace seed
