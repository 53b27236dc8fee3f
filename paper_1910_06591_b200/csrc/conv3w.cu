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

// ------------------------------------------------------------------ epilogues
template <int MODE, int NN>
struct W3FwdEpi {
  static constexpr int N = NN;
  static constexpr int RB = 2 * NN;
  PadGeo g;
  float in_scale;
  const float* bias;
  const uint8_t* res;
  uint8_t* out;
  uint8_t* outr;
  bf16* dense;
  __device__ void store(int64_t m, float (&v)[N]) const {
    int f, y, x;
    if (!g.split(m, f, y, x)) {
      if (MODE != W3_PLAIN) {
        const uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int j = 0; j < N / 8; ++j) {
          *chunk_at(out, m, RB, j) = z;
          if (MODE == W3_RES) *chunk_at(outr, m, RB, j) = z;
        }
      }
      return;
    }
#pragma unroll
    for (int q = 0; q < N; ++q) {
      v[q] = v[q] * in_scale + __ldg(bias + q);
      if (MODE == W3_RELU) v[q] = fmaxf(v[q], 0.f);
    }
    if (MODE == W3_RES) {
#pragma unroll
      for (int j = 0; j < N / 8; ++j) {
        float r[8];
        unpack8(*chunk_at(res, m, RB, j), r);
#pragma unroll
        for (int k = 0; k < 8; ++k) v[8 * j + k] += r[k];
      }
    }
#pragma unroll
    for (int j = 0; j < N / 8; ++j) *chunk_at(out, m, RB, j) = pack8(v + 8 * j);
    if (MODE == W3_RES) {
      float r[N];
#pragma unroll
      for (int q = 0; q < N; ++q) r[q] = fmaxf(__bfloat162float(__float2bfloat16_rn(v[q])), 0.f);
#pragma unroll
      for (int j = 0; j < N / 8; ++j) *chunk_at(outr, m, RB, j) = pack8(r + 8 * j);
      if (dense) {
        uint4* d = reinterpret_cast<uint4*>(dense + ((int64_t)f * g.H * g.W + (int64_t)y * g.W + x) * N);
#pragma unroll
        for (int j = 0; j < N / 8; ++j) d[j] = pack8(r + 8 * j);
      }
    }
  }
};

template <int MODE, int NN>
struct W3DgradEpi {
  static constexpr int N = NN;
  static constexpr int RB = 2 * NN;
  PadGeo g;
  const uint8_t* mask;
  const uint8_t* dres;
  uint8_t* dX;
  __device__ void store(int64_t m, float (&v)[N]) const {
    int f, y, x;
    if (!g.split(m, f, y, x)) {
      const uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int j = 0; j < N / 8; ++j) *chunk_at(dX, m, RB, j) = z;
      return;
    }
    if (MODE != D3W_PLAIN) {
#pragma unroll
      for (int j = 0; j < N / 8; ++j) {
        float mk[8];
        unpack8(*chunk_at(mask, m, RB, j), mk);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (!(mk[k] > 0.f)) v[8 * j + k] = 0.f;
      }
    }
    if (MODE == D3W_RES) {
#pragma unroll
      for (int j = 0; j < N / 8; ++j) {
        float r[8];
        unpack8(*chunk_at(dres, m, RB, j), r);
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
template <int MODE, int N, int RB, int NW>
static seed_status fwd_t(const Conv3wFwd& a, cudaStream_t st) {
  WinConvArgs w{};
  w.src = a.in; w.src_rows = a.rows; w.M = a.rows;
  w.wimg = reinterpret_cast<const uint8_t*>(a.wimg);
  for (int k = 0; k < NW; ++k)
    w.off[k] = NW == 9 ? ((k / 3) - 1) * a.g.Wp + (k % 3) - 1 : (k - 1) * a.g.Wp;
  W3FwdEpi<MODE, N> e{};
  e.g = a.g; e.in_scale = a.in_scale; e.bias = a.bias; e.res = a.res; e.out = a.out;
  e.outr = a.outr; e.dense = a.dense;
  return launch_win_conv<W3FwdEpi<MODE, N>, RB, NW>(w, e, st);
}

template <int MODE>
static seed_status fwd_mode(const Conv3wFwd& a, cudaStream_t st) {
  if (a.xim) {
    if (a.ch == 16 && a.cin_p == 16) return fwd_t<MODE, 16, 32, 3>(a, st);
    return SEED_E_UNSUPPORTED;
  }
  if (a.ch == 16 && a.cin_p == 16) return fwd_t<MODE, 16, 32, 9>(a, st);
  if (a.ch == 32 && a.cin_p == 16) return fwd_t<MODE, 32, 32, 9>(a, st);
  if (a.ch == 16 && a.cin_p == 32) return fwd_t<MODE, 16, 64, 9>(a, st);
  if (a.ch == 32 && a.cin_p == 32) return fwd_t<MODE, 32, 64, 9>(a, st);
  return SEED_E_UNSUPPORTED;
}

seed_status conv3w_forward(const Conv3wFwd& a, cudaStream_t st) {
  if (a.mode == W3_PLAIN) return fwd_mode<W3_PLAIN>(a, st);
  if (a.mode == W3_RELU && !a.xim) return fwd_mode<W3_RELU>(a, st);
  if (a.mode == W3_RES && !a.xim) return fwd_mode<W3_RES>(a, st);
  return SEED_E_UNSUPPORTED;
}

// ------------------------------------------------------------------ data gradient
template <int MODE, int N, int RB>
static seed_status dgrad_t(const Conv3wDgrad& a, cudaStream_t st) {
  WinConvArgs w{};
  w.src = a.dY; w.src_rows = a.rows; w.M = a.rows;
  w.wimg = reinterpret_cast<const uint8_t*>(a.wimg);
  for (int k = 0; k < 9; ++k) w.off[k] = -(((k / 3) - 1) * a.g.Wp + (k % 3) - 1);
  W3DgradEpi<MODE, N> e{};
  e.g = a.g; e.mask = a.mask; e.dres = a.dres; e.dX = a.dX;
  return launch_win_conv<W3DgradEpi<MODE, N>, RB, 9>(w, e, st);
}

template <int MODE>
static seed_status dgrad_mode(const Conv3wDgrad& a, cudaStream_t st) {
  if (a.cin == 16 && a.ch == 16) return dgrad_t<MODE, 16, 32>(a, st);
  if (a.cin == 16 && a.ch == 32) return dgrad_t<MODE, 16, 64>(a, st);
  if (a.cin == 32 && a.ch == 16) return dgrad_t<MODE, 32, 32>(a, st);
  if (a.cin == 32 && a.ch == 32) return dgrad_t<MODE, 32, 64>(a, st);
  return SEED_E_UNSUPPORTED;
}

seed_status conv3w_dgrad(const Conv3wDgrad& a, cudaStream_t st) {
  if (a.mode == D3W_PLAIN) return dgrad_mode<D3W_PLAIN>(a, st);
  if (a.mode == D3W_MASK) return dgrad_mode<D3W_MASK>(a, st);
  if (a.mode == D3W_RES) return dgrad_mode<D3W_RES>(a, st);
  return SEED_E_UNSUPPORTED;
}

// ------------------------------------------------------------------ weight gradient
static WinWgradArgs wgrad_args(const Conv3wWgrad& a) {
  WinWgradArgs w{};
  w.src = a.X; w.src_rows = a.rows; w.dy = a.dY; w.M = a.rows; w.part = a.part;
  if (a.xim) {
    w.ngroup = 1; w.goff[0] = -a.g.Wp; w.astride = a.g.Wp;
  } else {
    w.ngroup = 3;
    for (int k = 0; k < 3; ++k) w.goff[k] = (k - 1) * a.g.Wp - 1;
    w.astride = 1;
  }
  return w;
}

size_t conv3w_wgrad_part_bytes(int64_t rows, int ch, bool xim) {
  return win_wgrad_part_bytes_g(rows, ch, xim ? 1 : 3);
}

seed_status conv3w_wgrad(const Conv3wWgrad& a, cudaStream_t st) {
  const WinWgradArgs w = wgrad_args(a);
  W3Fin f{};
  f.xim = a.xim ? 1 : 0; f.Cp = a.cin_p; f.CI = a.cin; f.scale = a.scale; f.g_w = a.g_w;
  f.g_b = a.g_b;
  if (a.ch == 16 && a.cin_p == 16) return launch_win_wgrad<16, 32>(w, f, st);
  if (a.ch == 32 && a.cin_p == 16) return launch_win_wgrad<32, 32>(w, f, st);
  if (a.ch == 16 && a.cin_p == 32) return launch_win_wgrad<16, 64>(w, f, st);
  if (a.ch == 32 && a.cin_p == 32) return launch_win_wgrad<32, 64>(w, f, st);
  return SEED_E_UNSUPPORTED;
}

// ------------------------------------------------------------------ obs conversion
// one thread per (row, 16-byte chunk of 8 channels)
__global__ void conv3_obs_kernel(int64_t n, PadGeo g, int C, int Cp, int xim,
                                 const uint8_t* __restrict__ obs, uint8_t* __restrict__ X0) {
  pdl_wait();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int NC = Cp / 8, RB = 2 * Cp;
  const int j = (int)(i % NC);
  const int64_t m = i / NC;
  int f, y, x;
  float v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = 0.f;
  if (g.split(m, f, y, x)) {
    const uint8_t* fr = obs + (size_t)f * g.H * g.W * C;
    if (!xim && C % 8 == 0) {
      const uint2 u = __ldg(reinterpret_cast<const uint2*>(fr + ((size_t)y * g.W + x) * C + 8 * j));
      const uint32_t w[2] = {u.x, u.y};
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = (float)((w[k >> 2] >> (8 * (k & 3))) & 0xFF);
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int ch = 8 * j + k;
        if (!xim) {
          if (ch < C) v[k] = (float)__ldg(fr + ((size_t)y * g.W + x) * C + ch);
        } else if (ch < 3 * C) {
          const int kx = ch / C, c = ch % C, xx = x + kx - 1;
          if (xx >= 0 && xx < g.W) v[k] = (float)__ldg(fr + ((size_t)y * g.W + xx) * C + c);
        }
      }
    }
  }
  *chunk_at(X0, m, RB, j) = pack8(v);
}

seed_status conv3_obs(const uint8_t* obs, int64_t F, const PadGeo& g, int C, int Cp, bool xim,
                      uint8_t* X0, cudaStream_t st) {
  const int64_t n = F * g.P * (Cp / 8);
  if (n == 0) return SEED_OK;
  return launch_k(conv3_obs_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, n, g, C, Cp,
                  xim ? 1 : 0, obs, X0);
}

// ------------------------------------------------------------------ max-pool
__global__ void conv3w_pool_fwd_kernel(int64_t n, PadGeo gi, PadGeo go, int C, int pt, int pl,
                                       const uint8_t* __restrict__ conv, uint8_t* __restrict__ h0,
                                       uint8_t* __restrict__ hr0, uint8_t* __restrict__ arg) {
  pdl_wait();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int NC = C / 8, RB = 2 * C;
  const int j = (int)(i % NC);
  const int64_t m = i / NC;
  int f, oy, ox;
  if (!go.split(m, f, oy, ox)) {
    const uint4 z = make_uint4(0, 0, 0, 0);
    *chunk_at(h0, m, RB, j) = z;
    *chunk_at(hr0, m, RB, j) = z;
    return;
  }
  float best[8];
  uint32_t barg[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) { best[k] = -INFINITY; barg[k] = 0; }
#pragma unroll
  for (int ky = 0; ky < 3; ++ky) {
    const int y = oy * 2 - pt + ky;
    if (y < 0 || y >= gi.H) continue;
#pragma unroll
    for (int kx = 0; kx < 3; ++kx) {
      const int x = ox * 2 - pl + kx;
      if (x < 0 || x >= gi.W) continue;
      float v[8];
      unpack8(__ldg(chunk_at(conv, gi.row(f, y, x), RB, j)), v);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (v[k] > best[k]) {   // strict: the first maximum in (ky, kx) order wins
          best[k] = v[k];
          barg[k] = ky * 3 + kx;
        }
    }
  }
  float r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = fmaxf(best[k], 0.f);
  *chunk_at(h0, m, RB, j) = pack8(best);
  *chunk_at(hr0, m, RB, j) = pack8(r);
  uint2 a;
  a.x = barg[0] | (barg[1] << 8) | (barg[2] << 16) | (barg[3] << 24);
  a.y = barg[4] | (barg[5] << 8) | (barg[6] << 16) | (barg[7] << 24);
  *reinterpret_cast<uint2*>(arg + m * C + 8 * j) = a;
}

__global__ void conv3w_pool_bwd_kernel(int64_t n, PadGeo gi, PadGeo go, int C, int pt, int pl,
                                       const uint8_t* __restrict__ dout,
                                       const uint8_t* __restrict__ arg, uint8_t* __restrict__ din) {
  pdl_wait();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int NC = C / 8, RB = 2 * C;
  const int j = (int)(i % NC);
  const int64_t m = i / NC;
  int f, y, x;
  float s[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) s[k] = 0.f;
  if (gi.split(m, f, y, x)) {
    // windows (oy, ox) with oy*2 - pt <= y <= oy*2 - pt + 2, in ascending order
    const int oy_hi = (y + pt) >> 1, ox_hi = (x + pl) >> 1;
#pragma unroll
    for (int dy = 0; dy < 2; ++dy) {
      const int oy = oy_hi - 1 + dy;
      const int ky = y - (oy * 2 - pt);
      if (oy < 0 || oy >= go.H || ky < 0 || ky > 2) continue;
#pragma unroll
      for (int dx = 0; dx < 2; ++dx) {
        const int ox = ox_hi - 1 + dx;
        const int kx = x - (ox * 2 - pl);
        if (ox < 0 || ox >= go.W || kx < 0 || kx > 2) continue;
        const int64_t o = go.row(f, oy, ox);
        const uint2 a = __ldg(reinterpret_cast<const uint2*>(arg + o * C + 8 * j));
        float d[8];
        unpack8(__ldg(chunk_at(dout, o, RB, j)), d);
        const uint32_t want = (uint32_t)(ky * 3 + kx);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t ak = ((k < 4 ? a.x : a.y) >> (8 * (k & 3))) & 0xFF;
          if (ak == want) s[k] += d[k];
        }
      }
    }
  }
  *chunk_at(din, m, RB, j) = pack8(s);
}

seed_status conv3w_pool_fwd(int64_t F, const PadGeo& gi, const PadGeo& go, int C, int pt, int pl,
                            const uint8_t* conv, uint8_t* h0, uint8_t* hr0, uint8_t* arg,
                            cudaStream_t st) {
  const int64_t n = F * go.P * (C / 8);
  if (n == 0) return SEED_OK;
  return launch_k(conv3w_pool_fwd_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, n,
                  gi, go, C, pt, pl, conv, h0, hr0, arg);
}

seed_status conv3w_pool_bwd(int64_t F, const PadGeo& gi, const PadGeo& go, int C, int pt, int pl,
                            const uint8_t* dout, const uint8_t* arg, uint8_t* din,
                            cudaStream_t st) {
  const int64_t n = F * gi.P * (C / 8);
  if (n == 0) return SEED_OK;
  return launch_k(conv3w_pool_bwd_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, n,
                  gi, go, C, pt, pl, dout, arg, din);
}

}  // namespace seed
