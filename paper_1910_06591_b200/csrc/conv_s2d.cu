// conv_s2d.cu — see conv_s2d.cuh.  Atari-shallow torso (C14; P:591 network
// table, SURVEY.md §8(a) H1 forward / H9 backward) on tcgen05 with TMA bulk
// slabs.
#include <algorithm>
#include "conv_s2d.cuh"
#include "win_engine.cuh"

namespace seed {

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

__device__ void Conv2DgradS2dEpi::pre(int64_t p, uint4 (&pr)[PRE]) const {
  const uint8_t* srow = S1 + p * 128;
#pragma unroll
  for (int j = 0; j < 8; ++j) pr[j] = __ldg(reinterpret_cast<const uint4*>(srow + (swz_chunk(p, 128, j) << 4)));
}

__device__ void Conv2DgradS2dEpi::store(int64_t p, float (&v)[N], const uint4 (&pr)[PRE]) const {
  uint32_t f, rem, Y, X;
  P2.divmod((uint32_t)p, f, rem);
  W2.divmod(rem, Y, X);
  // ReLU mask of act1 (S1 row p, 64 channels = 4 conv1 pixels x 16; prefetched)
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint4 u = pr[j];
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
// groups a = 0, 1 (window rows a*Ws), atoms b = 0, 1 (window columns, LBO = one
// 128-byte row): accumulator row i = b*64 + s2d channel
__device__ void WinWgradFinish::weight(int a, int i, int n, float t) const {
  const int b = i >> 6, ch = i & 63;
  const int ky1 = ch / (g.s * g.C), kx1 = (ch / g.C) % g.s, c = ch % g.C;
  const int K = 2 * g.s, ky = g.s * a + ky1, kx = g.s * b + kx1;
  g_w[(((size_t)n * K + ky) * K + kx) * g.C + c] = t * scale;
}

size_t win_wgrad_part_bytes(int64_t M, int N) { return win3_wgrad_part_bytes(M, N, 2); }

// Both window rows in one MMA (win3_wgrad_kernel with 2 B atoms): D[(b, ch)][(j, n)] =
// sum_h S[h + b][ch] dY[h - Ws + j*Ws][n], window row a = 1 - j; the bias gradient
// from the epilogue warps' column sums of dY (B atom 1 = dY[h])
struct S2dFin2 {
  WinWgradFinish f;
  int CO;
  __device__ void weight3(int i, int n, float t) const { f.weight(1 - n / CO, i, n % CO, t); }
  __device__ void bias(int n, float t) const { f.bias(n, t); }
};
static Win3WgradArgs s2d_wgrad3_args(const uint8_t* src, int64_t rows, const uint8_t* dy, int wsp,
                                     float* part) {
  Win3WgradArgs a{};
  a.trig = 1;
  a.X = src; a.dy = dy; a.M = rows; a.part = part;
  a.boff = -wsp; a.bstride = wsp;
  return a;
}


// ------------------------------------------------------------------ obs -> S0
// 4 threads per S0 row, one obs row each: 16 input bytes (4 pixels x 4 channels,
// one load; a warp reads 128 contiguous bytes of each of 4 obs rows) -> output
// chunks 2r, 2r+1 of the row (a warp writes 8 whole rows, 1 KB contiguous)
__global__ void s2d_obs_kernel(int64_t nrows, FastDiv P, FastDiv Wd, int H, int W,
                               const uint8_t* __restrict__ obs, uint8_t* __restrict__ S0) {
  pdl_wait_trig();
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t g = t >> 2;
  if (g >= nrows) return;
  const int r = (int)(t & 3);
  uint32_t f, rem, Y, X;
  P.divmod((uint32_t)g, f, rem);
  Wd.divmod(rem, Y, X);
  const uint4 u = __ldg(reinterpret_cast<const uint4*>(obs + (((size_t)f * H + 4 * Y + r) * W + 4 * X) * 4));
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
  uint32_t o[8];
#pragma unroll
  for (int k = 0; k < 4; ++k) {   // bytes -> bf16 (exact): the float's high half
    const uint32_t b0 = w[k] & 0xFF, b1 = (w[k] >> 8) & 0xFF, b2 = (w[k] >> 16) & 0xFF, b3 = w[k] >> 24;
    o[2 * k] = (__float_as_uint((float)b0) >> 16) | (__float_as_uint((float)b1) & 0xFFFF0000u);
    o[2 * k + 1] = (__float_as_uint((float)b2) >> 16) | (__float_as_uint((float)b3) & 0xFFFF0000u);
  }
  uint8_t* row = S0 + g * 128;
  *reinterpret_cast<uint4*>(row + (swz_chunk(g, 128, 2 * r) << 4)) = make_uint4(o[0], o[1], o[2], o[3]);
  *reinterpret_cast<uint4*>(row + (swz_chunk(g, 128, 2 * r + 1) << 4)) = make_uint4(o[4], o[5], o[6], o[7]);
}

seed_status s2d_obs(const uint8_t* obs, int64_t F, int H, int W, uint8_t* S0, cudaStream_t st) {
  const int Hs = H / 4, Ws = W / 4;
  const int64_t n = F * Hs * Ws;
  if (n == 0) return SEED_OK;
  return launch_k(s2d_obs_kernel, dim3((unsigned)((n * 4 + 255) / 256)), dim3(256), 0, st, n,
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
  a.trig = 1;
  a.src = S0; a.src_rows = sg.rows1(F); a.M = sg.rows1(F);
  a.off[0] = 0; a.off[1] = 1; a.off[2] = g.Ws; a.off[3] = g.Ws + 1;
  a.wimg = reinterpret_cast<const uint8_t*>(w1img);
  Conv1S2dEpi e{};
  e.bias = b1; e.S1 = S1; e.P1 = FastDiv(g.P); e.W1 = FastDiv(g.Ws);
  e.Ho = g.Ho; e.Wo = g.Wo; e.W2s = sg.g2.Ws; e.P2 = sg.g2.P;
  return launch_win_conv<Conv1S2dEpi, 128, 4>(a, e, st);
}

seed_status shallow_s2d_conv2(const ShallowS2d& sg, int64_t F, const uint8_t* S1, const bf16* w2img,
                              const float* b2, bf16* act2, uint8_t* dY2z, cudaStream_t st) {
  const S2dGeo& g = sg.g2;
  WinConvArgs a{};
  a.trig = 1;
  a.src = S1; a.src_rows = sg.rows2(F); a.M = sg.rows2(F);
  a.off[0] = 0; a.off[1] = 1; a.off[2] = g.Ws; a.off[3] = g.Ws + 1;
  a.wimg = reinterpret_cast<const uint8_t*>(w2img);
  Conv2S2dEpi e{};
  e.bias = b2; e.act2 = act2; e.dY2z = dY2z; e.P2 = FastDiv(g.P); e.W2 = FastDiv(g.Ws);
  e.Ho = g.Ho; e.Wo = g.Wo; e.fc_in = sg.fc_in;
  return launch_win_conv<Conv2S2dEpi, 128, 4>(a, e, st);
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
  const Win3WgradArgs a = s2d_wgrad3_args(S1, sg.rows2(F), dY2, sg.g2.Ws, part);
  S2dFin2 f{};
  f.f.g = sg.g2; f.f.scale = 1.f; f.f.g_w = g_w2; f.f.g_b = g_b2; f.CO = 32;
  return launch_win3_wgrad<32, 128, S2dFin2, 2>(a, f, true, st);
}

seed_status shallow_s2d_conv2_dgrad(const ShallowS2d& sg, int64_t F, const uint8_t* dY2,
                                    const bf16* w2dg_img, const uint8_t* S1, uint8_t* dY1,
                                    cudaStream_t st) {
  const S2dGeo& g = sg.g2;
  WinConvArgs a{};
  a.trig = 1;
  a.src = dY2; a.src_rows = sg.rows2(F); a.M = sg.rows2(F);
  a.off[0] = 0; a.off[1] = -1; a.off[2] = -g.Ws; a.off[3] = -g.Ws - 1;
  a.wimg = reinterpret_cast<const uint8_t*>(w2dg_img);
  Conv2DgradS2dEpi e{};
  e.S1 = S1; e.dY1 = dY1; e.P2 = FastDiv(g.P); e.W2 = FastDiv(g.Ws); e.H2s = g.Hs; e.W2s = g.Ws;
  e.P1 = sg.g1.P; e.W1s = sg.g1.Ws; e.H1s = sg.g1.Hs;
  return launch_win_conv<Conv2DgradS2dEpi, 64, 4>(a, e, st);
}

seed_status shallow_s2d_conv1_wgrad(const ShallowS2d& sg, int64_t F, const uint8_t* S0,
                                    const uint8_t* dY1, float* part, float* g_w1, float* g_b1,
                                    cudaStream_t st) {
  const Win3WgradArgs a = s2d_wgrad3_args(S0, sg.rows1(F), dY1, sg.g1.Ws, part);
  S2dFin2 f{};
  f.f.g = sg.g1; f.f.scale = 1.f / 255.f; f.f.g_w = g_w1; f.f.g_b = g_b1; f.CO = 16;
  return launch_win3_wgrad<16, 128, S2dFin2, 2>(a, f, true, st);
}

}  // namespace seed
