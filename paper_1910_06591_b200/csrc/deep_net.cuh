// deep_net.cuh — the IMPALA-deep torso (configs[2] DMLab, configs[3] GRF; C14)
// as tcgen05 GEMM Problems + max-pool kernels.
//
// Section s: conv3x3 'same' (cin -> ch) -> maxpool 3x3/s2 'same' -> 2 x residual
// [h + conv(relu(conv(relu(h))))]; torso output relu(h) feeds the FC layer.
// Every 3x3 conv is an implicit GEMM with k = (ky, kx, c) and zero padding
// (nullptr chunks).  Activations bf16 NHWC; rows m = (f, y, x).
#pragma once
#include "shallow_net.cuh"

namespace seed {

struct Conv3Geo {
  int H, W;          // spatial (same in and out)
  int cin, cout;     // cin = padded input channels (multiple of 8)
  FastDiv hw, w;     // H*W, W
};

__device__ __forceinline__ void split_pix(const Conv3Geo& g, int m, int& f, int& y, int& x) {
  uint32_t uf, p, uy, ux;
  g.hw.divmod((uint32_t)m, uf, p);
  g.w.divmod(p, uy, ux);
  f = (int)uf; y = (int)uy; x = (int)ux;
}

enum { C3_PLAIN = 0, C3_RELU = 1, C3_RES = 2 };

// forward: out[m][n] = sum_{ky,kx,c} in[f][y+ky-1][x+kx-1][c] w[n][ky][kx][c] + b[n]
//   C3_PLAIN: out = acc * in_scale + b        (section conv; in_scale = 1/255 on obs)
//   C3_RELU:  out = relu(acc + b)              (u1 = relu(t0))
//   C3_RES:   out = res + acc + b, outr = relu(out)   (h <- h + t1)
template <int MODE>
struct Conv3Fwd {
  static constexpr bool ASYNC = true;
  const void* dummy = k_ones_chunk;
  static constexpr bool A_MN = false, B_MN = false;
  int M, N, K, kb_per_split;
  Conv3Geo g;
  int cshift;            // log2(cin)
  float in_scale;
  const bf16* in;
  const bf16* w;         // [cout][9*cin]
  const float* bias;
  const bf16* res;       // C3_RES: h_in [M][cout]
  bf16* out;             // [M][cout]
  bf16* outr;            // C3_RES: relu(out)
  __device__ const void* ptr_a(int m, int k) const {
    int f, y, x;
    split_pix(g, m, f, y, x);
    const int t = k >> cshift, c0 = k & (g.cin - 1);
    const int ky = t / 3, kx = t - 3 * ky;
    const int iy = y + ky - 1, ix = x + kx - 1;
    if (iy < 0 || ix < 0 || iy >= g.H || ix >= g.W) return nullptr;
    return in + (((size_t)f * g.H + iy) * g.W + ix) * g.cin + c0;
  }
  __device__ const void* ptr_b(int n, int k) const { return w + (size_t)n * K + k; }
  __device__ float post(int m, int n, float v) const {
    v = v * in_scale + bias[n];
    if (MODE == C3_RELU) v = fmaxf(v, 0.f);
    if (MODE == C3_RES) v += bf2f(res[(size_t)m * N + n]);
    return v;
  }
  __device__ void store(int m, int n, float v) const {
    const float o = post(m, n, v);
    out[(size_t)m * N + n] = to_bf(o);
    if (MODE == C3_RES) outr[(size_t)m * N + n] = to_bf(fmaxf(bf2f(to_bf(o)), 0.f));
  }
  static constexpr bool VEC_STORE = true;
  __device__ void store16(int m, int n0, float (&v)[16]) const {
    float r[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      v[q] = v[q] * in_scale + bias[n0 + q];
      if (MODE == C3_RELU) v[q] = fmaxf(v[q], 0.f);
    }
    if (MODE == C3_RES) {
      const uint4* rp = reinterpret_cast<const uint4*>(res + (size_t)m * N + n0);
      const uint4 a = rp[0], b = rp[1];
      const uint32_t wv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        v[2 * q] += bf16_lo(wv[q]);
        v[2 * q + 1] += bf16_hi(wv[q]);
      }
    }
    st_bf16x16(out + (size_t)m * N + n0, v);
    if (MODE == C3_RES) {
#pragma unroll
      for (int q = 0; q < 16; ++q) r[q] = fmaxf(bf2f(to_bf(v[q])), 0.f);
      st_bf16x16(outr + (size_t)m * N + n0, r);
    }
  }
};

enum { D3_PLAIN = 0, D3_MASK = 1, D3_RES = 2 };

// data gradient: dX[m][ci] = sum_{ky,kx,co} dY[f][y+1-ky][x+1-kx][co] w[co][ky][kx][ci]
//   D3_PLAIN: dX = acc;  D3_MASK: dX = acc * (mask > 0);  D3_RES: dX = dres + acc * (mask > 0)
template <int MODE>
struct Conv3Dgrad {
  static constexpr bool ASYNC = true;
  const void* dummy = k_ones_chunk;
  static constexpr bool A_MN = false, B_MN = false;
  int M, N, K, kb_per_split;
  Conv3Geo g;            // cin = this layer's cout (the dY channels), cout = ci
  int cshift;
  const bf16* dY;        // [M][g.cin]
  const bf16* wdg;       // [ci][3][3][co]
  const bf16* mask;      // [M][N]
  const bf16* dres;      // [M][N]
  bf16* dX;              // [M][N]
  __device__ const void* ptr_a(int m, int k) const {
    int f, y, x;
    split_pix(g, m, f, y, x);
    const int t = k >> cshift, c0 = k & (g.cin - 1);
    const int ky = t / 3, kx = t - 3 * ky;
    const int iy = y + 1 - ky, ix = x + 1 - kx;
    if (iy < 0 || ix < 0 || iy >= g.H || ix >= g.W) return nullptr;
    return dY + (((size_t)f * g.H + iy) * g.W + ix) * g.cin + c0;
  }
  __device__ const void* ptr_b(int n, int k) const { return wdg + (size_t)n * K + k; }
  __device__ void store(int m, int n, float v) const {
    const size_t i = (size_t)m * N + n;
    if (MODE != D3_PLAIN && !(bf2f(mask[i]) > 0.f)) v = 0.f;
    if (MODE == D3_RES) v += bf2f(dres[i]);
    dX[i] = to_bf(v);
  }
  static constexpr bool VEC_STORE = true;
  __device__ void store16(int m, int n0, float (&v)[16]) const {
    const size_t i = (size_t)m * N + n0;
    if (MODE != D3_PLAIN) relu_mask16(mask + i, v);
    if (MODE == D3_RES) {
      const uint4* rp = reinterpret_cast<const uint4*>(dres + i);
      const uint4 a = rp[0], b = rp[1];
      const uint32_t wv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        v[2 * q] += bf16_lo(wv[q]);
        v[2 * q + 1] += bf16_hi(wv[q]);
      }
    }
    st_bf16x16(dX + i, v);
  }
};

// weight gradient: dW^T[kin = (ky,kx,c)][co] = scale * sum_rows im2col(X)[row][kin] dY[row][co];
// written to the fp32 layout [co][3][3][creal] (padded channels c >= creal dropped)
struct Conv3Wgrad {
  static constexpr bool ASYNC = true;
  const void* dummy = k_ones_chunk;
  static constexpr bool A_MN = true, B_MN = true;
  int M, N, K, kb_per_split;
  Conv3Geo g;            // cin = padded input channels
  int cshift, creal;
  float scale;
  const bf16* X;         // [rows][cin]
  const bf16* dY;        // [rows][N]
  float* g_w;
  __device__ const void* ptr_a(int row, int m8) const {
    int f, y, x;
    split_pix(g, row, f, y, x);
    const int t = m8 >> cshift, c0 = m8 & (g.cin - 1);
    const int ky = t / 3, kx = t - 3 * ky;
    const int iy = y + ky - 1, ix = x + kx - 1;
    if (iy < 0 || ix < 0 || iy >= g.H || ix >= g.W) return nullptr;
    return X + (((size_t)f * g.H + iy) * g.W + ix) * g.cin + c0;
  }
  __device__ const void* ptr_b(int row, int n8) const { return dY + (size_t)row * N + n8; }
  __device__ void store(int m, int n, float v) const {
    const int t = m >> cshift, c = m & (g.cin - 1);
    if (c >= creal) return;
    g_w[((size_t)n * 9 + t) * creal + c] = v * scale;
  }
};

// max-pool 3x3 / stride 2 / TF 'same' (top/left pad = floor(total/2)), padding
// acts as -inf; argmax = first maximum in (ky, kx) row-major order.  Writes the
// pooled value, its relu copy and the window argmax (0..8).
__global__ void maxpool_fwd_kernel(int64_t n, int H, int W, int H2, int W2, int C, int pt, int pl,
                                   const bf16* __restrict__ in, bf16* __restrict__ out,
                                   bf16* __restrict__ outr, uint8_t* __restrict__ arg);
// gradient gather: dIn[f][y][x][c] = sum over windows whose argmax is (y, x)
__global__ void maxpool_bwd_kernel(int64_t n, int H, int W, int H2, int W2, int C, int pt, int pl,
                                   const bf16* __restrict__ dout, const uint8_t* __restrict__ arg,
                                   bf16* __restrict__ din);
// obs uint8 [N][H][W][C] -> bf16 [N][H][W][Cp] (channels zero-padded to Cp)
__global__ void obs_to_bf16_pad_kernel(int64_t npix, int C, int Cp, const uint8_t* __restrict__ obs,
                                       bf16* __restrict__ out);

}  // namespace seed
