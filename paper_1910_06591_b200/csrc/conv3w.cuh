// conv3w.cuh — the IMPALA-deep torso (configs[2] DMLab, configs[3] GRF; C14)
// as shifted-window GEMMs on tcgen05 (win_engine.cuh).
//
// Section s: conv3x3 'same' (cin -> ch) -> maxpool 3x3/s2 'same' -> 2 x residual
// [h + conv(relu(conv(relu(h))))]; relu(h) of the last section feeds the FC.
//
// Layout ("padded row space"): an activation at resolution H x W is stored as
// rows g = f*P + Y*Wp + X with Wp = W + 2, P = (H + 2)*Wp, pixel (y, x) at
// (Y, X) = (y + 1, x + 1); border rows hold zeros, so the 'same' zero padding
// of a 3x3 conv is read from memory.  A row is the pixel's C channels in bf16
// (RB = 2C = 32 or 64 bytes), stored pre-swizzled (swz_chunk).  A 3x3 conv is
// then 9 window GEMMs over the same rows at offsets (ky-1)*Wp + (kx-1)
// (forward), their negatives with the transposed weights (data gradient), and
// 3 groups (ky) x atoms (kx, LBO = one row) of the MN-major weight-gradient
// engine.  Section 0 with C <= 5 input channels (DMLab RGB) uses an x-im2col
// input instead: row channels (kx, c) (3C <= 16, zero-padded to 16), so the
// conv is 3 windows at offsets (ky-1)*Wp and its weight gradient 1 group whose
// atoms are the 3 ky rows (LBO = Wp rows).
// Epilogues write zeros on border rows (the outputs are the next conv's
// inputs); the max-pool kernels work on 16-byte chunks of 8 channels.
#pragma once
#include "common.cuh"
#include "win_engine.cuh"

namespace seed {

typedef __nv_bfloat16 bf16;

struct PadGeo {
  int H, W, Wp, P;       // interior size, padded row width, rows per frame
  FastDiv fP, fW;        // P, Wp
  static PadGeo make(int H, int W) {
    PadGeo g;
    g.H = H; g.W = W; g.Wp = W + 2; g.P = (H + 2) * (W + 2);
    g.fP = FastDiv((uint32_t)g.P); g.fW = FastDiv((uint32_t)g.Wp);
    return g;
  }
  // frame and unpadded pixel of row m; false on border rows
  __device__ __forceinline__ bool split(int64_t m, int& f, int& y, int& x) const {
    uint32_t uf, r, Y, X;
    fP.divmod((uint32_t)m, uf, r);
    fW.divmod(r, Y, X);
    f = (int)uf; y = (int)Y - 1; x = (int)X - 1;
    return y >= 0 && x >= 0 && y < H && x < W;
  }
  __host__ __device__ int64_t row(int64_t f, int y, int x) const {
    return f * P + (int64_t)(y + 1) * Wp + (x + 1);
  }
};

// obs uint8 [F][H][W][C] -> section-0 input rows (exact 0..255 in bf16):
//   xim = 0: channels c < C of 16 or 32 (Cp);  xim = 1: channel kx*C + c = pixel x+kx-1
seed_status conv3_obs(const uint8_t* obs, int64_t F, const PadGeo& g, int C, int Cp, bool xim,
                      uint8_t* X0, cudaStream_t st);

enum { W3_PLAIN = 0, W3_RELU = 1, W3_RES = 2, W3_PART = 3 };    // forward epilogues
enum { D3W_PLAIN = 0, D3W_MASK = 1, D3W_RES = 2, D3W_PART = 3 };  // data-gradient epilogues

// 128-channel tensors (the DMLab 4x torso) are stored as two 64-channel planes,
// each a padded row space of 128-byte rows (plane q at base + q * rows * 128); a
// 3x3 conv between such tensors is the sum over input planes p of the 64 -> 64
// convs into each output plane q.  The first input plane's conv stores its fp32
// accumulator (W3_PART / D3W_PART, `part_out`, [rows][64]); the second adds it
// (`part_in`) before its epilogue — one fp32 sum, one bf16 rounding, as a single
// conv over 128 input channels.

// Forward 3x3 conv (9 windows, or 3 for the x-im2col section-0 input).
//   W3_PLAIN: out = acc*in_scale + b  (section conv; border rows not written)
//   W3_RELU:  out = relu(acc + b)
//   W3_RES:   out = res + acc + b, outr (nullable) = relu(out), dense (nullable) =
//             relu(out) as [f][(y*W + x)*dense_ct + dense_off + c] (the FC input;
//             dense_ct 0 = ch)
//   W3_PART:  part_out[g][c] = acc*in_scale (fp32, every row); other modes add
//             part_in[g][c] (nullable) to acc*in_scale before the bias
// xf (win_engine.cuh): XF_RELU = the conv reads relu(in) (relu applied to the slab in
// shared memory); XF_U8 = `in` is ignored and the input rows are the uint8 obs
// [F][H][W][16] `obs_u8` expanded in shared memory (section 0 of the GRF net)
struct Conv3wFwd {
  int mode, cin_p, ch;    // cin_p = input row channels (16 / 32); ch = 16 / 32
  bool xim;
  int xf;
  const uint8_t* obs_u8;
  PadGeo g;
  int64_t rows;           // F*P
  float in_scale;
  const uint8_t* in;      // input rows (cin_p channels)
  const bf16* wimg;       // window image [NW][ch][cin_p] (pre-swizzled)
  const float* bias;
  const uint8_t* res;
  uint8_t* out;
  uint8_t* outr;
  bf16* dense;
  int dense_ct, dense_off;
  float* part_out;
  const float* part_in;
};
seed_status conv3w_forward(const Conv3wFwd& a, cudaStream_t st);

// Data gradient dX[g][ci] = sum_w dY[g - off_w] . Wdg_w[ci], into rows of cin channels
//   D3W_PLAIN: dX = acc;  D3W_MASK: dX = acc*(mask > 0);  D3W_RES: dX = dres + acc*(mask > 0)
//   D3W_PART: part_out[g][c] = acc; other modes: acc += part_in[g][c] (nullable) first
struct Conv3wDgrad {
  int mode, cin, ch;      // dX channels (16 / 32), dY channels
  PadGeo g;
  int64_t rows;
  const uint8_t* dY;
  const bf16* wimg;       // [9][cin][ch] (pre-swizzled)
  const uint8_t* mask;
  const uint8_t* dres;
  uint8_t* dX;
  float* part_out;
  const float* part_in;
};
seed_status conv3w_dgrad(const Conv3wDgrad& a, cudaStream_t st);

// Weight + bias gradient: dW[co][ky][kx][c] = scale * sum_g X[g + off][c] dY[g][co],
// db[co] = sum_g dY[g][co] (fixed-order split sum; part = scratch); xf as Conv3wFwd
// (XF_RELU: X = relu(rows), XF_U8: X from obs_u8)
struct Conv3wWgrad {
  int cin_p, cin, ch;     // X row channels, real input channels, dY channels
  bool xim;
  int xf;
  const uint8_t* obs_u8;
  PadGeo g;
  int64_t rows;
  float scale;
  const uint8_t* X;
  const uint8_t* dY;
  float* part;
  float* g_w;             // fp32 [ch][3][3][cin] (or the block [co_off..][..][..][c_off..] of
                          // a [..][3][3][ci_full] tensor: plane pairs of the 4x torso)
  float* g_b;             // fp32 [ch] (nullptr: no bias gradient)
  int ci_full, co_off, c_off;
};
seed_status conv3w_wgrad(const Conv3wWgrad& a, cudaStream_t st);
size_t conv3w_wgrad_part_bytes(int64_t rows, int ch, bool xim);

// max-pool 3x3 / stride 2 / TF 'same' (top/left pad pt/pl, padding = -inf, first
// maximum in (ky, kx) order): conv (gi rows) -> h0, hr0 = relu(h0) (nullable; go rows)
// and the window argmax (0..8) per (go row, channel)
seed_status conv3w_pool_fwd(int64_t F, const PadGeo& gi, const PadGeo& go, int C, int pt, int pl,
                            const uint8_t* conv, uint8_t* h0, uint8_t* hr0, uint8_t* arg,
                            cudaStream_t st);
// the 3x3 window max of 8 channels (one 16-byte chunk per tap, taps in (ky, kx)
// order, -inf for padding): packed bf16x2 v > best per half (strict: the first
// maximum wins), best / argmax selected through the 16-bit lane masks; rl =
// relu(best), arg = the 8 argmax bytes
__device__ __forceinline__ void pool_max9(const uint4 (&in)[9], uint4& best_o, uint4& rl_o, uint2& arg_o) {
  uint32_t best[4] = {in[0].x, in[0].y, in[0].z, in[0].w};
  uint32_t barg[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int q = 1; q < 9; ++q) {
    const uint32_t v[4] = {in[q].x, in[q].y, in[q].z, in[q].w};
    const uint32_t qq = (uint32_t)q * 0x00010001u;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const uint32_t gt = __hgt2_mask(*reinterpret_cast<const __nv_bfloat162*>(&v[p]),
                                      *reinterpret_cast<const __nv_bfloat162*>(&best[p]));
      best[p] = (v[p] & gt) | (best[p] & ~gt);
      barg[p] = (qq & gt) | (barg[p] & ~gt);
    }
  }
  uint32_t rl[4];
  const __nv_bfloat162 zero2 = __floats2bfloat162_rn(0.f, 0.f);
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const __nv_bfloat162 r2 = __hmax2(*reinterpret_cast<const __nv_bfloat162*>(&best[p]), zero2);
    rl[p] = *reinterpret_cast<const uint32_t*>(&r2);
  }
  best_o = make_uint4(best[0], best[1], best[2], best[3]);
  rl_o = make_uint4(rl[0], rl[1], rl[2], rl[3]);
  arg_o.x = __byte_perm(barg[0], barg[1], 0x6420);
  arg_o.y = __byte_perm(barg[2], barg[3], 0x6420);
}
constexpr uint32_t BF16X2_NEG_INF = 0xFF80FF80u;

// Section conv + max-pool in one kernel (conv3w_pool.cu): the conv of a band of
// whole image rows (or of several whole frames) accumulates in TMEM, is stored
// as bf16 into shared memory by the epilogue warps, which then pool it there and
// write h0 / hr0 / arg (borders zero) — the full-resolution conv output never
// goes to HBM.  `a` is the W3_PLAIN section conv; conv_dbg (nullable) also
// receives the conv rows (border rows unspecified) for the parity tests.
// SEED_E_UNSUPPORTED when the shape has no fused instantiation or does not fit
// (the caller then runs conv3w_forward + conv3w_pool_fwd).
seed_status conv3w_conv_pool(const Conv3wFwd& a, const PadGeo& go, int pt, int pl, uint8_t* h0,
                             uint8_t* hr0, uint8_t* arg, uint8_t* conv_dbg, cudaStream_t st);
// gradient gather into gi rows (borders zero)
seed_status conv3w_pool_bwd(int64_t F, const PadGeo& gi, const PadGeo& go, int C, int pt, int pl,
                            const uint8_t* dout, const uint8_t* arg, uint8_t* din,
                            cudaStream_t st);

// bf16 weight-image element position of source element e of W[CO][3][3][CI]
// (net.cuh IMG_WIN3: d0 = mode 0 forward [ky][kx][CO][RB] / 1 data gradient
// [ky][2-kx][CI][RB] / 2 x-im2col forward [ky][CO][RB]; d1 = CI, d2 = CO, d3 = RB bytes)
__host__ __device__ inline int64_t win3_img_pos(int mode, int CI, int CO, int RB, int64_t e64) {
  const int e = (int)e64;
  const int c = e % CI;
  int q = e / CI;
  const int kx = q % 3; q /= 3;
  const int ky = q % 3;
  const int co = q / 3;
  int row, k;
  if (mode == 0) { row = (ky * 3 + kx) * CO + co; k = c; }
  else if (mode == 1) { row = (ky * 3 + 2 - kx) * CI + c; k = co; }   // column taps reversed
  else { row = ky * CO + co; k = kx * CI + c; }
  return (int64_t)row * (RB / 2) + swz_chunk(row, RB, k / 8) * 8 + (k % 8);
}
__host__ __device__ inline int64_t win3_img_elems(int mode, int CI, int CO, int RB) {
  return (int64_t)(mode == 0 ? 9 * CO : mode == 1 ? 9 * CI : 3 * CO) * (RB / 2);
}
// Plane-pair images of a conv with more than 64 input or output channels: the
// 64 -> 64 sub-images (q = output plane, p = input plane) one after another, each
// 1024-byte aligned, sub-image (q, p) at index q * npi + p (mode 1 (data gradient)
// uses the same index: the dX plane p sums over the dY planes q).  RB = the
// sub-conv's row bytes (128).
__host__ __device__ inline int64_t win3p_sub_elems(int mode, int CI, int CO, int RB) {
  const int ci = CI > 64 ? 64 : CI, co = CO > 64 ? 64 : CO;
  return (win3_img_elems(mode, ci, co, RB) + 511) & ~(int64_t)511;
}
__host__ __device__ inline int64_t win3p_img_pos(int mode, int CI, int CO, int RB, int64_t e) {
  if (CI <= 64 && CO <= 64) return win3_img_pos(mode, CI, CO, RB, e);
  const int c = (int)(e % CI);
  const int64_t r = e / CI;
  const int k = (int)(r % 9), co = (int)(r / 9);
  const int ci_s = CI > 64 ? 64 : CI, co_s = CO > 64 ? 64 : CO, npi = CI > 64 ? 2 : 1;
  const int64_t es = ((int64_t)(co % 64) * 9 + k) * ci_s + c % 64;
  return ((co / 64) * npi + c / 64) * win3p_sub_elems(mode, CI, CO, RB) +
         win3_img_pos(mode, ci_s, co_s, RB, es);
}
inline int64_t win3p_img_elems(int mode, int CI, int CO, int RB) {
  return (int64_t)(CI > 64 ? 2 : 1) * (CO > 64 ? 2 : 1) * win3p_sub_elems(mode, CI, CO, RB);
}

}  // namespace seed
