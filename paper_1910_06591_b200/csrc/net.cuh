// net.cuh — host-side plans: parameter layout (include/seed.h), the bf16
// operand image ("lowp"), and the learner / inference workspace layouts.
#pragma once
#include <string.h>
#include "common.cuh"

namespace seed {

struct PTensor {
  char name[32];
  int ndim;
  int64_t shape[4];
  int64_t off, n;
};

// One bf16 operand image inside params_lowp.
enum { IMG_COPY_PAD = 0, IMG_CONV_DGRAD = 1, IMG_CHAN_PAD = 2, IMG_S2D = 3, IMG_WIN3 = 4 };
struct LowpImg {
  int kind;
  int64_t src;          // fp32 element offset of the source tensor
  int64_t dst;          // bf16 element offset in params_lowp
  int rows, cols, ld;   // COPY_PAD: dst[r][c] (ld) = src[r][c] (cols) for c < cols, else 0
  uint32_t cmul, cshr;  // cols as a multiply-high divisor (FastDiv of cols, < 2^31 dividends)
  int d0, d1, d2, d3;   // CONV_DGRAD: src [d0=CO][d1=KH][d2=KW][d3=CI] -> dst [CI][KH][KW][CO]
                        // CHAN_PAD: src [rows][taps=d1][d3=C] -> dst [rows][taps][d2=Cp] (0-padded)
                        // S2D: src W[CO=d2][2s][2s][C=d1] (s = d0) -> the pre-swizzled
                        //   space-to-depth window image (conv_s2d.cuh): d3 = 0 forward
                        //   [4][CO][64] (128-byte rows), d3 = 1 data gradient [4][64][CO]
                        // WIN3: src W[CO=d2][3][3][CI=d1] -> the pre-swizzled 3x3 window
                        //   image (conv3w.cuh win3_img_pos), mode d0, row bytes d3;
                        //   rows = CO, cols = ld = 9*CI (source elements)
};

// IMG_S2D: bf16 element position (inside the image) of source element e.
// Window w = (ky / s) * 2 + kx / s, s2d channel ch = ((ky % s) * s + kx % s) * C + c.
__host__ __device__ inline int64_t s2d_img_pos(const LowpImg& m, int64_t e64) {
  const int s = m.d0, C = m.d1, CO = m.d2, K = 2 * s;
  const int e = (int)e64;
  const int c = e % C;
  int q = e / C;
  const int kx = q % K; q /= K;
  const int ky = q % K;
  const int co = q / K;
  const int w = (ky / s) * 2 + kx / s, ch = ((ky % s) * s + kx % s) * C + c;
  int row, rb, k;
  if (m.d3 == 0) { row = w * CO + co; rb = 128; k = ch; }
  else { row = w * 64 + ch; rb = 2 * CO; k = co; }
  return (int64_t)row * (rb / 2) + swz_chunk(row, rb, k / 8) * 8 + (k % 8);
}
// row / column of element e of a COPY_PAD image (e < 2^31)
__host__ __device__ inline void img_rc(const LowpImg& m, uint32_t e, uint32_t& r, uint32_t& c) {
#ifdef __CUDA_ARCH__
  r = m.cmul ? (__umulhi(e, m.cmul) >> m.cshr) : e;
#else
  r = e / (uint32_t)m.cols;
#endif
  c = e - r * (uint32_t)m.cols;
}

// IMPALA-deep section (C14): conv3x3 (cin -> ch) at H x W, maxpool -> H2 x W2,
// residual blocks at H2 x W2 (conv3w.cuh).  cinp = channels of the input rows
// (16 / 32 / 64; 128 = two 64-channel planes); xim: section-0 x-im2col input (3 windows).
struct DeepSec {
  int H, W, cin, cinp, ch, H2, W2, pt, pl, xim;
  int t_w, t_b, t_rw[2][2], t_rb[2][2];              // tensor indices
  int64_t im_w, im_dg, im_rw[2][2], im_rdg[2][2];    // bf16 image offsets
};

struct NetPlan {
  int kind, H, W, C, A, U, D;
  int nt;
  PTensor t[64];
  int64_t P;
  // shallow-net geometry
  int oh1, ow1, oh2, ow2, fc_in, Kx, Kxp;
  // tensor indices
  int i_conv1w, i_conv1b, i_conv2w, i_conv2b, i_fcw, i_fcb, i_wx, i_wh, i_lb, i_hw, i_hb;
  int i_m0w, i_m0b, i_m1w, i_m1b;
  // IMPALA-deep sections
  int nsec;
  DeepSec sec[4];
  // lowp images
  int nimg;
  LowpImg img[64];
  int64_t lowp_elems;
  int64_t im_conv1, im_conv2, im_conv2dg, im_fc, im_wx, im_wh;  // bf16 offsets
                        // (shallow: im_conv1 / im_conv2 / im_conv2dg are IMG_S2D images)
};

seed_status make_net_plan(const seed_net_spec* s, NetPlan* p);
bool learner_supported(const NetPlan& p);

// Learner workspace: byte offsets (256-aligned) of every buffer.
struct LearnerWs {
  int T, B, T1, F;
  size_t total;
  // common
  size_t logits, values, vs, pg, dlogits, dvalues, loss_part, flag, norm_part, step_in, splitk,
      colsum_part, dH, hpart, splitk2;
  size_t splitk_bytes;
  // shallow
  size_t obs_bf16, act1, act2, X, xproj, H, Hprev, gates, Cst, dG, dfc, dY2, dY1;
  // shallow (conv_s2d.cuh): obs_bf16 = S0, act1 = S1, dY2 / dY1 pre-swizzled s2d rows
  // mlp
  size_t h1, h2, dh1, dh2;
  // deep torso (conv3w.cuh padded row spaces; obs_bf16 = section-0 input rows,
  // act2 = dense relu(h) of the last section, dY2 = that section's dhA), per section
  struct Sec {
    size_t conv, arg, h[3], hr[3], u1[2], dconv, dhA, dhB, dt0;
  } sec[4];
  size_t part3;   // fp32 [rows][64] partial sums of the plane-pair convs (0: none)
};
constexpr int NORM_BLOCKS = 296;
constexpr int COLSUM_BLOCKS = 148;

seed_status make_learner_ws(const NetPlan& p, int T, int B, LearnerWs* w);
int pick_splits(int M, int N, int BN, int K);
seed_status refresh_lowp(const NetPlan& p, const float* params, void* lowp, cudaStream_t st);

}  // namespace seed
