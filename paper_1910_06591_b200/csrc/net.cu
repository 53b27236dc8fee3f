// net.cu — network definitions (C14): parameter layout, bf16 operand image,
// workspace planning, and the parameter-query entry points of the C ABI.
#include <stdio.h>
#include <algorithm>
#include "gemm_tc.cuh"
#include "net.cuh"
#include "conv_s2d.cuh"
#include "conv3w.cuh"

namespace seed {

static void add_t(NetPlan* p, const char* name, int nd, int64_t a, int64_t b = 0, int64_t c = 0,
                  int64_t d = 0) {
  PTensor& t = p->t[p->nt];
  snprintf(t.name, sizeof(t.name), "%s", name);
  t.ndim = nd;
  t.shape[0] = a; t.shape[1] = b; t.shape[2] = c; t.shape[3] = d;
  int64_t n = 1;
  for (int i = 0; i < nd; ++i) n *= t.shape[i];
  t.n = n;
  t.off = p->P;
  p->P += n;
  p->nt++;
}

static int same_out(int n) { return (n + 1) / 2; }

seed_status make_net_plan(const seed_net_spec* s, NetPlan* p) {
  if (!s) return SEED_E_ARG;
  memset(p, 0, sizeof(*p));
  p->kind = s->kind;
  p->H = s->obs_h; p->W = s->obs_w; p->C = s->obs_c;
  p->A = s->num_actions;
  p->U = s->lstm_units;
  p->D = s->obs_h * s->obs_w * s->obs_c;
  if (p->A < 2 || p->A > 32 || p->H < 1 || p->W < 1 || p->C < 1) return SEED_E_SHAPE;
  const int A = p->A;
  if (s->kind == SEED_NET_MLP) {
    if (p->U != 0 || p->D > 256) return SEED_E_SHAPE;
    p->i_m0w = p->nt; add_t(p, "mlp0.w", 2, 64, p->D);
    p->i_m0b = p->nt; add_t(p, "mlp0.b", 1, 64);
    p->i_m1w = p->nt; add_t(p, "mlp1.w", 2, 64, 64);
    p->i_m1b = p->nt; add_t(p, "mlp1.b", 1, 64);
    p->i_hw = p->nt; add_t(p, "heads.w", 2, A + 1, 64);
    p->i_hb = p->nt; add_t(p, "heads.b", 1, A + 1);
    return SEED_OK;
  }
  if (p->U != 256) return SEED_E_SHAPE;  // LSTM256 (C14)
  int fh, fw, fc;
  if (s->kind == SEED_NET_ATARI_SHALLOW) {
    if (p->H < 12 || p->W < 12) return SEED_E_SHAPE;
    p->oh1 = (p->H - 8) / 4 + 1; p->ow1 = (p->W - 8) / 4 + 1;
    p->oh2 = (p->oh1 - 4) / 2 + 1; p->ow2 = (p->ow1 - 4) / 2 + 1;
    p->i_conv1w = p->nt; add_t(p, "conv1.w", 4, 16, 8, 8, p->C);
    p->i_conv1b = p->nt; add_t(p, "conv1.b", 1, 16);
    p->i_conv2w = p->nt; add_t(p, "conv2.w", 4, 32, 4, 4, 16);
    p->i_conv2b = p->nt; add_t(p, "conv2.b", 1, 32);
    fh = p->oh2; fw = p->ow2; fc = 32;
  } else if (s->kind == SEED_NET_IMPALA_DEEP || s->kind == SEED_NET_GFOOTBALL) {
    const int ns = s->kind == SEED_NET_IMPALA_DEEP ? 3 : 4;
    const int wm = s->torso_width <= 1 ? 1 : s->torso_width;
    if (wm != 1 && wm != 2 && wm != 4) return SEED_E_UNSUPPORTED;
    const int chs[4] = {16 * wm, 32 * wm, 32 * wm, 32 * wm};
    int cin = p->C, h = p->H, w = p->W;
    char nm[32];
    p->nsec = ns;
    for (int sct = 0; sct < ns; ++sct) {
      const int ch = chs[sct];
      DeepSec& d = p->sec[sct];
      d.H = h; d.W = w; d.cin = cin; d.ch = ch;
      d.xim = sct == 0 && 3 * cin <= 16;
      // input row channels; 128 = two 64-channel planes (conv3w.cuh)
      d.cinp = d.xim || cin <= 16 ? 16 : (cin <= 32 ? 32 : cin <= 64 ? 64 : 128);
      if (cin > 64 && cin != 128) return SEED_E_UNSUPPORTED;
      d.H2 = same_out(h); d.W2 = same_out(w);
      const int ph = std::max((d.H2 - 1) * 2 + 3 - h, 0), pw = std::max((d.W2 - 1) * 2 + 3 - w, 0);
      d.pt = ph / 2; d.pl = pw / 2;
      snprintf(nm, 32, "s%d.conv.w", sct); d.t_w = p->nt; add_t(p, nm, 4, ch, 3, 3, cin);
      snprintf(nm, 32, "s%d.conv.b", sct); d.t_b = p->nt; add_t(p, nm, 1, ch);
      for (int r = 0; r < 2; ++r)
        for (int j = 0; j < 2; ++j) {
          snprintf(nm, 32, "s%d.res%d.conv%d.w", sct, r, j); d.t_rw[r][j] = p->nt;
          add_t(p, nm, 4, ch, 3, 3, ch);
          snprintf(nm, 32, "s%d.res%d.conv%d.b", sct, r, j); d.t_rb[r][j] = p->nt;
          add_t(p, nm, 1, ch);
        }
      cin = ch; h = d.H2; w = d.W2;
    }
    fh = h; fw = w; fc = cin;
  } else {
    return SEED_E_UNSUPPORTED;
  }
  p->fc_in = fh * fw * fc;
  p->Kx = 256 + A + 1;
  p->Kxp = (int)align_up((size_t)p->Kx + 1, 32);  // + the all-ones column (bias grad)
  p->i_fcw = p->nt; add_t(p, "fc.w", 2, 256, p->fc_in);
  p->i_fcb = p->nt; add_t(p, "fc.b", 1, 256);
  p->i_wx = p->nt; add_t(p, "lstm.wx", 2, 4 * p->U, p->Kx);
  p->i_wh = p->nt; add_t(p, "lstm.wh", 2, 4 * p->U, p->U);
  p->i_lb = p->nt; add_t(p, "lstm.b", 1, 4 * p->U);
  p->i_hw = p->nt; add_t(p, "heads.w", 2, A + 1, p->U);
  p->i_hb = p->nt; add_t(p, "heads.b", 1, A + 1);
  // bf16 operand images (GEMM-ready, K padded to multiples of 8 / 32)
  int64_t off = 0;
  auto img = [&](int kind, int ti, int rows, int cols, int ld) {
    LowpImg& m = p->img[p->nimg++];
    m.kind = kind; m.src = p->t[ti].off; m.dst = off; m.rows = rows; m.cols = cols; m.ld = ld;
    const FastDiv fd((uint32_t)cols);
    m.cmul = fd.mul; m.cshr = fd.shr;
    const int64_t start = off;
    off += (int64_t)rows * ld;
    off = (int64_t)align_up((size_t)off, 64);
    return start;
  };
  if (s->kind == SEED_NET_ATARI_SHALLOW) {
    // space-to-depth window images (conv_s2d.cuh); 1024-byte aligned starts
    auto s2d_img = [&](int ti, int st, int C, int CO, int mode) {
      off = (int64_t)align_up((size_t)off, 512);
      const int64_t at = img(IMG_S2D, ti, 4 * CO, 64, 64);
      LowpImg& m = p->img[p->nimg - 1];
      m.d0 = st; m.d1 = C; m.d2 = CO; m.d3 = mode;
      return at;
    };
    p->im_conv1 = s2d_img(p->i_conv1w, 4, p->C, 16, 0);
    p->im_conv2 = s2d_img(p->i_conv2w, 2, 16, 32, 0);
    p->im_conv2dg = s2d_img(p->i_conv2w, 2, 16, 32, 1);
  } else {
    // 3x3 window images (conv3w.cuh), 1024-byte aligned starts
    auto win3_img = [&](int ti, int mode, int CI, int CO, int RB) {
      off = (int64_t)align_up((size_t)off, 512);
      LowpImg& m = p->img[p->nimg++];
      m.kind = IMG_WIN3; m.src = p->t[ti].off; m.dst = off;
      m.rows = CO; m.cols = 9 * CI; m.ld = 9 * CI;
      const FastDiv fd((uint32_t)m.cols);
      m.cmul = fd.mul; m.cshr = fd.shr;
      m.d0 = mode; m.d1 = CI; m.d2 = CO; m.d3 = RB;
      const int64_t start = off;
      off = (int64_t)align_up((size_t)(off + win3p_img_elems(mode, CI, CO, RB)), 64);
      return start;
    };
    // (more than 64 channels: plane-pair sub-images of 64 -> 64 convs, conv3w.cuh)
    for (int sct = 0; sct < p->nsec; ++sct) {
      DeepSec& d = p->sec[sct];
      const int ci_rb = 2 * std::min(d.cinp, 64), ch_rb = 2 * std::min(d.ch, 64);
      d.im_w = win3_img(d.t_w, d.xim ? 2 : 0, d.cin, d.ch, d.xim ? 32 : ci_rb);
      d.im_dg = sct > 0 ? win3_img(d.t_w, 1, d.cin, d.ch, ch_rb) : -1;
      for (int r = 0; r < 2; ++r)
        for (int j = 0; j < 2; ++j) {
          d.im_rw[r][j] = win3_img(d.t_rw[r][j], 0, d.ch, d.ch, ch_rb);
          d.im_rdg[r][j] = win3_img(d.t_rw[r][j], 1, d.ch, d.ch, ch_rb);
        }
    }
  }
  p->im_fc = img(IMG_COPY_PAD, p->i_fcw, 256, p->fc_in, p->fc_in);
  p->im_wx = img(IMG_COPY_PAD, p->i_wx, 4 * p->U, p->Kx, p->Kxp);
  p->im_wh = img(IMG_COPY_PAD, p->i_wh, 4 * p->U, p->U, p->U);
  p->lowp_elems = off;
  return SEED_OK;
}

bool learner_supported(const NetPlan& p) {
  if (p.kind == SEED_NET_MLP) return true;
  if (p.kind == SEED_NET_ATARI_SHALLOW) return shallow_s2d_supported(p.H, p.W, p.C);
  if (p.kind == SEED_NET_IMPALA_DEEP || p.kind == SEED_NET_GFOOTBALL)   // conv3w.cuh
    return p.C >= 1 && p.C <= 32 &&
           (p.sec[p.nsec - 1].ch == 32 || p.sec[p.nsec - 1].ch == 64 || p.sec[p.nsec - 1].ch == 128) &&
           p.fc_in % 8 == 0;
  return false;
}

static size_t bump(size_t& cur, size_t bytes) {
  const size_t at = cur;
  cur = align_up(cur + bytes, 256);
  return at;
}

int pick_splits(int M, int N, int BN, int K) {
  const int tiles = ceil_div(M, GEMM_BM) * ceil_div(N, BN);
  const int nkb = ceil_div(K, GEMM_BK);
  int s = ceil_div(148, tiles);
  const int cap = nkb / 4;
  if (s > cap) s = cap;
  if (s < 1) s = 1;
  return gemm_effective_splits(K, s);
}

seed_status make_learner_ws(const NetPlan& p, int T, int B, LearnerWs* w) {
  memset(w, 0, sizeof(*w));
  w->T = T; w->B = B; w->T1 = T + 1;
  const size_t F = (size_t)B * (T + 1);
  w->F = (int)F;
  const int A = p.A;
  size_t cur = 0;
  w->logits = bump(cur, F * A * 4);
  w->values = bump(cur, F * 4);
  w->vs = bump(cur, (size_t)B * T * 4);
  w->pg = bump(cur, (size_t)B * T * 4);
  w->dlogits = bump(cur, F * A * 4);
  w->dvalues = bump(cur, F * 4);
  w->loss_part = bump(cur, (size_t)B * 4 * 4);
  w->hpart = bump(cur, (size_t)B * 4 * (A + 1) * (std::max(p.U, 64) + 1) * 4);   // heads grad partials (b, cluster rank)
  w->flag = bump(cur, 16);
  w->norm_part = bump(cur, NORM_BLOCKS * 8 + 64);   // + clip/Adam coefficients, norm
  w->step_in = bump(cur, 8);
  // + tickets and split-K tile counters (zeroed at the start of every step)
  w->colsum_part = bump(cur, COLSUM_BLOCKS * 64 * 4 + 64 + GEMM_COUNTERS * 4);
  if (p.kind == SEED_NET_MLP) {
    w->h1 = bump(cur, F * 64 * 4);
    w->h2 = bump(cur, F * 64 * 4);
    w->dh1 = bump(cur, F * 64 * 4);
    w->dh2 = bump(cur, F * 64 * 4);
    w->total = cur;
    return SEED_OK;
  }
  const size_t U = p.U;
  w->dH = bump(cur, F * U * 4);
  if (p.nsec > 0) {
    const DeepSec& d0 = p.sec[0];
    w->obs_bf16 = bump(cur, F * (d0.H + 2) * (d0.W + 2) * d0.cinp * 2);
    for (int sct = 0; sct < p.nsec; ++sct) {
      const DeepSec& d = p.sec[sct];
      LearnerWs::Sec& b = w->sec[sct];
      const size_t sc = F * (d.H + 2) * (d.W + 2) * d.ch, sp = F * (d.H2 + 2) * (d.W2 + 2) * d.ch;
      b.conv = bump(cur, sc * 2);
      b.arg = bump(cur, sp);
      for (int k = 0; k < 3; ++k) {
        b.h[k] = bump(cur, sp * 2);
        b.hr[k] = bump(cur, sp * 2);
      }
      b.u1[0] = bump(cur, sp * 2);
      b.u1[1] = bump(cur, sp * 2);
      b.dconv = bump(cur, sc * 2);
      b.dhA = bump(cur, sp * 2);
      b.dhB = bump(cur, sp * 2);
      b.dt0 = bump(cur, sp * 2);
    }
    // fp32 partial sums of the plane-pair convs (128-channel sections): the largest
    // row space with two input planes
    size_t prow = 0;
    for (int sct = 0; sct < p.nsec; ++sct) {
      const DeepSec& d = p.sec[sct];
      if (d.cinp > 64 || d.ch > 64) prow = std::max(prow, (size_t)F * (d.H + 2) * (d.W + 2));
      if (d.ch > 64) prow = std::max(prow, (size_t)F * (d.H2 + 2) * (d.W2 + 2));
    }
    w->part3 = prow ? bump(cur, prow * 64 * 4) : 0;
    // the FC layer reads dense relu(h) of the last section (written by its last
    // residual epilogue) and writes its data gradient into that section's dhA
    w->act2 = bump(cur, F * p.fc_in * 2);
    w->dY2 = w->sec[p.nsec - 1].dhA;
  } else {
    const ShallowS2d sg = shallow_s2d_geometry(p.H, p.W, p.C);
    w->obs_bf16 = bump(cur, s2d_S0_bytes(sg, F));   // S0
    w->act1 = bump(cur, s2d_S1_bytes(sg, F));       // S1
    w->act2 = bump(cur, F * p.fc_in * 2);
    w->dY1 = bump(cur, s2d_dY1_bytes(sg, F));
    w->dY2 = bump(cur, s2d_dY2_bytes(sg, F));
  }
  w->X = bump(cur, F * p.Kxp * 2);
  w->xproj = bump(cur, F * 4 * U * 4);
  w->H = bump(cur, F * U * 4);
  w->Hprev = bump(cur, F * U * 2);
  w->gates = bump(cur, F * 4 * U * 4);
  w->Cst = bump(cur, F * U * 4);
  w->dG = bump(cur, F * 4 * U * 2);
  w->dfc = bump(cur, F * 256 * 2);
  // split-K partial buffer: max over the split GEMMs of the step
  const int Fi = (int)F;
  size_t sk = 0;
  auto need = [&](int M, int N, int BN, int K) {
    const int s = pick_splits(M, N, BN, K);
    if (s > 1) sk = std::max(sk, (size_t)s * M * N * 4);
  };
  need(Fi, 256, 128, p.fc_in);                         // fc forward
  need(Fi, 4 * (int)U, 128, p.Kxp);                    // lstm input projection
  need(4 * (int)U, p.Kxp + (int)U, 128, Fi);           // lstm weight grads
  need(Fi, 256, 128, 4 * (int)U);                      // dX (fc part)
  need(256, p.fc_in + 8, 128, Fi);                     // fc weight grads (+ bias column)
  need(Fi, p.fc_in, 128, 256);                         // fc dgrad
  if (p.nsec == 0) {                                  // s2d weight-gradient partials
    const ShallowS2d sg = shallow_s2d_geometry(p.H, p.W, p.C);
    sk = std::max(sk, win_wgrad_part_bytes(sg.rows1(F), 16));
    sk = std::max(sk, win_wgrad_part_bytes(sg.rows2(F), 32));
  }
  for (int sct = 0; sct < p.nsec; ++sct) {            // 3x3 weight grads (conv3w.cuh)
    const DeepSec& d = p.sec[sct];
    sk = std::max(sk, conv3w_wgrad_part_bytes(F * (d.H + 2) * (d.W + 2), d.ch, d.xim));
    sk = std::max(sk, conv3w_wgrad_part_bytes(F * (d.H2 + 2) * (d.W2 + 2), d.ch, false));
  }
  w->splitk_bytes = sk;
  w->splitk = bump(cur, sk + 16);
  w->splitk2 = bump(cur, sk + 16);   // partials of the second (aux-stream) backward branch
  w->total = cur;
  return SEED_OK;
}

// ------------------------------------------------------------------ lowp image refresh
// One launch for all images: image k owns blocks [first[k], first[k+1]) (its
// element count / (256 threads x 4)), so the large FC / LSTM images are spread over
// the GPU instead of 64 blocks striding through them (measured: 18 us at c4 with
// dim3(64, images) and 64-bit index arithmetic).
constexpr int REFRESH_PER = 4;   // elements per thread
struct ImgTable {
  int n;
  int first[65];
  LowpImg img[64];
};

__global__ void __launch_bounds__(256) refresh_lowp_multi(const float* __restrict__ params,
                                                          __nv_bfloat16* lowp, const ImgTable tab) {
  int k = 0;
  while (k + 1 < tab.n && (int)blockIdx.x >= tab.first[k + 1]) ++k;
  const LowpImg& m = tab.img[k];
  const int n = m.rows * m.ld;
  const int i0 = ((int)blockIdx.x - tab.first[k]) * 256 * REFRESH_PER + threadIdx.x;
#pragma unroll
  for (int u = 0; u < REFRESH_PER; ++u) {
    const int i = i0 + u * 256;
    if (i >= n) break;
    float v;
    if (m.kind == IMG_S2D) {   // bijective (s*s*C == 64): iterate the source elements
      lowp[m.dst + s2d_img_pos(m, i)] = __float2bfloat16_rn(params[m.src + i]);
      continue;
    }
    if (m.kind == IMG_WIN3) {  // source elements; padding positions stay zero
      lowp[m.dst + win3p_img_pos(m.d0, m.d1, m.d2, m.d3, i)] = __float2bfloat16_rn(params[m.src + i]);
      continue;
    }
    if (m.kind == IMG_COPY_PAD) {
      const int r = i / m.ld, c = i - r * m.ld;
      v = c < m.cols ? params[m.src + (int64_t)r * m.cols + c] : 0.f;
    } else if (m.kind == IMG_CHAN_PAD) {
      const int r = i / m.ld, q = i - r * m.ld;
      const int t = q / m.d2, c = q - t * m.d2;
      v = c < m.d3 ? params[m.src + ((int64_t)r * m.d1 + t) * m.d3 + c] : 0.f;
    } else {
      int q = i / m.d0;
      const int co = i - q * m.d0;
      const int kx = q % m.d2; q /= m.d2;
      const int ky = q % m.d1;
      const int ci = q / m.d1;
      v = params[m.src + (((int64_t)co * m.d1 + ky) * m.d2 + kx) * m.d3 + ci];
    }
    lowp[m.dst + i] = __float2bfloat16_rn(v);
  }
}

seed_status refresh_lowp(const NetPlan& p, const float* params, void* lowp, cudaStream_t st) {
  if (p.nimg == 0) return SEED_OK;
  if (p.nimg > 64) return SEED_E_UNSUPPORTED;
  ImgTable tab;
  tab.n = p.nimg;
  int blocks = 0;
  for (int k = 0; k < p.nimg; ++k) {
    tab.img[k] = p.img[k];
    tab.first[k] = blocks;
    const int64_t n = (int64_t)p.img[k].rows * p.img[k].ld;
    if (n >= (1ll << 31)) return SEED_E_SHAPE;
    blocks += (int)std::max<int64_t>(1, (n + 256 * REFRESH_PER - 1) / (256 * REFRESH_PER));
  }
  tab.first[p.nimg] = blocks;
  refresh_lowp_multi<<<blocks, 256, 0, st>>>(params, (__nv_bfloat16*)lowp, tab);
  return last_launch();
}

}  // namespace seed

using namespace seed;

extern "C" seed_status seed_net_param_count(const seed_net_spec* spec, int64_t* n) {
  if (!n) return SEED_E_ARG;
  NetPlan p;
  SEED_TRY(make_net_plan(spec, &p));
  *n = p.P;
  return SEED_OK;
}

extern "C" seed_status seed_net_param_tensor(const seed_net_spec* spec, int index, char* name,
                                             int* ndim, int64_t* shape, int64_t* offset) {
  NetPlan p;
  SEED_TRY(make_net_plan(spec, &p));
  if (index < 0 || index >= p.nt) return SEED_E_ARG;
  const PTensor& t = p.t[index];
  if (name) snprintf(name, 64, "%s", t.name);
  if (ndim) *ndim = t.ndim;
  if (shape)
    for (int i = 0; i < 4; ++i) shape[i] = i < t.ndim ? t.shape[i] : 0;
  if (offset) *offset = t.off;
  return SEED_OK;
}

extern "C" seed_status seed_net_lowp_bytes(const seed_net_spec* spec, size_t* bytes) {
  if (!bytes) return SEED_E_ARG;
  NetPlan p;
  SEED_TRY(make_net_plan(spec, &p));
  *bytes = align_up((size_t)p.lowp_elems * 2, 16);   // whole 16-byte chunks
  return SEED_OK;
}

extern "C" seed_status seed_net_refresh_lowp(const seed_net_spec* spec, const float* params,
                                             void* lowp, void* stream) {
  NetPlan p;
  SEED_TRY(make_net_plan(spec, &p));
  if (p.nimg == 0) return SEED_OK;
  if (!params || !lowp) return SEED_E_ARG;
  // image padding (channels, rows) is zero: clear once here, never in the step
  SEED_CUDA_TRY(cudaMemsetAsync(lowp, 0, (size_t)p.lowp_elems * 2, (cudaStream_t)stream));
  return refresh_lowp(p, params, lowp, (cudaStream_t)stream);
}

extern "C" seed_status seed_learner_workspace_size(const seed_net_spec* spec, int T, int B,
                                                   size_t* bytes) {
  if (!bytes) return SEED_E_ARG;
  NetPlan p;
  SEED_TRY(make_net_plan(spec, &p));
  if (!learner_supported(p)) return SEED_E_UNSUPPORTED;
  if (T < 1 || T > 256 || B < 1 || B > 1024) return SEED_E_SHAPE;
  LearnerWs w;
  SEED_TRY(make_learner_ws(p, T, B, &w));
  *bytes = w.total;
  return SEED_OK;
}
