// net.cu — network definitions (C14): parameter layout, bf16 operand image,
// workspace planning, and the parameter-query entry points of the C ABI.
#include <stdio.h>
#include "gemm_tc.cuh"
#include "net.cuh"

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
    const int chs[4] = {16, 32, 32, 32};
    int cin = p->C, h = p->H, w = p->W;
    char nm[32];
    for (int sct = 0; sct < ns; ++sct) {
      const int ch = chs[sct];
      snprintf(nm, 32, "s%d.conv.w", sct); add_t(p, nm, 4, ch, 3, 3, cin);
      snprintf(nm, 32, "s%d.conv.b", sct); add_t(p, nm, 1, ch);
      for (int r = 0; r < 2; ++r)
        for (int j = 0; j < 2; ++j) {
          snprintf(nm, 32, "s%d.res%d.conv%d.w", sct, r, j); add_t(p, nm, 4, ch, 3, 3, ch);
          snprintf(nm, 32, "s%d.res%d.conv%d.b", sct, r, j); add_t(p, nm, 1, ch);
        }
      cin = ch; h = same_out(h); w = same_out(w);
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
  if (s->kind == SEED_NET_ATARI_SHALLOW) {
    // bf16 operand images (GEMM-ready, K padded to multiples of 8 / 32)
    int64_t off = 0;
    auto img = [&](int kind, int ti, int rows, int cols, int ld) {
      LowpImg& m = p->img[p->nimg++];
      m.kind = kind; m.src = p->t[ti].off; m.dst = off; m.rows = rows; m.cols = cols; m.ld = ld;
      const int64_t start = off;
      off += (int64_t)rows * ld;
      off = (int64_t)align_up((size_t)off, 64);
      return start;
    };
    p->im_conv1 = img(IMG_COPY_PAD, p->i_conv1w, 16, 64 * p->C, 64 * p->C);
    p->im_conv2 = img(IMG_COPY_PAD, p->i_conv2w, 32, 256, 256);
    p->im_conv2dg = img(IMG_CONV_DGRAD, p->i_conv2w, 16, 512, 512);  // [ci][ky][kx][co]
    LowpImg& dg = p->img[p->nimg - 1];
    dg.d0 = 32; dg.d1 = 4; dg.d2 = 4; dg.d3 = 16;
    p->im_fc = img(IMG_COPY_PAD, p->i_fcw, 256, p->fc_in, p->fc_in);
    p->im_wx = img(IMG_COPY_PAD, p->i_wx, 4 * p->U, p->Kx, p->Kxp);
    p->im_wh = img(IMG_COPY_PAD, p->i_wh, 4 * p->U, p->U, p->U);
    p->lowp_elems = off;
  }
  return SEED_OK;
}

bool learner_supported(const NetPlan& p) {
  if (p.kind == SEED_NET_MLP) return true;
  if (p.kind == SEED_NET_ATARI_SHALLOW) return p.C == 4 && p.fc_in % 8 == 0 && (p.W * p.C) % 16 == 0;
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
  w->flag = bump(cur, 16);
  w->norm_part = bump(cur, NORM_BLOCKS * 8);
  w->step_in = bump(cur, 8);
  w->colsum_part = bump(cur, COLSUM_BLOCKS * 64 * 4 + 64);   // + ticket (zeroed at creation)
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
  w->obs_bf16 = bump(cur, F * p.H * p.W * p.C * 2);
  w->act1 = bump(cur, F * p.oh1 * p.ow1 * 16 * 2);
  w->act2 = bump(cur, F * p.fc_in * 2);
  w->X = bump(cur, F * p.Kxp * 2);
  w->xproj = bump(cur, F * 4 * U * 4);
  w->H = bump(cur, F * U * 4);
  w->Hprev = bump(cur, F * U * 2);
  w->gates = bump(cur, F * 4 * U * 4);
  w->Cst = bump(cur, F * U * 4);
  w->dG = bump(cur, F * 4 * U * 2);
  w->dfc = bump(cur, F * 256 * 2);
  w->dY2 = bump(cur, F * p.fc_in * 2);
  w->dY1 = bump(cur, F * p.oh1 * p.ow1 * 16 * 2);
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
  need(64 * p.C, 16, 16, Fi * p.oh1 * p.ow1);          // conv1 wgrad
  need(256, 32, 32, Fi * p.oh2 * p.ow2);              // conv2 wgrad
  w->splitk_bytes = sk;
  w->splitk = bump(cur, sk + 16);
  w->total = cur;
  return SEED_OK;
}

// ------------------------------------------------------------------ lowp image refresh
__global__ void refresh_lowp_kernel(const float* __restrict__ params, __nv_bfloat16* lowp,
                                    LowpImg img) {
  const int64_t n = (int64_t)img.rows * img.ld;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v;
    if (img.kind == IMG_COPY_PAD) {
      const int r = (int)(i / img.ld), c = (int)(i % img.ld);
      v = c < img.cols ? params[img.src + (int64_t)r * img.cols + c] : 0.f;
    } else {
      // dst [CI][KH][KW][CO] <- src [CO][KH][KW][CI]
      const int co = (int)(i % img.d0);
      int64_t q = i / img.d0;
      const int kx = (int)(q % img.d2); q /= img.d2;
      const int ky = (int)(q % img.d1);
      const int ci = (int)(q / img.d1);
      v = params[img.src + (((int64_t)co * img.d1 + ky) * img.d2 + kx) * img.d3 + ci];
    }
    lowp[img.dst + i] = __float2bfloat16_rn(v);
  }
}

seed_status refresh_lowp(const NetPlan& p, const float* params, void* lowp, cudaStream_t st) {
  for (int k = 0; k < p.nimg; ++k) {
    const int64_t n = (int64_t)p.img[k].rows * p.img[k].ld;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 4);
    refresh_lowp_kernel<<<blocks, 256, 0, st>>>(params, (__nv_bfloat16*)lowp, p.img[k]);
  }
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
  *bytes = (size_t)p.lowp_elems * 2;
  return SEED_OK;
}

extern "C" seed_status seed_net_refresh_lowp(const seed_net_spec* spec, const float* params,
                                             void* lowp, void* stream) {
  NetPlan p;
  SEED_TRY(make_net_plan(spec, &p));
  if (p.nimg == 0) return SEED_OK;
  if (!params || !lowp) return SEED_E_ARG;
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
