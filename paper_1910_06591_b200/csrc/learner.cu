// learner.cu — seed_learner_step: one synchronous SEED learner update on one
// GPU's [B][T+1] shard, with the DP gradient
// allreduce (H10) when a communicator is given.
//
// Atari-shallow path (configs[1]; C14), every dense contraction on tcgen05,
// rows f = b*(T+1)+t:
//   obs -> S0 (space-to-depth, bf16, pre-swizzled), conv1 / conv2 as 2x2
//   shifted-window GEMMs over TMA-loaded slabs (conv_s2d.cuh)
//   fc     GEMM           [F x 2592] . [2592 x 256]       (split-K)
//   Xproj  GEMM           [F x 288]  . [288 x 1024]       (+ bias; x = [fc, onehot, r, 1])
//   LSTM   persistent cluster kernel, T+1 serial steps (lstm.cu)
//   heads  fp32 warp-per-row; K2 fused log-softmax + V-trace + loss + output grads
//   heads backward; LSTM BPTT (cluster kernel)
//   dW_x|b|dW_h  one GEMM  [1024 x F] . [F x (288+256)]    (ones column -> bias grad)
//   dfc    GEMM  [F x 1024] . [1024 x 256]   (ReLU mask)
//   dW_fc|b  GEMM [256 x F] . [F x 2600]    (ones column -> bias grad)
//   dY2    GEMM  [F x 256] . [256 x 2592]   (ReLU mask; written in conv2 s2d row space)
//   dW2|db2, dY1 (masked), dW1|db1: window GEMMs (conv_s2d.cuh; all-ones operand
//   for the bias sums, fixed-order split-K finish)
//   [allreduce] -> global-norm clip + Adam -> bf16 operand image refresh
#include <string.h>
#include <utility>
#include "gemm_tc.cuh"
#include "learner_kernels.cuh"
#include "lstm.cuh"
#include "net.cuh"
#include "shallow_net.cuh"
#include "conv_s2d.cuh"
#include "conv3w.cuh"

namespace seed {

seed_status comm_allreduce(seed_comm* comm, float* data, int64_t n, cudaStream_t st);
seed_status comm_side(seed_comm* c, cudaStream_t* side, cudaStream_t* side2, cudaEvent_t* ev);
seed_status comm_allreduce2(seed_comm* comm, float* data, int64_t n, cudaStream_t st);
int comm_world(const seed_comm* c);

}  // namespace seed

// Caller-owned execution context (include/seed.h seed_exec): the second stream the
// independent backward GEMMs branch onto and the events of the fork / join edges.
// A step captured into a CUDA graph turns the edges into parallel graph branches.
struct seed_exec {
  int device;
  cudaStream_t aux;
  cudaEvent_t ev[8];
};

extern "C" seed_status seed_exec_create(seed_exec** out) {
  if (!out) return SEED_E_ARG;
  *out = nullptr;
  seed_exec* e = new seed_exec{};
  if (cudaGetDevice(&e->device) != cudaSuccess ||
      cudaStreamCreateWithFlags(&e->aux, cudaStreamNonBlocking) != cudaSuccess) {
    delete e;
    return SEED_E_CUDA;
  }
  for (int i = 0; i < 8; ++i)
    if (cudaEventCreateWithFlags(&e->ev[i], cudaEventDisableTiming) != cudaSuccess) {
      for (int k = 0; k < i; ++k) cudaEventDestroy(e->ev[k]);
      cudaStreamDestroy(e->aux);
      delete e;
      return SEED_E_CUDA;
    }
  *out = e;
  return SEED_OK;
}

extern "C" seed_status seed_exec_destroy(seed_exec* e) {
  if (!e) return SEED_OK;
  for (int i = 0; i < 8; ++i) cudaEventDestroy(e->ev[i]);
  cudaStreamDestroy(e->aux);
  delete e;
  return SEED_OK;
}

namespace seed {

// The step's second branch: the context's stream and events; without a context
// (or when tracing: phase marks need one stream) aux = st and no edges are made.
static seed_status aux_stream(const seed_exec* ex, cudaStream_t st, bool single, cudaStream_t* aux,
                              cudaEvent_t* ev8) {
  if (!ex || single) {
    *aux = st;
    return SEED_OK;
  }
  if (ex->device != current_device()) return SEED_E_ARG;
  *aux = ex->aux;
  for (int i = 0; i < 8; ++i) ev8[i] = ex->ev[i];
  return SEED_OK;
}

// DP gradient buckets (H10): 3 = LSTM+heads | FC | torso (default), 2 = core+FC | torso,
// 1 = one allreduce at the end.  SEED_DP_BUCKETS overrides (measurement; 3 measured
// best or equal at N=2: profiles/r01/dp_buckets_n2.txt).
static int dp_buckets() {
  static int b = -1;
  if (b < 0) {
    const char* e = getenv("SEED_DP_BUCKETS");
    b = e ? atoi(e) : 3;
    if (b < 1 || b > 3) b = 3;
  }
  return b;
}

struct Trace {
  void** events = nullptr;
  const char** names = nullptr;
  int* counts = nullptr;   // kernel launches of each phase (nullable)
  int max = 0, n = 0, launches = 0;
  bool capturing = false;
};

// Inside stream capture an event record must be an explicit graph node
// (cudaEventRecordExternal) to be recorded on every replay.
static inline void trace_record(const Trace* tr, void* ev, cudaStream_t st) {
  if (tr->capturing) cudaEventRecordWithFlags((cudaEvent_t)ev, st, cudaEventRecordExternal);
  else cudaEventRecord((cudaEvent_t)ev, st);
}

struct StepCtx {
  const NetPlan* p;
  LearnerWs w;
  uint8_t* ws;
  Geo g;
  Trace* tr = nullptr;
  cudaStream_t st;
  int max_ctas = 0;   // > 0 while collectives run concurrently (SMs left for NCCL)
  // H10 buckets: a gradient range that is final is allreduced on the comm's side
  // stream while the main stream continues (same bucket order on every rank)
  // The second bucket goes to a second communicator on its own stream (side2) when
  // the comm has one, so it reduces concurrently with the first.
  seed_comm* comm = nullptr;
  cudaStream_t side = nullptr, side2 = nullptr;
  cudaEvent_t ev[6] = {};
  int nbucket = 0;
  seed_status bucket(float* g, int64_t n, cudaStream_t from) {
    if (!side || n <= 0 || nbucket >= 3) return SEED_OK;
    const bool second = side2 && nbucket == 1;
    cudaStream_t s = second ? side2 : side;
    SEED_CUDA_TRY(cudaEventRecord(ev[nbucket], from));
    SEED_CUDA_TRY(cudaStreamWaitEvent(s, ev[nbucket], 0));
    ++nbucket;
    return second ? comm_allreduce2(comm, g, n, s) : comm_allreduce(comm, g, n, s);
  }
  // Independent backward GEMMs run as a second branch on `aux` (the caller's
  // seed_exec stream; inside a CUDA graph capture the event edges make it a
  // parallel branch of the graph).  aux == st without a seed_exec or when the step
  // is traced (phase marks need one stream) — then the branches simply run in order.
  cudaStream_t aux = nullptr;
  cudaEvent_t fev[8] = {};
  int nfev = 0;
  seed_status edge(cudaStream_t from, cudaStream_t to) {   // `to` waits for `from`'s work so far
    if (from == to) return SEED_OK;
    if (nfev >= 8) return SEED_E_ARG;
    SEED_CUDA_TRY(cudaEventRecord(fev[nfev], from));
    SEED_CUDA_TRY(cudaStreamWaitEvent(to, fev[nfev], 0));
    ++nfev;
    return SEED_OK;
  }
  template <class T>
  T* at(size_t off) const { return reinterpret_cast<T*>(ws + off); }
  // zeroed region after the column-sum partials: [0..15] tickets, then the
  // split-K tile counters (memset once per step, re-armed by their users)
  unsigned* tickets() const { return reinterpret_cast<unsigned*>(at<float>(w.colsum_part) + COLSUM_BLOCKS * 64); }
  unsigned* gemm_counters() const { return tickets() + 16; }
  // end of a phase of `k` kernel launches
  void mark(const char* name, int k = 1) const {
    if (!tr) return;
    tr->launches += k;
    if (tr->events && tr->n < tr->max) {
      trace_record(tr, tr->events[tr->n], st);
      if (tr->names) tr->names[tr->n] = name;
      if (tr->counts) tr->counts[tr->n] = k;
      tr->n++;
    }
  }
};

template <int BN, class Prob>
static seed_status gemm(const StepCtx& c, Prob pr, cudaStream_t st, const char* name) {
  const int s = pick_splits(pr.M, pr.N, BN, pr.K);
  // (the in-kernel last-CTA split reduction, launch_gemm's `cnt`, measured
  // slower here: few tiles -> the fixups serialise on a few SMs)
  float* part = (st == c.aux && c.aux != c.st) ? c.at<float>(c.w.splitk2) : c.at<float>(c.w.splitk);
  const seed_status r = launch_gemm<BN>(pr, s, st, part, c.max_ctas);
  c.mark(name, s > 1 ? 2 : 1);
  return r;
}

// Atari-shallow torso: obs -> act2 (H1), space-to-depth window convolutions
// (conv_s2d.cuh); conv2's epilogue also zeroes the padding rows of dY2
static seed_status shallow_forward(const StepCtx& c, const seed_batch* bt, const bf16* lowp,
                                   const float* params, cudaStream_t st) {
  const NetPlan& p = *c.p;
  const LearnerWs& w = c.w;
  const int F = w.F;
  const ShallowS2d sg = shallow_s2d_geometry(p.H, p.W, p.C);
  SEED_TRY(s2d_obs((const uint8_t*)bt->obs, F, p.H, p.W, c.at<uint8_t>(w.obs_bf16), st));
  c.mark("obs_s2d");
  SEED_TRY(shallow_s2d_conv1(sg, F, c.at<uint8_t>(w.obs_bf16), lowp + p.im_conv1,
                             params + p.t[p.i_conv1b].off, c.at<uint8_t>(w.act1), st));
  c.mark("conv1_fwd");
  SEED_TRY(shallow_s2d_conv2(sg, F, c.at<uint8_t>(w.act1), lowp + p.im_conv2,
                             params + p.t[p.i_conv2b].off, c.at<bf16>(w.act2),
                             c.at<uint8_t>(w.dY2), st));
  c.mark("conv2_fwd");
  return SEED_OK;
}

// FC + LSTM core + heads over the flattened torso output w.act2 (H2-H4)
static seed_status core_forward(const StepCtx& c, const seed_batch* bt, const bf16* lowp,
                                const float* params, cudaStream_t st) {
  const NetPlan& p = *c.p;
  const LearnerWs& w = c.w;
  const int F = w.F;
  {
    FcFwd pr{};
    pr.M = F; pr.N = 256; pr.K = p.fc_in; pr.Kxp = p.Kxp;
    pr.act2 = c.at<bf16>(w.act2); pr.w = lowp + p.im_fc;
    pr.bias = params + p.t[p.i_fcb].off; pr.X = c.at<bf16>(w.X);
    SEED_TRY(gemm<128>(c, pr, st, "fc_fwd"));
  }
  SEED_TRY(const_cast<StepCtx&>(c).edge(c.aux, st));   // join: X extras written
  {
    XprojFwd pr{};
    pr.M = F; pr.N = 4 * p.U; pr.K = p.Kxp;
    pr.X = c.at<bf16>(w.X); pr.w = lowp + p.im_wx;
    pr.bias = params + p.t[p.i_lb].off; pr.out = c.at<float>(w.xproj);
    SEED_TRY(gemm<128>(c, pr, st, "xproj_fwd"));
  }
  LstmFwdArgs la{};
  la.B = w.B; la.T1 = w.T1;
  la.xproj = c.at<float>(w.xproj);
  la.wh = lowp + p.im_wh;
  la.h0 = bt->h0; la.c0 = bt->c0; la.state_rows = nullptr;
  la.done = bt->done;
  la.H = c.at<float>(w.H); la.Hb = nullptr; la.Hprev = c.at<bf16>(w.Hprev);
  la.gates = c.at<float>(w.gates); la.C = c.at<float>(w.Cst);
  la.hT = la.cT = nullptr;
  SEED_TRY(lstm_forward(la, st));
  c.mark("lstm_fwd");
  return SEED_OK;   // the heads run inside the fused loss kernel
}

// heads + LSTM backward + FC backward, ending with w.dY2 = d(act2) (H8, H9 part)
static seed_status core_backward(const StepCtx& c, const seed_batch* bt, const bf16* lowp,
                                    const float* params, float* grads, cudaStream_t st) {
  const NetPlan& p = *c.p;
  const LearnerWs& w = c.w;
  const int F = w.F, U = p.U;
  // (heads backward: dH and the heads gradients come from the fused loss kernel)
  // LSTM BPTT
  LstmBwdArgs lb{};
  lb.B = w.B; lb.T1 = w.T1; lb.wh = lowp + p.im_wh;
  lb.gates = c.at<float>(w.gates); lb.C = c.at<float>(w.Cst); lb.c0 = bt->c0;
  lb.done = bt->done; lb.dH = c.at<float>(w.dH); lb.dG = c.at<bf16>(w.dG);
  SEED_TRY(lstm_backward(lb, st));
  c.mark("lstm_bwd");
  StepCtx& cc = const_cast<StepCtx&>(c);
  cudaStream_t ax = c.aux;
  // branch: LSTM weight gradient (aux) || FC input gradient (main)
  SEED_TRY(cc.edge(st, ax));
  {
    LstmWgrad pr{};
    pr.M = 4 * U; pr.N = p.Kxp + U; pr.K = F;
    pr.Kx = p.Kx; pr.Kxp = p.Kxp; pr.U = U;
    pr.dG = c.at<bf16>(w.dG); pr.X = c.at<bf16>(w.X); pr.Hprev = c.at<bf16>(w.Hprev);
    pr.g_wx = grads + p.t[p.i_wx].off; pr.g_b = grads + p.t[p.i_lb].off;
    pr.g_wh = grads + p.t[p.i_wh].off;
    SEED_TRY(gemm<128>(c, pr, ax, "lstm_wgrad"));
  }
  // LSTM + heads gradients are final: first DP bucket
  if (dp_buckets() >= 3) SEED_TRY(cc.bucket(grads + p.t[p.i_wx].off, p.P - p.t[p.i_wx].off, ax));
  {
    DxFc pr{};
    pr.M = F; pr.N = 256; pr.K = 4 * U; pr.Kxp = p.Kxp;
    pr.dG = c.at<bf16>(w.dG); pr.wx = lowp + p.im_wx; pr.X = c.at<bf16>(w.X);
    pr.dfc = c.at<bf16>(w.dfc);
    SEED_TRY(gemm<128>(c, pr, st, "dx_fc"));
  }
  // branch: FC weight gradient (aux, after the LSTM weight gradient) || FC data gradient (main)
  SEED_TRY(cc.edge(st, ax));
  {
    FcWgrad pr{};
    pr.M = 256; pr.N = p.fc_in + 8; pr.K = F; pr.fc_in = p.fc_in;
    pr.dfc = c.at<bf16>(w.dfc); pr.act2 = c.at<bf16>(w.act2);
    pr.g_w = grads + p.t[p.i_fcw].off; pr.g_b = grads + p.t[p.i_fcb].off;
    SEED_TRY(gemm<128>(c, pr, ax, "fc_wgrad"));
  }
  // FC gradients final: second bucket
  if (dp_buckets() >= 3) SEED_TRY(cc.bucket(grads + p.t[p.i_fcw].off, p.t[p.i_wx].off - p.t[p.i_fcw].off, ax));
  else if (dp_buckets() == 2) SEED_TRY(cc.bucket(grads + p.t[p.i_fcw].off, p.P - p.t[p.i_fcw].off, ax));
  {
    FcDgrad pr{};
    pr.M = F; pr.N = p.fc_in; pr.K = 256;
    pr.dfc = c.at<bf16>(w.dfc); pr.w = lowp + p.im_fc; pr.act2 = c.at<bf16>(w.act2);
    pr.dY2 = c.at<bf16>(w.dY2);
    if (p.nsec == 0) {   // Atari-shallow: conv2 output space rows (conv_s2d.cuh)
      const ShallowS2d sg = shallow_s2d_geometry(p.H, p.W, p.C);
      pr.dY2s = c.at<uint8_t>(w.dY2); pr.Wo = sg.g2.Wo; pr.W2s = sg.g2.Ws; pr.P2 = sg.g2.P;
      pr.g0 = 0;
    } else {             // IMPALA-deep: the last section's padded rows (conv3w.cuh)
      const DeepSec& d = p.sec[p.nsec - 1];
      const PadGeo g = PadGeo::make(d.H2, d.W2);
      pr.dY2s = c.at<uint8_t>(w.dY2); pr.Wo = d.W2; pr.W2s = g.Wp; pr.P2 = g.P; pr.g0 = g.Wp + 1;
      pr.CH = d.ch;
      // border rows are the next convs' zero padding; the GEMM writes interior rows only
      SEED_CUDA_TRY(cudaMemsetAsync(pr.dY2s, 0, (size_t)w.F * g.P * d.ch * 2, st));
    }
    SEED_TRY(gemm<128>(c, pr, st, "fc_dgrad"));
  }
  return SEED_OK;
}

// Atari-shallow torso backward from w.dY2 (H9): dW2|db2, dY1 (masked), dW1|db1
static seed_status shallow_backward(const StepCtx& c, const seed_batch* bt, const bf16* lowp,
                                    const float* params, float* grads, cudaStream_t st) {
  const NetPlan& p = *c.p;
  const LearnerWs& w = c.w;
  const int F = w.F;
  const ShallowS2d sg = shallow_s2d_geometry(p.H, p.W, p.C);
  StepCtx& cc = const_cast<StepCtx&>(c);
  cudaStream_t ax = c.aux;
  // branch: conv2 weight gradient (aux; needs dY2) || conv2 data + conv1 weight gradients (main)
  SEED_TRY(cc.edge(st, ax));
  float* part2 = ax != st ? c.at<float>(w.splitk2) : c.at<float>(w.splitk);
  SEED_TRY(shallow_s2d_conv2_wgrad(sg, F, c.at<uint8_t>(w.act1), c.at<uint8_t>(w.dY2), part2,
                                   grads + p.t[p.i_conv2w].off, grads + p.t[p.i_conv2b].off, ax));
  c.mark("conv2_wgrad", 2);
  SEED_TRY(shallow_s2d_conv2_dgrad(sg, F, c.at<uint8_t>(w.dY2), lowp + p.im_conv2dg,
                                   c.at<uint8_t>(w.act1), c.at<uint8_t>(w.dY1), st));
  c.mark("conv2_dgrad");
  SEED_TRY(shallow_s2d_conv1_wgrad(sg, F, c.at<uint8_t>(w.obs_bf16), c.at<uint8_t>(w.dY1),
                                   c.at<float>(w.splitk), grads + p.t[p.i_conv1w].off,
                                   grads + p.t[p.i_conv1b].off, st));
  c.mark("conv1_wgrad", 2);
  return SEED_OK;
}

// ------------------------------------------------------------------ IMPALA-deep torso
// conv3w.cuh: every activation in its padded row space (zero borders), 3x3
// convs as shifted-window tcgen05 GEMMs, bias gradients from the weight-gradient
// engine's all-ones operand.
// Section 0 reads the uint8 obs directly (converted to bf16 rows in shared memory,
// XF_U8) when they are 16 planes (GRF SMM); other inputs (DMLab RGB: the x-im2col
// rows) go through one conversion pass.  (Applying the residual stream's relu in
// shared memory instead of storing hr = relu(h), XF_RELU, was measured and is not
// used: the 16/32-channel convs are bound by shared-memory operand reads, and the
// in-place pass cost them more than the saved HBM writes: profiles/r02/xf_modes.md.)
// Measured slower (conv_fwd s0 432 -> 839 us, conv_wgrad s0 410 -> 938 us with the
// obs_bf16 pass (235 us) gone: the 16-channel convs are bound by shared-memory
// operand reads and the expansion's staging traffic and ALU work land on the same
// SMs; profiles/r02/xf_modes.md), so it is opt-in: SEED_XF_U8=1 (A/B measurement;
// parity-tested in tests/test_gpu_learner.py::test_learner_c4_u8_source_parity).
static bool deep_u8_input(const NetPlan& p) {
  static const bool on = [] {
    const char* e = getenv("SEED_XF_U8");
    return e && e[0] == '1';
  }();
  return on && !p.sec[0].xim && p.C == 16 && p.sec[0].cinp == 16;
}

// Section conv + max-pool fused (conv3w_pool.cu; the full-resolution conv output
// is not stored) unless SEED_FUSE_POOL=0 (A/B measurement).  SEED_STORE_CONV=1
// (read per call: the parity tests flip it) makes the fused kernel also write
// the conv rows to the workspace's "s<k>.conv" buffer.
static bool fuse_conv_pool() {
  static const bool on = [] {
    const char* e = getenv("SEED_FUSE_POOL");
    return !(e && e[0] == '0');
  }();
  return on;
}
static bool store_conv_rows() {
  const char* e = getenv("SEED_STORE_CONV");
  return e && e[0] == '1';
}

// ---- 128-channel sections (DMLab 4x torso): two 64-channel planes per tensor
// (conv3w.cuh); every conv is the plane-pair 64 -> 64 convs, the first input plane's
// fp32 sum carried to the second (W3_PART / D3W_PART, workspace part3).
static uint8_t* plane_at(const StepCtx& c, size_t off, int q, int64_t rows) {
  return c.at<uint8_t>(off) + (size_t)q * rows * 128;   // 64 bf16 channels per row
}
static int64_t w3_sub(const DeepSec& d, int mode, bool res) {
  const int ci = res ? d.ch : d.cin;
  const int rb = 2 * std::min(mode == 1 ? d.ch : (res ? d.ch : d.cinp), 64);
  return win3p_sub_elems(mode, ci, d.ch, rb);
}

static seed_status plane_section_forward(const StepCtx& c, int s, const bf16* lowp, const float* params,
                                         cudaStream_t st) {
  const NetPlan& p = *c.p;
  const LearnerWs& w = c.w;
  const int64_t F = w.F;
  const DeepSec& d = p.sec[s];
  const LearnerWs::Sec& b = w.sec[s];
  const PadGeo gi = PadGeo::make(d.H, d.W), go = PadGeo::make(d.H2, d.W2);
  const int64_t ri = F * gi.P, ro = F * go.P;
  const int npo = d.ch > 64 ? 2 : 1, npi = d.cinp > 64 ? 2 : 1;
  const int cpi = std::min(d.cinp, 64);
  float* part = c.at<float>(w.part3);
  if (d.xim || !part) return SEED_E_UNSUPPORTED;
  for (int q = 0; q < npo; ++q) {
    for (int pi = 0; pi < npi; ++pi) {
      Conv3wFwd a{};
      a.mode = pi + 1 < npi ? W3_PART : W3_PLAIN; a.cin_p = cpi; a.ch = 64; a.g = gi; a.rows = ri;
      a.in_scale = 1.f;
      a.in = npi > 1 ? plane_at(c, w.sec[s - 1].h[2], pi, ri) : c.at<uint8_t>(w.sec[s - 1].h[2]);
      a.wimg = lowp + d.im_w + (q * npi + pi) * w3_sub(d, 0, false);
      a.bias = params + p.t[d.t_b].off + 64 * q;
      a.out = plane_at(c, b.conv, q, ri);
      a.part_out = part; a.part_in = pi > 0 ? part : nullptr;
      SEED_TRY(conv3w_forward(a, st));
      c.mark("deep_conv_fwd");
    }
    SEED_TRY(conv3w_pool_fwd(F, gi, go, 64, d.pt, d.pl, plane_at(c, b.conv, q, ri), plane_at(c, b.h[0], q, ro),
                             plane_at(c, b.hr[0], q, ro), c.at<uint8_t>(b.arg) + (size_t)q * ro * 64, st));
    c.mark("deep_pool_fwd");
  }
  for (int r = 0; r < 2; ++r) {
    for (int j = 0; j < 2; ++j)   // conv0: relu(h) -> u1 (W3_RELU); conv1: u1 -> h + conv (W3_RES)
      for (int q = 0; q < npo; ++q)
        for (int pi = 0; pi < npo; ++pi) {
          Conv3wFwd a{};
          a.mode = pi + 1 < npo ? W3_PART : (j == 0 ? W3_RELU : W3_RES);
          a.cin_p = 64; a.ch = 64; a.g = go; a.rows = ro; a.in_scale = 1.f;
          a.in = plane_at(c, j == 0 ? b.hr[r] : b.u1[r], pi, ro);
          a.wimg = lowp + d.im_rw[r][j] + (q * npo + pi) * w3_sub(d, 0, true);
          a.bias = params + p.t[d.t_rb[r][j]].off + 64 * q;
          a.part_out = part; a.part_in = pi > 0 ? part : nullptr;
          if (j == 0) {
            a.out = plane_at(c, b.u1[r], q, ro);
          } else {
            a.res = plane_at(c, b.h[r], q, ro);
            a.out = plane_at(c, b.h[r + 1], q, ro); a.outr = plane_at(c, b.hr[r + 1], q, ro);
            if (s == p.nsec - 1 && r == 1) { a.dense = c.at<bf16>(w.act2); a.dense_ct = d.ch; a.dense_off = 64 * q; }
          }
          SEED_TRY(conv3w_forward(a, st));
          c.mark(j == 0 ? "deep_res_fwd0" : "deep_res_fwd1");
        }
  }
  return SEED_OK;
}

static seed_status plane_section_backward(const StepCtx& c, int s, const bf16* lowp, const float* params,
                                          float* grads, cudaStream_t st) {
  const NetPlan& p = *c.p;
  const LearnerWs& w = c.w;
  const int64_t F = w.F;
  const DeepSec& d = p.sec[s];
  const LearnerWs::Sec& b = w.sec[s];
  const PadGeo gi = PadGeo::make(d.H, d.W), go = PadGeo::make(d.H2, d.W2);
  const int64_t ri = F * gi.P, ro = F * go.P;
  const int npo = d.ch > 64 ? 2 : 1, npi = d.cinp > 64 ? 2 : 1;
  const int cpi = std::min(d.cinp, 64);
  float* part = c.at<float>(w.part3);
  float* wpart = c.at<float>(w.splitk);
  size_t cur = b.dhA, oth = b.dhB;
  auto wgrad = [&](const uint8_t* X, int xplanes, int cinp, const uint8_t* dY, int64_t rows, const PadGeo& g,
                   int ci_full, int ti_w, int ti_b, const char* name) -> seed_status {
    for (int q = 0; q < npo; ++q)
      for (int pi = 0; pi < xplanes; ++pi) {
        Conv3wWgrad wg{};
        wg.cin_p = cinp; wg.cin = cinp; wg.ch = 64; wg.g = g; wg.rows = rows; wg.scale = 1.f;
        wg.X = X + (size_t)pi * rows * 2 * cinp; wg.dY = dY + (size_t)q * rows * 128; wg.part = wpart;
        wg.g_w = grads + p.t[ti_w].off; wg.ci_full = ci_full; wg.co_off = 64 * q; wg.c_off = cinp * pi;
        wg.g_b = pi == 0 ? grads + p.t[ti_b].off + 64 * q : nullptr;
        SEED_TRY(conv3w_wgrad(wg, st));
        c.mark(name, 2);
      }
    return SEED_OK;
  };
  // dX plane pi = sum over dY planes q (D3W_PART then the final mode)
  auto dgrad = [&](int mode, const uint8_t* dY, int64_t rows, const PadGeo& g, int64_t im, int64_t sub,
                   int xplanes, const uint8_t* mask, const uint8_t* dres, uint8_t* dX, const char* name) -> seed_status {
    for (int pi = 0; pi < xplanes; ++pi)
      for (int q = 0; q < npo; ++q) {
        Conv3wDgrad dg{};
        dg.mode = q + 1 < npo ? D3W_PART : mode; dg.cin = 64; dg.ch = 64; dg.g = g; dg.rows = rows;
        dg.dY = dY + (size_t)q * rows * 128; dg.wimg = lowp + im + (q * xplanes + pi) * sub;
        dg.mask = mask ? mask + (size_t)pi * rows * 128 : nullptr;
        dg.dres = dres ? dres + (size_t)pi * rows * 128 : nullptr;
        dg.dX = dX + (size_t)pi * rows * 128;
        dg.part_out = part; dg.part_in = q > 0 ? part : nullptr;
        SEED_TRY(conv3w_dgrad(dg, st));
        c.mark(name);
      }
    return SEED_OK;
  };
  for (int r = 1; r >= 0; --r) {
    SEED_TRY(wgrad(c.at<uint8_t>(b.u1[r]), npo, 64, c.at<uint8_t>(cur), ro, go, d.ch, d.t_rw[r][1], d.t_rb[r][1],
                   "deep_res_wgrad1"));
    SEED_TRY(dgrad(D3W_MASK, c.at<uint8_t>(cur), ro, go, d.im_rdg[r][1], w3_sub(d, 1, true), npo,
                   c.at<uint8_t>(b.u1[r]), nullptr, c.at<uint8_t>(b.dt0), "deep_res_dgrad1"));
    SEED_TRY(wgrad(c.at<uint8_t>(b.hr[r]), npo, 64, c.at<uint8_t>(b.dt0), ro, go, d.ch, d.t_rw[r][0], d.t_rb[r][0],
                   "deep_res_wgrad0"));
    SEED_TRY(dgrad(D3W_RES, c.at<uint8_t>(b.dt0), ro, go, d.im_rdg[r][0], w3_sub(d, 1, true), npo,
                   c.at<uint8_t>(b.hr[r]), c.at<uint8_t>(cur), c.at<uint8_t>(oth), "deep_res_dgrad0"));
    std::swap(cur, oth);
  }
  for (int q = 0; q < npo; ++q) {
    SEED_TRY(conv3w_pool_bwd(F, gi, go, 64, d.pt, d.pl, plane_at(c, cur, q, ro),
                             c.at<uint8_t>(b.arg) + (size_t)q * ro * 64, plane_at(c, b.dconv, q, ri), st));
    c.mark("deep_pool_bwd");
  }
  if (s == 0 || d.xim) return SEED_E_UNSUPPORTED;   // plane sections follow a 64-channel section
  SEED_TRY(wgrad(c.at<uint8_t>(w.sec[s - 1].h[2]), npi, cpi, c.at<uint8_t>(b.dconv), ri, gi, d.cin, d.t_w, d.t_b,
                 "deep_conv_wgrad"));
  SEED_TRY(dgrad(D3W_PLAIN, c.at<uint8_t>(b.dconv), ri, gi, d.im_dg, w3_sub(d, 1, false), npi, nullptr, nullptr,
                 c.at<uint8_t>(w.sec[s - 1].dhA), "deep_conv_dgrad"));
  return SEED_OK;
}

static seed_status deep_forward(const StepCtx& c, const seed_batch* bt, const bf16* lowp,
                                const float* params, cudaStream_t st) {
  const NetPlan& p = *c.p;
  const LearnerWs& w = c.w;
  const int64_t F = w.F;
  const bool u8in = deep_u8_input(p);
  if (!u8in) {
    const DeepSec& d = p.sec[0];
    SEED_TRY(conv3_obs((const uint8_t*)bt->obs, F, PadGeo::make(d.H, d.W), p.C, d.cinp, d.xim,
                       c.at<uint8_t>(w.obs_bf16), st));
    c.mark("obs_bf16");
  }
  for (int s = 0; s < p.nsec; ++s) {
    const DeepSec& d = p.sec[s];
    const LearnerWs::Sec& b = w.sec[s];
    const PadGeo gi = PadGeo::make(d.H, d.W), go = PadGeo::make(d.H2, d.W2);
    if (d.ch > 64) {
      SEED_TRY(plane_section_forward(c, s, lowp, params, st));
      continue;
    }
    Conv3wFwd a{};
    a.mode = W3_PLAIN; a.cin_p = d.cinp; a.ch = d.ch; a.xim = d.xim; a.g = gi; a.rows = F * gi.P;
    a.in_scale = s == 0 ? 1.f / 255.f : 1.f;
    a.in = s == 0 ? c.at<uint8_t>(w.obs_bf16) : c.at<uint8_t>(w.sec[s - 1].h[2]);
    if (s == 0 && u8in) {
      a.xf = XF_U8;
      a.obs_u8 = (const uint8_t*)bt->obs;
    }
    a.wimg = lowp + d.im_w; a.bias = params + p.t[d.t_b].off; a.out = c.at<uint8_t>(b.conv);
    seed_status fs = SEED_E_UNSUPPORTED;
    if (fuse_conv_pool() && a.xf == XF_NONE) {
      fs = conv3w_conv_pool(a, go, d.pt, d.pl, c.at<uint8_t>(b.h[0]), c.at<uint8_t>(b.hr[0]),
                            c.at<uint8_t>(b.arg), store_conv_rows() ? c.at<uint8_t>(b.conv) : nullptr, st);
      if (fs != SEED_E_UNSUPPORTED) SEED_TRY(fs);
      if (fs == SEED_OK) c.mark("deep_conv_pool");
    }
    if (fs == SEED_E_UNSUPPORTED) {
      SEED_TRY(conv3w_forward(a, st));
      c.mark("deep_conv_fwd");
      SEED_TRY(conv3w_pool_fwd(F, gi, go, d.ch, d.pt, d.pl, c.at<uint8_t>(b.conv),
                               c.at<uint8_t>(b.h[0]), c.at<uint8_t>(b.hr[0]), c.at<uint8_t>(b.arg),
                               st));
      c.mark("deep_pool_fwd");
    }
    for (int r = 0; r < 2; ++r) {
      Conv3wFwd a0{};
      a0.mode = W3_RELU; a0.cin_p = d.ch; a0.ch = d.ch; a0.g = go; a0.rows = F * go.P;
      a0.in_scale = 1.f; a0.in = c.at<uint8_t>(b.hr[r]); a0.wimg = lowp + d.im_rw[r][0];
      a0.bias = params + p.t[d.t_rb[r][0]].off; a0.out = c.at<uint8_t>(b.u1[r]);
      SEED_TRY(conv3w_forward(a0, st));
      c.mark("deep_res_fwd0");
      Conv3wFwd a1 = a0;
      a1.mode = W3_RES; a1.xf = XF_NONE; a1.in = c.at<uint8_t>(b.u1[r]); a1.wimg = lowp + d.im_rw[r][1];
      a1.bias = params + p.t[d.t_rb[r][1]].off; a1.res = c.at<uint8_t>(b.h[r]);
      a1.out = c.at<uint8_t>(b.h[r + 1]); a1.outr = c.at<uint8_t>(b.hr[r + 1]);
      a1.dense = (s == p.nsec - 1 && r == 1) ? c.at<bf16>(w.act2) : nullptr;
      SEED_TRY(conv3w_forward(a1, st));
      c.mark("deep_res_fwd1");
    }
  }
  return SEED_OK;
}

static seed_status deep_backward(const StepCtx& c, const seed_batch* bt, const bf16* lowp,
                                 const float* params, float* grads, cudaStream_t st) {
  const NetPlan& p = *c.p;
  const LearnerWs& w = c.w;
  const int64_t F = w.F;
  float* part = c.at<float>(w.splitk);
  for (int s = p.nsec - 1; s >= 0; --s) {
    const DeepSec& d = p.sec[s];
    const LearnerWs::Sec& b = w.sec[s];
    const PadGeo gi = PadGeo::make(d.H, d.W), go = PadGeo::make(d.H2, d.W2);
    if (d.ch > 64) {
      SEED_TRY(plane_section_backward(c, s, lowp, params, grads, st));
      continue;
    }
    const int64_t Mr = F * go.P;
    size_t cur = b.dhA, oth = b.dhB;   // dh of h[2] arrives in dhA
    for (int r = 1; r >= 0; --r) {
      // t1 = conv1(u1): dt1 = dh
      Conv3wWgrad wg{};
      wg.cin_p = d.ch; wg.cin = d.ch; wg.ch = d.ch; wg.g = go; wg.rows = Mr; wg.scale = 1.f;
      wg.X = c.at<uint8_t>(b.u1[r]); wg.dY = c.at<uint8_t>(cur); wg.part = part;
      wg.g_w = grads + p.t[d.t_rw[r][1]].off; wg.g_b = grads + p.t[d.t_rb[r][1]].off;
      SEED_TRY(conv3w_wgrad(wg, st));
      c.mark("deep_res_wgrad1", 2);
      Conv3wDgrad dg{};
      dg.mode = D3W_MASK; dg.cin = d.ch; dg.ch = d.ch; dg.g = go; dg.rows = Mr;
      dg.dY = c.at<uint8_t>(cur); dg.wimg = lowp + d.im_rdg[r][1]; dg.mask = c.at<uint8_t>(b.u1[r]);
      dg.dX = c.at<uint8_t>(b.dt0);
      SEED_TRY(conv3w_dgrad(dg, st));
      c.mark("deep_res_dgrad1");
      // t0 = conv0(relu(h[r])): dh[r] = dh + dconv0 * (h[r] > 0)
      wg.X = c.at<uint8_t>(b.hr[r]); wg.dY = c.at<uint8_t>(b.dt0);
      wg.g_w = grads + p.t[d.t_rw[r][0]].off; wg.g_b = grads + p.t[d.t_rb[r][0]].off;
      SEED_TRY(conv3w_wgrad(wg, st));
      c.mark("deep_res_wgrad0", 2);
      Conv3wDgrad d0 = dg;
      d0.mode = D3W_RES; d0.dY = c.at<uint8_t>(b.dt0); d0.wimg = lowp + d.im_rdg[r][0];
      d0.mask = c.at<uint8_t>(b.hr[r]); d0.dres = c.at<uint8_t>(cur); d0.dX = c.at<uint8_t>(oth);
      SEED_TRY(conv3w_dgrad(d0, st));
      c.mark("deep_res_dgrad0");
      std::swap(cur, oth);
    }
    // max-pool backward into dconv, then the section conv
    SEED_TRY(conv3w_pool_bwd(F, gi, go, d.ch, d.pt, d.pl, c.at<uint8_t>(cur), c.at<uint8_t>(b.arg),
                             c.at<uint8_t>(b.dconv), st));
    c.mark("deep_pool_bwd");
    Conv3wWgrad wg{};
    wg.cin_p = d.cinp; wg.cin = d.cin; wg.ch = d.ch; wg.xim = d.xim; wg.g = gi; wg.rows = F * gi.P;
    wg.scale = s == 0 ? 1.f / 255.f : 1.f;
    wg.X = s == 0 ? c.at<uint8_t>(w.obs_bf16) : c.at<uint8_t>(w.sec[s - 1].h[2]);
    if (s == 0 && deep_u8_input(p)) {
      wg.xf = XF_U8;
      wg.obs_u8 = (const uint8_t*)bt->obs;
    }
    wg.dY = c.at<uint8_t>(b.dconv); wg.part = part;
    wg.g_w = grads + p.t[d.t_w].off; wg.g_b = grads + p.t[d.t_b].off;
    SEED_TRY(conv3w_wgrad(wg, st));
    c.mark("deep_conv_wgrad", 2);
    if (s > 0) {
      Conv3wDgrad dg{};
      dg.mode = D3W_PLAIN; dg.cin = d.cin; dg.ch = d.ch; dg.g = gi; dg.rows = F * gi.P;
      dg.dY = c.at<uint8_t>(b.dconv); dg.wimg = lowp + d.im_dg;
      dg.dX = c.at<uint8_t>(w.sec[s - 1].dhA);
      SEED_TRY(conv3w_dgrad(dg, st));
      c.mark("deep_conv_dgrad");
    }
  }
  return SEED_OK;
}

static seed_status mlp_forward(const StepCtx& c, const seed_batch* bt, const float* params,
                               cudaStream_t st) {
  const NetPlan& p = *c.p;
  const LearnerWs& w = c.w;
  const int F = w.F;
  SEED_TRY(launch_dense_fwd(F, p.D, 64, (const float*)bt->obs, params + p.t[p.i_m0w].off,
                            params + p.t[p.i_m0b].off, c.at<float>(w.h1), 64, nullptr, 1, st));
  SEED_TRY(launch_dense_fwd(F, 64, 64, c.at<float>(w.h1), params + p.t[p.i_m1w].off,
                            params + p.t[p.i_m1b].off, c.at<float>(w.h2), 64, nullptr, 1, st));
  c.mark("mlp_fwd", 2);   // the heads run inside the fused loss kernel
  return last_launch();
}

static seed_status mlp_backward(const StepCtx& c, const seed_batch* bt, const float* params,
                                float* grads, cudaStream_t st) {
  const NetPlan& p = *c.p;
  const LearnerWs& w = c.w;
  const int F = w.F;
  // dh2 (masked) and the heads gradients come from the fused loss kernel
  SEED_TRY(launch_dense_dgrad(F, 64, 64, c.at<float>(w.dh2), 64, nullptr,
                              params + p.t[p.i_m1w].off, c.at<float>(w.h1), c.at<float>(w.dh1), st));
  dense_wgrad_f32<<<dim3(64, ceil_div(65, 32)), 256, 0, st>>>(
      F, 64, 64, c.at<float>(w.dh2), 64, nullptr, c.at<float>(w.h1), grads + p.t[p.i_m1w].off,
      grads + p.t[p.i_m1b].off);
  dense_wgrad_f32<<<dim3(64, ceil_div(p.D + 1, 32)), 256, 0, st>>>(
      F, p.D, 64, c.at<float>(w.dh1), 64, nullptr, (const float*)bt->obs,
      grads + p.t[p.i_m0w].off, grads + p.t[p.i_m0b].off);
  c.mark("mlp_bwd", 3);
  return last_launch();
}



static seed_status learner_step_impl(const seed_net_spec* spec, int T, int B,
                                     const seed_batch* batch, const seed_train_state* state,
                                     const seed_hparams* hp, seed_comm* comm, const seed_exec* ex,
                                     void* ws, size_t ws_bytes, float* metrics, void* stream,
                                     Trace* tr) {
  NetPlan p;
  SEED_TRY(make_net_plan(spec, &p));
  if (!learner_supported(p)) return SEED_E_UNSUPPORTED;
  if (T < 1 || T > 256 || B < 1 || B > 1024) return SEED_E_SHAPE;
  if (!batch || !state || !hp || !ws || !metrics) return SEED_E_ARG;
  if (!batch->obs || !batch->action || !batch->reward || !batch->done || !batch->behaviour_logp ||
      !state->params || !state->grads || !state->adam_m || !state->adam_v || !state->step)
    return SEED_E_ARG;
  // fp32 master / grads / moments are read and written with float4 accesses
  if (!aligned16(state->params) || !aligned16(state->grads) || !aligned16(state->adam_m) ||
      !aligned16(state->adam_v) || !aligned16(ws))
    return SEED_E_ARG;
  if (p.kind != SEED_NET_MLP &&
      (!batch->prev_action || !batch->h0 || !batch->c0 || !state->params_lowp ||
       !aligned16(batch->obs) || !aligned16(state->params_lowp)))
    return SEED_E_ARG;
  if (!(hp->c_bar > 0.f) || !(hp->rho_bar >= hp->c_bar) || !(hp->lambda >= 0.f && hp->lambda <= 1.f) ||
      !(hp->max_grad_norm > 0.f))
    return SEED_E_ARG;
  StepCtx c;
  c.p = &p;
  SEED_TRY(make_learner_ws(p, T, B, &c.w));
  if (ws_bytes < c.w.total) return SEED_E_WORKSPACE;
  c.ws = (uint8_t*)ws;
  c.g = Geo{p.H, p.W, p.C, p.oh1, p.ow1, p.oh2, p.ow2, p.fc_in, p.Kx, p.Kxp,
             FastDiv((uint32_t)(p.oh1 * p.ow1)), FastDiv((uint32_t)p.ow1),
             FastDiv((uint32_t)(p.oh2 * p.ow2)), FastDiv((uint32_t)p.ow2)};
  cudaStream_t st = (cudaStream_t)stream;
  c.st = st;
  c.tr = tr;
  if (tr && tr->events && tr->max > 0) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    tr->capturing = cs == cudaStreamCaptureStatusActive;
    trace_record(tr, tr->events[0], st);
    if (tr->names) tr->names[0] = "begin";
    tr->n = 1;
  }
  const float* params = state->params;
  const bf16* lowp = (const bf16*)state->params_lowp;
  float* grads = state->grads;
  // column-sum completion ticket (re-armed by the kernel after each use)
  SEED_CUDA_TRY(cudaMemsetAsync(c.tickets(), 0, 64 + GEMM_COUNTERS * 4, st));

  if (p.kind == SEED_NET_MLP) {
    SEED_TRY(mlp_forward(c, batch, params, st));
  } else {
    SEED_TRY(aux_stream(ex, st, tr != nullptr, &c.aux, c.fev));
    // the LSTM-input extras (one-hot, reward, ones column) only read the batch:
    // an aux-stream branch beside the torso, joined before the input projection
    SEED_TRY(c.edge(st, c.aux));
    {
      const int E = p.Kxp - 256;
      const int64_t n = (int64_t)c.w.F * E;
      SEED_TRY(launch_k(core_extras_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, c.aux,
                        c.w.F, p.A, p.Kxp, batch->prev_action, batch->reward, batch->done,
                        c.at<bf16>(c.w.X)));
      c.mark("core_extras");
    }
    if (p.nsec > 0) SEED_TRY(deep_forward(c, batch, lowp, params, st));
    else SEED_TRY(shallow_forward(c, batch, lowp, params, st));
    SEED_TRY(core_forward(c, batch, lowp, params, st));
  }

  LossArgs la{};
  la.B = B; la.T = T; la.A = p.A;
  la.logits = c.at<float>(c.w.logits); la.values = c.at<float>(c.w.values);
  la.action = batch->action; la.blp = batch->behaviour_logp; la.reward = batch->reward;
  la.done = batch->done;
  la.discount = hp->discount; la.rho_bar = hp->rho_bar; la.c_bar = hp->c_bar;
  la.lam = hp->lambda; la.vf_coef = hp->vf_coef; la.ent_coef = hp->ent_coef;
  la.scale = hp->loss_scale;
  la.dlogits = c.at<float>(c.w.dlogits); la.dvalues = c.at<float>(c.w.dvalues);
  la.vs = c.at<float>(c.w.vs); la.pg = c.at<float>(c.w.pg); la.part = c.at<float>(c.w.loss_part);
  // heads forward + loss + heads backward (one kernel, then the weight-gradient sum)
  const bool mlp = p.kind == SEED_NET_MLP;
  la.H = mlp ? c.at<float>(c.w.h2) : c.at<float>(c.w.H);
  la.I = mlp ? 64 : p.U;
  la.hw = params + p.t[p.i_hw].off; la.hb = params + p.t[p.i_hb].off;
  la.hmask = mlp ? c.at<float>(c.w.h2) : nullptr;
  la.dH = mlp ? c.at<float>(c.w.dh2) : c.at<float>(c.w.dH);
  la.wpart = c.at<float>(c.w.hpart);
  la.g_w = grads + p.t[p.i_hw].off; la.g_b = grads + p.t[p.i_hb].off;
  SEED_TRY(launch_heads_loss(la, st));
  c.mark("heads_loss", 2);

  const bool dp = comm && comm_world(comm) > 1;
  if (p.kind == SEED_NET_MLP) {
    SEED_TRY(mlp_backward(c, batch, params, grads, st));
    if (dp) {
      SEED_TRY(comm_allreduce(comm, grads, p.P, st));
      c.mark("allreduce");
    }
  } else {
    // H10 overlapped with the rest of the backward: three buckets (LSTM+heads
    // after the LSTM weight gradient, FC after its weight gradient, the torso at
    // the end) reduced on the comm's side stream, joined before the clip.
    if (dp) {
      c.comm = comm;
      SEED_TRY(comm_side(comm, &c.side, &c.side2, c.ev));
    }
    SEED_TRY(core_backward(c, batch, lowp, params, grads, st));
    if (p.nsec > 0) SEED_TRY(deep_backward(c, batch, lowp, params, grads, st));
    else SEED_TRY(shallow_backward(c, batch, lowp, params, grads, st));
    SEED_TRY(c.edge(c.aux, st));   // join the aux branch
    if (dp) {
      SEED_TRY(c.bucket(grads, dp_buckets() >= 2 ? p.t[p.i_fcw].off : p.P, st));
      SEED_CUDA_TRY(cudaEventRecord(c.ev[3], c.side));
      SEED_CUDA_TRY(cudaStreamWaitEvent(st, c.ev[3], 0));
      if (c.side2) {
        SEED_CUDA_TRY(cudaEventRecord(c.ev[4], c.side2));
        SEED_CUDA_TRY(cudaStreamWaitEvent(st, c.ev[4], 0));
      }
      c.mark("allreduce_tail");
    }
  }

  double* npart = c.at<double>(c.w.norm_part);
  NormArgs na{};
  na.g = grads; na.P = p.P; na.part = npart;
  na.coef = reinterpret_cast<float*>(npart + NORM_BLOCKS); na.norm = npart + NORM_BLOCKS + 2;
  na.ticket = c.tickets() + 1;
  na.step = state->step; na.step_in = c.at<int64_t>(c.w.step_in);
  na.beta1 = hp->beta1; na.beta2 = hp->beta2; na.max_norm = hp->max_grad_norm;
  SEED_TRY(launch_k(grad_norm_kernel, dim3(NORM_BLOCKS), dim3(256), 0, st, na));
  c.mark("grad_norm");
  AdamArgs aa{};
  aa.P = p.P; aa.params = state->params; aa.grads = grads; aa.m = state->adam_m;
  aa.v = state->adam_v; aa.step = state->step; aa.step_in = c.at<int64_t>(c.w.step_in);
  aa.coef = na.coef; aa.norm = na.norm;
  aa.lr = hp->lr; aa.beta1 = hp->beta1; aa.beta2 = hp->beta2; aa.eps = hp->eps;
  aa.max_norm = hp->max_grad_norm; aa.loss_part = c.at<float>(c.w.loss_part); aa.B = B;
  aa.metrics = metrics;
  aa.lowp = (bf16*)state->params_lowp;
  const bool fused_lowp = p.nimg <= 8;    // Adam writes the operand image itself
  aa.nimg = fused_lowp ? p.nimg : 0;
  for (int k = 0; k < aa.nimg; ++k) aa.img[k] = p.img[k];
  SEED_TRY(launch_clip_adam(aa, st));
  c.mark("clip_adam");
  if (!fused_lowp) {
    SEED_TRY(refresh_lowp(p, state->params, state->params_lowp, st));
    c.mark("lowp_refresh");
  }
  return last_launch();
}

}  // namespace seed

extern "C" seed_status seed_learner_step(const seed_net_spec* spec, int T, int B,
                                         const seed_batch* batch, const seed_train_state* state,
                                         const seed_hparams* hp, seed_comm* comm, void* ws,
                                         size_t ws_bytes, float* metrics, void* stream) {
  return seed::learner_step_impl(spec, T, B, batch, state, hp, comm, nullptr, ws, ws_bytes, metrics,
                                 stream, nullptr);
}

extern "C" seed_status seed_learner_step_ex(const seed_net_spec* spec, int T, int B,
                                            const seed_batch* batch, const seed_train_state* state,
                                            const seed_hparams* hp, seed_comm* comm, seed_exec* exec,
                                            void* ws, size_t ws_bytes, float* metrics, void* stream) {
  return seed::learner_step_impl(spec, T, B, batch, state, hp, comm, exec, ws, ws_bytes, metrics,
                                 stream, nullptr);
}

extern "C" seed_status seed_learner_step_traced(const seed_net_spec* spec, int T, int B,
                                                const seed_batch* batch,
                                                const seed_train_state* state,
                                                const seed_hparams* hp, seed_comm* comm,
                                                void* ws, size_t ws_bytes, float* metrics,
                                                void* stream, void** events, int max_events,
                                                const char** names_out, int* n_events_out,
                                                int* n_launches_out, int* launch_counts_out) {
  seed::Trace tr;
  tr.events = events;
  tr.names = names_out;
  tr.counts = launch_counts_out;
  tr.max = events ? max_events : 0;
  const seed_status r = seed::learner_step_impl(spec, T, B, batch, state, hp, comm, nullptr, ws,
                                                ws_bytes, metrics, stream, &tr);
  if (n_events_out) *n_events_out = tr.n;
  if (n_launches_out) *n_launches_out = tr.launches;
  return r;
}

namespace seed {

}  // namespace seed

using namespace seed;

extern "C" seed_status seed_learner_outputs(const seed_net_spec* spec, int T, int B, void* ws,
                                            float** logits, float** values, float** vs,
                                            float** pg) {
  NetPlan p;
  SEED_TRY(make_net_plan(spec, &p));
  if (!learner_supported(p)) return SEED_E_UNSUPPORTED;
  if (!ws) return SEED_E_ARG;
  LearnerWs w;
  SEED_TRY(make_learner_ws(p, T, B, &w));
  uint8_t* b = (uint8_t*)ws;
  if (logits) *logits = (float*)(b + w.logits);
  if (values) *values = (float*)(b + w.values);
  if (vs) *vs = (float*)(b + w.vs);
  if (pg) *pg = (float*)(b + w.pg);
  return SEED_OK;
}

extern "C" seed_status seed_learner_debug_buffer(const seed_net_spec* spec, int T, int B, void* ws,
                                                 const char* name, void** ptr, size_t* bytes) {
  NetPlan p;
  SEED_TRY(make_net_plan(spec, &p));
  if (!learner_supported(p)) return SEED_E_UNSUPPORTED;
  if (!ws || !name || !ptr) return SEED_E_ARG;
  LearnerWs w;
  SEED_TRY(make_learner_ws(p, T, B, &w));
  const size_t F = w.F, U = p.U;
  struct Ent { const char* n; size_t off, bytes; };
  const bool mlp = p.kind == SEED_NET_MLP;
  const Ent ents[] = {
      {"dlogits", w.dlogits, F * p.A * 4}, {"dvalues", w.dvalues, F * 4},
      {"act1", mlp ? 0 : w.act1, F * p.oh1 * p.ow1 * 16 * 2}, {"act2", mlp ? 0 : w.act2, F * p.fc_in * 2},
      {"X", mlp ? 0 : w.X, F * p.Kxp * 2}, {"xproj", mlp ? 0 : w.xproj, F * 4 * U * 4},
      {"H", mlp ? 0 : w.H, F * U * 4}, {"Hprev", mlp ? 0 : w.Hprev, F * U * 2},
      {"gates", mlp ? 0 : w.gates, F * 4 * U * 4}, {"C", mlp ? 0 : w.Cst, F * U * 4},
      {"dH", mlp ? 0 : w.dH, F * U * 4}, {"dG", mlp ? 0 : w.dG, F * 4 * U * 2},
      {"dfc", mlp ? 0 : w.dfc, F * 256 * 2}, {"dY2", mlp ? 0 : w.dY2, F * p.fc_in * 2},
      {"dY1", mlp ? 0 : w.dY1, F * p.oh1 * p.ow1 * 16 * 2},
      {"obs_bf16", w.obs_bf16, p.nsec > 0 ? F * (p.sec[0].H + 2) * (p.sec[0].W + 2) * p.sec[0].cinp * 2 : 16},
      {"h1", mlp ? w.h1 : 0, F * 64 * 4}, {"h2", mlp ? w.h2 : 0, F * 64 * 4},
      {"dh1", mlp ? w.dh1 : 0, F * 64 * 4}, {"dh2", mlp ? w.dh2 : 0, F * 64 * 4}};
  for (const Ent& e : ents)
    if (strcmp(e.n, name) == 0 && e.off) {
      *ptr = (uint8_t*)ws + e.off;
      if (bytes) *bytes = e.bytes;
      return SEED_OK;
    }
  // deep torso: "s<k>.<buf>" with buf in conv, arg, h0..h2, hr0..hr2, u10, u11, dconv, dhA, dhB, dt0
  if (p.nsec > 0 && name[0] == 's' && name[1] >= '0' && name[1] < '0' + p.nsec && name[2] == '.') {
    const int k = name[1] - '0';
    const DeepSec& d = p.sec[k];
    const LearnerWs::Sec& b = w.sec[k];
    // conv3w.cuh padded, pre-swizzled row spaces
    const size_t sc = F * (d.H + 2) * (d.W + 2) * d.ch * 2, sp = F * (d.H2 + 2) * (d.W2 + 2) * d.ch * 2;
    const char* bn = name + 3;
    struct E2 { const char* n; size_t off, bytes; };
    const E2 e2[] = {{"conv", b.conv, sc}, {"arg", b.arg, sp / 2}, {"h0", b.h[0], sp},
                     {"h1", b.h[1], sp}, {"h2", b.h[2], sp}, {"hr0", b.hr[0], sp},
                     {"hr1", b.hr[1], sp}, {"hr2", b.hr[2], sp}, {"u10", b.u1[0], sp},
                     {"u11", b.u1[1], sp}, {"dconv", b.dconv, sc}, {"dhA", b.dhA, sp},
                     {"dhB", b.dhB, sp}, {"dt0", b.dt0, sp}};
    for (const E2& e : e2)
      if (strcmp(e.n, bn) == 0) {
        *ptr = (uint8_t*)ws + e.off;
        if (bytes) *bytes = e.bytes;
        return SEED_OK;
      }
  }
  return SEED_E_ARG;
}

// ============================================================================
// R2D2 learner step (hyper-parameters
// P:586-622): burn-in, online / target forward passes, n-step double-Q targets
// with value rescaling and priorities (seed_r2d2_targets), dueling heads, the
// importance-weighted squared-TD backward, clip (80) + Adam.  The network is the
// configured one (seed_net_spec) with dueling heads read from its A+1 outputs:
// Q(a) = V + A_a - mean_j A_j (C35).
// ============================================================================
extern "C" seed_status seed_r2d2_targets(int T, int B, int A, int n, const float* q_online,
                                         const float* q_target, const int32_t* actions,
                                         const float* rewards, const float* discounts, float eta,
                                         float rescale_eps, const float* is_weights, float loss_scale,
                                         float* y, float* delta, float* priority, float* dq,
                                         float* loss_part, void* stream);

namespace seed {

// trained step t of a [B][T+1] window uses reward[t+1] and gamma (1 - done[t+1]) (C5)
__global__ void r2d2_rewards_kernel(int B, int T, float gamma, const float* __restrict__ reward,
                                    const uint8_t* __restrict__ done, float* __restrict__ r,
                                    float* __restrict__ disc) {
  pdl_wait_trig();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B * T) return;
  const int b = i / T, t = i % T;
  const int s = b * (T + 1) + t + 1;
  r[i] = reward[s];
  disc[i] = done[s] ? 0.f : gamma;
}

// dueling combine: Q[f][a] = V[f] + A[f][a] - mean_j A[f][j]  (warp per row)
__global__ void dueling_q_kernel(int F, int A, const float* __restrict__ adv, const float* __restrict__ val,
                                 float* __restrict__ q) {
  pdl_wait_trig();
  const int f = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (f >= F) return;
  float s = 0.f;
  for (int j = lane; j < A; j += 32) s += adv[(size_t)f * A + j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mean = s / (float)A, v = val[f];
  for (int j = lane; j < A; j += 32) q[(size_t)f * A + j] = v + adv[(size_t)f * A + j] - mean;
}

// its backward: dV = sum_a dQ_a, dA_j = dQ_j - (1/A) sum_a dQ_a
__global__ void dueling_bwd_kernel(int F, int A, const float* __restrict__ dq, float* __restrict__ dadv,
                                   float* __restrict__ dval) {
  pdl_wait_trig();
  const int f = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (f >= F) return;
  float s = 0.f;
  for (int j = lane; j < A; j += 32) s += dq[(size_t)f * A + j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  for (int j = lane; j < A; j += 32) dadv[(size_t)f * A + j] = dq[(size_t)f * A + j] - s / (float)A;
  if (lane == 0) dval[f] = s;
}

// last LSTM state of each burn-in window -> the trained window's initial state
__global__ void last_state_kernel(int B, int T1, int U, const float* __restrict__ H,
                                  const float* __restrict__ C, float* __restrict__ h0,
                                  float* __restrict__ c0) {
  pdl_wait_trig();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B * U) return;
  const int b = i / U, u = i % U;
  const size_t r = ((size_t)b * T1 + T1 - 1) * U + u;
  h0[i] = H[r];
  c0[i] = C[r];
}

// R2D2 loss partials in the clip + Adam kernel's [B][4] layout: {loss_b, 0, 0, nonfinite}
__global__ void r2d2_loss_part_kernel(int B, const float* __restrict__ loss, float* __restrict__ part) {
  pdl_wait_trig();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const float l = loss[b];
  part[b * 4 + 0] = l;
  part[b * 4 + 1] = 0.f;
  part[b * 4 + 2] = 0.f;
  part[b * 4 + 3] = isfinite(l) ? 0.f : 1.f;
}

// workspace: [burn-in online | burn-in target | trained online | trained target |
//             R2D2 extras]
struct R2d2Ws {
  LearnerWs wbo, wbt, wto, wtt;
  size_t obo, obt, oto, ott;
  size_t qo, qt, adv, val, y, delta, dq, dadv, dval, loss, lpart, r, disc, h0o, c0o, h0t, c0t;
  size_t total;
};

static seed_status make_r2d2_ws(const NetPlan& p, int burn_in, int T, int B, R2d2Ws* w) {
  size_t cur = 0;
  auto take = [&](size_t bytes) {
    const size_t at = cur;
    cur = align_up(cur + bytes, 256);
    return at;
  };
  if (burn_in > 0) {
    SEED_TRY(make_learner_ws(p, burn_in - 1, B, &w->wbo));
    w->wbt = w->wbo;
    w->obo = take(w->wbo.total);
    w->obt = take(w->wbt.total);
  }
  SEED_TRY(make_learner_ws(p, T, B, &w->wto));
  w->wtt = w->wto;
  w->oto = take(w->wto.total);
  w->ott = take(w->wtt.total);
  const size_t F = (size_t)B * (T + 1), A = p.A, U = p.U;
  w->qo = take(F * A * 4); w->qt = take(F * A * 4);
  w->adv = take(F * A * 4); w->val = take(F * 4);
  w->y = take((size_t)B * T * 4); w->delta = take((size_t)B * T * 4);
  w->dq = take(F * A * 4); w->dadv = take(F * A * 4); w->dval = take(F * 4);
  w->loss = take((size_t)B * 4); w->lpart = take((size_t)B * 16);
  w->r = take((size_t)B * T * 4); w->disc = take((size_t)B * T * 4);
  w->h0o = take((size_t)B * U * 4); w->c0o = take((size_t)B * U * 4);
  w->h0t = take((size_t)B * U * 4); w->c0t = take((size_t)B * U * 4);
  w->total = cur;
  return SEED_OK;
}

// torso + core forward of one [B][T+1] window into a workspace (no loss): the LSTM
// outputs H / C rows, and (heads) A advantages + 1 value per row
static seed_status r2d2_forward(const NetPlan& p, const LearnerWs& lw, uint8_t* wsb, int T, int B,
                                const seed_batch* bt, const bf16* lowp, const float* params,
                                cudaStream_t st) {
  StepCtx c;
  c.p = &p;
  c.w = lw;
  c.ws = wsb;
  c.g = Geo{p.H, p.W, p.C, p.oh1, p.ow1, p.oh2, p.ow2, p.fc_in, p.Kx, p.Kxp,
            FastDiv((uint32_t)(p.oh1 * p.ow1)), FastDiv((uint32_t)p.ow1),
            FastDiv((uint32_t)(p.oh2 * p.ow2)), FastDiv((uint32_t)p.ow2)};
  c.st = st;
  c.aux = st;
  SEED_CUDA_TRY(cudaMemsetAsync(c.tickets(), 0, 64 + GEMM_COUNTERS * 4, st));
  {
    const int E = p.Kxp - 256;
    const int64_t n = (int64_t)lw.F * E;
    SEED_TRY(launch_k(core_extras_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, lw.F, p.A,
                      p.Kxp, bt->prev_action, bt->reward, bt->done, c.at<bf16>(lw.X)));
  }
  if (p.nsec > 0) SEED_TRY(deep_forward(c, bt, lowp, params, st));
  else SEED_TRY(shallow_forward(c, bt, lowp, params, st));
  return core_forward(c, bt, lowp, params, st);
}

static seed_status r2d2_step_impl(const seed_net_spec* spec, int burn_in, int T, int B,
                                  const seed_batch* burn, const seed_batch* train,
                                  const seed_train_state* state, const float* tparams,
                                  const void* tlowp, const float* is_weights,
                                  const seed_r2d2_hparams* hp, seed_comm* comm, const seed_exec* ex,
                                  void* ws, size_t ws_bytes, float* prio_out, float* metrics,
                                  void* stream) {
  NetPlan p;
  SEED_TRY(make_net_plan(spec, &p));
  if (p.kind == SEED_NET_MLP || !learner_supported(p)) return SEED_E_UNSUPPORTED;
  if (T < 1 || T > 256 || B < 1 || B > 1024 || burn_in < 0 || burn_in > 256) return SEED_E_SHAPE;
  if (!train || !state || !hp || !ws || !metrics || !prio_out || !tparams || !tlowp) return SEED_E_ARG;
  if (burn_in > 0 && (!burn || !burn->obs || !burn->prev_action || !burn->reward || !burn->done ||
                      !burn->h0 || !burn->c0 || !aligned16(burn->obs)))
    return SEED_E_ARG;
  if (!train->obs || !train->action || !train->prev_action || !train->reward || !train->done ||
      !aligned16(train->obs) || (burn_in == 0 && (!train->h0 || !train->c0)))
    return SEED_E_ARG;
  if (!state->params || !state->grads || !state->adam_m || !state->adam_v || !state->step ||
      !state->params_lowp || !aligned16(state->params) || !aligned16(state->grads) ||
      !aligned16(state->adam_m) || !aligned16(state->adam_v) || !aligned16(state->params_lowp) ||
      !aligned16(tlowp) || !aligned16(ws))
    return SEED_E_ARG;
  if (!(hp->max_grad_norm > 0.f) || hp->n < 1 || !(hp->rescale_eps > 0.f) || !(hp->eta >= 0.f && hp->eta <= 1.f))
    return SEED_E_ARG;
  R2d2Ws w;
  SEED_TRY(make_r2d2_ws(p, burn_in, T, B, &w));
  if (ws_bytes < w.total) return SEED_E_WORKSPACE;
  uint8_t* base = (uint8_t*)ws;
  auto at = [&](size_t off) { return base + off; };
  cudaStream_t st = (cudaStream_t)stream;
  const bf16* lowp = (const bf16*)state->params_lowp;
  const bf16* tl = (const bf16*)tlowp;
  const float* params = state->params;
  float* grads = state->grads;
  const int U = p.U, A = p.A, F = B * (T + 1);
  // 1. burn-in (no gradient): the stored state warmed over the first burn_in steps,
  //    by the online and by the target network
  seed_batch to = *train, tt = *train;
  if (burn_in > 0) {
    SEED_TRY(r2d2_forward(p, w.wbo, at(w.obo), burn_in - 1, B, burn, lowp, params, st));
    SEED_TRY(r2d2_forward(p, w.wbt, at(w.obt), burn_in - 1, B, burn, tl, tparams, st));
    const int n = B * U;
    SEED_TRY(launch_k(last_state_kernel, dim3((unsigned)ceil_div(n, 256)), dim3(256), 0, st, B, burn_in, U,
                      (const float*)at(w.obo + w.wbo.H), (const float*)at(w.obo + w.wbo.Cst),
                      (float*)at(w.h0o), (float*)at(w.c0o)));
    SEED_TRY(launch_k(last_state_kernel, dim3((unsigned)ceil_div(n, 256)), dim3(256), 0, st, B, burn_in, U,
                      (const float*)at(w.obt + w.wbt.H), (const float*)at(w.obt + w.wbt.Cst),
                      (float*)at(w.h0t), (float*)at(w.c0t)));
    to.h0 = (const float*)at(w.h0o); to.c0 = (const float*)at(w.c0o);
    tt.h0 = (const float*)at(w.h0t); tt.c0 = (const float*)at(w.c0t);
  }
  // 2. trained window: online and target forward, dueling heads
  SEED_TRY(r2d2_forward(p, w.wto, at(w.oto), T, B, &to, lowp, params, st));
  SEED_TRY(r2d2_forward(p, w.wtt, at(w.ott), T, B, &tt, tl, tparams, st));
  const float* Ho = (const float*)at(w.oto + w.wto.H);
  const float* Ht = (const float*)at(w.ott + w.wtt.H);
  const int64_t hw = p.t[p.i_hw].off, hb = p.t[p.i_hb].off;
  const unsigned rows_blocks = (unsigned)ceil_div(F * 32, 256);
  SEED_TRY(launch_dense_fwd(F, U, A + 1, Ho, params + hw, params + hb, (float*)at(w.adv), A,
                            (float*)at(w.val), 0, st));
  SEED_TRY(launch_k(dueling_q_kernel, dim3(rows_blocks), dim3(256), 0, st, F, A, (const float*)at(w.adv),
                    (const float*)at(w.val), (float*)at(w.qo)));
  SEED_TRY(launch_dense_fwd(F, U, A + 1, Ht, tparams + hw, tparams + hb, (float*)at(w.adv), A,
                            (float*)at(w.val), 0, st));
  SEED_TRY(launch_k(dueling_q_kernel, dim3(rows_blocks), dim3(256), 0, st, F, A, (const float*)at(w.adv),
                    (const float*)at(w.val), (float*)at(w.qt)));
  // 3. targets, TD errors, priorities, IS-weighted loss gradient
  SEED_TRY(launch_k(r2d2_rewards_kernel, dim3((unsigned)ceil_div(B * T, 256)), dim3(256), 0, st, B, T,
                    hp->discount, train->reward, train->done, (float*)at(w.r), (float*)at(w.disc)));
  SEED_TRY(seed_r2d2_targets(T, B, A, hp->n, (const float*)at(w.qo), (const float*)at(w.qt),
                             train->action, (const float*)at(w.r), (const float*)at(w.disc), hp->eta,
                             hp->rescale_eps, is_weights, hp->loss_scale, (float*)at(w.y),
                             (float*)at(w.delta), prio_out, (float*)at(w.dq), (float*)at(w.loss), st));
  // 4. dueling + heads backward (the heads forward of the online net is recomputed
  //    into adv / val above only for the target; H is the online core output)
  SEED_TRY(launch_k(dueling_bwd_kernel, dim3(rows_blocks), dim3(256), 0, st, F, A, (const float*)at(w.dq),
                    (float*)at(w.dadv), (float*)at(w.dval)));
  dense_wgrad_f32<<<dim3(A + 1, ceil_div(U + 1, 32)), 256, 0, st>>>(
      F, U, A + 1, (const float*)at(w.dadv), A, (const float*)at(w.dval), Ho, grads + hw, grads + hb);
  SEED_TRY(launch_dense_dgrad(F, U, A + 1, (const float*)at(w.dadv), A, (const float*)at(w.dval),
                              params + hw, nullptr, (float*)at(w.oto + w.wto.dH), st));
  // 5. core + torso backward on the online workspace, then the optimizer
  StepCtx c;
  c.p = &p;
  c.w = w.wto;
  c.ws = at(w.oto);
  c.g = Geo{p.H, p.W, p.C, p.oh1, p.ow1, p.oh2, p.ow2, p.fc_in, p.Kx, p.Kxp,
            FastDiv((uint32_t)(p.oh1 * p.ow1)), FastDiv((uint32_t)p.ow1),
            FastDiv((uint32_t)(p.oh2 * p.ow2)), FastDiv((uint32_t)p.ow2)};
  c.st = st;
  SEED_TRY(aux_stream(ex, st, false, &c.aux, c.fev));
  const bool dp = comm && comm_world(comm) > 1;
  if (dp) {
    c.comm = comm;
    SEED_TRY(comm_side(comm, &c.side, &c.side2, c.ev));
  }
  SEED_TRY(core_backward(c, &to, lowp, params, grads, st));
  if (p.nsec > 0) SEED_TRY(deep_backward(c, &to, lowp, params, grads, st));
  else SEED_TRY(shallow_backward(c, &to, lowp, params, grads, st));
  SEED_TRY(c.edge(c.aux, st));
  if (dp) {
    SEED_TRY(c.bucket(grads, dp_buckets() >= 2 ? p.t[p.i_fcw].off : p.P, st));
    SEED_CUDA_TRY(cudaEventRecord(c.ev[3], c.side));
    SEED_CUDA_TRY(cudaStreamWaitEvent(st, c.ev[3], 0));
    if (c.side2) {
      SEED_CUDA_TRY(cudaEventRecord(c.ev[4], c.side2));
      SEED_CUDA_TRY(cudaStreamWaitEvent(st, c.ev[4], 0));
    }
  }
  SEED_TRY(launch_k(r2d2_loss_part_kernel, dim3((unsigned)ceil_div(B, 256)), dim3(256), 0, st, B,
                    (const float*)at(w.loss), (float*)at(w.lpart)));
  double* npart = c.at<double>(c.w.norm_part);
  NormArgs na{};
  na.g = grads; na.P = p.P; na.part = npart;
  na.coef = reinterpret_cast<float*>(npart + NORM_BLOCKS); na.norm = npart + NORM_BLOCKS + 2;
  na.ticket = c.tickets() + 1;
  na.step = state->step; na.step_in = c.at<int64_t>(c.w.step_in);
  na.beta1 = hp->beta1; na.beta2 = hp->beta2; na.max_norm = hp->max_grad_norm;
  SEED_TRY(launch_k(grad_norm_kernel, dim3(NORM_BLOCKS), dim3(256), 0, st, na));
  AdamArgs aa{};
  aa.P = p.P; aa.params = state->params; aa.grads = grads; aa.m = state->adam_m;
  aa.v = state->adam_v; aa.step = state->step; aa.step_in = c.at<int64_t>(c.w.step_in);
  aa.coef = na.coef; aa.norm = na.norm;
  aa.lr = hp->lr; aa.beta1 = hp->beta1; aa.beta2 = hp->beta2; aa.eps = hp->eps;
  aa.max_norm = hp->max_grad_norm; aa.loss_part = (const float*)at(w.lpart); aa.B = B;
  aa.metrics = metrics;
  aa.lowp = (bf16*)state->params_lowp;
  const bool fused_lowp = p.nimg <= 8;
  aa.nimg = fused_lowp ? p.nimg : 0;
  for (int k = 0; k < aa.nimg; ++k) aa.img[k] = p.img[k];
  SEED_TRY(launch_clip_adam(aa, st));
  if (!fused_lowp) SEED_TRY(refresh_lowp(p, state->params, state->params_lowp, st));
  return last_launch();
}

}  // namespace seed

extern "C" seed_status seed_r2d2_workspace_size(const seed_net_spec* spec, int burn_in, int T, int B,
                                                size_t* bytes) {
  if (!bytes) return SEED_E_ARG;
  NetPlan p;
  SEED_TRY(make_net_plan(spec, &p));
  if (p.kind == SEED_NET_MLP || !learner_supported(p)) return SEED_E_UNSUPPORTED;
  if (T < 1 || T > 256 || B < 1 || B > 1024 || burn_in < 0 || burn_in > 256) return SEED_E_SHAPE;
  R2d2Ws w;
  SEED_TRY(make_r2d2_ws(p, burn_in, T, B, &w));
  *bytes = w.total;
  return SEED_OK;
}

extern "C" seed_status seed_r2d2_learner_step(const seed_net_spec* spec, int burn_in, int T, int B,
                                              const seed_batch* burn, const seed_batch* train,
                                              const seed_train_state* online, const float* target_params,
                                              const void* target_lowp, const float* is_weights,
                                              const seed_r2d2_hparams* hp, seed_comm* comm,
                                              seed_exec* exec, void* ws, size_t ws_bytes,
                                              float* priorities_out, float* metrics, void* stream) {
  return seed::r2d2_step_impl(spec, burn_in, T, B, burn, train, online, target_params, target_lowp,
                              is_weights, hp, comm, exec, ws, ws_bytes, priorities_out, metrics, stream);
}
