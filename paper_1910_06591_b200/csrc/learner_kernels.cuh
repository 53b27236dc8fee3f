// learner_kernels.cuh — the non-GEMM kernels of the learner step: fp32 dense
// layers (the configs[0] MLP and the policy/value heads), the fused policy
// loss (K2: log-softmax + V-trace scan + loss + output gradients), column sums
// for conv bias gradients, LSTM core-input extras, global-norm clip + Adam (K9).
#pragma once
#include "common.cuh"
#include "vtrace_scan.cuh"
#include "net.cuh"

namespace seed {

// Y[r][o] = act(b[o] + sum_i X[r][i] W[o][i]); warp per row, lane per output
// (I <= 256, O <= 64; dynamic smem (I*O + 8*I)*4).  Optional split output:
// columns o < A go to Y (ld A), column A to Yv (heads: logits / value).
__global__ void dense_fwd_f32(int R, int I, int O, const float* __restrict__ X,
                              const float* __restrict__ W, const float* __restrict__ b,
                              float* __restrict__ Y, int ldy, float* __restrict__ Yv, int relu);

// dX[r][i] = (sum_o dY(r,o) W[o][i]) * (mask ? mask[r][i] > 0 : 1), dY(r,o) = o < ldy ?
// dy[r*ldy+o] : dv[r] (dv used for the last column when non-null).  Block = 8
// rows (grid ceil(R/8)), dynamic smem (O*I + 8*O)*4.
__global__ void dense_dgrad_f32(int R, int I, int O, const float* __restrict__ dy, int ldy,
                                const float* __restrict__ dv, const float* __restrict__ W,
                                const float* __restrict__ mask, float* __restrict__ dX);

seed_status launch_dense_fwd(int R, int I, int O, const float* X, const float* W, const float* b,
                             float* Y, int ldy, float* Yv, int relu, cudaStream_t st);
seed_status launch_dense_dgrad(int R, int I, int O, const float* dy, int ldy, const float* dv,
                               const float* W, const float* mask, float* dX, cudaStream_t st);

// gW[o][i] = sum_r dY(r,o) X[r][i];  gb[o] = sum_r dY(r,o)  (grid (O, ceil((I+1)/32)), 256
// threads; fixed-order reduction)
__global__ void dense_wgrad_f32(int R, int I, int O, const float* __restrict__ dy, int ldy,
                                const float* __restrict__ dv, const float* __restrict__ X,
                                float* __restrict__ gW, float* __restrict__ gb);

struct LossArgs {
  int B, T, A;
  float* logits;         // [B][T+1][A] (input of policy_loss_kernel, output of the fused kernel)
  float* values;         // [B][T+1]
  const int32_t* action;
  const float* blp;
  const float* reward;
  const uint8_t* done;   // [B][T+1]
  float discount, rho_bar, c_bar, lam, vf_coef, ent_coef, scale;
  float* dlogits;        // [B][T+1][A]
  float* dvalues;        // [B][T+1]
  float* vs;             // [B][T]
  float* pg;             // [B][T]
  float* part;           // [B][4]: scaled pg, baseline, entropy terms, nonfinite
  // fused heads (launch_heads_loss): the heads forward (H4) runs inside the loss
  // kernel, which also forms the heads backward (H8): logits / values above
  // become outputs, and
  const float* H;        // [B*(T+1)][I] fp32 core output
  int I;                 // I <= 256, I % 4 == 0
  const float* hw;       // [A+1][I] heads weights (row A = value head)
  const float* hb;       // [A+1]
  const float* hmask;    // nullable: dH zeroed where hmask <= 0 (ReLU input)
  float* dH;             // [B*(T+1)][I]
  float* wpart;          // [B][A+1][I+1] per-trajectory heads weight | bias gradients
  float* g_w;            // [A+1][I] heads weight gradient (fixed-order sum over b)
  float* g_b;            // [A+1]
};
seed_status launch_policy_loss(const LossArgs& a, cudaStream_t st);
seed_status launch_heads_loss(const LossArgs& a, cudaStream_t st);

// X[f][256 + j] for j in [0, Kxp-256): onehot(prev_action), clip(reward), 1, 0 pad (C15)
__global__ void core_extras_kernel(int F, int A, int Kxp, const int32_t* __restrict__ prev_action,
                                   const float* __restrict__ reward,
                                   const uint8_t* __restrict__ done, __nv_bfloat16* X);


struct AdamArgs {
  int64_t P;
  float* params;
  const float* grads;
  float* m;
  float* v;
  int64_t* step;
  const int64_t* step_in;
  const float* coef;       // grad_norm_kernel output
  const double* norm;
  float lr, beta1, beta2, eps, max_norm;
  const float* loss_part;  // [B][4]
  int B;
  float* metrics;          // [8]
  __nv_bfloat16* lowp;     // bf16 operand images refreshed in the same pass
  int nimg;
  LowpImg img[8];
};
seed_status launch_clip_adam(const AdamArgs& a, cudaStream_t st);
// Global-norm partials; the last block (integer ticket, re-armed by itself)
// reduces them in block order and writes the clip + Adam coefficients
// coef = {clip scale, 1 - beta1^t, 1 - beta2^t, finite} and the norm (double).
struct NormArgs {
  const float* g;
  int64_t P;
  double* part;            // [NORM_BLOCKS]
  float* coef;             // [4]
  double* norm;
  unsigned* ticket;
  const int64_t* step;
  int64_t* step_in;
  float beta1, beta2, max_norm;
};
__global__ void grad_norm_kernel(const NormArgs a);

}  // namespace seed
