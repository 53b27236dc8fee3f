// lstm.cuh — persistent cluster LSTM core (H3 forward, H8 BPTT) declarations.
#pragma once
#include "common.cuh"

namespace seed {

constexpr int LSTM_U = 256;        // hidden units (C14)
constexpr int LSTM_CLUSTER = 8;    // CTAs per cluster; CTA r owns units [32r, 32r+32)
constexpr int LSTM_BB = 32;        // batch rows per cluster

struct LstmFwdArgs {
  int B, T1;
  const float* xproj;          // [B*T1][4U] = Wx x_t + b (gate order i,f,g,o)
  const __nv_bfloat16* wh;     // [4U][U] bf16
  const float* h0;             // [*][U]
  const float* c0;             // [*][U]
  const int32_t* state_rows;   // nullable: batch row b reads h0/c0 row state_rows[b]
  const uint8_t* done;         // [B][T1]; reset (h,c) <- 0 before step t when done[b][t]
  float* H;                    // [B*T1][U] fp32 h_t
  __nv_bfloat16* Hb;           // nullable [B*T1][U] bf16 h_t
  __nv_bfloat16* Hprev;        // nullable [B*T1][U] bf16 reset-aware h_{t-1}
  float* gates;                // nullable [B*T1][4U] post-activation i,f,g,o
  float* C;                    // nullable [B*T1][U] c_t
  float* hT;                   // nullable: final h written to hT[state_rows[b]] (or row b)
  float* cT;
};

struct LstmBwdArgs {
  int B, T1;
  const __nv_bfloat16* wh;     // [4U][U]
  const float* gates;          // [B*T1][4U]
  const float* C;              // [B*T1][U]
  const float* c0;             // [B][U]
  const uint8_t* done;         // [B][T1]
  const float* dH;             // [B*T1][U] dL/dh_t from the heads
  __nv_bfloat16* dG;           // out [B*T1][4U] dL/d(pre-activation gates), bf16
};

// Activations on the SFU's tanh.approx.f32 (one MUFU op; max rel. error ~2^-11, far
// inside the bf16 tolerance C22): sigmoid(x) = 0.5 * tanh(0.5 x) + 0.5.  Shared by
// the cluster kernels and the inference cell (infer.cu), so the policy that acts
// and the learner's recomputation use the same cell arithmetic.
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sigm(float x) { return fmaf(0.5f, tanh_fast(0.5f * x), 0.5f); }

seed_status lstm_forward(const LstmFwdArgs& a, cudaStream_t st);
seed_status lstm_backward(const LstmBwdArgs& a, cudaStream_t st);

}  // namespace seed
