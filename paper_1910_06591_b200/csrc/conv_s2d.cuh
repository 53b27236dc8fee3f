// conv_s2d.cuh — the Atari-shallow torso (C14: conv 8x8/4 -> 16, conv 4x4/2 ->
// 32) as space-to-depth "shifted-window" GEMMs on tcgen05.
//
// A stride-s convolution with a 2s x 2s kernel equals a 2x2 stride-1
// convolution over the space-to-depth image S (s x s pixel blocks folded into
// s*s*C channels; both Atari layers give 64 channels = one 128-byte bf16 row):
//   out[f][oy][ox][co] = sum_{a,b in {0,1}} S[f][oy+a][ox+b][:] . W'_{ab}[co][:]
//   W'_{ab}[co][(ky'*s + kx')*C + c] = W[co][s*a + ky'][s*b + kx'][c]
// Rows of S are numbered g = f*Hs*Ws + Y*Ws + X, and the outputs use the same
// padded numbering (ox = Ws-1 / oy = Hs-1 rows are computed and discarded), so
// window (a, b) of the 128 output rows starting at m0 is the contiguous row
// range starting at m0 + a*Ws + b.  Each CTA copies one contiguous "slab" of
// rows with a single TMA bulk copy (cp.async.bulk) and the MMA reads the four
// windows from it through shifted shared-memory descriptors.  Buffers are
// stored pre-swizzled (the 128B / 64B / 32B swizzle of the byte address), so a
// linear copy that preserves the address phase mod 1024 lands every row in the
// canonical UMMA layout (verified: scripts/probe_umma_layouts.cu).
//
// Kernels: s2d_obs_kernel (uint8 obs -> S0), win_conv_kernel (forward /
// data-gradient: persistent, TMA slab ring, double-buffered TMEM accumulators),
// win3_wgrad_kernel with 2 B atoms (weight + bias gradient: split over rows, one
// MMA per 16 rows — A = MN-major slab whose two 64-channel atoms are the window
// columns b (LBO = one 128-byte row), B = dY rows whose two atoms are the window
// rows a (LBO = Ws rows); bias from the epilogue warps' column sums of dY) +
// win3_wgrad_finish (fixed-order split sum).
#pragma once
#include "common.cuh"
#include "win_engine.cuh"

namespace seed {

typedef __nv_bfloat16 bf16;

// geometry of one space-to-depth layer
struct S2dGeo {
  int s, C, CO;        // stride, input channels, output channels (s*s*C == 64)
  int Hs, Ws, P;       // s2d image (rows per frame P = Hs*Ws)
  int Ho, Wo;          // valid outputs (Hs-1, Ws-1)
};

// conv1 epilogue: relu(acc/255 + b) of the valid rows -> S1 (conv2's s2d input)
struct Conv1S2dEpi {
  static constexpr int N = 16;
  const float* bias;
  uint8_t* S1;
  FastDiv P1, W1;        // conv1 s2d rows per frame (441), row width (21)
  int Ho, Wo, W2s, P2;   // 20, 20, 10, 100
  __device__ void store(int64_t m, float (&v)[N]) const;
};
// conv2 epilogue: relu(acc + b) of the valid rows -> act2 [F][Ho*Wo*32] (FC input);
// the invalid (padding) rows zero the matching rows of dY2 (optional)
struct Conv2S2dEpi {
  static constexpr int N = 32;
  const float* bias;
  bf16* act2;
  uint8_t* dY2z;         // nullable: dY2 rows (64 B) zeroed where the row is padding
  FastDiv P2, W2;        // 100, 10
  int Ho, Wo, fc_in;
  __device__ void store(int64_t m, float (&v)[N]) const;
};
// conv2 data gradient in conv2-input s2d space: dS1[p] masked by S1[p] > 0 and
// scattered to dY1 rows of conv1 output space (32-byte rows, 32B swizzle); the
// padding rows of conv1 output space receive zeros
struct Conv2DgradS2dEpi {
  static constexpr int N = 64;
  static constexpr int PRE = 8;   // the S1 row (ReLU mask), prefetched by the engine
  const uint8_t* S1;
  uint8_t* dY1;
  FastDiv P2, W2;        // 100, 10
  int H2s, W2s;          // 10, 10
  int P1, W1s, H1s;      // 441, 21, 21 (conv1 output rows, padded numbering)
  __device__ void pre(int64_t m, uint4 (&p)[PRE]) const;
  __device__ void store(int64_t m, float (&v)[N], const uint4 (&p)[PRE]) const;
};

struct WinWgradFinish {
  S2dGeo g;
  float scale;           // weight-gradient scale (1/255 for conv1)
  float* g_w;            // fp32 [CO][2s][2s][C]
  float* g_b;            // fp32 [CO]
  __device__ void weight(int grp, int i, int n, float v) const;
  __device__ void bias(int n, float v) const { g_b[n] = v; }
};
size_t win_wgrad_part_bytes(int64_t M, int N);

// uint8 obs [F][H][W][4] -> S0 pre-swizzled bf16 rows [F*Hs*Ws][64] (exact 0..255)
seed_status s2d_obs(const uint8_t* obs, int64_t F, int H, int W, uint8_t* S0, cudaStream_t st);

// the shallow torso, forward (shared by the learner and inference)
struct ShallowS2d {
  S2dGeo g1, g2;
  int fc_in;
  int64_t rows1(int64_t F) const { return F * g1.P; }
  int64_t rows2(int64_t F) const { return F * g2.P; }
};
ShallowS2d shallow_s2d_geometry(int H, int W, int C);
bool shallow_s2d_supported(int H, int W, int C);
// obs -> S0 -> S1 -> act2 (dY2z nullable)
seed_status shallow_s2d_forward(const ShallowS2d& sg, int64_t F, const uint8_t* obs,
                                const bf16* w1img, const float* b1, const bf16* w2img,
                                const float* b2, uint8_t* S0, uint8_t* S1, bf16* act2,
                                uint8_t* dY2z, cudaStream_t st);
// the three launches of the forward, separately (phase marks)
seed_status shallow_s2d_conv1(const ShallowS2d& sg, int64_t F, const uint8_t* S0, const bf16* w1img,
                              const float* b1, uint8_t* S1, cudaStream_t st);
seed_status shallow_s2d_conv2(const ShallowS2d& sg, int64_t F, const uint8_t* S1, const bf16* w2img,
                              const float* b2, bf16* act2, uint8_t* dY2z, cudaStream_t st);
// backward pieces: dW2|db2 (from S1, dY2), dY1 (from dY2, W2 dgrad image, S1 mask),
// dW1|db1 (from S0, dY1; scale 1/255)
seed_status shallow_s2d_conv2_wgrad(const ShallowS2d& sg, int64_t F, const uint8_t* S1,
                                    const uint8_t* dY2, float* part, float* g_w2, float* g_b2,
                                    cudaStream_t st);
seed_status shallow_s2d_conv2_dgrad(const ShallowS2d& sg, int64_t F, const uint8_t* dY2,
                                    const bf16* w2dg_img, const uint8_t* S1, uint8_t* dY1,
                                    cudaStream_t st);
seed_status shallow_s2d_conv1_wgrad(const ShallowS2d& sg, int64_t F, const uint8_t* S0,
                                    const uint8_t* dY1, float* part, float* g_w1, float* g_b1,
                                    cudaStream_t st);
// buffer sizes (bytes) for F frames
size_t s2d_S0_bytes(const ShallowS2d& sg, int64_t F);   // F*P1 rows x 128
size_t s2d_S1_bytes(const ShallowS2d& sg, int64_t F);   // F*P2 rows x 128
size_t s2d_dY2_bytes(const ShallowS2d& sg, int64_t F);  // F*P2 rows x 64
size_t s2d_dY1_bytes(const ShallowS2d& sg, int64_t F);  // F*P1 rows x 32

}  // namespace seed
