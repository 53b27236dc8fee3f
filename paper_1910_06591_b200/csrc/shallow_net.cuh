// shallow_net.cuh — the FC / LSTM-input GEMM Problems (gemm_tc.cuh concept) of
// the torso+core (C14), shared by the learner step (learner.cu) and centralized
// inference (infer.cu).  Activations bf16, rows f = b*(T+1)+t (learner) or
// request index (inference).  The Atari-shallow convolutions themselves are
// the space-to-depth window GEMMs of conv_s2d.cuh.
#pragma once
#include "gemm_tc.cuh"

namespace seed {

typedef __nv_bfloat16 bf16;

__device__ __forceinline__ bf16 to_bf(float v) { return __float2bfloat16_rn(v); }
__device__ __forceinline__ float bf2f(bf16 v) { return __bfloat162float(v); }

struct Geo {
  int H, W, C, oh1, ow1, oh2, ow2, fc_in, Kx, Kxp;
  FastDiv hw1, w1, hw2, w2;   // oh1*ow1, ow1, oh2*ow2, ow2
};
// row of conv1 output (f, oy, ox) / conv2 output
__device__ __forceinline__ void split_row(const FastDiv& hw, const FastDiv& w, int m, uint32_t& f,
                                          uint32_t& oy, uint32_t& ox) {
  uint32_t p;
  hw.divmod((uint32_t)m, f, p);
  w.divmod(p, oy, ox);
}

// 16 fp32 -> 16 bf16 (two 16-byte stores)
__device__ __forceinline__ void st_bf16x16(bf16* dst, const float (&v)[16]) {
  uint4 a, b;
  a.x = pack_bf16(v[0], v[1]); a.y = pack_bf16(v[2], v[3]);
  a.z = pack_bf16(v[4], v[5]); a.w = pack_bf16(v[6], v[7]);
  b.x = pack_bf16(v[8], v[9]); b.y = pack_bf16(v[10], v[11]);
  b.z = pack_bf16(v[12], v[13]); b.w = pack_bf16(v[14], v[15]);
  reinterpret_cast<uint4*>(dst)[0] = a;
  reinterpret_cast<uint4*>(dst)[1] = b;
}
// mask v[q] by (src[q] > 0) for 16 bf16 values of a ReLU output
__device__ __forceinline__ void relu_mask16(const bf16* src, float (&v)[16]) {
  const uint4 a = reinterpret_cast<const uint4*>(src)[0];
  const uint4 b = reinterpret_cast<const uint4*>(src)[1];
  const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (!(bf16_lo(w[q]) > 0.f)) v[2 * q] = 0.f;
    if (!(bf16_hi(w[q]) > 0.f)) v[2 * q + 1] = 0.f;
  }
}


// fc: X[f][0:256] = relu(act2[f] . Wfc^T + b)
struct FcFwd {
  static constexpr bool ASYNC = true;
  static constexpr bool TMA = true;   // plain K-major A [M][K] and B [N][K]: tensor-map tiles
  CUtensorMap ta, tb;
  const void* dummy = k_ones_chunk;
  static constexpr bool A_MN = false, B_MN = false;
  int M, N, K, kb_per_split;
  int Kxp;
  const bf16* act2;
  const bf16* w;
  const float* bias;
  bf16* X;
  bool tmaps(int bn) { return tmap_kmajor(&ta, act2, M, K, K, 128) && tmap_kmajor(&tb, w, N, K, K, bn); }
  __device__ const void* ptr_a(int m, int k) const { return act2 + (size_t)m * K + k; }
  __device__ const void* ptr_b(int n, int k) const { return w + (size_t)n * K + k; }
  __device__ void store(int m, int n, float v) const {
    X[(size_t)m * Kxp + n] = to_bf(fmaxf(v + bias[n], 0.f));
  }
  static constexpr bool VEC_STORE = true;
  __device__ void store16(int m, int n0, float (&v)[16]) const {
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = fmaxf(v[q] + bias[n0 + q], 0.f);
    st_bf16x16(X + (size_t)m * Kxp + n0, v);
  }
};

// LSTM input projection: xproj[f][n] = X[f] . Wx[n] + b[n]
struct XprojFwd {
  static constexpr bool ASYNC = true;
  static constexpr bool TMA = true;   // plain K-major A [M][K] and B [N][K]: tensor-map tiles
  CUtensorMap ta, tb;
  const void* dummy = k_ones_chunk;
  static constexpr bool A_MN = false, B_MN = false;
  int M, N, K, kb_per_split;
  const bf16* X;
  const bf16* w;
  const float* bias;
  float* out;
  bool tmaps(int bn) { return tmap_kmajor(&ta, X, M, K, K, 128) && tmap_kmajor(&tb, w, N, K, K, bn); }
  __device__ const void* ptr_a(int m, int k) const { return X + (size_t)m * K + k; }
  __device__ const void* ptr_b(int n, int k) const { return w + (size_t)n * K + k; }
  __device__ void store(int m, int n, float v) const { out[(size_t)m * N + n] = v + bias[n]; }
  static constexpr bool ROW_OUT = true;   // coalesced staged epilogue (gemm_tc.cuh)
  __device__ float* out_row(int m) const { return out + (size_t)m * N; }
  __device__ float post(int, int n, float v) const { return v + bias[n]; }
  static constexpr bool VEC_STORE = true;
  __device__ void store16(int m, int n0, float (&v)[16]) const {
    float4* o = reinterpret_cast<float4*>(out + (size_t)m * N + n0);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      o[q] = make_float4(v[4 * q] + bias[n0 + 4 * q], v[4 * q + 1] + bias[n0 + 4 * q + 1],
                         v[4 * q + 2] + bias[n0 + 4 * q + 2], v[4 * q + 3] + bias[n0 + 4 * q + 3]);
  }
};

// [dWx | db | dWh] = dG^T . [X | Hprev]   (M = 4U gate rows, K = F rows)
struct LstmWgrad {
  static constexpr bool ASYNC = true;
  const void* dummy = k_ones_chunk;
  static constexpr bool A_MN = true, B_MN = true;
  int M, N, K, kb_per_split;
  int Kx, Kxp, U;
  const bf16* dG;
  const bf16* X;
  const bf16* Hprev;
  float* g_wx;
  float* g_b;
  float* g_wh;
  __device__ const void* ptr_a(int row, int m8) const { return dG + (size_t)row * M + m8; }
  __device__ const void* ptr_b(int row, int n8) const {
    return n8 < Kxp ? (const void*)(X + (size_t)row * Kxp + n8)
                    : (const void*)(Hprev + (size_t)row * U + n8 - Kxp);
  }
  __device__ void store(int m, int n, float v) const {
    if (n < Kx) g_wx[(size_t)m * Kx + n] = v;
    else if (n == Kx) g_b[m] = v;
    else if (n >= Kxp) g_wh[(size_t)m * U + (n - Kxp)] = v;
  }
};

// dfc = (dG . Wx)[:, 0:256] masked by fc > 0
struct DxFc {
  static constexpr bool ASYNC = true;
  const void* dummy = k_ones_chunk;
  static constexpr bool A_MN = false, B_MN = true;
  int M, N, K, kb_per_split;
  int Kxp;
  const bf16* dG;
  const bf16* wx;
  const bf16* X;
  bf16* dfc;
  __device__ const void* ptr_a(int m, int k) const { return dG + (size_t)m * K + k; }
  __device__ const void* ptr_b(int k, int n8) const { return wx + (size_t)k * Kxp + n8; }
  __device__ void store(int m, int n, float v) const {
    dfc[(size_t)m * 256 + n] = to_bf(bf2f(X[(size_t)m * Kxp + n]) > 0.f ? v : 0.f);
  }
  static constexpr bool VEC_STORE = true;
  __device__ void store16(int m, int n0, float (&v)[16]) const {
    relu_mask16(X + (size_t)m * Kxp + n0, v);
    st_bf16x16(dfc + (size_t)m * 256 + n0, v);
  }
};

// [dWfc | dbfc] = dfc^T . [act2 | 1]
struct FcWgrad {
  static constexpr bool ASYNC = true;
  const void* dummy = k_ones_chunk;
  static constexpr bool A_MN = true, B_MN = true;
  int M, N, K, kb_per_split;
  int fc_in;
  const bf16* dfc;
  const bf16* act2;
  float* g_w;
  float* g_b;
  __device__ const void* ptr_a(int row, int m8) const { return dfc + (size_t)row * 256 + m8; }
  __device__ const void* ptr_b(int row, int n8) const {
    if (n8 < fc_in) return act2 + (size_t)row * fc_in + n8;
    return k_ones_chunk;  // bf16 1.0 in column fc_in, zeros after
  }
  __device__ void store(int m, int n, float v) const {
    if (n < fc_in) g_w[(size_t)m * fc_in + n] = v;
    else if (n == fc_in) g_b[m] = v;
  }
};

// dY2 = (dfc . Wfc) masked by act2 > 0
struct FcDgrad {
  static constexpr bool ASYNC = true;
  const void* dummy = k_ones_chunk;
  static constexpr bool A_MN = false, B_MN = true;
  int M, N, K, kb_per_split;
  const bf16* dfc;
  const bf16* w;
  const bf16* act2;
  bf16* dY2;             // plain [M][N] layout (deep torso), or
  uint8_t* dY2s;         // non-null: Atari-shallow conv2 output space, pre-swizzled
                         // rows of 2*CH bytes g = f*P2 + g0 + y*W2s + x (conv_s2d.cuh;
                         // deep torso: conv3w.cuh padded rows, g0 = W2s + 1)
  int Wo, W2s, P2, g0;
  int CH = 32;           // channels per dY2s pixel (32; 64 for the 2x DMLab torso; 128
                         // for the 4x: two planes of 64-channel rows, conv3w.cuh)
  __device__ const void* ptr_a(int m, int k) const { return dfc + (size_t)m * 256 + k; }
  __device__ const void* ptr_b(int k, int n8) const { return w + (size_t)k * N + n8; }
  // the row holding channel n % CH of pixel n / CH (its plane's row for CH = 128)
  __device__ uint8_t* s2d_row(int m, int n, int64_t& g) const {
    const int pix = n / CH;
    g = (int64_t)m * P2 + g0 + (pix / Wo) * W2s + pix % Wo;
    if (CH > 64) return dY2s + (size_t)((n % CH) >> 6) * M * P2 * 128 + g * 128;
    return dY2s + g * (2 * CH);
  }
  __device__ int row_bytes() const { return CH > 64 ? 128 : 2 * CH; }
  __device__ void store(int m, int n, float v) const {
    const size_t i = (size_t)m * N + n;
    const bf16 o = to_bf(bf2f(act2[i]) > 0.f ? v : 0.f);
    if (dY2s) {
      int64_t g;
      uint8_t* row = s2d_row(m, n, g);
      const int c = (n % CH) & (row_bytes() / 2 - 1);
      *reinterpret_cast<bf16*>(row + (swz_chunk(g, row_bytes(), c >> 3) << 4) + (c & 7) * 2) = o;
    } else {
      dY2[i] = o;
    }
  }
  static constexpr bool VEC_STORE = true;
  __device__ void store16(int m, int n0, float (&v)[16]) const {
    const size_t i = (size_t)m * N + n0;
    relu_mask16(act2 + i, v);
    if (dY2s) {
      int64_t g;
      uint8_t* row = s2d_row(m, n0, g);
      const int j0 = ((n0 % CH) & (row_bytes() / 2 - 1)) >> 3;
      uint4 a, b;
      a.x = pack_bf16(v[0], v[1]); a.y = pack_bf16(v[2], v[3]);
      a.z = pack_bf16(v[4], v[5]); a.w = pack_bf16(v[6], v[7]);
      b.x = pack_bf16(v[8], v[9]); b.y = pack_bf16(v[10], v[11]);
      b.z = pack_bf16(v[12], v[13]); b.w = pack_bf16(v[14], v[15]);
      *reinterpret_cast<uint4*>(row + (swz_chunk(g, row_bytes(), j0) << 4)) = a;
      *reinterpret_cast<uint4*>(row + (swz_chunk(g, row_bytes(), j0 + 1) << 4)) = b;
    } else {
      st_bf16x16(dY2 + i, v);
    }
  }
};

}  // namespace seed
