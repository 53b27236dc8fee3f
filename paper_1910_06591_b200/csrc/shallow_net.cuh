// shallow_net.cuh — the Atari IMPALA-shallow network (C14) as tcgen05 GEMM
// Problems (gemm_tc.cuh concept), shared by the learner step (learner.cu) and
// centralized inference (infer.cu).  Activations are bf16 NHWC, rows
// f = b*(T+1)+t (learner) or request index (inference).
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


// obs (uint8) -> bf16 (exact integers 0..255; the 1/255 scale is applied in the
// conv1 epilogue / weight gradient), 16 values per thread.
static __global__ void obs_to_bf16_kernel(const uint8_t* __restrict__ obs, bf16* __restrict__ out,
                                   int64_t n16) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(obs) + i);
    uint4* o = reinterpret_cast<uint4*>(out) + 2 * i;
    o[0] = u8x8_to_bf16(make_uint2(v.x, v.y));
    o[1] = u8x8_to_bf16(make_uint2(v.z, v.w));
  }
}

// conv1: A(m = (f, oy, ox), k = (ky, kx, c)) = obs[f][4oy+ky][4ox+kx][c]
// (8 consecutive k = 2 pixels x 4 channels = 16 contiguous bytes of obs_bf16)
struct Conv1Fwd {
  static constexpr bool ASYNC = true;
  const void* dummy = k_ones_chunk;
  static constexpr bool A_MN = false, B_MN = false;
  int M, N, K, kb_per_split;
  Geo g;
  const bf16* obs;
  const bf16* w;
  const float* bias;
  bf16* out;
  __device__ const void* ptr_a(int m, int k) const {
    uint32_t f, oy, ox;
    split_row(g.hw1, g.w1, m, f, oy, ox);
    const int ky = k >> 5, kx = (k & 31) >> 2;   // k = (ky*8 + kx)*4 + c, C == 4
    return obs + (((size_t)f * g.H + oy * 4 + ky) * g.W + ox * 4 + kx) * 4;
  }
  __device__ const void* ptr_b(int n, int k) const { return w + (size_t)n * K + k; }
  __device__ void store(int m, int n, float v) const {
    out[(size_t)m * 16 + n] = to_bf(fmaxf(v * (1.f / 255.f) + bias[n], 0.f));
  }
  static constexpr bool VEC_STORE = true;
  __device__ void store16(int m, int n0, float (&v)[16]) const {
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = fmaxf(v[q] * (1.f / 255.f) + bias[n0 + q], 0.f);
    st_bf16x16(out + (size_t)m * 16 + n0, v);
  }
};

// conv2: A(m = (f, oy, ox), k = (ky, kx, c)) = act1[f][2oy+ky][2ox+kx][c]
struct Conv2Fwd {
  static constexpr bool ASYNC = true;
  const void* dummy = k_ones_chunk;
  static constexpr bool A_MN = false, B_MN = false;
  int M, N, K, kb_per_split;
  Geo g;
  const bf16* act1;
  const bf16* w;
  const float* bias;
  bf16* out;
  __device__ const void* ptr_a(int m, int k) const {
    uint32_t f, oy, ox;
    split_row(g.hw2, g.w2, m, f, oy, ox);
    const int ky = k >> 6, kx = (k >> 4) & 3, c0 = k & 15;
    return act1 + (((size_t)f * g.oh1 + oy * 2 + ky) * g.ow1 + ox * 2 + kx) * 16 + c0;
  }
  __device__ const void* ptr_b(int n, int k) const { return w + (size_t)n * 256 + k; }
  __device__ void store(int m, int n, float v) const {
    out[(size_t)m * 32 + n] = to_bf(fmaxf(v + bias[n], 0.f));
  }
  static constexpr bool VEC_STORE = true;
  __device__ void store16(int m, int n0, float (&v)[16]) const {
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = fmaxf(v[q] + bias[n0 + q], 0.f);
    st_bf16x16(out + (size_t)m * 32 + n0, v);
  }
};

// fc: X[f][0:256] = relu(act2[f] . Wfc^T + b)
struct FcFwd {
  static constexpr bool ASYNC = true;
  const void* dummy = k_ones_chunk;
  static constexpr bool A_MN = false, B_MN = false;
  int M, N, K, kb_per_split;
  int Kxp;
  const bf16* act2;
  const bf16* w;
  const float* bias;
  bf16* X;
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
  const void* dummy = k_ones_chunk;
  static constexpr bool A_MN = false, B_MN = false;
  int M, N, K, kb_per_split;
  const bf16* X;
  const bf16* w;
  const float* bias;
  float* out;
  __device__ const void* ptr_a(int m, int k) const { return X + (size_t)m * K + k; }
  __device__ const void* ptr_b(int n, int k) const { return w + (size_t)n * K + k; }
  __device__ void store(int m, int n, float v) const { out[(size_t)m * N + n] = v + bias[n]; }
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
  bf16* dY2;
  __device__ const void* ptr_a(int m, int k) const { return dfc + (size_t)m * 256 + k; }
  __device__ const void* ptr_b(int k, int n8) const { return w + (size_t)k * N + n8; }
  __device__ void store(int m, int n, float v) const {
    const size_t i = (size_t)m * N + n;
    dY2[i] = to_bf(bf2f(act2[i]) > 0.f ? v : 0.f);
  }
  static constexpr bool VEC_STORE = true;
  __device__ void store16(int m, int n0, float (&v)[16]) const {
    const size_t i = (size_t)m * N + n0;
    relu_mask16(act2 + i, v);
    st_bf16x16(dY2 + i, v);
  }
};

// dW2^T[kin][co] = sum_rows im2col(act1)[row][kin] dY2[row][co]
struct Conv2Wgrad {
  static constexpr bool ASYNC = true;
  const void* dummy = k_ones_chunk;
  static constexpr bool A_MN = true, B_MN = true;
  int M, N, K, kb_per_split;
  Geo g;
  const bf16* act1;
  const bf16* dY2;
  float* g_w;
  __device__ const void* ptr_a(int row, int m8) const {
    uint32_t f, oy, ox;
    split_row(g.hw2, g.w2, row, f, oy, ox);
    const int ky = m8 >> 6, kx = (m8 >> 4) & 3, c0 = m8 & 15;
    return act1 + (((size_t)f * g.oh1 + oy * 2 + ky) * g.ow1 + ox * 2 + kx) * 16 + c0;
  }
  __device__ const void* ptr_b(int row, int n8) const { return dY2 + (size_t)row * 32 + n8; }
  __device__ void store(int m, int n, float v) const { g_w[(size_t)n * 256 + m] = v; }
};

// dY1 = transposed conv of dY2, masked by act1 > 0, as a sub-pixel GEMM: the
// stride-2 4x4 kernel splits into 4 output parity classes (py, px); class pixels
// y = 2qy + py, x = 2qx + px receive only taps ky = py + 2kyi, kx = px + 2kxi
// (kyi, kxi in {0,1}) from dY2[qy - kyi][qx - kxi], so K = 2*2*32 = 128 with no
// zero taps.  Rows m = ((class * F + f) * QH + qy) * QW + qx; all four classes run
// in one launch with N = 64 = 4 classes x 16 channels (B rows 16c..16c+15 hold
// class c's taps) and each row keeps only its own class's 16 columns.
struct Conv2Dgrad {
  static constexpr bool ASYNC = true;
  const void* dummy = k_ones_chunk;
  static constexpr bool A_MN = false, B_MN = false;
  int M, N, K, kb_per_split;
  Geo g;
  int F, QH, QW;         // QH = ceil(oh1/2), QW = ceil(ow1/2)
  FastDiv fcls, fq, fqw; // F*QH*QW, QH*QW, QW
  const bf16* dY2;
  const bf16* wdg;  // [16 ci][4 ky][4 kx][32 co]
  const bf16* act1;
  bf16* dY1;
  __device__ void decode(int m, int& cls, int& f, int& y, int& x) const {
    uint32_t c, rem, ff, q, qy, qx;
    fcls.divmod((uint32_t)m, c, rem);
    fq.divmod(rem, ff, q);
    fqw.divmod(q, qy, qx);
    cls = (int)c; f = (int)ff;
    y = 2 * (int)qy + (cls >> 1);
    x = 2 * (int)qx + (cls & 1);
  }
  __device__ const void* ptr_a(int m, int k) const {
    int cls, f, y, x;
    decode(m, cls, f, y, x);
    if (y >= g.oh1 || x >= g.ow1) return nullptr;
    const int kyi = k >> 6, kxi = (k >> 5) & 1, co0 = k & 31;
    const int oy = (y >> 1) - kyi, ox = (x >> 1) - kxi;
    if (oy < 0 || ox < 0 || oy >= g.oh2 || ox >= g.ow2) return nullptr;
    return dY2 + (((size_t)f * g.oh2 + oy) * g.ow2 + ox) * 32 + co0;
  }
  __device__ const void* ptr_b(int n, int k) const {
    const int cls = n >> 4, ci = n & 15;
    const int ky = (cls >> 1) + 2 * (k >> 6), kx = (cls & 1) + 2 * ((k >> 5) & 1);
    return wdg + (size_t)ci * 512 + (ky * 4 + kx) * 32 + (k & 31);
  }
  __device__ size_t pix(int m, bool& ok) const {
    int cls, f, y, x;
    decode(m, cls, f, y, x);
    ok = y < g.oh1 && x < g.ow1;
    return ((size_t)f * g.oh1 + y) * g.ow1 + x;
  }
  __device__ void store(int m, int n, float v) const {
    int cls, f, y, x;
    decode(m, cls, f, y, x);
    if ((n >> 4) != cls || y >= g.oh1 || x >= g.ow1) return;
    const size_t i = (((size_t)f * g.oh1 + y) * g.ow1 + x) * 16 + (n & 15);
    dY1[i] = to_bf(bf2f(act1[i]) > 0.f ? v : 0.f);
  }
  static constexpr bool VEC_STORE = true;
  __device__ void store16(int m, int n0, float (&v)[16]) const {
    int cls, f, y, x;
    decode(m, cls, f, y, x);
    if ((n0 >> 4) != cls || y >= g.oh1 || x >= g.ow1) return;
    const size_t i = (((size_t)f * g.oh1 + y) * g.ow1 + x) * 16;
    relu_mask16(act1 + i, v);
    st_bf16x16(dY1 + i, v);
  }
};

// dW1^T[kin][co] = (1/255) sum_rows im2col(obs)[row][kin] dY1[row][co]
struct Conv1Wgrad {
  static constexpr bool ASYNC = true;
  const void* dummy = k_ones_chunk;
  static constexpr bool A_MN = true, B_MN = true;
  int M, N, K, kb_per_split;
  Geo g;
  const bf16* obs;
  const bf16* dY1;
  float* g_w;
  __device__ const void* ptr_a(int row, int m8) const {
    uint32_t f, oy, ox;
    split_row(g.hw1, g.w1, row, f, oy, ox);
    const int ky = m8 >> 5, kx = (m8 & 31) >> 2;   // C == 4
    return obs + (((size_t)f * g.H + oy * 4 + ky) * g.W + ox * 4 + kx) * 4;
  }
  __device__ const void* ptr_b(int row, int n8) const { return dY1 + (size_t)row * 16 + n8; }
  __device__ void store(int m, int n, float v) const {
    g_w[(size_t)n * M + m] = v * (1.f / 255.f);
  }
};


}  // namespace seed
