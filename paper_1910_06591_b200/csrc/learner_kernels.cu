// learner_kernels.cu — see learner_kernels.cuh.
#include <algorithm>
#include "learner_kernels.cuh"
#include "net.cuh"
#include "conv3w.cuh"

namespace seed {

// Warp per row, lane = output (O <= 64: two outputs per lane), row staged in
// shared memory, weights staged transposed [I][O] (conflict-free), 4 partial
// accumulators per output.  I <= 256.
__global__ void __launch_bounds__(256) dense_fwd_f32(int R, int I, int O, const float* __restrict__ X,
                                                     const float* __restrict__ W,
                                                     const float* __restrict__ b,
                                                     float* __restrict__ Y, int ldy,
                                                     float* __restrict__ Yv, int relu) {
  pdl_wait_trig();
  extern __shared__ float shf[];
  float* Wt = shf;                  // [I][O]
  float* xs = shf + I * O;          // [8][I]
  for (int q = threadIdx.x; q < I * O; q += blockDim.x) {
    const int o = q / I, i = q % I;
    Wt[i * O + o] = W[q];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* xw = xs + warp * I;
  for (int r = blockIdx.x * 8 + warp; r < R; r += gridDim.x * 8) {
    for (int i = lane; i < I; i += 32) xw[i] = X[(size_t)r * I + i];
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int o = lane + 32 * h;
      if (o < O) {
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
        int i = 0;
        for (; i + 3 < I; i += 4) {
          a0 += xw[i] * Wt[i * O + o];
          a1 += xw[i + 1] * Wt[(i + 1) * O + o];
          a2 += xw[i + 2] * Wt[(i + 2) * O + o];
          a3 += xw[i + 3] * Wt[(i + 3) * O + o];
        }
        for (; i < I; ++i) a0 += xw[i] * Wt[i * O + o];
        float y = ((a0 + a1) + (a2 + a3)) + b[o];
        if (relu) y = fmaxf(y, 0.f);
        if (Yv && o == O - 1) Yv[r] = y;
        else Y[(size_t)r * ldy + o] = y;
      }
    }
    __syncwarp();
  }
}

__device__ __forceinline__ float dy_at(const float* dy, int ldy, const float* dv, int r, int o) {
  return (dv && o == ldy) ? dv[r] : dy[(size_t)r * ldy + o];
}

// block = DG_ROWS rows x all I columns; W [O][I] and the dY rows staged in shared memory
constexpr int DG_ROWS = 8;
__global__ void __launch_bounds__(256) dense_dgrad_f32(int R, int I, int O, const float* __restrict__ dy,
                                                       int ldy, const float* __restrict__ dv,
                                                       const float* __restrict__ W,
                                                       const float* __restrict__ mask,
                                                       float* __restrict__ dX) {
  pdl_wait_trig();
  extern __shared__ float shf[];
  float* Ws = shf;              // [O][I]
  float* ds = shf + O * I;      // [DG_ROWS][O]
  for (int q = threadIdx.x; q < O * I; q += blockDim.x) Ws[q] = W[q];
  const int r0 = blockIdx.x * DG_ROWS;
  for (int q = threadIdx.x; q < DG_ROWS * O; q += blockDim.x) {
    const int rr = r0 + q / O, o = q % O;
    ds[q] = rr < R ? dy_at(dy, ldy, dv, rr, o) : 0.f;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < DG_ROWS * I; q += blockDim.x) {
    const int rl = q / I, i = q % I, r = r0 + rl;
    if (r >= R) continue;
    float s0 = 0.f, s1 = 0.f;
    int o = 0;
    for (; o + 1 < O; o += 2) {
      s0 += ds[rl * O + o] * Ws[o * I + i];
      s1 += ds[rl * O + o + 1] * Ws[(o + 1) * I + i];
    }
    if (o < O) s0 += ds[rl * O + o] * Ws[o * I + i];
    float sres = s0 + s1;
    const size_t idx = (size_t)r * I + i;
    if (mask && !(mask[idx] > 0.f)) sres = 0.f;
    dX[idx] = sres;
  }
}

// grid (O, ceil((I+1)/32)), block 256 = 32 columns x 8 row groups; each thread
// keeps 4 independent accumulators, the 8 row groups are summed in fixed order.
__global__ void __launch_bounds__(256) dense_wgrad_f32(int R, int I, int O, const float* __restrict__ dy,
                                                       int ldy, const float* __restrict__ dv,
                                                       const float* __restrict__ X,
                                                       float* __restrict__ gW, float* __restrict__ gb) {
  pdl_wait_trig();
  const int o = blockIdx.x;
  const int lane = threadIdx.x & 31, rg = threadIdx.x >> 5;
  const int i = blockIdx.y * 32 + lane;
  const bool isb = i == I, valid = i <= I;
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  if (valid) {
    int r = rg;
    for (; r + 24 < R; r += 32) {
      const float d0 = dy_at(dy, ldy, dv, r, o), d1 = dy_at(dy, ldy, dv, r + 8, o);
      const float d2 = dy_at(dy, ldy, dv, r + 16, o), d3 = dy_at(dy, ldy, dv, r + 24, o);
      const float x0 = isb ? 1.f : X[(size_t)r * I + i];
      const float x1 = isb ? 1.f : X[(size_t)(r + 8) * I + i];
      const float x2 = isb ? 1.f : X[(size_t)(r + 16) * I + i];
      const float x3 = isb ? 1.f : X[(size_t)(r + 24) * I + i];
      a0 += d0 * x0; a1 += d1 * x1; a2 += d2 * x2; a3 += d3 * x3;
    }
    for (; r < R; r += 8) a0 += dy_at(dy, ldy, dv, r, o) * (isb ? 1.f : X[(size_t)r * I + i]);
  }
  __shared__ float sh[8][33];
  sh[rg][lane] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  if (rg == 0 && valid) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += sh[k][lane];
    if (isb) gb[o] = t;
    else gW[(size_t)o * I + i] = t;
  }
}

seed_status launch_dense_fwd(int R, int I, int O, const float* X, const float* W, const float* b,
                             float* Y, int ldy, float* Yv, int relu, cudaStream_t st) {
  if (I > 256 || O > 64) return SEED_E_SHAPE;
  static PerDevice attr;
  SEED_TRY(smem_optin(attr, dense_fwd_f32, (256 * 64 + 8 * 256) * 4));
    const size_t smem = (size_t)(I * O + 8 * I) * 4;
  const int blocks = std::min(ceil_div(R, 8), 148 * 4);
  return launch_k(dense_fwd_f32, dim3(blocks), dim3(256), smem, st, R, I, O, X, W, b, Y, ldy, Yv, relu);
}

seed_status launch_dense_dgrad(int R, int I, int O, const float* dy, int ldy, const float* dv,
                               const float* W, const float* mask, float* dX, cudaStream_t st) {
  if (I > 256 || O > 64) return SEED_E_SHAPE;
  static PerDevice attr;
  SEED_TRY(smem_optin(attr, dense_dgrad_f32, (256 * 64 + DG_ROWS * 64) * 4));
    const size_t smem = (size_t)(O * I + DG_ROWS * O) * 4;
  return launch_k(dense_dgrad_f32, dim3(ceil_div(R, DG_ROWS)), dim3(256), smem, st, R, I, O, dy, ldy, dv,
                  W, mask, dX);
}

// ------------------------------------------------------------------ K2 policy loss
// One block per trajectory b (T <= 256):
//  1. warps compute the per-step policy statistics (lane = action): log-sum-exp,
//     target log-prob, entropy H_t (H5);
//  2. warp 0 runs the V-trace scan (vtrace_chunk, 4 steps per lane, H6) and the
//     loss sums;
//  3. all threads write the closed-form output gradients (H7).
__global__ void __launch_bounds__(256) policy_loss_kernel(const LossArgs a) {
  pdl_wait_trig();
  __shared__ float s_lse[256], s_tlp[256], s_H[256], s_pg[256];
  const int b = blockIdx.x;
  const int T = a.T, T1 = a.T + 1, A = a.A;
  const size_t row0 = (size_t)b * T1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = warp; t < T; t += 8) {
    const float z = lane < A ? a.logits[(row0 + t) * A + lane] : -INFINITY;
    const float mx = warp_max(z);
    const float e = lane < A ? expf(z - mx) : 0.f;
    const float se = warp_sum(e);
    const float lse = mx + logf(se);
    const float lp = z - lse;
    const float H = -warp_sum(lane < A ? expf(lp) * lp : 0.f);
    const int act = a.action[row0 + t];
    const float tl = __shfl_sync(0xffffffffu, lp, act & 31);
    if (lane == 0) {
      s_lse[t] = lse;
      s_tlp[t] = tl;
      s_H[t] = H;
    }
  }
  __syncthreads();
  if (warp == 0) {
    VtraceLaneState st;
    st.init(a.values[row0 + T]);
    bool bad = !isfinite(st.carry_vs);
    float sum_pg = 0.f, sum_b = 0.f, sum_h = 0.f;
    const int nch = (T + 127) / 128;
    for (int ch = nch - 1; ch >= 0; --ch) {
      const int t0 = ch * 128 + 4 * lane;
      float d[4], r[4], g[4], v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int t = t0 + j;
        d[j] = r[j] = g[j] = v[j] = 0.f;
        if (t < T) {
          d[j] = s_tlp[t] - a.blp[row0 + t];
          r[j] = a.reward[row0 + t + 1];
          g[j] = a.discount * (a.done[row0 + t + 1] ? 0.f : 1.f);
          v[j] = a.values[row0 + t];
        }
      }
      float vs[4], pg[4];
      bad |= vtrace_chunk<32>(st, lane, t0, T, d, r, g, v, a.rho_bar, a.c_bar, a.lam, vs, pg);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int t = t0 + j;
        if (t >= T) continue;
        s_pg[t] = pg[j];
        a.vs[(size_t)b * T + t] = vs[j];
        a.pg[(size_t)b * T + t] = pg[j];
        a.dvalues[row0 + t] = a.scale * a.vf_coef * (v[j] - vs[j]);
        sum_pg += -pg[j] * s_tlp[t];
        sum_b += (vs[j] - v[j]) * (vs[j] - v[j]);
        sum_h += s_H[t];
      }
    }
    sum_pg = warp_sum(sum_pg);
    sum_b = warp_sum(sum_b);
    sum_h = warp_sum(sum_h);
    const unsigned anybad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
      float* pp = a.part + (size_t)b * 4;
      pp[0] = a.scale * sum_pg;
      pp[1] = a.scale * 0.5f * a.vf_coef * sum_b;
      pp[2] = -a.scale * a.ent_coef * sum_h;
      pp[3] = anybad ? 1.f : 0.f;
      a.dvalues[row0 + T] = 0.f;   // bootstrap is a constant (C4)
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < T1 * A; q += blockDim.x) {
    const int t = q / A, k = q % A;
    const size_t idx = (row0 + t) * A + k;
    if (t == T) {
      a.dlogits[idx] = 0.f;
      continue;
    }
    const float lp = a.logits[idx] - s_lse[t];
    const float p = expf(lp);
    const float onehot = (k == a.action[row0 + t]) ? 1.f : 0.f;
    a.dlogits[idx] = a.scale * (-s_pg[t] * (onehot - p) + a.ent_coef * p * (lp + s_H[t]));
  }
}

// ------------------------------------------------------------------ fused heads + loss
// One block per trajectory b.  Phase 1: logits | value = H W^T + b (H4; warp per
// row, lane = output, H rows staged 32 at a time).  Phase 2: the policy loss of
// policy_loss_kernel on those values (H5-H7).  Phase 3: dH = [dlogits|dvalue] W
// (thread = hidden unit, W row in registers) and the per-trajectory weight /
// bias gradient partials (summed over b in order by heads_wgrad_finish).
constexpr int HL_RC = 32;
constexpr int HL_THREADS = 512;
constexpr int HL_CL = 4;   // CTAs (thread-block cluster) per trajectory
#ifdef SEED_LSTM_PROF
__device__ long long g_heads_prof[8];
#define HL_STAMP(I) \
  if (blockIdx.x == 0 && threadIdx.x == 0) g_heads_prof[I] = clock64();
extern "C" int seed_debug_heads_prof(long long* out) {
  return cudaMemcpyFromSymbol(out, g_heads_prof, sizeof(g_heads_prof)) == cudaSuccess ? 0 : 5;
}
#else
#define HL_STAMP(I)
#endif

// MINB = 2 (64 registers, two CTAs per SM) when the trajectories' clusters exceed one
// wave of 148 SMs at one CTA each (c4: B = 128 -> 512 CTAs, 81 -> 69 us); below that
// the 99-register form is faster (c2: 24 vs 27 us)
// CL = CTAs (cluster) per trajectory: 4, or 2 when B is large enough that 4 would
// need more than one wave even at two CTAs per SM
template <int MINB, int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(HL_THREADS, MINB)
    heads_loss_kernel(const LossArgs a) {
  HL_STAMP(0)
  extern __shared__ float hsm[];
  const int I = a.I, A = a.A, A1 = A + 1, A1p = A1 | 1;
  const int T = a.T, T1 = T + 1, b = blockIdx.x / CL;
  const int cr = (int)cluster_rank();
  const int Rr = (T1 + CL - 1) / CL, rb0 = min(T1, cr * Rr), rb1 = min(T1, rb0 + Rr);
  const size_t row0 = (size_t)b * T1;
  float* Wt = hsm;                  // [I][A1p]
  float* sL = Wt + I * A1p;         // [T1][A1p]: logits | value, then their gradients
  float* Hc = hsm + (((size_t)I * A1p + (size_t)T1 * A1p + 3) & ~(size_t)3);   // [HL_RC][I], 16-B aligned
  __shared__ float s_lse[256], s_tlp[256], s_H[256], s_pg[256], s_dv[257];
  __shared__ int s_act[256];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NW = HL_THREADS / 32;
  // per-trajectory scalars used by phase 2, loaded up front (off the critical path)
  for (int t = tid; t < T; t += HL_THREADS) s_act[t] = a.action[row0 + t];
  float pre_blp[8], pre_r[8], pre_g[8];   // warp 0, V-trace chunk inputs (T <= 256)
  if (warp == 0) {
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int t = c * 128 + 4 * lane + j;
        const bool ok = t < T;
        pre_blp[c * 4 + j] = ok ? a.blp[row0 + t] : 0.f;
        pre_r[c * 4 + j] = ok ? a.reward[row0 + t + 1] : 0.f;
        pre_g[c * 4 + j] = ok ? a.discount * (a.done[row0 + t + 1] ? 0.f : 1.f) : 0.f;
      }
  }
  // W^T staged with float4 loads (I % 4 == 0: a float4 never crosses a row)
  for (int q4 = tid; q4 < A1 * I / 4; q4 += HL_THREADS) {
    const float4 w4 = __ldg(reinterpret_cast<const float4*>(a.hw) + q4);
    const int q = q4 * 4, o = q / I, i = q - o * I;
    Wt[i * A1p + o] = w4.x;
    Wt[(i + 1) * A1p + o] = w4.y;
    Wt[(i + 2) * A1p + o] = w4.z;
    Wt[(i + 3) * A1p + o] = w4.w;
  }
  // everything above reads the batch and the heads weights (last written by the
  // previous step's Adam, >= 2 kernels back); H comes from the preceding kernel
  pdl_wait_trig();
  cluster_sync_all();   // every CTA of the cluster runs before any DSMEM store
  // ---- phase 1: heads forward of this CTA's rows, one (row, output) dot product
  // per thread; results stored into all CL CTAs' sL (DSMEM all-gather)
  for (int r0 = rb0; r0 < rb1; r0 += HL_RC) {
    const int nr = min(HL_RC, rb1 - r0);
    __syncthreads();
    const float4* src = reinterpret_cast<const float4*>(a.H + (row0 + r0) * I);
    for (int q = tid; q < nr * I / 4; q += HL_THREADS) reinterpret_cast<float4*>(Hc)[q] = src[q];
    __syncthreads();
    for (int q = tid; q < nr * A1; q += HL_THREADS) {
      const int rr = q / A1, o = q - rr * A1;
      const float* hr = Hc + rr * I;
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll 4
      for (int i = 0; i < I; i += 4) {
        const float4 h4 = *reinterpret_cast<const float4*>(hr + i);
        a0 += h4.x * Wt[i * A1p + o];
        a1 += h4.y * Wt[(i + 1) * A1p + o];
        a2 += h4.z * Wt[(i + 2) * A1p + o];
        a3 += h4.w * Wt[(i + 3) * A1p + o];
      }
      const float y = ((a0 + a1) + (a2 + a3)) + a.hb[o];
      const int t = r0 + rr;
      const uint32_t la = smem_u32(sL + t * A1p + o);
#pragma unroll
      for (int d = 0; d < CL; ++d) st_cluster_f32(mapa_u32(la, d), y);
      if (o < A) a.logits[(row0 + t) * A + o] = y;
      else a.values[row0 + t] = y;
    }
  }
  cluster_sync_all();   // all rows' logits | values present in every CTA
  HL_STAMP(1)
  // ---- phase 2: policy statistics, V-trace, losses (as policy_loss_kernel)
  for (int t = warp; t < T; t += NW) {
    const float z = lane < A ? sL[t * A1p + lane] : -INFINITY;
    const float mx = warp_max(z);
    const float e = lane < A ? expf(z - mx) : 0.f;
    const float se = warp_sum(e);
    const float lse = mx + logf(se);
    const float lp = z - lse;
    const float Hn = -warp_sum(lane < A ? expf(lp) * lp : 0.f);
    const int act = s_act[t];
    const float tl = __shfl_sync(0xffffffffu, lp, act & 31);
    if (lane == 0) {
      s_lse[t] = lse;
      s_tlp[t] = tl;
      s_H[t] = Hn;
    }
  }
  __syncthreads();
  HL_STAMP(2)
  if (warp == 0) {
    VtraceLaneState st;
    st.init(sL[T * A1p + A]);
    bool bad = !isfinite(st.carry_vs);
    float sum_pg = 0.f, sum_b = 0.f, sum_h = 0.f;
    const int nch = (T + 127) / 128;
#pragma unroll
    for (int ch = 1; ch >= 0; --ch) {   // static chunk index: the prefetched inputs stay in registers
      if (ch >= nch) continue;
      const int t0 = ch * 128 + 4 * lane;
      float d[4], r[4], g[4], v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int t = t0 + j;
        d[j] = r[j] = g[j] = v[j] = 0.f;
        if (t < T) {
          d[j] = s_tlp[t] - pre_blp[ch * 4 + j];
          r[j] = pre_r[ch * 4 + j];
          g[j] = pre_g[ch * 4 + j];
          v[j] = sL[t * A1p + A];
        }
      }
      float vs[4], pg[4];
      bad |= vtrace_chunk<32>(st, lane, t0, T, d, r, g, v, a.rho_bar, a.c_bar, a.lam, vs, pg);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int t = t0 + j;
        if (t >= T) continue;
        s_pg[t] = pg[j];
        const float dv = a.scale * a.vf_coef * (v[j] - vs[j]);
        s_dv[t] = dv;
        if (cr == 0) {   // phase 2 runs redundantly in every CTA; rank 0 writes
          a.vs[(size_t)b * T + t] = vs[j];
          a.pg[(size_t)b * T + t] = pg[j];
          a.dvalues[row0 + t] = dv;
        }
        sum_pg += -pg[j] * s_tlp[t];
        sum_b += (vs[j] - v[j]) * (vs[j] - v[j]);
        sum_h += s_H[t];
      }
    }
    sum_pg = warp_sum(sum_pg);
    sum_b = warp_sum(sum_b);
    sum_h = warp_sum(sum_h);
    const unsigned anybad = __any_sync(0xffffffffu, bad);
    if (lane == 0 && cr == 0) {
      float* pp = a.part + (size_t)b * 4;
      pp[0] = a.scale * sum_pg;
      pp[1] = a.scale * 0.5f * a.vf_coef * sum_b;
      pp[2] = -a.scale * a.ent_coef * sum_h;
      pp[3] = anybad ? 1.f : 0.f;
      a.dvalues[row0 + T] = 0.f;   // bootstrap is a constant (C4)
    }
    if (lane == 0) s_dv[T] = 0.f;
  }
  __syncthreads();
  HL_STAMP(3)
  for (int q = tid; q < T1 * A1; q += HL_THREADS) {
    const int t = q / A1, k = q - t * A1;
    float d;
    if (k == A) {
      d = s_dv[t];
    } else if (t == T) {
      d = 0.f;
      if (cr == 0) a.dlogits[(row0 + t) * A + k] = 0.f;
    } else {
      const float lp = sL[t * A1p + k] - s_lse[t];
      const float p = expf(lp);
      const float onehot = (k == s_act[t]) ? 1.f : 0.f;
      d = a.scale * (-s_pg[t] * (onehot - p) + a.ent_coef * p * (lp + s_H[t]));
      if (cr == 0) a.dlogits[(row0 + t) * A + k] = d;
    }
    sL[t * A1p + k] = d;
  }
  // ---- phase 3: dH and the per-trajectory weight / bias gradients; thread =
  // (hidden unit i, row parity rg); the two row-parity partials are added in order
  HL_STAMP(4)
  constexpr int AMAX = 33;
  const int ci = tid & 255, rg = tid >> 8;
  const bool col = ci < I;
  float wreg[AMAX], acc[AMAX];
#pragma unroll
  for (int o = 0; o < AMAX; ++o) {
    wreg[o] = (col && o < A1) ? Wt[ci * A1p + o] : 0.f;
    acc[o] = 0.f;
  }
  for (int r0 = rb0; r0 < rb1; r0 += HL_RC) {
    const int nr = min(HL_RC, rb1 - r0);
    __syncthreads();
    const float4* src = reinterpret_cast<const float4*>(a.H + (row0 + r0) * I);
    for (int q = tid; q < nr * I / 4; q += HL_THREADS) reinterpret_cast<float4*>(Hc)[q] = src[q];
    __syncthreads();
    if (col) {
      for (int rr = rg; rr < nr; rr += 2) {
        const int t = r0 + rr;
        const float h = Hc[rr * I + ci];
        const float* dl = sL + t * A1p;
        float dh = 0.f;
#pragma unroll
        for (int o = 0; o < AMAX; ++o) {
          if (o < A1) {
            const float d = dl[o];
            dh += d * wreg[o];
            acc[o] += d * h;
          }
        }
        const size_t idx = (row0 + t) * I + ci;
        if (a.hmask && !(a.hmask[idx] > 0.f)) dh = 0.f;
        a.dH[idx] = dh;
      }
    }
  }
  __syncthreads();   // Hc free: row-parity-1 partials go through it
  HL_STAMP(5)
  float* red = Hc;   // [A1][I]
  if (col && rg == 1) {
#pragma unroll
    for (int o = 0; o < AMAX; ++o)
      if (o < A1) red[o * I + ci] = acc[o];
  }
  __syncthreads();
  if (col && rg == 0) {
#pragma unroll
    for (int o = 0; o < AMAX; ++o)
      if (o < A1) acc[o] += red[o * I + ci];
  }
  float sb = 0.f;
  if (tid < A1)
    for (int t = rb0; t < rb1; ++t) sb += sL[t * A1p + tid];
  // one partial per (trajectory, cluster rank), written straight to global (a DSMEM
  // gather into rank 0 cost two cluster barriers and ~5K remote stores per CTA);
  // heads_wgrad_finish sums them in (b, rank) order
  {
    const int n = A1 * (I + 1);
    float* wp = a.wpart + ((size_t)b * CL + cr) * n;
    if (col && rg == 0) {
#pragma unroll
      for (int o = 0; o < AMAX; ++o)
        if (o < A1) wp[o * (I + 1) + ci] = acc[o];
    }
    if (tid < A1) wp[tid * (I + 1) + I] = sb;
  }
  // (the last DSMEM access, phase 1's all-gather, completed at its cluster barrier)
  HL_STAMP(6)
}

// heads weight / bias gradient: fixed-order sum of the per-(trajectory, cluster
// rank) partials.  Block = 32 outputs x 8 groups; group g adds partials
// g, g+8, ... in order, then the 8 group sums are added in order.
__global__ void __launch_bounds__(256) heads_wgrad_finish(int NP, int A1, int I, const float* __restrict__ wpart,
                                                          float* __restrict__ g_w, float* __restrict__ g_b) {
  pdl_wait_trig();
  const int n = A1 * (I + 1);
  const int q = blockIdx.x * 32 + (threadIdx.x & 31), g = threadIdx.x >> 5;
  __shared__ float sh[8][33];
  float s = 0.f;
  if (q < n) {
#pragma unroll 4
    for (int b = g; b < NP; b += 8) s += __ldcg(wpart + (size_t)b * n + q);
  }
  sh[g][threadIdx.x & 31] = s;
  __syncthreads();
  if (g == 0 && q < n) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += sh[k][threadIdx.x];
    const int o = q / (I + 1), i = q - o * (I + 1);
    if (i < I) g_w[(size_t)o * I + i] = t;
    else g_b[o] = t;
  }
}

seed_status launch_heads_loss(const LossArgs& a, cudaStream_t st) {
  if (a.T > 256 || a.A > 32 || a.I > 256 || (a.I & 3)) return SEED_E_SHAPE;
  const int A1p = (a.A + 1) | 1;
  // Hc holds HL_RC rows of H, later the [A+1][I] row-parity partials (A+1 <= HL_RC+1)
  const size_t smem = ((((size_t)a.I * A1p + (size_t)(a.T + 1) * A1p + 3) & ~(size_t)3) +
                       (size_t)(HL_RC + 1) * a.I) * 4;
  const int smax = (int)std::max<size_t>((256 * 33 + 257 * 33 + 4 + (HL_RC + 1) * 256) * 4,
                                          (size_t)HL_CL * 33 * 257 * 4);
  int cl = HL_CL;
  if (a.B * HL_CL > 2 * 148) {          // more than one wave at two CTAs per SM
    cl = 2;
    static PerDevice attr;
    SEED_TRY(smem_optin(attr, heads_loss_kernel<2, 2>, smax));
    SEED_TRY(launch_k(heads_loss_kernel<2, 2>, dim3(a.B * 2), dim3(HL_THREADS), smem, st, a));
  } else if (a.B * HL_CL > 148) {
    static PerDevice attr2;
    SEED_TRY(smem_optin(attr2, heads_loss_kernel<2, HL_CL>, smax));
    SEED_TRY(launch_k(heads_loss_kernel<2, HL_CL>, dim3(a.B * HL_CL), dim3(HL_THREADS), smem, st, a));
  } else {
    static PerDevice attr1;
    SEED_TRY(smem_optin(attr1, heads_loss_kernel<1, HL_CL>, smax));
    SEED_TRY(launch_k(heads_loss_kernel<1, HL_CL>, dim3(a.B * HL_CL), dim3(HL_THREADS), smem, st, a));
  }
  const int n = (a.A + 1) * (a.I + 1);
  return launch_k(heads_wgrad_finish, dim3(ceil_div(n, 32)), dim3(256), 0, st, a.B * cl, a.A + 1,
                  a.I, (const float*)a.wpart, a.g_w, a.g_b);
}

seed_status launch_policy_loss(const LossArgs& a, cudaStream_t st) {
  if (a.T > 256 || a.A > 32) return SEED_E_SHAPE;
  return launch_k(policy_loss_kernel, dim3(a.B), dim3(256), 0, st, a);
}

// ------------------------------------------------------------------ LSTM input extras
__global__ void core_extras_kernel(int F, int A, int Kxp, const int32_t* __restrict__ prev_action,
                                   const float* __restrict__ reward,
                                   const uint8_t* __restrict__ done, __nv_bfloat16* X) {
  pdl_wait_trig();
  const int E = Kxp - 256;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)F * E) return;
  const int f = (int)(idx / E), j = (int)(idx % E);
  const bool dn = done[f] != 0;
  float v = 0.f;
  if (j < A) v = (!dn && prev_action[f] == j) ? 1.f : 0.f;
  else if (j == A) v = dn ? 0.f : fminf(fmaxf(reward[f], -1.f), 1.f);
  else if (j == A + 1) v = 1.f;  // all-ones column: its weight-grad row is the bias grad
  X[(size_t)f * Kxp + 256 + j] = __float2bfloat16_rn(v);
}


// ------------------------------------------------------------------ K9 clip + Adam
__device__ __forceinline__ double block_sum_double(double v, double* sh8) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh8[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += sh8[k];   // fixed order
  return t;   // valid in thread 0
}

__global__ void __launch_bounds__(256) grad_norm_kernel(const NormArgs a) {
  pdl_wait_trig();
  // 4 float4 per thread, all loads issued first; squares and sums in double
  const int64_t P4 = a.P / 4;
  const float4* g4 = reinterpret_cast<const float4*>(a.g);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double s = 0.0;
  for (int64_t base = t0; base < P4; base += 4 * stride) {
    float4 x[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t i = base + q * stride;
      x[q] = i < P4 ? g4[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      s += ((double)x[q].x * x[q].x + (double)x[q].y * x[q].y) +
           ((double)x[q].z * x[q].z + (double)x[q].w * x[q].w);   // fp64: no fp32 overflow
  }
  if (blockIdx.x == 0 && threadIdx.x < a.P - 4 * P4) {
    const double x = a.g[4 * P4 + threadIdx.x];
    s += x * x;
  }
  __shared__ double sh8[8];
  __shared__ bool last;
  const double bs = block_sum_double(s, sh8);
  if (threadIdx.x == 0) {
    a.part[blockIdx.x] = bs;
    __threadfence();
    last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double t = 0.0;
  for (int k = threadIdx.x; k < (int)gridDim.x; k += 256) t += __ldcg(a.part + k);
  __syncthreads();   // sh8 reuse
  const double tot = block_sum_double(t, sh8);
  if (threadIdx.x == 0) {
    const double norm = sqrt(tot);
    const bool finite = isfinite(norm);
    const int64_t st = *a.step;
    const int64_t tt = st + 1;
    *a.step_in = st;
    *a.norm = norm;
    a.coef[0] = finite && norm > (double)a.max_norm ? (float)((double)a.max_norm / norm) : 1.f;
    a.coef[1] = (float)(1.0 - pow((double)a.beta1, (double)tt));
    a.coef[2] = (float)(1.0 - pow((double)a.beta2, (double)tt));
    a.coef[3] = finite ? 1.f : 0.f;
    *a.ticket = 0;
  }
}

// bf16 operand images of the updated parameters (net.cuh LowpImg), written by
// the Adam kernel so no separate refresh pass is needed.
__device__ __forceinline__ void lowp_write(const AdamArgs& a, int64_t i, float v) {
  for (int k = 0; k < a.nimg; ++k) {
    const LowpImg& m = a.img[k];
    const int64_t n = (int64_t)m.rows * m.cols;
    const int64_t e = i - m.src;
    if (e < 0 || e >= n) continue;
    int64_t dst;
    if (m.kind == IMG_S2D) {
      dst = s2d_img_pos(m, e);
    } else if (m.kind == IMG_WIN3) {
      dst = win3p_img_pos(m.d0, m.d1, m.d2, m.d3, e);
    } else if (m.kind == IMG_COPY_PAD) {
      uint32_t r, c;
      img_rc(m, (uint32_t)e, r, c);
      dst = (int64_t)r * m.ld + c;
    } else {  // src [CO][KH][KW][CI] -> dst [CI][KH][KW][CO]
      const int ci = (int)(e % m.d3);
      int64_t q = e / m.d3;
      const int kx = (int)(q % m.d2); q /= m.d2;
      const int ky = (int)(q % m.d1);
      const int co = (int)(q / m.d1);
      dst = (((int64_t)ci * m.d1 + ky) * m.d2 + kx) * m.d0 + co;
    }
    a.lowp[m.dst + dst] = __float2bfloat16_rn(v);
  }
}

// 4 consecutive parameters per thread (float4 when aligned); the bf16 image of
// the group is found once per group.
__device__ __forceinline__ int find_img(const uint32_t (*bounds)[2], int nimg, uint32_t i) {
  for (int k = 0; k < nimg; ++k)
    if (i >= bounds[k][0] && i < bounds[k][1]) return k;
  return -1;
}

constexpr int ADAM_GPT = 2;   // float4 groups per thread, all loads in flight together

struct AdamIn { float4 g, m, v, p; };
__device__ __forceinline__ AdamIn adam_load(const AdamArgs& a, int64_t gi) {
  const int64_t i0 = gi * 4;
  AdamIn r;
  if (i0 + 3 < a.P) {
    r.g = reinterpret_cast<const float4*>(a.grads)[gi];
    r.m = reinterpret_cast<const float4*>(a.m)[gi];
    r.v = reinterpret_cast<const float4*>(a.v)[gi];
    r.p = reinterpret_cast<const float4*>(a.params)[gi];
  } else {
    float* g = &r.g.x; float* m = &r.m.x; float* v = &r.v.x; float* p = &r.p.x;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const bool ok = i0 + q < a.P;
      g[q] = ok ? a.grads[i0 + q] : 0.f;
      m[q] = ok ? a.m[i0 + q] : 0.f;
      v[q] = ok ? a.v[i0 + q] : 0.f;
      p[q] = ok ? a.params[i0 + q] : 0.f;
    }
  }
  return r;
}

__global__ void __launch_bounds__(256) adam_kernel(const AdamArgs a) {
  pdl_wait_trig();
  __shared__ uint32_t bounds[8][2];   // source parameter range of each bf16 image
  if (threadIdx.x < a.nimg) {
    bounds[threadIdx.x][0] = (uint32_t)a.img[threadIdx.x].src;
    bounds[threadIdx.x][1] =
        (uint32_t)(a.img[threadIdx.x].src + (int64_t)a.img[threadIdx.x].rows * a.img[threadIdx.x].cols);
  }
  __syncthreads();
  const bool finite = a.coef[3] != 0.f;
  if (finite) {
    // bias corrections as reciprocals; one (fast, 2-ulp) division per parameter —
    // the IEEE-division slow path (zero / denormal operands) is kept off the loop
    const float scale = a.coef[0], ibc1 = 1.f / a.coef[1], ibc2 = 1.f / a.coef[2];
    const int64_t ngroups = (a.P + 3) / 4;
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    for (int64_t g0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g0 < ngroups; g0 += ADAM_GPT * T) {
      AdamIn in[ADAM_GPT];
#pragma unroll
      for (int k = 0; k < ADAM_GPT; ++k)
        if (g0 + k * T < ngroups) in[k] = adam_load(a, g0 + k * T);
#pragma unroll
      for (int k = 0; k < ADAM_GPT; ++k) {
        const int64_t gi = g0 + k * T;
        if (gi >= ngroups) break;
        const int64_t i0 = gi * 4;
        float g[4] = {in[k].g.x, in[k].g.y, in[k].g.z, in[k].g.w};
        float m[4] = {in[k].m.x, in[k].m.y, in[k].m.z, in[k].m.w};
        float v[4] = {in[k].v.x, in[k].v.y, in[k].v.z, in[k].v.w};
        float p[4] = {in[k].p.x, in[k].p.y, in[k].p.z, in[k].p.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float gg = g[q] * scale;
          m[q] = a.beta1 * m[q] + (1.f - a.beta1) * gg;
          v[q] = a.beta2 * v[q] + (1.f - a.beta2) * gg * gg;
          p[q] = p[q] - __fdividef(a.lr * (m[q] * ibc1), sqrtf(v[q] * ibc2) + a.eps);
        }
        if (i0 + 3 < a.P) {
          reinterpret_cast<float4*>(a.m)[gi] = make_float4(m[0], m[1], m[2], m[3]);
          reinterpret_cast<float4*>(a.v)[gi] = make_float4(v[0], v[1], v[2], v[3]);
          reinterpret_cast<float4*>(a.params)[gi] = make_float4(p[0], p[1], p[2], p[3]);
        } else {
          for (int q = 0; q < 4 && i0 + q < a.P; ++q) {
            a.m[i0 + q] = m[q];
            a.v[i0 + q] = v[q];
            a.params[i0 + q] = p[q];
          }
        }
        if (a.nimg) {
          const int k0 = find_img(bounds, a.nimg, (uint32_t)i0);
          const int k3 = find_img(bounds, a.nimg, (uint32_t)min(i0 + 3, a.P - 1));
          bool done = false;
          if (k0 >= 0 && k0 == k3 && a.img[k0].kind == IMG_COPY_PAD) {
            const LowpImg& im = a.img[k0];
            uint32_t r, c;
            img_rc(im, (uint32_t)(i0 - im.src), r, c);
            if ((int)c + 3 < im.cols) {   // the group stays in one image row
              __nv_bfloat16* d = a.lowp + im.dst + (int64_t)r * im.ld + c;
              d[0] = __float2bfloat16_rn(p[0]); d[1] = __float2bfloat16_rn(p[1]);
              d[2] = __float2bfloat16_rn(p[2]); d[3] = __float2bfloat16_rn(p[3]);
              done = true;
            }
          }
          if (!done)
            for (int q = 0; q < 4 && i0 + q < a.P; ++q) lowp_write(a, i0 + q, p[q]);
        }
      }
    }
  }
  if (blockIdx.x == 0) {
    // per-trajectory loss partials: strided over the block's threads, then a
    // fixed-order block reduction (was one thread looping over B: the kernel's
    // straggler at B = 128)
    double q0 = 0, q1 = 0, q2 = 0;
    int nf = 0;
    for (int b = threadIdx.x; b < a.B; b += blockDim.x) {
      q0 += a.loss_part[b * 4 + 0];
      q1 += a.loss_part[b * 4 + 1];
      q2 += a.loss_part[b * 4 + 2];
      nf |= a.loss_part[b * 4 + 3] != 0.f;
    }
    __shared__ double sh8[8];
    const double l0 = block_sum_double(q0, sh8);
    __syncthreads();
    const double l1 = block_sum_double(q1, sh8);
    __syncthreads();
    const double l2 = block_sum_double(q2, sh8);
    const int anynf = __syncthreads_or(nf);
    if (threadIdx.x != 0) return;
    const float nonfin = (finite && !anynf) ? 0.f : 1.f;
    const int64_t ver = *a.step_in + (finite ? 1 : 0);
    const double norm = *a.norm;
    a.metrics[0] = (float)(l0 + l1 + l2);
    a.metrics[1] = (float)l0;
    a.metrics[2] = (float)l1;
    a.metrics[3] = (float)l2;
    a.metrics[4] = (float)norm;
    a.metrics[5] = finite ? 1.f : 0.f;
    a.metrics[6] = (float)ver;
    a.metrics[7] = nonfin;
    *a.step = ver;
  }
}

seed_status launch_clip_adam(const AdamArgs& a, cudaStream_t st) {
  const int64_t groups = (a.P + 3) / 4;
  return launch_k(adam_kernel, dim3((unsigned)std::min<int64_t>((groups + 256 * ADAM_GPT - 1) / (256 * ADAM_GPT),
                                                                 148 * 8)),
                  dim3(256), 0, st, a);
}

}  // namespace seed
