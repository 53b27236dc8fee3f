// learner_kernels.cu — see learner_kernels.cuh.
#include "learner_kernels.cuh"
#include "net.cuh"

namespace seed {

__global__ void dense_fwd_f32(int R, int I, int O, const float* __restrict__ X,
                              const float* __restrict__ W, const float* __restrict__ b,
                              float* __restrict__ Y, int ldy, float* __restrict__ Yv, int relu) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= R) return;
  const float* x = X + (size_t)warp * I;
  float xv[8];
  const int nq = (I + 31) / 32;  // I <= 256
#pragma unroll
  for (int q = 0; q < 8; ++q) xv[q] = (q < nq && lane + 32 * q < I) ? x[lane + 32 * q] : 0.f;
  for (int o = 0; o < O; ++o) {
    const float* w = W + (size_t)o * I;
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < nq && lane + 32 * q < I) s += xv[q] * w[lane + 32 * q];
    s = warp_sum(s);
    if (lane == 0) {
      float y = s + b[o];
      if (relu) y = fmaxf(y, 0.f);
      if (Yv && o == O - 1) Yv[warp] = y;
      else Y[(size_t)warp * ldy + o] = y;
    }
  }
}

__device__ __forceinline__ float dy_at(const float* dy, int ldy, const float* dv, int r, int o) {
  return (dv && o == ldy) ? dv[r] : dy[(size_t)r * ldy + o];
}

__global__ void dense_dgrad_f32(int R, int I, int O, const float* __restrict__ dy, int ldy,
                                const float* __restrict__ dv, const float* __restrict__ W,
                                const float* __restrict__ mask, float* __restrict__ dX) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)R * I) return;
  const int r = (int)(idx / I), i = (int)(idx % I);
  float s = 0.f;
  for (int o = 0; o < O; ++o) s += dy_at(dy, ldy, dv, r, o) * W[(size_t)o * I + i];
  if (mask && !(mask[idx] > 0.f)) s = 0.f;
  dX[idx] = s;
}

// grid (O, ceil((I+1)/32)), block 256 = 32 columns x 8 row groups; each thread
// keeps 4 independent accumulators, the 8 row groups are summed in fixed order.
__global__ void __launch_bounds__(256) dense_wgrad_f32(int R, int I, int O, const float* __restrict__ dy,
                                                       int ldy, const float* __restrict__ dv,
                                                       const float* __restrict__ X,
                                                       float* __restrict__ gW, float* __restrict__ gb) {
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

// ------------------------------------------------------------------ K2 policy loss
// Group of G lanes per trajectory; lane owns 4 consecutive trained steps of a
// chunk (the vtrace_chunk scheme), computes log-softmax / target log-prob /
// entropy of its steps, feeds the V-trace scan, then writes the output
// gradients (H7 closed forms) and its share of the loss sums.
template <int G>
__global__ void __launch_bounds__(256) policy_loss_kernel(const LossArgs a) {
  const int gid = (blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int lane = threadIdx.x % G;
  const bool active = gid < a.B;
  const int b = active ? gid : a.B - 1;
  const int T = a.T, T1 = a.T + 1, A = a.A;
  const size_t row0 = (size_t)b * T1;
  VtraceLaneState st;
  st.init(a.values[row0 + T]);
  bool bad = !isfinite(st.carry_vs);
  float sum_pg = 0.f, sum_b = 0.f, sum_h = 0.f;
  const int CH = 4 * G;
  const int nch = (T + CH - 1) / CH;
  for (int ch = nch - 1; ch >= 0; --ch) {
    const int t0 = ch * CH + 4 * lane;
    float d[4], r[4], g[4], v[4], tl[4], H[4], lse4[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int t = t0 + j;
      d[j] = r[j] = g[j] = v[j] = tl[j] = H[j] = lse4[j] = 0.f;
      if (t < T) {
        const float* z = a.logits + (row0 + t) * A;
        float mx = -INFINITY;
        for (int k = 0; k < A; ++k) mx = fmaxf(mx, z[k]);
        float se = 0.f;
        for (int k = 0; k < A; ++k) se += expf(z[k] - mx);
        const float lse = mx + logf(se);
        float h = 0.f;
        for (int k = 0; k < A; ++k) {
          const float lp = z[k] - lse;
          h -= expf(lp) * lp;
        }
        const int act = a.action[row0 + t];
        tl[j] = z[act] - lse;
        lse4[j] = lse;
        H[j] = h;
        d[j] = tl[j] - a.blp[row0 + t];
        r[j] = a.reward[row0 + t + 1];
        g[j] = a.discount * (a.done[row0 + t + 1] ? 0.f : 1.f);
        v[j] = a.values[row0 + t];
      }
    }
    float vs[4], pg[4];
    bad |= vtrace_chunk<G>(st, lane, t0, T, d, r, g, v, a.rho_bar, a.c_bar, a.lam, vs, pg);
    if (active) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int t = t0 + j;
        if (t >= T) continue;
        a.vs[(size_t)b * T + t] = vs[j];
        a.pg[(size_t)b * T + t] = pg[j];
        sum_pg += -pg[j] * tl[j];
        sum_b += (vs[j] - v[j]) * (vs[j] - v[j]);
        sum_h += H[j];
        a.dvalues[row0 + t] = a.scale * a.vf_coef * (v[j] - vs[j]);
        const float* z = a.logits + (row0 + t) * A;
        float* dz = a.dlogits + (row0 + t) * A;
        const int act = a.action[row0 + t];
        for (int k = 0; k < A; ++k) {
          const float lp = z[k] - lse4[j];  // log pi(k | x_t)
          const float p = expf(lp);
          const float onehot = (k == act) ? 1.f : 0.f;
          dz[k] = a.scale * (-pg[j] * (onehot - p) + a.ent_coef * p * (lp + H[j]));
        }
      }
    }
  }
  // row T: no loss term, zero gradients (bootstrap is a constant, C4)
  if (active) {
    for (int k = lane; k < A; k += G) a.dlogits[(row0 + T) * A + k] = 0.f;
    if (lane == 0) a.dvalues[row0 + T] = 0.f;
  }
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) {
    sum_pg += __shfl_xor_sync(0xffffffffu, sum_pg, off, G);
    sum_b += __shfl_xor_sync(0xffffffffu, sum_b, off, G);
    sum_h += __shfl_xor_sync(0xffffffffu, sum_h, off, G);
  }
  const unsigned anybad = __any_sync(0xffffffffu, bad);  // warp-wide is fine: flag only
  if (active && lane == 0) {
    float* pp = a.part + (size_t)b * 4;
    pp[0] = a.scale * sum_pg;
    pp[1] = a.scale * 0.5f * a.vf_coef * sum_b;
    pp[2] = -a.scale * a.ent_coef * sum_h;
    pp[3] = anybad ? 1.f : 0.f;
  }
}

template <int G>
static void launch_loss_g(const LossArgs& a, cudaStream_t st) {
  const long long threads = (long long)a.B * G;
  policy_loss_kernel<G><<<(int)((threads + 255) / 256), 256, 0, st>>>(a);
}

seed_status launch_policy_loss(const LossArgs& a, cudaStream_t st) {
  switch (vtrace_group_size(a.T)) {
    case 1: launch_loss_g<1>(a, st); break;
    case 2: launch_loss_g<2>(a, st); break;
    case 4: launch_loss_g<4>(a, st); break;
    case 8: launch_loss_g<8>(a, st); break;
    case 16: launch_loss_g<16>(a, st); break;
    default: launch_loss_g<32>(a, st); break;
  }
  return last_launch();
}

// ------------------------------------------------------------------ LSTM input extras
__global__ void core_extras_kernel(int F, int A, int Kxp, const int32_t* __restrict__ prev_action,
                                   const float* __restrict__ reward,
                                   const uint8_t* __restrict__ done, __nv_bfloat16* X) {
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

// ------------------------------------------------------------------ column sums
__global__ void colsum_part_kernel(const __nv_bfloat16* __restrict__ X, int64_t R, int C,
                                   float* __restrict__ part) {
  // blockDim 256: thread (rl, c) with rl in [0, 256/C)
  const int RL = 256 / C;
  const int c = threadIdx.x % C, rl = threadIdx.x / C;
  const int64_t per = (R + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * per, r1 = min(R, r0 + per);
  float s = 0.f;
  if (rl < RL)
    for (int64_t r = r0 + rl; r < r1; r += RL) s += __bfloat162float(X[r * C + c]);
  __shared__ float sh[256];
  sh[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x < C) {
    float t = 0.f;
    for (int k = 0; k < RL; ++k) t += sh[k * C + threadIdx.x];
    part[blockIdx.x * C + threadIdx.x] = t;
  }
}

__global__ void colsum_final_kernel(const float* __restrict__ part, int nb, int C,
                                    float* __restrict__ out) {
  const int c = threadIdx.x;
  if (c >= C) return;
  float s = 0.f;
  for (int k = 0; k < nb; ++k) s += part[k * C + c];
  out[c] = s;
}

seed_status colsum_bf16(const __nv_bfloat16* X, int64_t R, int C, float* part, float* out,
                        cudaStream_t st) {
  if (C > 64 || 256 % C) return SEED_E_SHAPE;
  colsum_part_kernel<<<COLSUM_BLOCKS, 256, 0, st>>>(X, R, C, part);
  colsum_final_kernel<<<1, 64, 0, st>>>(part, COLSUM_BLOCKS, C, out);
  return last_launch();
}

// ------------------------------------------------------------------ K9 clip + Adam
__global__ void grad_norm_kernel(const float* __restrict__ g, int64_t P, double* __restrict__ part,
                                 const int64_t* step, int64_t* step_in) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = g[i];
    s += x * x;
  }
  __shared__ double sh[256];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[blockIdx.x] = sh[0];
    if (blockIdx.x == 0) *step_in = *step;
  }
}

__global__ void adam_kernel(const AdamArgs a) {
  __shared__ double tot;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < a.nblocks_norm; ++k) s += a.norm_part[k];
    tot = s;
  }
  __syncthreads();
  const double norm = sqrt(tot);
  const bool finite = isfinite(norm);
  const int64_t t = *a.step_in + 1;
  if (finite) {
    const float scale = norm > (double)a.max_norm ? (float)((double)a.max_norm / norm) : 1.f;
    const float bc1 = (float)(1.0 - pow((double)a.beta1, (double)t));
    const float bc2 = (float)(1.0 - pow((double)a.beta2, (double)t));
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.P;
         i += (int64_t)gridDim.x * blockDim.x) {
      const float g = a.grads[i] * scale;
      const float m = a.beta1 * a.m[i] + (1.f - a.beta1) * g;
      const float v = a.beta2 * a.v[i] + (1.f - a.beta2) * g * g;
      a.m[i] = m;
      a.v[i] = v;
      a.params[i] -= a.lr * (m / bc1) / (sqrtf(v / bc2) + a.eps);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double l0 = 0, l1 = 0, l2 = 0;
    float nonfin = finite ? 0.f : 1.f;
    for (int b = 0; b < a.B; ++b) {
      l0 += a.loss_part[b * 4 + 0];
      l1 += a.loss_part[b * 4 + 1];
      l2 += a.loss_part[b * 4 + 2];
      if (a.loss_part[b * 4 + 3] != 0.f) nonfin = 1.f;
    }
    const int64_t ver = *a.step_in + (finite ? 1 : 0);
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
  adam_kernel<<<148 * 4, 256, 0, st>>>(a);
  return last_launch();
}

}  // namespace seed
