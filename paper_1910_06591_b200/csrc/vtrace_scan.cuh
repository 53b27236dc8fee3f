// vtrace_scan.cuh — the lane-group V-trace chunk step shared by K1 (seed_vtrace)
// and K2 (the fused policy loss).  See vtrace.cu for the scheme.
#pragma once
#include "common.cuh"

namespace seed {

struct VtraceLaneState {
  float carry_acc;  // acc = vs - V at the first step right of the current chunk (0 past T)
  float carry_vs;   // vs at that step (bootstrap past T)
  float carry_v;    // V at that step (bootstrap past T)
  __device__ void init(float bootstrap) {
    carry_acc = 0.f;
    carry_vs = bootstrap;
    carry_v = bootstrap;
  }
};

// Process one chunk of 4*G steps: lane `lane` owns steps t0..t0+3 (t0 = chunk
// base + 4*lane).  d = target_logp - behaviour_logp, r, g (discount), v (value)
// for the 4 steps (anything for steps >= T).  Writes vs/pg for the 4 steps and
// returns true when a non-finite input was seen.  All G lanes must call it.
template <int G>
__device__ __forceinline__ bool vtrace_chunk(VtraceLaneState& st, int lane, int t0, int T,
                                             const float (&d)[4], const float (&r)[4],
                                             const float (&g)[4], const float (&v)[4],
                                             float rho_bar, float c_bar, float lam,
                                             float (&vs)[4], float (&pg)[4]) {
  const unsigned FULL = 0xffffffffu;
  bool bad = false;
  // V_{t+1} for each owned step: next lane's first value / the carried value.
  float v_right = __shfl_down_sync(FULL, v[0], 1, G);
  if (lane == G - 1) v_right = st.carry_v;
  float a[4], bq[4], rho[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int t = t0 + j;
    const bool valid = t < T;
    float vnext = (j < 3) ? v[j + 1] : v_right;
    if (t + 1 >= T) vnext = st.carry_v;  // only reached at t == T-1 with carry = bootstrap
    const float ratio = expf(d[j]);
    const float rh = fminf(rho_bar, ratio);
    const float cc = lam * fminf(c_bar, ratio);
    const float delta = rh * (r[j] + g[j] * vnext - v[j]);
    a[j] = valid ? g[j] * cc : 1.f;
    bq[j] = valid ? delta : 0.f;
    rho[j] = rh;
    if (valid) bad |= !(isfinite(d[j]) && isfinite(r[j]) && isfinite(g[j]) && isfinite(v[j]));
  }
  // compose this lane's maps right-to-left: acc_in(left) = B + A * acc_in(right)
  float A = 1.f, Bm = 0.f;
#pragma unroll
  for (int j = 3; j >= 0; --j) {
    Bm = bq[j] + a[j] * Bm;
    A = a[j] * A;
  }
  // inclusive suffix scan of maps over lanes lane..G-1
#pragma unroll
  for (int off = 1; off < G; off <<= 1) {
    const float A2 = __shfl_down_sync(FULL, A, off, G);
    const float B2 = __shfl_down_sync(FULL, Bm, off, G);
    if (lane + off < G) {
      Bm = Bm + A * B2;
      A = A * A2;
    }
  }
  // exclusive: maps of lanes > lane, applied to the carry
  float Ae = __shfl_down_sync(FULL, A, 1, G);
  float Be = __shfl_down_sync(FULL, Bm, 1, G);
  if (lane == G - 1) {
    Ae = 1.f;
    Be = 0.f;
  }
  float acc = Be + Ae * st.carry_acc;
  float accs[4];
#pragma unroll
  for (int j = 3; j >= 0; --j) {
    acc = bq[j] + a[j] * acc;
    accs[j] = acc;
    vs[j] = v[j] + acc;
  }
  float vs_right = __shfl_down_sync(FULL, vs[0], 1, G);
  if (lane == G - 1) vs_right = st.carry_vs;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int t = t0 + j;
    float vsn = (j < 3) ? vs[j + 1] : vs_right;
    if (t + 1 >= T) vsn = st.carry_vs;
    pg[j] = rho[j] * (r[j] + g[j] * vsn - v[j]);
  }
  // carries for the chunk to the left: values at this chunk's first step
  st.carry_acc = __shfl_sync(FULL, accs[0], 0, G);
  st.carry_vs = __shfl_sync(FULL, vs[0], 0, G);
  st.carry_v = __shfl_sync(FULL, v[0], 0, G);
  return bad;
}

int vtrace_group_size(int T);

}  // namespace seed
