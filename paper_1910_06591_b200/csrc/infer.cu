// infer.cu — centralized batched inference (H12, H13): seed_infer and
// seed_assemble_batch.
//
// P:125 "Inference threads receive a batch of observations, rewards and episode
// termination flags. They load the recurrent states and send the data to the
// inference TPU core. The sampled actions and new recurrent states are
// received ... the latest recurrent states are stored.  When a trajectory is
// fully unrolled it is added to a FIFO queue"; S:434-442 (serve_inference).
//
// One call over n requests (unique actor ids):
//   pre      gather last_action / (h, c) of each actor (pre-reset copy kept for
//            the unroll store, C19), core-input extras onehot(prev a), clip(r),
//            zeroed on done (C15)
//   torso    obs -> bf16, conv1, conv2, fc on the tcgen05 engine (shallow_net.cuh)
//   core     one GEMM for the single LSTM step: [x | h_{t-1}] . [W_x | W_h]^T + b
//            (h_{t-1} from the table rows, reset on done)
//   cell+heads+sample  one CTA per request: the cell (new (h, c) written back to
//            the table row), logits / value (fp32), then softmax, CDF,
//            a = min{j : u < CDF_j} (C18) and the behaviour log-prob; u from the
//            caller or Philox4x32-10 keyed (seed, counter, actor id)
//   record   (optional) obs/action/reward/done/log-prob into each actor's
//            current unroll buffer; a completed unroll (T+1 slots) is pushed to
//            the ready ring at a position given by a block-wide prefix sum in
//            request order (deterministic) and slot T is copied into slot 0
//            of the actor's other buffer (C17)
#include "learner_kernels.cuh"
#include "lstm.cuh"
#include "net.cuh"
#include "shallow_net.cuh"
#include "conv_s2d.cuh"

namespace seed {

struct InferWs {
  int n;
  size_t total, obs_bf16, act1, act2, X, xproj, H, logits, values, hpre, cpre, prev, splitk, hb;
};

static size_t ibump(size_t& cur, size_t bytes) {
  const size_t at = cur;
  cur = align_up(cur + bytes, 256);
  return at;
}

static seed_status make_infer_ws(const NetPlan& p, int n, InferWs* w) {
  memset(w, 0, sizeof(*w));
  w->n = n;
  size_t cur = 0;
  const size_t N = n;
  const ShallowS2d sg = shallow_s2d_geometry(p.H, p.W, p.C);
  w->obs_bf16 = ibump(cur, s2d_S0_bytes(sg, N));   // S0 (conv_s2d.cuh)
  w->act1 = ibump(cur, s2d_S1_bytes(sg, N));       // S1
  w->act2 = ibump(cur, N * p.fc_in * 2);
  w->X = ibump(cur, N * p.Kxp * 2);
  w->xproj = ibump(cur, N * 4 * p.U * 4);
  w->H = ibump(cur, N * p.U * 4);
  w->logits = ibump(cur, N * p.A * 4);
  w->values = ibump(cur, N * 4);
  w->hpre = ibump(cur, N * p.U * 4);
  w->cpre = ibump(cur, N * p.U * 4);
  w->prev = ibump(cur, N * 4);
  w->hb = ibump(cur, N * p.U * 2);
  size_t sk = 0;
  auto need = [&](int M, int Nn, int BN, int K) {
    const int s = pick_splits(M, Nn, BN, K);
    if (s > 1) sk = std::max(sk, (size_t)s * M * Nn * 4);
  };
  need(n, 256, 128, p.fc_in);
  need(n, 4 * p.U, 128, p.Kxp + p.U);
  w->splitk = ibump(cur, sk + 16);
  w->total = cur;
  return SEED_OK;
}

// ------------------------------------------------------------------ pre
__global__ void infer_pre_kernel(int n, int A, int U, int Kxp, int num_actors,
                                 const int32_t* __restrict__ ids,
                                 const float* __restrict__ reward, const uint8_t* __restrict__ done,
                                 const float* __restrict__ th, const float* __restrict__ tc,
                                 const int32_t* __restrict__ tla, float* __restrict__ hpre,
                                 float* __restrict__ cpre, int32_t* __restrict__ prev,
                                 __nv_bfloat16* __restrict__ X, __nv_bfloat16* __restrict__ hb) {
  pdl_wait_trig();
  const int E = Kxp - 256;
  const int per = U + E;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * per) return;
  const int i = (int)(idx / per), j = (int)(idx % per);
  const int a = ids[i];
  // an out-of-range actor id reads no table row (zero state, no previous action);
  // the cell kernel reports it (action -1, NaN log-prob) and writes nothing
  const bool valid = a >= 0 && a < num_actors;
  if (j < U) {
    const float h = valid ? th[(size_t)a * U + j] : 0.f;
    hpre[(size_t)i * U + j] = h;
    cpre[(size_t)i * U + j] = valid ? tc[(size_t)a * U + j] : 0.f;
    hb[(size_t)i * U + j] = __float2bfloat16_rn(done[i] ? 0.f : h);   // reset on done (C15)
    return;
  }
  const int e = j - U;
  const bool dn = done[i] != 0;
  const int pa = valid ? tla[a] : -1;
  if (e == 0) prev[i] = pa;
  float v = 0.f;
  if (e < A) v = (!dn && pa == e) ? 1.f : 0.f;
  else if (e == A) v = dn ? 0.f : fminf(fmaxf(reward[i], -1.f), 1.f);
  else if (e == A + 1) v = 1.f;
  X[(size_t)i * Kxp + 256 + e] = __float2bfloat16_rn(v);
}

// ------------------------------------------------------------------ Philox4x32-10
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

// ------------------------------------------------------------------ core + heads + sample
// The single-step LSTM as one GEMM: gates = [x | h_{t-1}] . [W_x | W_h]^T + b
// (K = Kxp + U; both operand rows are read through the engine's gather, so no
// concatenated copy exists), then one CTA per request runs the cell, writes the
// new state into its table row, the heads (fp32) and the sampling.
struct GatesFwd {
  static constexpr bool ASYNC = true;
  const void* dummy = k_ones_chunk;
  static constexpr bool A_MN = false, B_MN = false;
  int M, N, K, kb_per_split;
  int Kxp, U;
  const bf16* X;         // [n][Kxp]: fc | onehot(prev a) | clip(r) | 1 | 0-pad
  const bf16* hb;        // [n][U]: h_{t-1}, zero on done
  const bf16* wx;        // [4U][Kxp]
  const bf16* wh;        // [4U][U]
  const float* bias;
  float* out;            // [n][4U] pre-activation gates
  __device__ const void* ptr_a(int m, int k) const {
    return k < Kxp ? X + (size_t)m * Kxp + k : hb + (size_t)m * U + (k - Kxp);
  }
  __device__ const void* ptr_b(int n, int k) const {
    return k < Kxp ? wx + (size_t)n * Kxp + k : wh + (size_t)n * U + (k - Kxp);
  }
  __device__ void store(int m, int n, float v) const { out[(size_t)m * N + n] = v + bias[n]; }
  static constexpr bool ROW_OUT = true;
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

constexpr int ICH_THREADS = 256;   // = LSTM_U: thread j owns hidden unit j

// CTA i = request i: cell (gate order i, f, g, o; c reset on done, C15), new (h, c)
// into table row ids[i]; logits | value = W h + b (fp32, fixed-order block sum);
// warp 0 samples a = min{j : u < CDF_j} (C18) and writes the behaviour log-prob.
// With `part` (the gates GEMM's split-K partials [splits][n][4U]) the pre-activation
// gates are summed here, splits in z order, then + bias — the arithmetic of the
// GEMM's fixed-order finish, without its launch.
// R2D2 actors: the A+1 outputs are dueling heads (C35:
// advantages 0..A-1, value A), Q_a = V + A_a - mean_j A_j, and the action is
// epsilon-greedy with the per-actor epsilon_i = base^(1 + alpha * i / (N - 1)) of
// actor i of N (0.4, 7).  u0 = uniforms[2r] (explore if u0 < epsilon_i),
// u1 = uniforms[2r+1] (the random action floor(u1 * A)); the greedy action is the
// first maximum of Q; the behaviour log-prob is log(eps/A + (1 - eps)[a = greedy]).
struct EpsGreedy {
  int on;
  float base, alpha;
  int n_eps;
};

__global__ void __launch_bounds__(ICH_THREADS) infer_cell_heads_kernel(
    EpsGreedy eg, int A, const float* __restrict__ gates, const float* __restrict__ part, int splits,
    const float* __restrict__ gbias, const float* __restrict__ cpre,
    const uint8_t* __restrict__ done, const int32_t* __restrict__ ids, const float* __restrict__ hw,
    const float* __restrict__ hbias, const float* __restrict__ uniforms, uint64_t seed,
    uint64_t counter, float* __restrict__ th, float* __restrict__ tc, int32_t* __restrict__ tla,
    int32_t* __restrict__ action_out, float* __restrict__ blp_out, float* __restrict__ logits_out,
    int num_actors) {
  pdl_wait_trig();
  constexpr int U = LSTM_U, NW = ICH_THREADS / 32;
  const int i = blockIdx.x, j = threadIdx.x, warp = j >> 5, lane = j & 31;
  const int A1 = A + 1;
  __shared__ float red[NW][33];
  __shared__ float lg[33];
  float gv[4];
  if (part) {
    const size_t MN = (size_t)gridDim.x * 4 * U;
    const float* pz = part + (size_t)i * 4 * U + j;
#pragma unroll
    for (int k = 0; k < 4; ++k) gv[k] = 0.f;
    for (int z = 0; z < splits; ++z)
#pragma unroll
      for (int k = 0; k < 4; ++k) gv[k] += __ldcs(pz + (size_t)z * MN + k * U);
#pragma unroll
    for (int k = 0; k < 4; ++k) gv[k] += __ldg(gbias + k * U + j);
  } else {
    const float* g = gates + (size_t)i * 4 * U;
#pragma unroll
    for (int k = 0; k < 4; ++k) gv[k] = g[k * U + j];
  }
  const float c0 = done[i] ? 0.f : cpre[(size_t)i * U + j];
  const float gi = sigm(gv[0]), gf = sigm(gv[1]), gg = tanh_fast(gv[2]), go = sigm(gv[3]);
  const float c = gf * c0 + gi * gg;
  const float h = go * tanh_fast(c);
  const int a = ids[i];
  if (a < 0 || a >= num_actors) {   // out-of-range actor id: reported, nothing written
    if (j == 0) {
      action_out[i] = -1;
      blp_out[i] = __int_as_float(0x7fffffff);
    }
    if (logits_out && j < A) logits_out[(size_t)i * A + j] = __int_as_float(0x7fffffff);
    return;
  }
  th[(size_t)a * U + j] = h;
  tc[(size_t)a * U + j] = c;
  for (int o = 0; o < A1; ++o) {
    const float v = warp_sum(h * __ldg(hw + (size_t)o * U + j));
    if (lane == 0) red[warp][o] = v;
  }
  __syncthreads();
  if (j < A1) {
    float t = __ldg(hbias + j);
#pragma unroll
    for (int w = 0; w < NW; ++w) t += red[w][j];   // fixed order
    lg[j] = t;
    if (logits_out && j < A) logits_out[(size_t)i * A + j] = t;
  }
  __syncthreads();
  if (warp == 0 && eg.on) {
    const float adv = lane < A ? lg[lane] : 0.f;
    const float mean = warp_sum(adv) / (float)A;
    const float q = lane < A ? (lg[A] + adv) - mean : -INFINITY;
    if (logits_out && lane < A) logits_out[(size_t)i * A + lane] = q;
    const float qmax = warp_max(q);
    const unsigned ism = __ballot_sync(0xffffffffu, lane < A && q == qmax);
    const int greedy = ism ? __ffs(ism) - 1 : 0;
    float u0, u1;
    if (uniforms) {
      u0 = uniforms[2 * i];
      u1 = uniforms[2 * i + 1];
    } else {
      const uint4 r = philox4x32_10(
          make_uint4((uint32_t)counter, (uint32_t)(counter >> 32), (uint32_t)a, 0u),
          make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
      u0 = (float)(r.x >> 8) * (1.f / 16777216.f);
      u1 = (float)(r.y >> 8) * (1.f / 16777216.f);
    }
    const float eps = eg.n_eps > 1 ? powf(eg.base, 1.f + eg.alpha * (float)a / (float)(eg.n_eps - 1)) : eg.base;
    const int act = u0 < eps ? min((int)(u1 * (float)A), A - 1) : greedy;
    if (lane == 0) {
      action_out[i] = act;
      blp_out[i] = logf(eps / (float)A + (act == greedy ? 1.f - eps : 0.f));
      tla[a] = act;
    }
  } else if (warp == 0) {
    const float z = lane < A ? lg[lane] : -INFINITY;
    const float mx = warp_max(z);
    const float e = lane < A ? expf(z - mx) : 0.f;
    const float se = warp_sum(e);
    float cdf = e / se;   // inclusive prefix sum of the probabilities, fp32, action order
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const float t = __shfl_up_sync(0xffffffffu, cdf, o);
      if (lane >= o) cdf += t;
    }
    float u;
    if (uniforms) {
      u = uniforms[i];
    } else {
      const uint4 r = philox4x32_10(
          make_uint4((uint32_t)counter, (uint32_t)(counter >> 32), (uint32_t)a, 0u),
          make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
      u = (float)(r.x >> 8) * (1.f / 16777216.f);
    }
    const unsigned hit = __ballot_sync(0xffffffffu, lane < A && u < cdf);
    const int act = hit ? (__ffs(hit) - 1) : A - 1;
    const float za = __shfl_sync(0xffffffffu, z, act);
    if (lane == 0) {
      action_out[i] = act;
      blp_out[i] = za - mx - logf(se);
      tla[a] = act;
    }
  }
}

// ------------------------------------------------------------------ unroll store
__global__ void infer_store_obs_kernel(int n, int64_t obs16, const uint8_t* __restrict__ obs,
                                       const int32_t* __restrict__ ids, seed_unroll_store st) {
  const int T1 = st.T + 1;
  const int64_t total = (int64_t)n * obs16;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx / obs16);
    const int64_t q = idx % obs16;
    const int a = ids[i];
    if (a < 0 || a >= st.num_actors) continue;
    const int buf = st.cur[a], slot = st.fill[a];
    const uint4 v = reinterpret_cast<const uint4*>(obs)[idx];
    uint4* base = reinterpret_cast<uint4*>(st.obs);
    base[(((int64_t)a * 2 + buf) * T1 + slot) * obs16 + q] = v;
    if (slot == st.T) base[(((int64_t)a * 2 + (1 - buf)) * T1 + 0) * obs16 + q] = v;
  }
}

// single block, blockDim >= n (n <= 1024): request order defines ring order
__global__ void infer_store_record_kernel(int n, int U, const int32_t* __restrict__ ids,
                                          const int32_t* __restrict__ action,
                                          const int32_t* __restrict__ prev,
                                          const float* __restrict__ reward,
                                          const uint8_t* __restrict__ done,
                                          const float* __restrict__ blp,
                                          const float* __restrict__ hpre,
                                          const float* __restrict__ cpre, seed_unroll_store st) {
  const int i = threadIdx.x;
  const int T1 = st.T + 1;
  int a = 0, buf = 0, slot = 0;
  bool completed = false;
  const bool valid = i < n && ids[i] >= 0 && ids[i] < st.num_actors;
  if (valid) {
    a = ids[i];
    buf = st.cur[a];
    slot = st.fill[a];
    completed = slot == st.T;
  }
  // block-wide exclusive prefix count of completions (request order)
  __shared__ int warp_tot[32];
  __shared__ int base_pos;
  const int lane = i & 31, wid = i >> 5;
  const unsigned bal = __ballot_sync(0xffffffffu, completed);
  const int within = __popc(bal & ((1u << lane) - 1u));
  if (lane == 0) warp_tot[wid] = __popc(bal);
  if (i == 0) base_pos = st.ready_count[0];
  __syncthreads();
  int before = 0;
  for (int w = 0; w < wid; ++w) before += warp_tot[w];
  if (valid) {
    const int64_t s0 = ((int64_t)a * 2 + buf) * T1 + slot;
    st.action[s0] = action[i];
    st.prev_action[s0] = prev[i];
    st.reward[s0] = reward[i];
    st.done[s0] = done[i];
    st.behaviour_logp[s0] = blp[i];
    if (slot == 0) {
      for (int u = 0; u < U; ++u) {
        st.h0[((int64_t)a * 2 + buf) * U + u] = hpre[(size_t)i * U + u];
        st.c0[((int64_t)a * 2 + buf) * U + u] = cpre[(size_t)i * U + u];
      }
    }
    if (completed) {
      const int pos = (base_pos + before + within) % st.ring_capacity;
      st.ready_ring[pos] = a * 2 + buf;
      const int nb = 1 - buf;
      // buffer generations: the entry carries buf's generation; nb is
      // being reused from here on (its slot 0 is written below), so its generation
      // advances and a not-yet-assembled entry of nb becomes detectably stale
      st.ready_gen[pos] = st.gen[a * 2 + buf];
      st.gen[a * 2 + nb] += 1;
      const int64_t d0 = ((int64_t)a * 2 + nb) * T1;
      st.action[d0] = action[i];
      st.prev_action[d0] = prev[i];
      st.reward[d0] = reward[i];
      st.done[d0] = done[i];
      st.behaviour_logp[d0] = blp[i];
      for (int u = 0; u < U; ++u) {   // state before slot T's step = before slot 0 (C19)
        st.h0[((int64_t)a * 2 + nb) * U + u] = hpre[(size_t)i * U + u];
        st.c0[((int64_t)a * 2 + nb) * U + u] = cpre[(size_t)i * U + u];
      }
      st.cur[a] = nb;
      st.fill[a] = 1;
    } else {
      st.fill[a] = slot + 1;
    }
  }
  __syncthreads();
  if (i == 0) {
    int tot = 0;
    for (int w = 0; w < (n + 31) / 32; ++w) tot += warp_tot[w];
    st.ready_count[0] = base_pos + tot;
  }
}

// ------------------------------------------------------------------ assemble
__global__ void assemble_kernel(seed_unroll_store st, int64_t obs16, int U, int B, seed_batch out) {
  const int b = blockIdx.y;
  const int T1 = st.T + 1;
  const int consumed = st.ready_count[1];
  const int pos = (consumed + b) % st.ring_capacity;
  const int e = st.ready_ring[pos];
  const int a = e >> 1, buf = e & 1;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // the unroll's buffer was reused (refilled) after it was pushed: stale
    if (st.gen[e] != st.ready_gen[pos]) atomicAdd(&st.ready_count[2], 1);
    // fewer than B unrolls pushed and not yet consumed
    if (b == 0 && st.ready_count[0] - consumed < B) atomicAdd(&st.ready_count[3], 1);
  }
  const int64_t src = ((int64_t)a * 2 + buf) * T1;
  const uint4* so = reinterpret_cast<const uint4*>(st.obs) + src * obs16;
  uint4* dob = reinterpret_cast<uint4*>(const_cast<void*>(out.obs)) + (int64_t)b * T1 * obs16;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < T1 * obs16;
       q += (int64_t)gridDim.x * blockDim.x)
    dob[q] = so[q];
  if (blockIdx.x == 0) {
    for (int t = threadIdx.x; t < T1; t += blockDim.x) {
      const int64_t d = (int64_t)b * T1 + t;
      const_cast<int32_t*>(out.action)[d] = st.action[src + t];
      const_cast<int32_t*>(out.prev_action)[d] = st.prev_action[src + t];
      const_cast<float*>(out.reward)[d] = st.reward[src + t];
      const_cast<uint8_t*>(out.done)[d] = st.done[src + t];
      const_cast<float*>(out.behaviour_logp)[d] = st.behaviour_logp[src + t];
    }
    for (int u = threadIdx.x; u < U; u += blockDim.x) {
      const_cast<float*>(out.h0)[(int64_t)b * U + u] = st.h0[((int64_t)a * 2 + buf) * U + u];
      const_cast<float*>(out.c0)[(int64_t)b * U + u] = st.c0[((int64_t)a * 2 + buf) * U + u];
    }
  }
}

__global__ void assemble_advance_kernel(int* ready_count, int B) { ready_count[1] += B; }

}  // namespace seed

using namespace seed;

extern "C" seed_status seed_infer_workspace_size(const seed_net_spec* spec, int max_n,
                                                 size_t* bytes) {
  if (!bytes) return SEED_E_ARG;
  NetPlan p;
  SEED_TRY(make_net_plan(spec, &p));
  if (p.kind != SEED_NET_ATARI_SHALLOW || !learner_supported(p)) return SEED_E_UNSUPPORTED;
  if (max_n < 1 || max_n > 1024) return SEED_E_SHAPE;
  InferWs w;
  SEED_TRY(make_infer_ws(p, max_n, &w));
  *bytes = w.total;
  return SEED_OK;
}

static seed_status infer_impl(const seed_net_spec* spec, const void* params_lowp,
                              const float* params, const seed_state_table* table, int n,
                              const int32_t* actor_ids, const uint8_t* obs,
                              const float* reward, const uint8_t* done,
                              const float* uniforms, uint64_t seed, uint64_t counter,
                              int32_t* action_out, float* blp_out, float* logits_out,
                              const seed_unroll_store* store, void* ws, size_t ws_bytes,
                              void* stream, const EpsGreedy& eg) {
  NetPlan p;
  SEED_TRY(make_net_plan(spec, &p));
  if (p.kind != SEED_NET_ATARI_SHALLOW || !learner_supported(p)) return SEED_E_UNSUPPORTED;
  if (n < 1 || n > 1024) return SEED_E_SHAPE;
  if (table && table->num_actors < 1) return SEED_E_ARG;
  if (store && (!store->gen || !store->ready_gen || store->num_actors != table->num_actors ||
                store->ring_capacity < 1))
    return SEED_E_ARG;
  if (!params_lowp || !params || !table || !actor_ids || !obs || !reward || !done ||
      !action_out || !blp_out || !ws || !table->h || !table->c || !table->last_action)
    return SEED_E_ARG;
  if (!aligned16(obs) || !aligned16(ws) || !aligned16(params_lowp)) return SEED_E_ARG;
  InferWs w;
  SEED_TRY(make_infer_ws(p, n, &w));
  if (ws_bytes < w.total) return SEED_E_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* base = (uint8_t*)ws;
  auto at = [&](size_t off) { return base + off; };
  const bf16* lowp = (const bf16*)params_lowp;
  const int U = p.U, A = p.A;
  float* splitk = (float*)at(w.splitk);
  {
    const int64_t tot = (int64_t)n * (U + p.Kxp - 256);
    SEED_TRY(launch_k(infer_pre_kernel, dim3((unsigned)((tot + 255) / 256)), dim3(256), 0, st, n, A, U,
                      p.Kxp, table->num_actors, actor_ids, reward, done, (const float*)table->h, (const float*)table->c,
                      (const int32_t*)table->last_action, (float*)at(w.hpre), (float*)at(w.cpre),
                      (int32_t*)at(w.prev), (bf16*)at(w.X), (bf16*)at(w.hb)));
  }
  SEED_TRY(shallow_s2d_forward(shallow_s2d_geometry(p.H, p.W, p.C), n, obs, lowp + p.im_conv1,
                               params + p.t[p.i_conv1b].off, lowp + p.im_conv2,
                               params + p.t[p.i_conv2b].off, (uint8_t*)at(w.obs_bf16),
                               (uint8_t*)at(w.act1), (bf16*)at(w.act2), nullptr, st));
  {
    FcFwd pr{};
    pr.M = n; pr.N = 256; pr.K = p.fc_in; pr.Kxp = p.Kxp;
    pr.act2 = (const bf16*)at(w.act2); pr.w = lowp + p.im_fc;
    pr.bias = params + p.t[p.i_fcb].off; pr.X = (bf16*)at(w.X);
    SEED_TRY(launch_gemm<128>(pr, pick_splits(pr.M, pr.N, 128, pr.K), st, splitk));
  }
  int gsplits = 1;
  {
    GatesFwd pr{};
    pr.M = n; pr.N = 4 * U; pr.K = p.Kxp + U; pr.Kxp = p.Kxp; pr.U = U;
    pr.X = (const bf16*)at(w.X); pr.hb = (const bf16*)at(w.hb);
    pr.wx = lowp + p.im_wx; pr.wh = lowp + p.im_wh;
    pr.bias = params + p.t[p.i_lb].off; pr.out = (float*)at(w.xproj);
    gsplits = gemm_effective_splits(pr.K, pick_splits(pr.M, pr.N, 128, pr.K));
    SEED_TRY(launch_gemm<128>(pr, gsplits, st, splitk, 0, nullptr, /*run_finish=*/false));
  }
  SEED_TRY(launch_k(infer_cell_heads_kernel, dim3(n), dim3(ICH_THREADS), 0, st, eg, A,
                    (const float*)at(w.xproj), gsplits > 1 ? (const float*)splitk : nullptr, gsplits,
                    params + p.t[p.i_lb].off, (const float*)at(w.cpre), done, actor_ids,
                    params + p.t[p.i_hw].off, params + p.t[p.i_hb].off, uniforms, seed, counter,
                    table->h, table->c, table->last_action, action_out, blp_out, logits_out,
                    table->num_actors));
  if (store) {
    const int64_t obs16 = (int64_t)p.H * p.W * p.C / 16;
    infer_store_obs_kernel<<<(int)std::min<int64_t>((n * obs16 + 255) / 256, 148 * 8), 256, 0,
                             st>>>(n, obs16, obs, actor_ids, *store);
    infer_store_record_kernel<<<1, ((n + 31) / 32) * 32, 0, st>>>(
        n, U, actor_ids, action_out, (const int32_t*)at(w.prev), reward, done, blp_out,
        (const float*)at(w.hpre), (const float*)at(w.cpre), *store);
  }
  return last_launch();
}

extern "C" seed_status seed_infer(const seed_net_spec* spec, const void* params_lowp,
                                  const float* params, const seed_state_table* table, int n,
                                  const int32_t* actor_ids, const uint8_t* obs,
                                  const float* reward, const uint8_t* done,
                                  const float* uniforms, uint64_t seed, uint64_t counter,
                                  int32_t* action_out, float* blp_out, float* logits_out,
                                  const seed_unroll_store* store, void* ws, size_t ws_bytes,
                                  void* stream) {
  const EpsGreedy off{0, 0.f, 0.f, 0};
  return infer_impl(spec, params_lowp, params, table, n, actor_ids, obs, reward, done, uniforms, seed,
                    counter, action_out, blp_out, logits_out, store, ws, ws_bytes, stream, off);
}

extern "C" seed_status seed_infer_eps_greedy(const seed_net_spec* spec, const void* params_lowp,
                                             const float* params, const seed_state_table* table, int n,
                                             const int32_t* actor_ids, const uint8_t* obs,
                                             const float* reward, const uint8_t* done,
                                             const float* uniforms, uint64_t seed, uint64_t counter,
                                             float eps_base, float eps_alpha, int num_actors_eps,
                                             int32_t* action_out, float* blp_out, float* q_out,
                                             const seed_unroll_store* store, void* ws, size_t ws_bytes,
                                             void* stream) {
  if (!(eps_base >= 0.f && eps_base <= 1.f) || !(eps_alpha >= 0.f) || num_actors_eps < 1) return SEED_E_ARG;
  const EpsGreedy eg{1, eps_base, eps_alpha, num_actors_eps};
  return infer_impl(spec, params_lowp, params, table, n, actor_ids, obs, reward, done, uniforms, seed,
                    counter, action_out, blp_out, q_out, store, ws, ws_bytes, stream, eg);
}

extern "C" seed_status seed_assemble_batch(const seed_unroll_store* store, int obs_bytes,
                                           int lstm_units, int B, const seed_batch* out,
                                           void* stream) {
  if (!store || !out || B < 1 || obs_bytes <= 0 || obs_bytes % 16 || lstm_units < 1 ||
      !store->gen || !store->ready_gen || store->ring_capacity < 1)
    return SEED_E_ARG;
  if (!out->obs || !out->action || !out->prev_action || !out->reward || !out->done ||
      !out->behaviour_logp || !out->h0 || !out->c0)
    return SEED_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t obs16 = obs_bytes / 16;
  dim3 grid((unsigned)std::min<int64_t>((store->T + 1) * obs16 / 256 + 1, 64), B);
  assemble_kernel<<<grid, 256, 0, st>>>(*store, obs16, lstm_units, B, *out);
  assemble_advance_kernel<<<1, 1, 0, st>>>(store->ready_count, B);
  return last_launch();
}
