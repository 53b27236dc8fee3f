// r2d2.cu — the R2D2 pieces of SEED's Q-learning path (
// P:149-153 "fully implementing R2D2", hyper-parameters P:586-622):
//   seed_r2d2_targets  n-step double-Q targets with value rescaling, TD errors,
//                      sequence priorities and the importance-weighted loss gradient
//   seed_replay_*      the learner-resident prioritized sequence replay ("keep
//                      the replay buffer on the learner"): a sum tree over p^alpha in
//                      HBM, FIFO insertion at the max priority, priority updates with
//                      generation tags, proportional sampling with importance weights,
//                      and the gather of the sampled sequences' bytes.
// Everything fp32 on the device; reductions in fixed order (C21).
#include <algorithm>
#include "common.cuh"

namespace seed {

// h and h^-1 in cancellation-free fp32 forms (algebraically identical to P:611 /
// S:204): sqrt(1+u) - 1 = u / (sqrt(1+u) + 1), and with r = sqrt(1+z),
// z = 4 eps (|y| + 1 + eps), d = r - 1 = z / (r + 1):
//   s = (r - 1) / (2 eps) = 2 (|y| + 1 + eps) / (r + 1),
//   s - 1 = (2|y| + 2 eps - d) / (r + 1),  h^-1(y) = sign(y) (s - 1)(s + 1).
// (The textbook forms lose ~1e-4 relative to cancellation in fp32.)
__device__ __forceinline__ float rescale_h(float x, float eps) {
  const float ax = fabsf(x);
  return copysignf(ax / (sqrtf(ax + 1.f) + 1.f), x) + eps * x;
}
__device__ __forceinline__ float rescale_hinv(float y, float eps) {
  const float ay = fabsf(y);
  const float z = 4.f * eps * (ay + 1.f + eps);
  const float r = sqrtf(1.f + z);
  const float d = z / (r + 1.f);
  const float sm1 = (2.f * ay + (2.f * eps - d)) / (r + 1.f);
  return copysignf(sm1 * (2.f + sm1), y);
}

__device__ __forceinline__ float warp_max_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// one warp per trajectory; lane = step t (chunks of 32)
struct R2d2Args {
  int T, B, A, n;
  float eta, eps, scale;
  const float* qo;        // [B][T+1][A]
  const float* qt;        // [B][T+1][A]
  const int32_t* act;     // [B][T+1]
  const float* rew;       // [B][T]
  const float* disc;      // [B][T]
  const float* w;         // nullable [B]
  float* y;               // [B][T]
  float* delta;           // [B][T]
  float* prio;            // [B]
  float* dq;              // nullable [B][T+1][A]
  float* loss;            // nullable [B]
};

// one CTA per sequence with its q_online / q_target rows staged in shared memory
// (coalesced float4 loads; the per-step argmax then reads shared memory)
__global__ void __launch_bounds__(128) r2d2_targets_smem_kernel(const R2d2Args a) {
  pdl_wait();
  extern __shared__ float sq[];
  const int b = blockIdx.x, T = a.T, A = a.A, T1 = T + 1, tid = threadIdx.x;
  const int nq = T1 * A;
  float* so = sq;
  float* st = sq + ((nq + 3) & ~3);
  const float* qo = a.qo + (size_t)b * nq;
  const float* qt = a.qt + (size_t)b * nq;
  if (((reinterpret_cast<uintptr_t>(qo) | reinterpret_cast<uintptr_t>(qt)) & 15) == 0 && (nq & 3) == 0) {
    for (int i = tid; i < nq / 4; i += blockDim.x) {
      reinterpret_cast<float4*>(so)[i] = __ldcs(reinterpret_cast<const float4*>(qo) + i);
      reinterpret_cast<float4*>(st)[i] = __ldcs(reinterpret_cast<const float4*>(qt) + i);
    }
  } else {
    for (int i = tid; i < nq; i += blockDim.x) {
      so[i] = __ldcs(qo + i);
      st[i] = __ldcs(qt + i);
    }
  }
  if (a.dq) {
    float* d = a.dq + (size_t)b * nq;
    for (int i = tid; i < nq; i += blockDim.x) d[i] = 0.f;
  }
  __syncthreads();
  const float* rw = a.rew + (size_t)b * T;
  const float* ds = a.disc + (size_t)b * T;
  const float wb = a.w ? a.w[b] : 1.f;
  float dmax = 0.f, dsum = 0.f, lsum = 0.f;
  for (int t = tid; t < T; t += blockDim.x) {
    const int m = min(a.n, T - t);
    float G = 0.f, g = 1.f;
    for (int k = 0; k < m; ++k) {
      G += g * rw[t + k];
      g *= ds[t + k];
    }
    const float* qn = so + (t + m) * A;
    int astar = 0;
    float best = qn[0];
    for (int j = 1; j < A; ++j) {
      const float v = qn[j];
      if (v > best) { best = v; astar = j; }
    }
    G += g * rescale_hinv(st[(t + m) * A + astar], a.eps);
    const float yt = rescale_h(G, a.eps);
    const int at = a.act[(size_t)b * T1 + t];
    const float q = so[t * A + at];
    const float dt = yt - q;
    a.y[(size_t)b * T + t] = yt;
    a.delta[(size_t)b * T + t] = dt;
    dmax = fmaxf(dmax, fabsf(dt));
    dsum += fabsf(dt);
    lsum += 0.5f * dt * dt;
    if (a.dq) a.dq[(size_t)b * nq + t * A + at] = a.scale * wb * (q - yt);
  }
  // fixed-order block reduction (4 warps)
  __shared__ float red[3][4];
  dmax = warp_max_f(dmax);
  dsum = warp_sum_f(dsum);
  lsum = warp_sum_f(lsum);
  if ((tid & 31) == 0) { red[0][tid >> 5] = dmax; red[1][tid >> 5] = dsum; red[2][tid >> 5] = lsum; }
  __syncthreads();
  if (tid == 0) {
    float mx = red[0][0], sm = red[1][0], ls = red[2][0];
    for (int w = 1; w < 4; ++w) { mx = fmaxf(mx, red[0][w]); sm += red[1][w]; ls += red[2][w]; }
    a.prio[b] = a.eta * mx + (1.f - a.eta) * (sm / (float)T);
    if (a.loss) a.loss[b] = a.scale * wb * ls;
  }
}

__global__ void __launch_bounds__(256) r2d2_targets_kernel(const R2d2Args a) {
  pdl_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= a.B) return;
  const int b = warp, T = a.T, A = a.A, T1 = T + 1;
  const float* qo = a.qo + (size_t)b * T1 * A;
  const float* qt = a.qt + (size_t)b * T1 * A;
  const float* rw = a.rew + (size_t)b * T;
  const float* ds = a.disc + (size_t)b * T;
  const float wb = a.w ? a.w[b] : 1.f;
  float dmax = 0.f, dsum = 0.f, lsum = 0.f;
  for (int t0 = 0; t0 < T1; t0 += 32) {
    const int t = t0 + lane;
    if (a.dq && t < T1) {   // dq row t: zero except the taken action (row T all zero)
      float* d = a.dq + ((size_t)b * T1 + t) * A;
      for (int j = 0; j < A; ++j) d[j] = 0.f;
    }
    if (t >= T) continue;
    const int m = min(a.n, T - t);
    float G = 0.f, g = 1.f;
    for (int k = 0; k < m; ++k) {
      G += g * rw[t + k];
      g *= ds[t + k];
    }
    const float* qn = qo + (size_t)(t + m) * A;   // double Q: online network selects
    int astar = 0;
    float best = qn[0];
    for (int j = 1; j < A; ++j) {
      const float v = qn[j];
      if (v > best) { best = v; astar = j; }       // first maximum
    }
    G += g * rescale_hinv(qt[(size_t)(t + m) * A + astar], a.eps);
    const float yt = rescale_h(G, a.eps);
    const int at = a.act[(size_t)b * T1 + t];
    const float q = qo[(size_t)t * A + at];
    const float dt = yt - q;
    a.y[(size_t)b * T + t] = yt;
    a.delta[(size_t)b * T + t] = dt;
    dmax = fmaxf(dmax, fabsf(dt));
    dsum += fabsf(dt);
    lsum += 0.5f * dt * dt;
    if (a.dq) a.dq[((size_t)b * T1 + t) * A + at] = a.scale * wb * (q - yt);
  }
  dmax = warp_max_f(dmax);
  dsum = warp_sum_f(dsum);
  lsum = warp_sum_f(lsum);
  if (lane == 0) {
    a.prio[b] = a.eta * dmax + (1.f - a.eta) * (dsum / (float)T);
    if (a.loss) a.loss[b] = a.scale * wb * lsum;
  }
}

// ------------------------------------------------------------------ replay sum tree
// tree[1] = root; node k has children 2k, 2k+1; leaves tree[C + i] = p_i^alpha.
// Every change is followed by a rebuild of the internal nodes: one CTA per 2048
// leaves builds its subtree in shared memory (fixed pairwise order), the last CTA
// to finish (ticket) builds the levels above — deterministic, exact per level, no
// drift from incremental updates.
constexpr int RP_SUB = 2048;   // leaves per subtree CTA
constexpr int RP_THREADS = 1024;

__global__ void __launch_bounds__(RP_THREADS) replay_rebuild_kernel(float* tree, int C,
                                                                    unsigned* ticket) {
  pdl_wait();
  __shared__ float s[RP_SUB];
  __shared__ bool last;
  const int tid = threadIdx.x;
  const int sub = min(C, RP_SUB);
  int first = C + blockIdx.x * sub;   // first node of the current level of this subtree
  for (int i = tid; i < sub; i += blockDim.x) s[i] = tree[first + i];
  __syncthreads();
  // each level: node i = s[2i] + s[2i+1] (w <= 1024 = blockDim: one node per thread)
  for (int w = sub >> 1; w >= 1; w >>= 1) {
    first >>= 1;
    const float v = tid < w ? s[2 * tid] + s[2 * tid + 1] : 0.f;
    __syncthreads();
    if (tid < w) {
      s[tid] = v;
      tree[first + tid] = v;
    }
    __syncthreads();
  }
  if (gridDim.x == 1) return;
  // the levels above the subtree roots tree[C/sub .. C/sub + grid): the last CTA
  __threadfence();
  if (tid == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  int n = gridDim.x;
  first = C / sub;
  for (int i = tid; i < n; i += blockDim.x) s[i] = __ldcg(tree + first + i);
  __syncthreads();
  for (int w = n >> 1; w >= 1; w >>= 1) {
    first >>= 1;
    const float v = tid < w ? s[2 * tid] + s[2 * tid + 1] : 0.f;
    __syncthreads();
    if (tid < w) {
      s[tid] = v;
      tree[first + tid] = v;
    }
    __syncthreads();
  }
  if (tid == 0) *ticket = 0;   // re-armed for the next rebuild
}

// new sequences: FIFO slots at the max priority seen (1 before any update)
__global__ void replay_insert_kernel(int n, int slots, int C, float alpha, float* tree,
                                     const float* maxp, int32_t* size, int32_t* gen,
                                     int32_t* out_slots, int32_t* out_gens) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int next = size[1];
  if (i < n) {
    const int slot = (next + i) % slots;
    const float p = *maxp > 0.f ? *maxp : 1.f;
    tree[C + slot] = powf(p, alpha);
    const int gsl = gen[slot] + 1;   // the slot's previous sequence (if any) is evicted
    gen[slot] = gsl;
    if (out_slots) out_slots[i] = slot;
    if (out_gens) out_gens[i] = gsl;
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // (single block: n <= 1024, checked on the host)
    size[1] = (next + n) % slots;
    size[0] = min(slots, size[0] + n);
  }
}

// new priorities for sampled sequences; entries whose generation no longer matches
// (the slot was refilled since the sample) are skipped; non-finite / negative
// priorities are skipped and counted in size[2]
__global__ void replay_update_kernel(int n, int C, float alpha, const int32_t* slots,
                                     const int32_t* gens, const float* prio, float* tree,
                                     float* maxp, const int32_t* gen, int32_t* size) {
  pdl_wait();
  const int i = threadIdx.x;
  float m = 0.f;
  if (i < n) {
    const int slot = slots[i];
    const float p = prio[i];
    if (!(p >= 0.f) || isinf(p)) {
      atomicAdd(&size[2], 1);
    } else if (gens == nullptr || gen[slot] == gens[i]) {
      tree[C + slot] = powf(p, alpha);
      m = p;
    }
  }
  // block max (n <= 1024, one block) -> running max priority
  __shared__ float red[32];
  m = warp_max_f(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x + 31) / 32 ? red[threadIdx.x] : 0.f;
    v = warp_max_f(v);
    if (threadIdx.x == 0 && v > *maxp) *maxp = v;
  }
}

__device__ __forceinline__ uint4 philox10(uint4 c, uint2 k) {
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

// one thread per draw: descend the tree with x = u * root; importance weights
// (N P(i))^-beta normalised by the batch max (one block, B <= 1024)
__global__ void replay_sample_kernel(int Bn, int C, float beta, const float* tree,
                                     const int32_t* size, const int32_t* gen, const float* uniforms,
                                     uint64_t seed, uint64_t counter, int32_t* out_slots,
                                     int32_t* out_gens, float* out_w) {
  pdl_wait();
  const int i = threadIdx.x;
  const float total = tree[1];
  const int N = max(size[0], 1);
  float w = 0.f;
  int node = 1;
  if (i < Bn) {
    float u;
    if (uniforms) {
      u = uniforms[i];
    } else {
      const uint4 r = philox10(make_uint4((uint32_t)counter, (uint32_t)(counter >> 32), (uint32_t)i, 1u),
                               make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
      u = (float)(r.x >> 8) * (1.f / 16777216.f);
    }
    float x = fminf(u * total, nextafterf(total, 0.f));
    while (node < C) {
      const float l = tree[2 * node];
      if (x < l) {
        node = 2 * node;
      } else {
        x -= l;
        // rounding can push x past the right subtree: never descend into an empty one
        node = tree[2 * node + 1] > 0.f ? 2 * node + 1 : 2 * node;
      }
    }
    const int slot = node - C;
    const float P = tree[node] / total;
    w = powf((float)N * P, -beta);
    out_slots[i] = slot;
    if (out_gens) out_gens[i] = gen[slot];
  }
  __shared__ float red[32];
  float m = warp_max_f(w);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x + 31) / 32 ? red[threadIdx.x] : 0.f;
    v = warp_max_f(v);
    __syncwarp();
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  if (i < Bn) out_w[i] = w / red[0];
}

// gather the sampled sequences' bytes: dst[b] = src[slots[b]] (uint4 granules)
__global__ void replay_gather_kernel(const uint4* __restrict__ src, int64_t slot16, const int32_t* slots,
                                     int Bn, uint4* __restrict__ dst) {
  pdl_wait();
  const int b = blockIdx.y;
  const uint4* s = src + (int64_t)slots[b] * slot16;
  uint4* d = dst + (int64_t)b * slot16;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < slot16;
       q += (int64_t)gridDim.x * blockDim.x)
    d[q] = __ldcs(s + q);
}

// the inverse: dst[slots[b]] = src[b] (payload of newly inserted sequences)
__global__ void replay_scatter_kernel(const uint4* __restrict__ src, int64_t slot16, const int32_t* slots,
                                      int Bn, uint4* __restrict__ dst) {
  pdl_wait();
  const int b = blockIdx.y;
  const uint4* s = src + (int64_t)b * slot16;
  uint4* d = dst + (int64_t)slots[b] * slot16;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < slot16;
       q += (int64_t)gridDim.x * blockDim.x)
    d[q] = __ldcs(s + q);
}

static bool pow2(int c) { return c > 0 && (c & (c - 1)) == 0; }

}  // namespace seed

using namespace seed;

extern "C" seed_status seed_r2d2_targets(int T, int B, int A, int n, const float* q_online,
                                         const float* q_target, const int32_t* actions,
                                         const float* rewards, const float* discounts, float eta,
                                         float rescale_eps, const float* is_weights, float loss_scale,
                                         float* y, float* delta, float* priority, float* dq,
                                         float* loss_part, void* stream) {
  if (T < 1 || B < 1 || A < 2 || A > 4096 || n < 1) return SEED_E_SHAPE;
  if (!q_online || !q_target || !actions || !rewards || !discounts || !y || !delta || !priority)
    return SEED_E_ARG;
  if (!(rescale_eps > 0.f) || !(eta >= 0.f && eta <= 1.f)) return SEED_E_ARG;
  R2d2Args a{T, B, A, n, eta, rescale_eps, loss_scale, q_online, q_target, actions, rewards,
             discounts, is_weights, y, delta, priority, dq, loss_part};
  const size_t smem = 2 * align_up((size_t)(T + 1) * A, 4) * 4;
  if (smem <= 96 * 1024) {
    static PerDevice attr;
    SEED_TRY(smem_optin(attr, r2d2_targets_smem_kernel, 96 * 1024));
    return launch_k(r2d2_targets_smem_kernel, dim3((unsigned)B), dim3(128), smem, (cudaStream_t)stream, a);
  }
  const int warps_per_block = 8;
  return launch_k(r2d2_targets_kernel, dim3((unsigned)ceil_div(B, warps_per_block)),
                  dim3(32 * warps_per_block), 0, (cudaStream_t)stream, a);
}

extern "C" seed_status seed_replay_check(const seed_replay* r) {
  if (!r || !pow2(r->capacity) || r->slots < 1 || r->slots > r->capacity || !r->tree ||
      !r->max_priority || !r->size || !r->gen || !r->ticket)
    return SEED_E_ARG;
  if (r->capacity > RP_SUB && (r->capacity / RP_SUB) > RP_SUB) return SEED_E_SHAPE;
  return SEED_OK;
}

static seed_status rebuild(const seed_replay* r, cudaStream_t st) {
  const int sub = std::min(r->capacity, RP_SUB);
  return launch_k(replay_rebuild_kernel, dim3((unsigned)(r->capacity / sub)), dim3(RP_THREADS), 0, st,
                  r->tree, r->capacity, r->ticket);
}

extern "C" seed_status seed_replay_insert(const seed_replay* r, int n, float alpha,
                                          int32_t* out_slots, int32_t* out_gens, void* stream) {
  SEED_TRY(seed_replay_check(r));
  if (n < 1 || n > 1024 || n > r->slots) return SEED_E_SHAPE;
  if (!(alpha >= 0.f)) return SEED_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  SEED_TRY(launch_k(replay_insert_kernel, dim3(1), dim3(((n + 31) / 32) * 32), 0, st, n, r->slots,
                    r->capacity, alpha, r->tree, (const float*)r->max_priority, r->size, r->gen,
                    out_slots, out_gens));
  return rebuild(r, st);
}

extern "C" seed_status seed_replay_update(const seed_replay* r, int n, const int32_t* slots,
                                          const int32_t* gens, const float* priorities, float alpha,
                                          void* stream) {
  SEED_TRY(seed_replay_check(r));
  if (n < 1 || n > 1024) return SEED_E_SHAPE;
  if (!slots || !priorities || !(alpha >= 0.f)) return SEED_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  SEED_TRY(launch_k(replay_update_kernel, dim3(1), dim3(((n + 31) / 32) * 32), 0, st, n, r->capacity,
                    alpha, slots, gens, priorities, r->tree, r->max_priority, (const int32_t*)r->gen,
                    r->size));
  return rebuild(r, st);
}

extern "C" seed_status seed_replay_sample(const seed_replay* r, int B, float beta,
                                          const float* uniforms, uint64_t seed, uint64_t counter,
                                          int32_t* out_slots, int32_t* out_gens, float* out_weights,
                                          void* stream) {
  SEED_TRY(seed_replay_check(r));
  if (B < 1 || B > 1024) return SEED_E_SHAPE;
  if (!out_slots || !out_weights || !(beta >= 0.f)) return SEED_E_ARG;
  return launch_k(replay_sample_kernel, dim3(1), dim3(((B + 31) / 32) * 32), 0, (cudaStream_t)stream,
                  B, r->capacity, beta, (const float*)r->tree, (const int32_t*)r->size,
                  (const int32_t*)r->gen, uniforms, seed, counter, out_slots, out_gens, out_weights);
}

extern "C" seed_status seed_replay_gather(const void* src, size_t slot_bytes, const int32_t* slots,
                                          int B, void* dst, void* stream) {
  if (!src || !slots || !dst || B < 1 || B > 65535 || slot_bytes == 0 || slot_bytes % 16) return SEED_E_ARG;
  if (!aligned16(src) || !aligned16(dst)) return SEED_E_ARG;
  const int64_t s16 = (int64_t)(slot_bytes / 16);
  const unsigned gx = (unsigned)std::min<int64_t>((s16 + 255) / 256, 64);
  return launch_k(replay_gather_kernel, dim3(gx, (unsigned)B), dim3(256), 0, (cudaStream_t)stream,
                  (const uint4*)src, s16, slots, B, (uint4*)dst);
}

extern "C" seed_status seed_replay_scatter(const void* src, size_t slot_bytes, const int32_t* slots,
                                           int B, void* dst, void* stream) {
  if (!src || !slots || !dst || B < 1 || B > 65535 || slot_bytes == 0 || slot_bytes % 16) return SEED_E_ARG;
  if (!aligned16(src) || !aligned16(dst)) return SEED_E_ARG;
  const int64_t s16 = (int64_t)(slot_bytes / 16);
  const unsigned gx = (unsigned)std::min<int64_t>((s16 + 255) / 256, 64);
  return launch_k(replay_scatter_kernel, dim3(gx, (unsigned)B), dim3(256), 0, (cudaStream_t)stream,
                  (const uint4*)src, s16, slots, B, (uint4*)dst);
}
