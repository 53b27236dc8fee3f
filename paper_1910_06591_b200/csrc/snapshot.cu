// snapshot.cu — versioned parameter publication for inference that runs
// concurrently with training (P:98 / P:111 "the
// inference ... uses the latest parameters", P:125, P:238 inference on
// dedicated cores while the learner trains; S:37-42 ParamSnapshot.version,
// S:109, S:465 single-copy semantics).
//
// A single-producer / single-consumer triple buffer in device memory.  Slot k
// holds one complete parameter set: the bf16 operand image (params_lowp) then
// the fp32 params, plus its version.  Three indices partition {0, 1, 2}:
//   back   — owned by the producer (the learner's stream), being written;
//   middle — the last completely written slot, with a FRESH bit;
//   front  — owned by the consumer (the inference stream), being read.
// publish: copy into back; then version[back] = step, fence, and ONE atomic
//   exchange  middle <- back | FRESH, back <- old middle.
// acquire: if middle has FRESH, ONE atomic exchange  middle <- front,
//   front <- old middle (which is FRESH: only the consumer clears the bit),
//   then copy slot[front] into the consumer's private image when it changed.
// Neither side ever waits for the other, and a slot the consumer can read is
// never written: the consumer sees whole updates only (never a torn one), and
// always the latest complete one at its acquire.
#include <algorithm>
#include "common.cuh"
#include "net.cuh"

namespace seed {

constexpr int32_t SNAP_FRESH = 0x100;
enum { SNAP_BACK = 0, SNAP_MIDDLE = 1, SNAP_FRONT = 2, SNAP_CHANGED = 3 };

// params_lowp bytes (seed_net_lowp_bytes: whole 16-byte chunks) and the slot offset
// of the fp32 params
static size_t snap_lowp16(const NetPlan& p) { return align_up((size_t)p.lowp_elems * 2, 16) / 16; }
static size_t snap_lowp_bytes(const NetPlan& p) { return align_up((size_t)p.lowp_elems * 2, 256); }

struct SnapSlots {
  uint8_t* s[3];
};

// producer, step 1: the current parameters into slot[back] (uint4 copies)
__global__ void snap_copy_in_kernel(SnapSlots sl, const int32_t* __restrict__ state,
                                    const uint4* __restrict__ lowp, int64_t n_lowp16,
                                    const float* __restrict__ params, int64_t n_params,
                                    int64_t params_off) {
  pdl_wait();
  uint8_t* dst = sl.s[state[SNAP_BACK] & 3];
  uint4* d16 = reinterpret_cast<uint4*>(dst);
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < n_lowp16; i += stride) d16[i] = lowp[i];
  float* dp = reinterpret_cast<float*>(dst + params_off);
  const int64_t n4 = n_params / 4;
  for (int64_t i = tid; i < n4; i += stride)
    reinterpret_cast<float4*>(dp)[i] = reinterpret_cast<const float4*>(params)[i];
  for (int64_t i = 4 * n4 + tid; i < n_params; i += stride) dp[i] = params[i];
}

// producer, step 2: stamp the version and hand the slot over (one thread)
__global__ void snap_publish_kernel(int32_t* state, int64_t* version, const int64_t* step) {
  pdl_wait();
  const int32_t back = state[SNAP_BACK] & 3;
  version[back] = step ? *step : version[back] + 1;
  __threadfence();   // slot contents and version before the index exchange
  const int32_t old = atomicExch(&state[SNAP_MIDDLE], back | SNAP_FRESH);
  state[SNAP_BACK] = old & 3;
}

// consumer, step 1: take the freshest complete slot (one thread)
__global__ void snap_acquire_kernel(int32_t* state, const int64_t* version, int64_t* version_out) {
  pdl_wait();
  int32_t changed = 0;
  const int32_t mid = atomicAdd(&state[SNAP_MIDDLE], 0);
  if (mid & SNAP_FRESH) {
    const int32_t got = atomicExch(&state[SNAP_MIDDLE], state[SNAP_FRONT] & 3);
    state[SNAP_FRONT] = got & 3;
    changed = 1;
  }
  __threadfence();
  state[SNAP_CHANGED] = changed;
  if (version_out) *version_out = *(volatile const int64_t*)&version[state[SNAP_FRONT] & 3];
}

// consumer, step 2: slot[front] into the consumer's private image when it changed
__global__ void snap_copy_out_kernel(SnapSlots sl, const int32_t* __restrict__ state, int64_t n_lowp16,
                                     int64_t n_params, int64_t params_off, uint4* __restrict__ lowp_out,
                                     float* __restrict__ params_out, int force) {
  pdl_wait();
  if (!force && !state[SNAP_CHANGED]) return;
  const uint8_t* src = sl.s[state[SNAP_FRONT] & 3];
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint4* s16 = reinterpret_cast<const uint4*>(src);
  for (int64_t i = tid; i < n_lowp16; i += stride) lowp_out[i] = __ldcg(s16 + i);
  const float* sp = reinterpret_cast<const float*>(src + params_off);
  const int64_t n4 = n_params / 4;
  for (int64_t i = tid; i < n4; i += stride)
    reinterpret_cast<float4*>(params_out)[i] = __ldcg(reinterpret_cast<const float4*>(sp) + i);
  for (int64_t i = 4 * n4 + tid; i < n_params; i += stride) params_out[i] = __ldcg(sp + i);
}

__global__ void snap_init_kernel(int32_t* state, int64_t* version) {
  state[SNAP_BACK] = 0;
  state[SNAP_MIDDLE] = 1;
  state[SNAP_FRONT] = 2;
  state[SNAP_CHANGED] = 0;
  version[0] = version[1] = version[2] = -1;
}

static int copy_blocks(int64_t bytes) {
  return (int)std::min<int64_t>(std::max<int64_t>(bytes / (256 * 16 * 4), 1), 4 * 148);
}

static seed_status snap_check(const seed_net_spec* spec, const seed_param_snapshot* s, NetPlan* p) {
  SEED_TRY(make_net_plan(spec, p));
  if (!s || !s->state || !s->version) return SEED_E_ARG;
  for (int k = 0; k < 3; ++k)
    if (!s->slots[k] || !aligned16(s->slots[k])) return SEED_E_ARG;
  return SEED_OK;
}

}  // namespace seed

using namespace seed;

extern "C" seed_status seed_param_snapshot_bytes(const seed_net_spec* spec, size_t* slot_bytes) {
  if (!slot_bytes) return SEED_E_ARG;
  NetPlan p;
  SEED_TRY(make_net_plan(spec, &p));
  *slot_bytes = snap_lowp_bytes(p) + align_up((size_t)p.P * 4, 256);
  return SEED_OK;
}

extern "C" seed_status seed_param_snapshot_init(seed_param_snapshot* s, void* stream) {
  if (!s || !s->state || !s->version) return SEED_E_ARG;
  snap_init_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(s->state, s->version);
  return last_launch();
}

extern "C" seed_status seed_param_publish(const seed_net_spec* spec, const seed_train_state* state,
                                          seed_param_snapshot* s, void* stream) {
  NetPlan p;
  SEED_TRY(snap_check(spec, s, &p));
  if (!state || !state->params || !state->params_lowp || !aligned16(state->params) ||
      !aligned16(state->params_lowp))
    return SEED_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t lb = snap_lowp_bytes(p);
  SnapSlots sl{{(uint8_t*)s->slots[0], (uint8_t*)s->slots[1], (uint8_t*)s->slots[2]}};
  SEED_TRY(launch_k(snap_copy_in_kernel, dim3(copy_blocks(lb + p.P * 4)), dim3(256), 0, st, sl,
                    (const int32_t*)s->state, (const uint4*)state->params_lowp, (int64_t)snap_lowp16(p),
                    (const float*)state->params, (int64_t)p.P, (int64_t)lb));
  return launch_k(snap_publish_kernel, dim3(1), dim3(1), 0, st, s->state, s->version,
                  (const int64_t*)state->step);
}

extern "C" seed_status seed_param_acquire(const seed_net_spec* spec, seed_param_snapshot* s,
                                          void* lowp_out, float* params_out, int64_t* version_out,
                                          int force_copy, void* stream) {
  NetPlan p;
  SEED_TRY(snap_check(spec, s, &p));
  if (!lowp_out || !params_out || !aligned16(lowp_out) || !aligned16(params_out)) return SEED_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t lb = snap_lowp_bytes(p);
  SnapSlots sl{{(uint8_t*)s->slots[0], (uint8_t*)s->slots[1], (uint8_t*)s->slots[2]}};
  SEED_TRY(launch_k(snap_acquire_kernel, dim3(1), dim3(1), 0, st, s->state,
                    (const int64_t*)s->version, version_out));
  return launch_k(snap_copy_out_kernel, dim3(copy_blocks(lb + p.P * 4)), dim3(256), 0, st, sl,
                  (const int32_t*)s->state, (int64_t)snap_lowp16(p), (int64_t)p.P, (int64_t)lb,
                  (uint4*)lowp_out, params_out, force_copy);
}
