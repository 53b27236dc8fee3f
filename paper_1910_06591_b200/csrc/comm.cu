// comm.cu — data-parallel communicator (H10; "applies the gradients ...
// synchronously"): a thin owner of an ncclComm_t.  NCCL is resolved at run
// time with dlopen("libnccl.so.2") so the library follows whichever NCCL the
// process (torch) already loaded and has no link-time NCCL dependency.
#include <dlfcn.h>
#include <stdio.h>
#include <algorithm>
#include <string.h>
#include "common.cuh"

namespace {
struct NcclUid { char internal[128]; };
typedef void* ncclComm_t;
typedef int (*GetUid_t)(NcclUid*);
typedef int (*InitRank_t)(ncclComm_t*, int, NcclUid, int);
typedef int (*AllReduce_t)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t);
typedef int (*Destroy_t)(ncclComm_t);
typedef int (*Split_t)(ncclComm_t, int, int, ncclComm_t*, void*);
constexpr int kNcclFloat32 = 7, kNcclSum = 0;

struct Nccl {
  bool ok = false;
  GetUid_t get_uid = nullptr;
  InitRank_t init_rank = nullptr;
  AllReduce_t all_reduce = nullptr;
  Destroy_t destroy = nullptr;
  Split_t split = nullptr;   // optional (NCCL >= 2.18)
};

// resolved once per process (thread-safe static initialisation)
static Nccl load_nccl() {
  Nccl n;
  {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      n.get_uid = (GetUid_t)dlsym(h, "ncclGetUniqueId");
      n.init_rank = (InitRank_t)dlsym(h, "ncclCommInitRank");
      n.all_reduce = (AllReduce_t)dlsym(h, "ncclAllReduce");
      n.destroy = (Destroy_t)dlsym(h, "ncclCommDestroy");
      n.split = (Split_t)dlsym(h, "ncclCommSplit");
      n.ok = n.get_uid && n.init_rank && n.all_reduce && n.destroy;
    }
  }
  return n;
}
const Nccl& nccl() {
  static const Nccl n = load_nccl();
  return n;
}
}  // namespace

constexpr int COMM_EVENTS = 6;
constexpr int PEER_MAX = 8;
// 128 x 256 measured best standalone (4.9 MB in 31-33 us at N=2 vs NCCL's 39 us);
// inside the learner step it still loses to NCCL (its CTAs compete with the
// backward's persistent kernels for SMs), so it is opt-in (SEED_PEER=1)
constexpr int PEER_BLOCKS = 128, PEER_THREADS = 256;
// Exchange buffer of one rank (device, IPC-exported): in[max] | out[max] | ctrl
struct PeerCtrl {
  unsigned cntA[PEER_MAX];    // cross-GPU arrivals per source rank (one per call), barrier 1
  unsigned cntB[PEER_MAX];    // barrier 2
  unsigned localA, localB;    // this GPU's block arrivals
  unsigned relA, relB;        // this GPU's release flags (= calls passed)
  unsigned epoch;             // completed calls (read at kernel start)
  unsigned error;             // set on a timed-out wait
  unsigned long long stamp[10];   // block 0 globaltimer stamps of the last call (diagnostics)
};
struct seed_comm {
  ncclComm_t comm;
  int rank, world;
  cudaStream_t side;          // all of this comm's collectives inside a learner step
  cudaEvent_t ev[COMM_EVENTS];   // bucket forks ..., joins
  // a second communicator (ncclCommSplit of the first) on its own side stream, so
  // two gradient buckets reduce concurrently (NCCL serialises one communicator's
  // collectives); null when the split is unavailable or SEED_DP_COMMS=1
  ncclComm_t comm2 = nullptr;
  cudaStream_t side2 = nullptr;
  // peer-memory allreduce
  int64_t peer_max = 0;
  uint8_t* peer_local = nullptr;            // this rank's buffer (cudaMalloc)
  uint8_t* peer_map[PEER_MAX] = {};         // every rank's buffer in this process
  bool peer_on = false;
};

namespace seed {
struct PeerArgs {
  float* data;
  int64_t n;
  int me, world;
  int64_t max;
  uint8_t* buf[PEER_MAX];     // rank r's exchange buffer as mapped here
};

__device__ __forceinline__ float* peer_in(const PeerArgs& a, int r) {
  return reinterpret_cast<float*>(a.buf[r]);
}
__device__ __forceinline__ float* peer_out(const PeerArgs& a, int r) {
  return reinterpret_cast<float*>(a.buf[r]) + a.max;
}
__device__ __forceinline__ PeerCtrl* peer_ctrl(const PeerArgs& a, int r) {
  return reinterpret_cast<PeerCtrl*>(reinterpret_cast<float*>(a.buf[r]) + 2 * a.max);
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Hierarchical barrier across all blocks of all ranks: blocks arrive on this
// GPU's counter (device scope); block 0 waits for them, then (release, system
// scope) signals every rank once and waits for every rank's signal; the other
// blocks wait for block 0's local release flag.  Waits are bounded (2 s).
template <int WHICH>
__device__ void peer_barrier(const PeerArgs& a, unsigned ep) {
  PeerCtrl* mine = peer_ctrl(a, a.me);
  unsigned* local = WHICH == 0 ? &mine->localA : &mine->localB;
  unsigned* rel = WHICH == 0 ? &mine->relA : &mine->relB;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(local) : "memory");
    const uint64_t t0 = gtimer();
    if (blockIdx.x == 0) {
      const unsigned lt = (ep + 1) * gridDim.x;
      while (ld_acquire_gpu(local) < lt)
        if (gtimer() - t0 > 2000000000ull) { atomicExch(&mine->error, 1u); break; }
      mine->stamp[WHICH * 4 + 0] = gtimer();
      mine->stamp[WHICH * 4 + 1] = gtimer();
      // release (system scope, cumulative over what this thread observed: every
      // block's writes, through the acquire above) — no separate full fence
      for (int r = 0; r < a.world; ++r) {
        PeerCtrl* pc = peer_ctrl(a, r);
        unsigned* dst = (WHICH == 0 ? pc->cntA : pc->cntB) + a.me;
        asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(dst) : "memory");
      }
      mine->stamp[WHICH * 4 + 2] = gtimer();
      const unsigned* cnt = WHICH == 0 ? mine->cntA : mine->cntB;
      for (int src = 0; src < a.world; ++src)
        while (ld_acquire_sys(cnt + src) < ep + 1)
          if (gtimer() - t0 > 2000000000ull) { atomicExch(&mine->error, 1u); break; }
      mine->stamp[WHICH * 4 + 3] = gtimer();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(rel), "r"(ep + 1) : "memory");
    } else {
      while (ld_acquire_gpu(rel) < ep + 1)
        if (gtimer() - t0 > 2000000000ull) { atomicExch(&mine->error, 1u); break; }
    }
  }
  __syncthreads();
}

template <int W>
__global__ void __launch_bounds__(PEER_THREADS) peer_allreduce_kernel(const PeerArgs a) {
  pdl_wait();
  const unsigned ep = *(volatile unsigned*)&peer_ctrl(a, a.me)->epoch;
  if (blockIdx.x == 0 && threadIdx.x == 0) peer_ctrl(a, a.me)->stamp[8] = gtimer();
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // 1. this rank's values into its exchange buffer
  const int64_t n4 = a.n / 4;
  const float4* d4 = reinterpret_cast<const float4*>(a.data);
  float4* in4 = reinterpret_cast<float4*>(peer_in(a, a.me));
  for (int64_t i = tid; i < n4; i += 4 * stride) {
    float4 t[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) t[u] = i + u * stride < n4 ? d4[i + u * stride] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 4; ++u) if (i + u * stride < n4) in4[i + u * stride] = t[u];
  }
  for (int64_t i = 4 * n4 + tid; i < a.n; i += stride) peer_in(a, a.me)[i] = a.data[i];
  peer_barrier<0>(a, ep);
  // 2. my slice [lo, hi): sum over ranks in rank order, write into every rank's out
  const int64_t per = ((a.n + a.world - 1) / a.world + 3) / 4 * 4;
  const int64_t lo = std::min<int64_t>(a.n, per * a.me), hi = std::min<int64_t>(a.n, lo + per);
  // 4 float4 per thread per round, every load issued before the sums (NVLink
  // latency is hidden by bytes in flight, not by threads alone)
  constexpr int U = W <= 2 ? 8 : (W <= 4 ? 4 : 2);
  for (int64_t i0 = lo + 4 * tid; i0 < hi; i0 += 4 * U * stride) {
    float4 v[W][U];
#pragma unroll
    for (int r = 0; r < W; ++r)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + 4 * u * stride;
        v[r][u] = i + 4 <= hi ? __ldcv(reinterpret_cast<const float4*>(peer_in(a, r) + i))
                              : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + 4 * u * stride;
      if (i >= hi) break;
      if (i + 4 <= hi) {
        float4 s4 = v[0][u];
#pragma unroll
        for (int r = 1; r < W; ++r) {
          s4.x += v[r][u].x; s4.y += v[r][u].y; s4.z += v[r][u].z; s4.w += v[r][u].w;
        }
#pragma unroll
        for (int r = 0; r < W; ++r) *reinterpret_cast<float4*>(peer_out(a, r) + i) = s4;
      } else {
        for (int64_t k = i; k < hi; ++k) {
          float s1 = __ldcv(peer_in(a, 0) + k);
          for (int r = 1; r < W; ++r) s1 += __ldcv(peer_in(a, r) + k);
          for (int r = 0; r < W; ++r) peer_out(a, r)[k] = s1;
        }
      }
    }
  }
  peer_barrier<1>(a, ep);
  // 3. the full sum back into the caller's buffer
  const float4* o4 = reinterpret_cast<const float4*>(peer_out(a, a.me));
  float4* w4 = reinterpret_cast<float4*>(a.data);
  for (int64_t i = tid; i < n4; i += 4 * stride) {
    float4 t[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) t[u] = i + u * stride < n4 ? __ldcv(o4 + i + u * stride) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 4; ++u) if (i + u * stride < n4) w4[i + u * stride] = t[u];
  }
  for (int64_t i = 4 * n4 + tid; i < a.n; i += stride) a.data[i] = __ldcv(peer_out(a, a.me) + i);
  // a barrier timeout (this call or an earlier one: the flag is sticky) leaves the
  // sum partial: each block poisons the first value it wrote with NaN, so the global
  // norm is non-finite and clip + Adam skip the update (metrics[7] = 1)
  if (threadIdx.x == 0 && *(volatile unsigned*)&peer_ctrl(a, a.me)->error) {
    if (tid < n4) a.data[4 * tid] = __int_as_float(0x7fffffff);
    else if (4 * n4 + tid < a.n) a.data[4 * n4 + tid] = __int_as_float(0x7fffffff);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) peer_ctrl(a, a.me)->epoch = ep + 1;   // all blocks read ep
}
}  // namespace seed

namespace seed {
static bool aligned_f4(const float* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
}

namespace seed {
seed_status comm_allreduce(seed_comm* c, float* data, int64_t n, cudaStream_t st);
seed_status comm_side(seed_comm* c, cudaStream_t* side, cudaStream_t* side2, cudaEvent_t* ev) {
  if (!c || c->world == 1 || !c->side) return SEED_E_ARG;
  *side = c->side;
  *side2 = c->comm2 ? c->side2 : nullptr;
  for (int i = 0; i < COMM_EVENTS; ++i) ev[i] = c->ev[i];
  return SEED_OK;
}
seed_status comm_allreduce2(seed_comm* c, float* data, int64_t n, cudaStream_t st) {
  if (!c || !data) return SEED_E_ARG;
  if (c->world == 1) return SEED_OK;
  if (!c->comm2) return comm_allreduce(c, data, n, st);
  return nccl().all_reduce(data, data, (size_t)n, kNcclFloat32, kNcclSum, c->comm2, st) == 0
             ? SEED_OK
             : SEED_E_NCCL;
}
int comm_world(const seed_comm* c) { return c ? c->world : 1; }

seed_status comm_allreduce(seed_comm* c, float* data, int64_t n, cudaStream_t st) {
  if (!c || !data) return SEED_E_ARG;
  if (c->world == 1) return SEED_OK;
  if (c->peer_on && n <= c->peer_max && aligned_f4(data)) {
    PeerArgs a{};
    a.data = data; a.n = n; a.me = c->rank; a.world = c->world; a.max = c->peer_max;
    for (int r = 0; r < c->world; ++r) a.buf[r] = c->peer_map[r];
    switch (c->world) {
      case 2: return launch_k(peer_allreduce_kernel<2>, dim3(PEER_BLOCKS), dim3(PEER_THREADS), 0, st, a);
      case 3: return launch_k(peer_allreduce_kernel<3>, dim3(PEER_BLOCKS), dim3(PEER_THREADS), 0, st, a);
      case 4: return launch_k(peer_allreduce_kernel<4>, dim3(PEER_BLOCKS), dim3(PEER_THREADS), 0, st, a);
      case 5: return launch_k(peer_allreduce_kernel<5>, dim3(PEER_BLOCKS), dim3(PEER_THREADS), 0, st, a);
      case 6: return launch_k(peer_allreduce_kernel<6>, dim3(PEER_BLOCKS), dim3(PEER_THREADS), 0, st, a);
      case 7: return launch_k(peer_allreduce_kernel<7>, dim3(PEER_BLOCKS), dim3(PEER_THREADS), 0, st, a);
      default: return launch_k(peer_allreduce_kernel<8>, dim3(PEER_BLOCKS), dim3(PEER_THREADS), 0, st, a);
    }
  }
  if (!nccl().ok) return SEED_E_NCCL;
  return nccl().all_reduce(data, data, (size_t)n, kNcclFloat32, kNcclSum, c->comm, st) == 0
             ? SEED_OK
             : SEED_E_NCCL;
}
}  // namespace seed

extern "C" seed_status seed_comm_get_unique_id(void* id128) {
  if (!id128) return SEED_E_ARG;
  if (!nccl().ok) return SEED_E_NCCL;
  NcclUid u;
  if (nccl().get_uid(&u) != 0) return SEED_E_NCCL;
  memcpy(id128, &u, sizeof(u));
  return SEED_OK;
}

extern "C" seed_status seed_comm_init(const void* id128, int rank, int world, seed_comm** out) {
  if (!id128 || !out || world < 1 || rank < 0 || rank >= world) return SEED_E_ARG;
  seed_comm* c = new seed_comm{};
  c->rank = rank;
  c->world = world;
  if (world > 1) {
    if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess) {
      delete c;
      return SEED_E_CUDA;
    }
    for (int i = 0; i < COMM_EVENTS; ++i)
      if (cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming) != cudaSuccess) {
        delete c;
        return SEED_E_CUDA;
      }
    if (!nccl().ok) {
      delete c;
      return SEED_E_NCCL;
    }
    NcclUid u;
    memcpy(&u, id128, sizeof(u));
    if (nccl().init_rank(&c->comm, world, u, rank) != 0) {
      delete c;
      return SEED_E_NCCL;
    }
    const char* e = getenv("SEED_DP_COMMS");   // collective decision: same env on every rank
    if (nccl().split && !(e && e[0] == '1')) {
      if (nccl().split(c->comm, 0, rank, &c->comm2, nullptr) != 0 ||
          cudaStreamCreateWithFlags(&c->side2, cudaStreamNonBlocking) != cudaSuccess)
        c->comm2 = nullptr;
    }
  }
  *out = c;
  return SEED_OK;
}

extern "C" seed_status seed_comm_destroy(seed_comm* c) {
  if (!c) return SEED_E_ARG;
  if (c->comm2 && nccl().ok) nccl().destroy(c->comm2);
  if (c->comm && nccl().ok) nccl().destroy(c->comm);
  if (c->side2) cudaStreamDestroy(c->side2);
  for (int r = 0; r < c->world && r < PEER_MAX; ++r)
    if (c->peer_map[r] && c->peer_map[r] != c->peer_local) cudaIpcCloseMemHandle(c->peer_map[r]);
  if (c->peer_local) cudaFree(c->peer_local);
  for (int i = 0; i < COMM_EVENTS; ++i)
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
  if (c->side) cudaStreamDestroy(c->side);
  delete c;
  return SEED_OK;
}

extern "C" seed_status seed_comm_allreduce_f32(seed_comm* c, float* data, int64_t n, void* stream) {
  return seed::comm_allreduce(c, data, n, (cudaStream_t)stream);
}

extern "C" seed_status seed_comm_peer_setup(seed_comm* c, int64_t max_floats, void* handle_out) {
  if (!c || max_floats <= 0 || !handle_out || c->world > PEER_MAX) return SEED_E_ARG;
  if (c->peer_local) return SEED_E_ARG;
  max_floats = (max_floats + 3) / 4 * 4;
  const size_t bytes = (size_t)2 * max_floats * 4 + sizeof(PeerCtrl);
  if (cudaMalloc(&c->peer_local, bytes) != cudaSuccess) return SEED_E_CUDA;
  if (cudaMemset(c->peer_local, 0, bytes) != cudaSuccess) return SEED_E_CUDA;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, c->peer_local) != cudaSuccess) return SEED_E_CUDA;
  static_assert(sizeof(h) == 64, "IPC handle size");
  memcpy(handle_out, &h, 64);
  c->peer_max = max_floats;
  return SEED_OK;
}

extern "C" seed_status seed_comm_peer_open(seed_comm* c, const void* handles) {
  if (!c || !handles || !c->peer_local) return SEED_E_ARG;
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank) {
      c->peer_map[r] = c->peer_local;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, (const uint8_t*)handles + 64 * r, 64);
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return SEED_E_CUDA;
    c->peer_map[r] = (uint8_t*)p;
  }
  if (cudaDeviceSynchronize() != cudaSuccess) return SEED_E_CUDA;
  c->peer_on = true;
  return SEED_OK;
}

extern "C" seed_status seed_comm_peer_status(seed_comm* c) {
  if (!c) return SEED_E_ARG;
  if (!c->peer_local) return SEED_OK;
  if (cudaDeviceSynchronize() != cudaSuccess) return SEED_E_CUDA;
  PeerCtrl ctl;
  if (cudaMemcpy(&ctl, c->peer_local + (size_t)2 * c->peer_max * 4, sizeof(ctl),
                 cudaMemcpyDeviceToHost) != cudaSuccess)
    return SEED_E_CUDA;
  if (getenv("SEED_PEER_DEBUG")) {
    const unsigned long long b = ctl.stamp[8];
    fprintf(stderr, "[peer rank %d] start->A.local %llu ns, A.fence %llu, A.signal %llu, A.wait %llu | "
            "B.local %llu, B.fence %llu, B.signal %llu, B.wait %llu\n", c->rank, ctl.stamp[0] - b,
            ctl.stamp[1] - ctl.stamp[0], ctl.stamp[2] - ctl.stamp[1], ctl.stamp[3] - ctl.stamp[2],
            ctl.stamp[4] - ctl.stamp[3], ctl.stamp[5] - ctl.stamp[4], ctl.stamp[6] - ctl.stamp[5],
            ctl.stamp[7] - ctl.stamp[6]);
  }
  return ctl.error ? SEED_E_NCCL : SEED_OK;
}
