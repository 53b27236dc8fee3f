// comm.cu — data-parallel communicator (H10; "applies the gradients ...
// synchronously"): a thin owner of an ncclComm_t.  NCCL is resolved at run
// time with dlopen("libnccl.so.2") so the library follows whichever NCCL the
// process (torch) already loaded and has no link-time NCCL dependency.
#include <dlfcn.h>
#include <string.h>
#include "common.cuh"

namespace {
struct NcclUid { char internal[128]; };
typedef void* ncclComm_t;
typedef int (*GetUid_t)(NcclUid*);
typedef int (*InitRank_t)(ncclComm_t*, int, NcclUid, int);
typedef int (*AllReduce_t)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t);
typedef int (*Destroy_t)(ncclComm_t);
constexpr int kNcclFloat32 = 7, kNcclSum = 0;

struct Nccl {
  bool ok = false;
  GetUid_t get_uid = nullptr;
  InitRank_t init_rank = nullptr;
  AllReduce_t all_reduce = nullptr;
  Destroy_t destroy = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      n.get_uid = (GetUid_t)dlsym(h, "ncclGetUniqueId");
      n.init_rank = (InitRank_t)dlsym(h, "ncclCommInitRank");
      n.all_reduce = (AllReduce_t)dlsym(h, "ncclAllReduce");
      n.destroy = (Destroy_t)dlsym(h, "ncclCommDestroy");
      n.ok = n.get_uid && n.init_rank && n.all_reduce && n.destroy;
    }
  }
  return n;
}
}  // namespace

constexpr int COMM_EVENTS = 4;
struct seed_comm {
  ncclComm_t comm;
  int rank, world;
  cudaStream_t side;          // all of this comm's collectives inside a learner step
  cudaEvent_t ev[COMM_EVENTS];   // bucket forks ..., join
};

namespace seed {
seed_status comm_side(seed_comm* c, cudaStream_t* side, cudaEvent_t* ev) {
  if (!c || c->world == 1 || !c->side) return SEED_E_ARG;
  *side = c->side;
  for (int i = 0; i < COMM_EVENTS; ++i) ev[i] = c->ev[i];
  return SEED_OK;
}
int comm_world(const seed_comm* c) { return c ? c->world : 1; }

seed_status comm_allreduce(seed_comm* c, float* data, int64_t n, cudaStream_t st) {
  if (!c || !data) return SEED_E_ARG;
  if (c->world == 1) return SEED_OK;
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
  seed_comm* c = new seed_comm{nullptr, rank, world, nullptr, {}};
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
  }
  *out = c;
  return SEED_OK;
}

extern "C" seed_status seed_comm_destroy(seed_comm* c) {
  if (!c) return SEED_E_ARG;
  if (c->comm && nccl().ok) nccl().destroy(c->comm);
  for (int i = 0; i < COMM_EVENTS; ++i)
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
  if (c->side) cudaStreamDestroy(c->side);
  delete c;
  return SEED_OK;
}

extern "C" seed_status seed_comm_allreduce_f32(seed_comm* c, float* data, int64_t n, void* stream) {
  return seed::comm_allreduce(c, data, n, (cudaStream_t)stream);
}
