// abi.cu — status strings and version of the libseed C ABI (include/seed.h).
#include "common.cuh"

extern "C" const char* seed_status_string(int s) {
  switch (s) {
    case SEED_OK: return "ok";
    case SEED_E_ARG: return "invalid argument";
    case SEED_E_SHAPE: return "unsupported shape";
    case SEED_E_NONFINITE: return "non-finite value";
    case SEED_E_CUDA: return "CUDA error";
    case SEED_E_NCCL: return "NCCL error";
    case SEED_E_UNSUPPORTED: return "unsupported in this build";
    case SEED_E_WORKSPACE: return "workspace too small";
    default: return "unknown status";
  }
}

extern "C" int seed_abi_version(void) { return 1; }

namespace seed {
static thread_local cudaError_t g_last_cuda_error = cudaSuccess;
void note_cuda_error(cudaError_t e) { g_last_cuda_error = e; }
}  // namespace seed

extern "C" const char* seed_last_cuda_error(void) {
  return cudaGetErrorString(seed::g_last_cuda_error);
}
