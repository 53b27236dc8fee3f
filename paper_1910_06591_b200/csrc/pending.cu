// pending.cu — ABI entry points not built yet in this revision (return UNSUPPORTED).
#include "common.cuh"
extern "C" {
seed_status seed_infer_workspace_size(const seed_net_spec*, int, size_t*) { return SEED_E_UNSUPPORTED; }
seed_status seed_infer(const seed_net_spec*, const void*, const float*, const seed_state_table*, int, const int32_t*, const uint8_t*, const float*, const uint8_t*, const float*, uint64_t, uint64_t, int32_t*, float*, float*, const seed_unroll_store*, void*, size_t, void*) { return SEED_E_UNSUPPORTED; }
seed_status seed_assemble_batch(const seed_unroll_store*, int, int, int, const seed_batch*, void*) { return SEED_E_UNSUPPORTED; }
}
