// pending.cu — ABI entry points not built yet in this revision (return UNSUPPORTED).
#include "common.cuh"
extern "C" {
seed_status seed_net_param_count(const seed_net_spec*, int64_t*) { return SEED_E_UNSUPPORTED; }
seed_status seed_net_param_tensor(const seed_net_spec*, int, char*, int*, int64_t*, int64_t*) { return SEED_E_UNSUPPORTED; }
seed_status seed_net_lowp_bytes(const seed_net_spec*, size_t*) { return SEED_E_UNSUPPORTED; }
seed_status seed_net_refresh_lowp(const seed_net_spec*, const float*, void*, void*) { return SEED_E_UNSUPPORTED; }
seed_status seed_learner_workspace_size(const seed_net_spec*, int, int, size_t*) { return SEED_E_UNSUPPORTED; }
seed_status seed_learner_step(const seed_net_spec*, int, int, const seed_batch*, const seed_train_state*, const seed_hparams*, seed_comm*, void*, size_t, float*, void*) { return SEED_E_UNSUPPORTED; }
seed_status seed_learner_outputs(const seed_net_spec*, int, int, void*, float**, float**, float**, float**) { return SEED_E_UNSUPPORTED; }
seed_status seed_comm_get_unique_id(void*) { return SEED_E_UNSUPPORTED; }
seed_status seed_comm_init(const void*, int, int, seed_comm**) { return SEED_E_UNSUPPORTED; }
seed_status seed_comm_destroy(seed_comm*) { return SEED_E_UNSUPPORTED; }
seed_status seed_comm_allreduce_f32(seed_comm*, float*, int64_t, void*) { return SEED_E_UNSUPPORTED; }
seed_status seed_infer_workspace_size(const seed_net_spec*, int, size_t*) { return SEED_E_UNSUPPORTED; }
seed_status seed_infer(const seed_net_spec*, const void*, const float*, const seed_state_table*, int, const int32_t*, const uint8_t*, const float*, const uint8_t*, const float*, uint64_t, uint64_t, int32_t*, float*, float*, const seed_unroll_store*, void*, size_t, void*) { return SEED_E_UNSUPPORTED; }
seed_status seed_assemble_batch(const seed_unroll_store*, int, int, int, const seed_batch*, void*) { return SEED_E_UNSUPPORTED; }
}
