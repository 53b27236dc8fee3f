/*
 * seed.h — C ABI of libseed.so, the B200 (sm_100a) hot path of SEED
 * (Espeholt et al., arXiv 1910.06591): the centralized data-parallel learner
 * step over [T+1][B] unroll batches, V-trace, and centralized batched inference
 * with an on-device per-actor recurrent-state table.
 *
 * Citations: P:NNN = line of /root/reference/PAPER.md, S:NNN = line of
 * /root/reference/SPEC.md, C# = reading
 *
 * ---- conventions (apply to every call) -----------------------------------
 * Memory:    every tensor pointer is caller-owned DEVICE memory unless a
 *            parameter says "host".  The library never allocates inside a hot
 *            call; scratch comes from a caller workspace sized by the matching
 *            *_workspace_size() query.  The library keeps no pointer after a
 *            call returns (except inside a seed_comm, which owns an NCCL comm).
 * Streams:   `stream` is a cudaStream_t passed as void*; NULL = legacy default
 *            stream.  All calls are asynchronous on that stream.
 * Errors:    return codes only (seed_status); nothing is thrown across the ABI.
 *            Host-checkable argument errors return synchronously and launch
 *            nothing.  Data-dependent numeric problems are reported through
 *            device-side flags/metrics and never force a host sync.
 * Layout:    batch-major, trajectory-contiguous, row-major: [B][T] and
 *            [B][T+1][...]; bootstrap values separate [B].  16-byte aligned
 *            pointers are required (torch allocations satisfy this).
 * Threads:   no global mutable state: the second stream and events a learner step
 *            branches onto belong to a caller-owned seed_exec, the NCCL comms to a
 *            caller-owned seed_comm.  The only process-wide data are idempotent
 *            per-device caches (kernel shared-memory opt-ins, SM counts) and
 *            environment switches for A/B measurement, read once (SEED_PDL,
 *            SEED_DP_BUCKETS, SEED_DP_COMMS, SEED_FUSE_POOL=0 unfused section conv +
 *            max-pool, SEED_CP_KX / SEED_CP_EW its column-tap-stacked form / epilogue
 *            warps, SEED_KX, SEED_XF_U8, SEED_DEEP_TRIG early PDL triggers of the 3x3
 *            kernels, SEED_PEER_DEBUG) or per call
 *            (SEED_STORE_CONV=1: the fused section conv + max-pool also stores the
 *            conv rows, a test hook).  Calls on
 *            different streams with disjoint buffers (and distinct seed_exec /
 *            seed_comm handles) are independent; one process may drive several
 *            devices (each call runs on the device current at the call).
 */
#ifndef SEED_H_
#define SEED_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SEED_OK = 0,
  SEED_E_ARG = 1,          /* null / misaligned pointer, bad hyper-parameter   */
  SEED_E_SHAPE = 2,        /* T, B, A, n out of the supported range            */
  SEED_E_NONFINITE = 3,    /* reserved: numeric problems are device flags      */
  SEED_E_CUDA = 4,         /* a CUDA runtime call failed (launch, attribute)   */
  SEED_E_NCCL = 5,         /* NCCL missing or an NCCL call failed              */
  SEED_E_UNSUPPORTED = 6,  /* net kind / size not built into this library      */
  SEED_E_WORKSPACE = 7     /* ws_bytes smaller than the *_workspace_size query */
} seed_status;

const char* seed_status_string(int status);
/* Diagnostics: the CUDA error string behind the last SEED_E_CUDA returned to
 * this thread (thread-local; "no error" if none). */
const char* seed_last_cuda_error(void);
/* Library ABI version (this header): 1. */
int seed_abi_version(void);

/* ===========================================================================
 * seed_vtrace — V-trace targets (H6).
 * Definition: S:140 (the IMPALA recursion cited at P:143-145; PAPER.md prints
 * no formula, reading C1):
 *   ratio_t = exp(target_logp_t - behaviour_logp_t)
 *   rho_t   = min(rho_bar, ratio_t);  c_t = lambda * min(c_bar, ratio_t)   (C2)
 *   delta_t = rho_t (r_t + gamma_t V_{t+1} - V_t),   V_T := bootstrap     (C4)
 *   vs_t    = V_t + delta_t + gamma_t c_t (vs_{t+1} - V_{t+1}), vs_T - V_T := 0
 *   pg_t    = rho_t (r_t + gamma_t vs_{t+1} - V_t),  vs_T := bootstrap    (C3)
 * Arguments: all [B][T] float32 row-major (trajectory b contiguous), bootstrap
 *   [B].  discounts gamma_t = gamma * (1 - done_{t->t+1}) (C5).
 *   rho_bar, c_bar may be +INFINITY (no clipping); require c_bar > 0,
 *   rho_bar >= c_bar, 0 <= lambda <= 1 (C6) else SEED_E_ARG.
 *   T >= 1, B >= 1 else SEED_E_SHAPE.  T % 4 == 0 takes the float4 path.
 * Outputs: vs, pg_advantages [B][T] (may not alias inputs).
 *   nonfinite_flag: nullable device int32; set to 1 (never cleared) when any
 *   target-behaviour log-prob difference, reward, discount, value or
 *   bootstrap is NaN/Inf (C7).  Outputs are still written.
 * ======================================================================== */
seed_status seed_vtrace(int T, int B,
                        const float* behaviour_logp, const float* target_logp,
                        const float* rewards, const float* discounts,
                        const float* values, const float* bootstrap_value,
                        float rho_bar, float c_bar, float lambda,
                        float* vs, float* pg_advantages,
                        int* nonfinite_flag, void* stream);

/* ===========================================================================
 * Networks (C14).  Flat fp32 parameter layout = the tensors below, row-major,
 * concatenated in this order (query with seed_net_param_tensor):
 *  SEED_NET_MLP (configs[0]): mlp0.w[64][D] mlp0.b[64] mlp1.w[64][64] mlp1.b[64]
 *      heads.w[A+1][64] heads.b[A+1];  D = obs_h*obs_w*obs_c, obs fp32.
 *  SEED_NET_ATARI_SHALLOW (configs[1], 84x84x4 uint8):
 *      conv1.w[16][8][8][C] conv1.b[16]  (8x8 stride 4 valid, ReLU)
 *      conv2.w[32][4][4][16] conv2.b[32] (4x4 stride 2 valid, ReLU)
 *      fc.w[256][9*9*32] fc.b[256]        (input flattened (y, x, c); ReLU)
 *      lstm.wx[4U][256+A+1] lstm.wh[4U][U] lstm.b[4U]   (gates [i,f,g,o], C15)
 *      heads.w[A+1][U] heads.b[A+1]       (rows 0..A-1 logits, row A value)
 *  SEED_NET_IMPALA_DEEP / SEED_NET_GFOOTBALL (configs[2]/[3]): per section s
 *      s{s}.conv.w[ch][3][3][cin] .b, then res{0,1}.conv{0,1}.w[ch][3][3][ch] .b;
 *      then fc / lstm / heads as above.  seed_learner_step supports every
 *      kind; seed_infer supports SEED_NET_ATARI_SHALLOW (configs[4]) and returns
 *      SEED_E_UNSUPPORTED for the others.
 *  Observations enter as obs/255 (uint8 nets).  LSTM core input
 *  x_t = [fc_t, onehot(prev_action_t), clip(reward_t,-1,1)], one-hot and reward
 *  zeroed when done_t, and (h,c) reset to 0 before step t when done_t
 *  (C15).
 * ======================================================================== */
enum { SEED_NET_MLP = 0, SEED_NET_ATARI_SHALLOW = 1, SEED_NET_IMPALA_DEEP = 2,
       SEED_NET_GFOOTBALL = 3 };

typedef struct {
  int kind;                       /* SEED_NET_*                                  */
  int obs_h, obs_w, obs_c;        /* MLP: 1, 1, D                                */
  int num_actions;                /* A >= 2                               */
  int lstm_units;                 /* 0 for the MLP; 256 for the conv nets        */
  int torso_width;                /* IMPALA-deep channel multiplier: 0/1 = (16, 32,
                                     32[, 32]), 2 = DMLab "Medium 2x" (32, 64, 64),
                                     4 = DMLab "Large 4x" (64, 128, 128; P:411,
                                     P:432-434); others SEED_E_UNSUPPORTED        */
} seed_net_spec;

seed_status seed_net_param_count(const seed_net_spec* spec, int64_t* n_out /* host */);
/* Describe parameter tensor `index` (0-based).  name_out: host char[64];
 * shape_out: host int64[4] (unused dims 0); offset_out: element offset in the
 * flat vector.  Returns SEED_E_ARG when index >= tensor count. */
seed_status seed_net_param_tensor(const seed_net_spec* spec, int index, char* name_out,
                                  int* ndim_out, int64_t* shape_out, int64_t* offset_out);
/* Bytes of the library-private low-precision operand image (bf16 weights in
 * the GEMM-ready layout) that seed_train_state.params_lowp points to. */
seed_status seed_net_lowp_bytes(const seed_net_spec* spec, size_t* bytes_out);
/* Rebuild params_lowp from fp32 params (call once after initialising params;
 * seed_learner_step keeps it in sync afterwards). */
seed_status seed_net_refresh_lowp(const seed_net_spec* spec, const float* params,
                                  void* params_lowp, void* stream);

/* ===========================================================================
 * seed_learner_step — one synchronous learner update (H0-H11; P:125
 * "computes gradients ... and applies the gradients ... synchronously").
 * Forward over the whole [B][T+1] batch, V-trace targets (stop-gradient), loss
 *   L = loss_scale * sum_{b,t<T} [ -pg_t log pi(a_t|x_t)
 *                                  + 1/2 vf_coef (vs_t - V_t)^2 - ent_coef H_t ]
 * (C8-C10), backward, optional NCCL allreduce (sum) of the flat
 * grads across the comm's ranks (C20: loss_scale = 1/(N B T) makes the
 * sum a global mean), global-norm clip, Adam (C11-C12), bf16
 * shadow refresh, step += 1.  A non-finite gradient norm skips the update
 * and leaves params, moments and step unchanged.
 * Trained steps t = 0..T-1 use reward[t+1], discount gamma*(1-done[t+1]),
 * behaviour_logp[t], action[t]; bootstrap = V(x_T) (C5).
 * ======================================================================== */
typedef struct {
  float discount;        /* gamma (.99)                         */
  float lambda;          /* V-trace lambda                     */
  float rho_bar, c_bar;  /* C6: 1, 1                                   */
  float vf_coef;         /* .5                                  */
  float ent_coef;
  float loss_scale;      /* 1/(N*B*T) for a global mean                */
  float lr, beta1, beta2, eps;   /* Adam (C12)                         */
  float max_grad_norm;   /* C11: 40                                    */
} seed_hparams;

typedef struct {
  const void* obs;             /* uint8 [B][T+1][H][W][C]; MLP: fp32 [B][T+1][D] */
  const int32_t* action;       /* [B][T+1]  a_t taken at obs t                  */
  const int32_t* prev_action;  /* [B][T+1]  action before obs t (<0 = none)     */
  const float* reward;         /* [B][T+1]  reward received with obs t          */
  const uint8_t* done;         /* [B][T+1]  1: obs t starts a new episode (C5)  */
  const float* behaviour_logp; /* [B][T+1]  log mu(a_t|x_t) recorded at inference */
  const float* h0;             /* [B][U]    LSTM state before slot 0 (C19)      */
  const float* c0;             /* [B][U]                                        */
} seed_batch;

/* params, grads, adam_m, adam_v, params_lowp and obs must be 16-byte aligned
 * (float4 / bulk-copy accesses); SEED_E_ARG otherwise.
 * params_lowp is rewritten in place by every applied update (inside the clip +
 * Adam kernel, on `stream`).  A seed_infer reading the same params_lowp on
 * another stream must be ordered against the step by the caller; for
 * inference running concurrently with training use the versioned snapshot
 * (seed_param_publish / seed_param_acquire below), which never exposes a
 * half-written update. */
typedef struct {
  float* params;       /* [P] fp32 master (flat layout above)          */
  float* grads;        /* [P] fp32: receives the (allreduced, unclipped) grads */
  float* adam_m;       /* [P]                                          */
  float* adam_v;       /* [P]                                          */
  void* params_lowp;   /* seed_net_lowp_bytes() bytes                  */
  int64_t* step;       /* device int64: ParamSnapshot.version */
} seed_train_state;

typedef struct seed_comm seed_comm;  /* wraps an ncclComm_t */

/* Execution context of a learner step (caller-owned; create on the device the
 * steps run on): a second CUDA stream of that device and the events of the
 * fork / join edges, onto which the step branches its independent backward
 * GEMMs (inside a CUDA-graph capture the edges become parallel graph branches).
 * One seed_exec must not be used by two steps at the same time.
 * seed_learner_step == seed_learner_step_ex with exec = NULL: everything on
 * `stream`, in order (same results; no overlap of the branches). */
typedef struct seed_exec seed_exec;
seed_status seed_exec_create(seed_exec** out);
seed_status seed_exec_destroy(seed_exec* exec);

seed_status seed_learner_workspace_size(const seed_net_spec* spec, int T, int B,
                                        size_t* bytes_out);
/* metrics: device float[8] = {loss, pg, baseline, entropy, grad_norm,
 * applied (1/0), version (after the step), nonfinite (1/0)}; loss terms are
 * this rank's (scaled) sums, grad_norm is of the allreduced gradient.
 * comm == NULL: single GPU.  Shapes: 1 <= T <= 256, 1 <= B <= 1024 (MLP: B*(T+1)
 * <= 65536), 2 <= A <= 32; SEED_E_SHAPE otherwise. */
seed_status seed_learner_step(const seed_net_spec* spec, int T, int B,
                              const seed_batch* batch, const seed_train_state* state,
                              const seed_hparams* hp, seed_comm* comm,
                              void* workspace, size_t ws_bytes, float* metrics,
                              void* stream);
seed_status seed_learner_step_ex(const seed_net_spec* spec, int T, int B,
                                 const seed_batch* batch, const seed_train_state* state,
                                 const seed_hparams* hp, seed_comm* comm, seed_exec* exec,
                                 void* workspace, size_t ws_bytes, float* metrics,
                                 void* stream);
/* Bench / profiling hook: identical to seed_learner_step, and additionally
 * records events[0] (cudaEvent_t as void*) before the first kernel and
 * events[i] after the i-th phase of the step (a phase = one kernel, or a
 * split-K GEMM + its fixed-order reduction).  names_out (host, nullable,
 * max_events entries) receives static phase names (names_out[i] ends at
 * events[i]); *n_events_out (host) the number of events recorded and
 * *n_launches_out (host, nullable) the number of kernels the step launched;
 * launch_counts_out (host, nullable, max_events entries) the number of kernels of
 * each phase (launch_counts_out[i] for the phase ending at events[i]). */
seed_status seed_learner_step_traced(const seed_net_spec* spec, int T, int B,
                                     const seed_batch* batch, const seed_train_state* state,
                                     const seed_hparams* hp, seed_comm* comm,
                                     void* workspace, size_t ws_bytes, float* metrics,
                                     void* stream, void** events, int max_events,
                                     const char** names_out, int* n_events_out,
                                     int* n_launches_out, int* launch_counts_out);
/* Views into a workspace after seed_learner_step (for tests / metrics):
 * logits [B][T+1][A], values [B][T+1], vs [B][T], pg_adv [B][T] (fp32). */
seed_status seed_learner_outputs(const seed_net_spec* spec, int T, int B, void* workspace,
                                 float** logits, float** values, float** vs,
                                 float** pg_adv);

/* Test hook: device pointer + byte size of a named internal buffer of the
 * learner workspace (after a step): "act1", "act2", "X", "xproj", "H",
 * "Hprev", "gates", "C", "dlogits", "dvalues", "dH", "dG", "dfc", "dY2",
 * "dY1", "h1", "h2", "dh1", "dh2".  SEED_E_ARG if the name is unknown for
 * this net. */
seed_status seed_learner_debug_buffer(const seed_net_spec* spec, int T, int B, void* workspace,
                                      const char* name, void** ptr_out, size_t* bytes_out);

/* ===========================================================================
 * Data-parallel communicator.  The caller broadcasts the
 * 128-byte unique id (host buffer) from rank 0 via torch.distributed.
 * NCCL is loaded at run time (libnccl.so.2); SEED_E_NCCL if unavailable.
 * ======================================================================== */
seed_status seed_comm_get_unique_id(void* id128 /* host, 128 bytes */);
seed_status seed_comm_init(const void* id128, int rank, int world, seed_comm** out);
seed_status seed_comm_destroy(seed_comm* comm);
/* In-place sum allreduce of n fp32 device values (metrics, probes). */
seed_status seed_comm_allreduce_f32(seed_comm* comm, float* data, int64_t n, void* stream);

/* Peer-memory allreduce over NVLink (H10 without NCCL; one process per GPU,
 * every pair of GPUs peer-capable).  Two-phase setup:
 *   seed_comm_peer_setup: allocates this rank's exchange buffer (2*max_floats
 *     fp32 + counters; freed by seed_comm_destroy) and writes its 64-byte CUDA
 *     IPC handle to handle_out (host);
 *   the caller all-gathers the handles (rank order) over its process group;
 *   seed_comm_peer_open: maps every peer's buffer (handles = world*64 bytes,
 *     host) and switches this comm's allreduce (n <= max_floats) to the peer
 *     kernel: copy in -> cross-GPU arrival counters -> each rank sums its 1/N
 *     slice over the ranks in rank order and writes it into every rank's
 *     buffer -> counters -> copy out.  Results are bit-identical on all ranks.
 * Waits are bounded (2 s): on timeout the kernel sets a sticky device error flag
 * that seed_comm_peer_status reports (SEED_E_NCCL) instead of hanging, and
 * poisons the (partial) result with NaN, so a learner step's global norm is
 * non-finite and the update is skipped (metrics[7] = 1).
 * All ranks must call every allreduce in the same order. */
seed_status seed_comm_peer_setup(seed_comm* comm, int64_t max_floats, void* handle_out /* 64 B */);
seed_status seed_comm_peer_open(seed_comm* comm, const void* handles /* world*64 B */);
seed_status seed_comm_peer_status(seed_comm* comm);   /* synchronizes; SEED_OK or SEED_E_NCCL */

/* ===========================================================================
 * Centralized inference (H12-H13; "load the recurrent states ... the
 * latest recurrent states are stored").
 * For each request i (actor a = actor_ids[i], unique within a call):
 *   (h, c, prev) <- table[a]; if done[i]: h = c = 0, prev = none, reward = 0
 *   forward one step with params_lowp; action = min{ j : u_i < CDF_j } over
 *   softmax(logits) (C18; A-1 if none); behaviour_logp = log pi(action);
 *   table[a] <- (h', c', action).  Rows of actors not in the call are untouched.
 * uniforms: nullable [n]; NULL = counter-based Philox4x32-10 keyed
 *   (seed, counter, actor_id) (C18).
 * store: nullable unroll store; each step is recorded (C17, C19) and completed
 *   unrolls (T+1 slots, slot T copied into slot 0 of the next) are pushed to
 *   the ready ring.
 * actor_ids: must be unique within a call.  An id outside [0, num_actors) is
 *   reported on the device, not trusted: that request reads no table row,
 *   writes nothing (table, store), and gets action_out = -1, behaviour_logp_out
 *   (and its logits_out row) = NaN.
 * ======================================================================== */
typedef struct {
  float* h;              /* [num_actors][U] */
  float* c;              /* [num_actors][U] */
  int32_t* last_action;  /* [num_actors]; < 0 = none */
  int num_actors;
} seed_state_table;

typedef struct {
  int T;                   /* unroll length; buffers hold T+1 slots           */
  int num_actors;
  uint8_t* obs;            /* [num_actors][2][T+1][obs_bytes]                 */
  int32_t* action;         /* [num_actors][2][T+1]                            */
  int32_t* prev_action;    /* [num_actors][2][T+1]                            */
  float* reward;           /* [num_actors][2][T+1]                            */
  uint8_t* done;           /* [num_actors][2][T+1]                            */
  float* behaviour_logp;   /* [num_actors][2][T+1]                            */
  float* h0;               /* [num_actors][2][U]                              */
  float* c0;               /* [num_actors][2][U]                              */
  int32_t* fill;           /* [num_actors]  slots filled in the current buffer */
  int32_t* cur;            /* [num_actors]  current buffer 0/1                */
  int32_t* ready_ring;     /* [ring_capacity] entries actor*2 + buffer        */
  int32_t* ready_count;    /* device int32[4]: {pushed total, consumed total,
                              stale unrolls assembled, short assembles}       */
  int ring_capacity;
  int32_t* gen;            /* [num_actors][2] buffer generations (zeroed)     */
  int32_t* ready_gen;      /* [ring_capacity] generation of each ring entry   */
} seed_unroll_store;
/* Lifetime (C29): each actor has two unroll buffers.  A completed unroll stays
 * valid until the actor completes its NEXT unroll (T more steps): from then on
 * its buffer is refilled.  The learner must assemble it before that, and the
 * ring must not wrap over unconsumed entries (ring_capacity >= the number of
 * unrolls pushed but not yet assembled).  seed_assemble_batch checks both on the
 * device: an entry whose buffer was reused since it was pushed (generation
 * mismatch) increments ready_count[2]; asking for more unrolls than are pushed
 * and unconsumed increments ready_count[3].  The batch is still written (the
 * counters are the report; nothing forces a host sync). */

seed_status seed_infer_workspace_size(const seed_net_spec* spec, int max_n, size_t* bytes_out);
seed_status seed_infer(const seed_net_spec* spec, const void* params_lowp, const float* params,
                       const seed_state_table* table, int n, const int32_t* actor_ids,
                       const uint8_t* obs, const float* reward, const uint8_t* done,
                       const float* uniforms, uint64_t seed, uint64_t counter,
                       int32_t* action_out, float* behaviour_logp_out, float* logits_out,
                       const seed_unroll_store* store, void* workspace, size_t ws_bytes,
                       void* stream);
/* R2D2 actors (P:591 dueling heads, P:614 per-actor
 * epsilon-greedy): the same batched step (state table, unroll store, workspace as
 * seed_infer), but the net's A+1 outputs are read as dueling heads (C35: A advantages
 * then the value), Q_a = V + A_a - mean_j A_j (written to q_out [n][A] if non-NULL),
 * and the action is epsilon-greedy with epsilon_i = eps_base^(1 + eps_alpha * i /
 * (num_actors_eps - 1)) for table row i (0.4, 7; num_actors_eps = 1: eps_base):
 * uniforms [n][2] (device, or NULL: Philox4x32-10 keyed by seed, counter and the row,
 * outputs x, y): explore when uniforms[r][0] < epsilon_i, then action =
 * floor(uniforms[r][1] * A) (clamped to A-1), else the first maximum of Q.
 * behaviour_logp_out = log(epsilon_i / A + (1 - epsilon_i) [action = greedy]).
 * SEED_E_ARG for eps_base outside [0, 1], eps_alpha < 0 or num_actors_eps < 1. */
seed_status seed_infer_eps_greedy(const seed_net_spec* spec, const void* params_lowp, const float* params,
                                  const seed_state_table* table, int n, const int32_t* actor_ids,
                                  const uint8_t* obs, const float* reward, const uint8_t* done,
                                  const float* uniforms, uint64_t seed, uint64_t counter,
                                  float eps_base, float eps_alpha, int num_actors_eps,
                                  int32_t* action_out, float* behaviour_logp_out, float* q_out,
                                  const seed_unroll_store* store, void* workspace, size_t ws_bytes,
                                  void* stream);
/* Host side of the inference batch (H12).  A seed_stager
 * is a caller-owned pool of `threads` host worker threads.  seed_stage_requests
 * packs the n requests' observations — obs_ptrs[i] (host) points to request i's
 * obs_bytes bytes wherever the transport left them — into contiguous pinned
 * staging (pinned_obs, n*obs_bytes page-locked host bytes), chunk by chunk
 * (`chunk` requests, <= 0: 128), and issues each chunk's host->device copy into
 * dev_obs on `stream` as soon as the chunk is packed, so the copies overlap the
 * packing of later chunks.  Optional metadata (all three host arrays non-NULL or
 * all NULL) goes in one copy into dev_meta (9n bytes, 16-B aligned): int32 actor
 * ids at byte 0, fp32 rewards at byte 4n, uint8 dones at byte 8n — the seed_infer
 * argument layouts.  Returns once every copy is issued; the staging must stay
 * untouched until the stream reaches them.  One call at a time per stager. */
typedef struct seed_stager seed_stager;
seed_status seed_stager_create(int threads, seed_stager** out);
seed_status seed_stager_destroy(seed_stager* stager);
seed_status seed_stage_requests(seed_stager* stager, int n, const uint8_t* const* obs_ptrs,
                                size_t obs_bytes, const int32_t* actor_ids, const float* rewards,
                                const uint8_t* dones, uint8_t* pinned_obs, uint8_t* pinned_meta,
                                uint8_t* dev_obs, uint8_t* dev_meta, int chunk, void* stream);

/* Actor transport + server-side batching ("the
 * connection from actor to learner is kept open and metadata sent only once",
 * P:136 the batching module; wire format SEEDWire v1: frames =
 * u32 LE length (of type byte + payload) | u8 type | payload; Hello 0x01 (u32
 * actor_id, u32 num_envs), StepRequest 0x02 (u32 env_id, f32 reward, u8 done, u32
 * obs_count, obs_count f32 — rounded and clamped to 0..255 bytes), ActionResponse
 * 0x03 (u32 env_id, u32 action), Error 0x00 (u16 code, u16 length, UTF-8); plus
 * StepRequest-u8 0x04 = StepRequest with obs_count uint8 pixels; max frame 16 MiB).
 * Host-only: a TCP server on 127.0.0.1:port (0 = any free port, returned in
 * *port_out) whose I/O thread accepts actors, gives each Hello num_envs consecutive
 * state-table rows (at most max_rows in all), and queues StepRequests (obs_count
 * must equal obs_bytes; one in-flight request per (actor, env), else Error +
 * close).  seed_wire_next_batch blocks until max_batch requests are queued, or the
 * oldest has waited max_wait_us, or timeout_us passes, and copies up to max_batch
 * of them in arrival order into host buffers (obs_out [n][obs_bytes], rows_out =
 * state-table rows for seed_infer's actor_ids, reward_out, done_out; *n_out may
 * be 0).  seed_wire_reply sends each request's action to its connection (exactly
 * once; SEED_E_ARG for a row with no request waiting).  stats6: batches, requests,
 * batches by size / deadline / timeout trigger, protocol errors.  The server's
 * calls are thread-safe; destroy joins the I/O thread and closes every socket. */
typedef struct seed_wire_server seed_wire_server;
seed_status seed_wire_server_create(int port, int max_batch, int max_wait_us, int obs_bytes, int max_rows,
                                    seed_wire_server** out, int* port_out);
seed_status seed_wire_server_destroy(seed_wire_server* server);
seed_status seed_wire_next_batch(seed_wire_server* server, int timeout_us, uint8_t* obs_out /* host */,
                                 int32_t* rows_out, float* reward_out, uint8_t* done_out, int* n_out);
seed_status seed_wire_reply(seed_wire_server* server, int n, const int32_t* rows /* host */,
                            const int32_t* actions /* host */);
seed_status seed_wire_server_stats(seed_wire_server* server, int64_t* stats6 /* host */,
                                   int* rows_assigned);

/* Gather B completed unrolls (entries ready_ring[consumed .. consumed+B)) into
 * the seed_batch layout buffers given in `out` (device pointers, cast away
 * const), and advance the consumed counter.  The caller must only ask for
 * unrolls already pushed (host-visible count). */
seed_status seed_assemble_batch(const seed_unroll_store* store, int obs_bytes, int lstm_units,
                                int B, const seed_batch* out, void* stream);

/* ===========================================================================
 * Versioned parameter snapshots: inference concurrent with training (SURVEY
 * §8(f) row 2; P:98, P:111 inference with the latest parameters
 * inference on cores of its own while the learner trains; S:37-42 the version
 * is ParamSnapshot.version, S:109 / S:465 single-copy semantics).
 * A single-producer (learner) / single-consumer (inference) triple buffer in
 * device memory: three slots of seed_param_snapshot_bytes() bytes each (the
 * params_lowp image, then the fp32 params), their versions, and an index word.
 * seed_param_publish (producer's stream, after seed_learner_step): copies
 *   params_lowp + params into the producer's slot, stamps version = *step,
 *   and hands the slot over with one atomic exchange.
 * seed_param_acquire (consumer's stream, before seed_infer): takes the latest
 *   handed-over slot with one atomic exchange when there is a newer one, and
 *   copies it into the consumer's private lowp_out / params_out (which
 *   seed_infer then reads) when it changed (always if force_copy != 0);
 *   *version_out (nullable, device int64) = the version now held.
 * Neither side waits for the other; a slot the consumer can read is never
 * written, so inference always runs on one whole update (never a torn one)
 * and on the newest one published before its acquire.  One producer stream and
 * one consumer stream per snapshot.  Call seed_param_snapshot_init once
 * (version -1 = nothing published yet).
 * ======================================================================== */
typedef struct {
  void* slots[3];          /* device, seed_param_snapshot_bytes() each, 16-B aligned */
  int32_t* state;          /* device int32[4] (library-private index word)        */
  int64_t* version;        /* device int64[3]: version held by each slot           */
} seed_param_snapshot;
seed_status seed_param_snapshot_bytes(const seed_net_spec* spec, size_t* slot_bytes);
seed_status seed_param_snapshot_init(seed_param_snapshot* snap, void* stream);
seed_status seed_param_publish(const seed_net_spec* spec, const seed_train_state* state,
                               seed_param_snapshot* snap, void* stream);
seed_status seed_param_acquire(const seed_net_spec* spec, seed_param_snapshot* snap,
                               void* lowp_out, float* params_out, int64_t* version_out,
                               int force_copy, void* stream);

/* ===========================================================================
 * R2D2 on SEED ("fully implementing R2D2",
 * hyper-parameters P:586-622).
 *
 * seed_r2d2_targets — n-step double-Q targets with value rescaling (P:149, P:611,
 * P:613), TD errors, sequence priorities and the importance-weighted
 * squared-TD loss gradient, one warp per sequence:
 *   h(x) = sign(x)(sqrt(|x|+1) - 1) + eps x,  h^-1 its closed-form inverse
 *   for t < T, m = min(n, T - t):  a* = argmax_a q_online[t+m][a] (first maximum)
 *     G_t = sum_{k<m} (prod_{j<k} gamma_{t+j}) r_{t+k}
 *           + (prod_{j<m} gamma_{t+j}) h^-1(q_target[t+m][a*])
 *     y_t = h(G_t);  delta_t = y_t - q_online[t][a_t]
 *   priority_b = eta max_t |delta_t| + (1 - eta) mean_t |delta_t|
 *   loss_part_b = loss_scale w_b sum_t delta_t^2 / 2;
 *   dq[b][t][a_t] = loss_scale w_b (q_online[t][a_t] - y_t), 0 elsewhere, row T zero.
 * Arguments: q_online, q_target [B][T+1][A] fp32 (rescaled values of the trained
 *   part, after burn-in); actions [B][T+1] int32; rewards, discounts [B][T]
 *   (gamma_t = gamma (1 - done_{t+1}), C5 — an episode end zeroes the rest of the
 *   window, the sequence end shortens it: reading C32); is_weights nullable [B]
 *   (1 if NULL); dq, loss_part nullable.  T, B >= 1, 2 <= A <= 4096, n >= 1 else
 *   SEED_E_SHAPE; eps > 0, 0 <= eta <= 1 else SEED_E_ARG.
 * ======================================================================== */
seed_status seed_r2d2_targets(int T, int B, int A, int n, const float* q_online,
                              const float* q_target, const int32_t* actions,
                              const float* rewards, const float* discounts, float eta,
                              float rescale_eps, const float* is_weights, float loss_scale,
                              float* y, float* delta, float* priority, float* dq,
                              float* loss_part, void* stream);

/* seed_r2d2_learner_step — one R2D2 learner update:
 *   burn-in: the sequences' stored (h0, c0) warmed over their first burn_in steps
 *      by the online and by the target network, with no gradient;
 *   trained window [B][T+1]: online and target forward passes, dueling heads read
 *     from the net's A+1 outputs (Q(a) = V + A_a - mean_j A_j; reading C35),
 *     seed_r2d2_targets (n-step double Q, value rescaling, priorities -> priorities_out,
 *     IS-weighted squared-TD gradient), the dueling / heads / core / torso backward,
 *     the optional DP allreduce (comm), global-norm clip (80) and Adam
 *     (lr 1e-4, eps 1e-3) of the online parameters; version += 1 if finite.
 * The target parameters (target_params fp32 [P] + target_lowp image) are read only;
 * the caller copies the online parameters into them every 2500 updates.
 * burn: [B][burn_in] frames (obs, prev_action, reward, done, h0 / c0 = the stored
 *   state at the sequence start); NULL iff burn_in == 0 (then train's h0 / c0).
 * train: [B][T+1] frames (obs, action, prev_action, reward, done); trained step t
 *   uses reward[t+1] and discount gamma (1 - done[t+1]) (C5).
 * is_weights: nullable [B] importance weights (seed_replay_sample).
 * metrics: device float[8] as seed_learner_step (loss in [0] and [1]).
 * Supports the conv nets (not SEED_NET_MLP). */
typedef struct {
  float discount;        /* gamma (.997)                         */
  int n;                 /* n-step (5)                           */
  float eta;             /* priority mixing (.9)                 */
  float rescale_eps;     /* value rescaling epsilon (1e-3)       */
  float loss_scale;      /* e.g. 1/(N*B*T)                              */
  float lr, beta1, beta2, eps;   /* Adam                                */
  float max_grad_norm;   /* 80                                   */
} seed_r2d2_hparams;
seed_status seed_r2d2_workspace_size(const seed_net_spec* spec, int burn_in, int T, int B,
                                     size_t* bytes_out);
seed_status seed_r2d2_learner_step(const seed_net_spec* spec, int burn_in, int T, int B,
                                   const seed_batch* burn, const seed_batch* train,
                                   const seed_train_state* online, const float* target_params,
                                   const void* target_lowp, const float* is_weights,
                                   const seed_r2d2_hparams* hp, seed_comm* comm, seed_exec* exec,
                                   void* workspace, size_t ws_bytes, float* priorities_out,
                                   float* metrics, void* stream);

/* Learner-resident prioritized sequence replay ("keep the replay buffer on
 * the learner"; priority exponent alpha P:602, importance exponent beta P:603;
 * S:287-333), entirely in HBM: a sum tree over p_i^alpha (leaves tree[C + i],
 * root tree[1]; rebuilt in fixed pairwise order after every change — exact per
 * level, deterministic), FIFO slots, and per-slot generations so that priority
 * updates for a sequence evicted since its sample are skipped.  All fields are
 * caller-owned device memory, zero-initialised before first use. */
typedef struct {
  int capacity;            /* sum-tree leaves C: power of two >= slots, C/2048 <= 2048 */
  int slots;               /* sequences held (FIFO ring)                               */
  float* tree;             /* device fp32 [2*C]                                        */
  float* max_priority;     /* device fp32 [1]: max priority seen (new sequences')     */
  int32_t* size;           /* device int32 [4]: {stored, next slot, rejected
                              priorities (negative / non-finite), 0}                  */
  int32_t* gen;            /* device int32 [slots]: generation of each slot           */
  unsigned* ticket;        /* device uint32 [1]                                       */
} seed_replay;
/* SEED_OK if the descriptor is well-formed (host check only). */
seed_status seed_replay_check(const seed_replay* replay);
/* n (<= 1024) new sequences take the next FIFO slots (evicting the oldest) at the
 * max priority seen so far (1 before any update); out_slots / out_gens (nullable
 * device [n]) receive their slots and generations — the caller then writes the
 * sequence payload into those slots. */
seed_status seed_replay_insert(const seed_replay* replay, int n, float alpha,
                               int32_t* out_slots, int32_t* out_gens, void* stream);
/* New raw priorities p (>= 0, finite) for n (<= 1024) sampled sequences; an entry
 * whose generation differs from the slot's current one (gens non-NULL) is skipped;
 * invalid priorities are skipped and counted in size[2]; the max priority is
 * raised to the largest applied p. */
seed_status seed_replay_update(const seed_replay* replay, int n, const int32_t* slots,
                               const int32_t* gens, const float* priorities, float alpha,
                               void* stream);
/* B (<= 1024) i.i.d. proportional draws: x = u * root, descend the tree (left if
 * x < left sum, else subtract it and go right); u from `uniforms` (nullable [B]) or
 * Philox4x32-10 keyed (seed) with counter (counter, draw index, 1);
 * out_weights[b] = (N P(slot))^-beta / max over the batch, N = stored sequences.
 * Requires at least one positive priority (stored > 0). */
seed_status seed_replay_sample(const seed_replay* replay, int B, float beta,
                               const float* uniforms, uint64_t seed, uint64_t counter,
                               int32_t* out_slots, int32_t* out_gens, float* out_weights,
                               void* stream);
/* dst[b] = src[slots[b]] for slot_bytes-sized records (multiple of 16, 16-B aligned
 * pointers): the sampled sequences' payload into a contiguous training batch. */
seed_status seed_replay_gather(const void* src, size_t slot_bytes, const int32_t* slots, int B,
                               void* dst, void* stream);
/* The inverse: dst[slots[b]] = src[b] (the payload of sequences just inserted). */
seed_status seed_replay_scatter(const void* src, size_t slot_bytes, const int32_t* slots, int B,
                                void* dst, void* stream);

/* ===========================================================================
 * Test / benchmark hooks (not part of the method):
 * seed_debug_gemm: D[M][N] (fp32, row-major) = A . B^T with A [M][K], B [N][K]
 * bf16 row-major (a_t / b_t != 0: A given as [K][M] / B as [K][N]), on the
 * tcgen05 engine the learner uses.  Requires K % 8 == 0, M % 8 == 0 and
 * N % 8 == 0.  splits < 0 selects the register-staged producer with |splits|
 * K splits (default: the cp.async producer).
 * ======================================================================== */
seed_status seed_debug_gemm(int M, int N, int K, const void* A, int a_t, const void* B,
                            int b_t, float* D, int bn, int splits, void* workspace,
                            void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SEED_H_ */
