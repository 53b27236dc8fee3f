"""ctypes declarations for libseed.so (include/seed.h).  Argument marshalling only."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SEED_LIB", os.path.join(HERE, "libseed.so"))

c_int, c_float, c_void_p, c_size_t = C.c_int, C.c_float, C.c_void_p, C.c_size_t
c_int64, c_uint64 = C.c_int64, C.c_uint64
P = C.POINTER


class NetSpec(C.Structure):
    _fields_ = [("kind", c_int), ("obs_h", c_int), ("obs_w", c_int), ("obs_c", c_int),
                ("num_actions", c_int), ("lstm_units", c_int), ("torso_width", c_int)]


class HParams(C.Structure):
    _fields_ = [(n, c_float) for n in ("discount", "lam", "rho_bar", "c_bar", "vf_coef",
                                       "ent_coef", "loss_scale", "lr", "beta1", "beta2", "eps",
                                       "max_grad_norm")]


class Batch(C.Structure):
    _fields_ = [(n, c_void_p) for n in ("obs", "action", "prev_action", "reward", "done",
                                        "behaviour_logp", "h0", "c0")]


class TrainState(C.Structure):
    _fields_ = [(n, c_void_p) for n in ("params", "grads", "adam_m", "adam_v", "params_lowp",
                                        "step")]


class StateTable(C.Structure):
    _fields_ = [("h", c_void_p), ("c", c_void_p), ("last_action", c_void_p),
                ("num_actors", c_int)]


class UnrollStore(C.Structure):
    _fields_ = [("T", c_int), ("num_actors", c_int)] + \
        [(n, c_void_p) for n in ("obs", "action", "prev_action", "reward", "done",
                                 "behaviour_logp", "h0", "c0", "fill", "cur", "ready_ring",
                                 "ready_count")] + [("ring_capacity", c_int), ("gen", c_void_p),
                                                    ("ready_gen", c_void_p)]


class Replay(C.Structure):
    _fields_ = [("capacity", c_int), ("slots", c_int)] + \
        [(n, c_void_p) for n in ("tree", "max_priority", "size", "gen", "ticket")]


class R2d2HParams(C.Structure):
    _fields_ = [("discount", c_float), ("n", c_int), ("eta", c_float), ("rescale_eps", c_float),
                ("loss_scale", c_float), ("lr", c_float), ("beta1", c_float), ("beta2", c_float),
                ("eps", c_float), ("max_grad_norm", c_float)]


class ParamSnapshot(C.Structure):
    _fields_ = [("slots", c_void_p * 3), ("state", c_void_p), ("version", c_void_p)]


_SIGS = {
    "seed_status_string": (C.c_char_p, [c_int]),
    "seed_abi_version": (c_int, []),
    "seed_last_cuda_error": (C.c_char_p, []),
    "seed_vtrace": (c_int, [c_int, c_int] + [c_void_p] * 6 + [c_float] * 3 +
                    [c_void_p, c_void_p, c_void_p, c_void_p]),
    "seed_net_param_count": (c_int, [P(NetSpec), P(c_int64)]),
    "seed_net_param_tensor": (c_int, [P(NetSpec), c_int, C.c_char_p, P(c_int), P(c_int64),
                                      P(c_int64)]),
    "seed_net_lowp_bytes": (c_int, [P(NetSpec), P(c_size_t)]),
    "seed_net_refresh_lowp": (c_int, [P(NetSpec), c_void_p, c_void_p, c_void_p]),
    "seed_learner_workspace_size": (c_int, [P(NetSpec), c_int, c_int, P(c_size_t)]),
    "seed_learner_step": (c_int, [P(NetSpec), c_int, c_int, P(Batch), P(TrainState),
                                  P(HParams), c_void_p, c_void_p, c_size_t, c_void_p,
                                  c_void_p]),
    "seed_exec_create": (c_int, [P(c_void_p)]),
    "seed_exec_destroy": (c_int, [c_void_p]),
    "seed_learner_step_ex": (c_int, [P(NetSpec), c_int, c_int, P(Batch), P(TrainState),
                                     P(HParams), c_void_p, c_void_p, c_void_p, c_size_t, c_void_p,
                                     c_void_p]),
    "seed_param_snapshot_bytes": (c_int, [P(NetSpec), P(c_size_t)]),
    "seed_param_snapshot_init": (c_int, [P(ParamSnapshot), c_void_p]),
    "seed_param_publish": (c_int, [P(NetSpec), P(TrainState), P(ParamSnapshot), c_void_p]),
    "seed_param_acquire": (c_int, [P(NetSpec), P(ParamSnapshot), c_void_p, c_void_p, c_void_p,
                                   c_int, c_void_p]),
    "seed_r2d2_targets": (c_int, [c_int, c_int, c_int, c_int] + [c_void_p] * 5 +
                          [c_float, c_float, c_void_p, c_float] + [c_void_p] * 6),
    "seed_r2d2_workspace_size": (c_int, [P(NetSpec), c_int, c_int, c_int, P(c_size_t)]),
    "seed_r2d2_learner_step": (c_int, [P(NetSpec), c_int, c_int, c_int, c_void_p, P(Batch),
                                       P(TrainState), c_void_p, c_void_p, c_void_p,
                                       P(R2d2HParams), c_void_p, c_void_p, c_void_p, c_size_t,
                                       c_void_p, c_void_p, c_void_p]),
    "seed_replay_check": (c_int, [P(Replay)]),
    "seed_replay_insert": (c_int, [P(Replay), c_int, c_float, c_void_p, c_void_p, c_void_p]),
    "seed_replay_update": (c_int, [P(Replay), c_int, c_void_p, c_void_p, c_void_p, c_float,
                                   c_void_p]),
    "seed_replay_sample": (c_int, [P(Replay), c_int, c_float, c_void_p, c_uint64, c_uint64,
                                   c_void_p, c_void_p, c_void_p, c_void_p]),
    "seed_replay_gather": (c_int, [c_void_p, c_size_t, c_void_p, c_int, c_void_p, c_void_p]),
    "seed_replay_scatter": (c_int, [c_void_p, c_size_t, c_void_p, c_int, c_void_p, c_void_p]),
    "seed_learner_step_traced": (c_int, [P(NetSpec), c_int, c_int, P(Batch), P(TrainState),
                                         P(HParams), c_void_p, c_void_p, c_size_t, c_void_p,
                                         c_void_p, P(c_void_p), c_int, P(C.c_char_p), P(c_int),
                                         P(c_int), c_void_p]),
    "seed_learner_outputs": (c_int, [P(NetSpec), c_int, c_int, c_void_p, P(c_void_p),
                                     P(c_void_p), P(c_void_p), P(c_void_p)]),
    "seed_learner_debug_buffer": (c_int, [P(NetSpec), c_int, c_int, c_void_p, C.c_char_p,
                                          P(c_void_p), P(c_size_t)]),
    "seed_comm_get_unique_id": (c_int, [c_void_p]),
    "seed_comm_init": (c_int, [c_void_p, c_int, c_int, P(c_void_p)]),
    "seed_comm_destroy": (c_int, [c_void_p]),
    "seed_comm_allreduce_f32": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "seed_comm_peer_setup": (c_int, [c_void_p, c_int64, c_void_p]),
    "seed_comm_peer_open": (c_int, [c_void_p, c_void_p]),
    "seed_comm_peer_status": (c_int, [c_void_p]),
    "seed_infer_workspace_size": (c_int, [P(NetSpec), c_int, P(c_size_t)]),
    "seed_infer": (c_int, [P(NetSpec), c_void_p, c_void_p, P(StateTable), c_int, c_void_p,
                           c_void_p, c_void_p, c_void_p, c_void_p, c_uint64, c_uint64,
                           c_void_p, c_void_p, c_void_p, P(UnrollStore), c_void_p, c_size_t,
                           c_void_p]),
    "seed_infer_eps_greedy": (c_int, [P(NetSpec), c_void_p, c_void_p, P(StateTable), c_int, c_void_p,
                                      c_void_p, c_void_p, c_void_p, c_void_p, c_uint64, c_uint64,
                                      c_float, c_float, c_int,
                                      c_void_p, c_void_p, c_void_p, P(UnrollStore), c_void_p, c_size_t,
                                      c_void_p]),
    "seed_stager_create": (c_int, [c_int, P(c_void_p)]),
    "seed_stager_destroy": (c_int, [c_void_p]),
    "seed_stage_requests": (c_int, [c_void_p, c_int, c_void_p, c_size_t, c_void_p, c_void_p, c_void_p,
                                    c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p]),
    "seed_assemble_batch": (c_int, [P(UnrollStore), c_int, c_int, c_int, P(Batch), c_void_p]),
    "seed_wire_server_create": (c_int, [c_int, c_int, c_int, c_int, c_int, P(c_void_p), P(c_int)]),
    "seed_wire_server_destroy": (c_int, [c_void_p]),
    "seed_wire_next_batch": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p, P(c_int)]),
    "seed_wire_reply": (c_int, [c_void_p, c_int, c_void_p, c_void_p]),
    "seed_wire_server_stats": (c_int, [c_void_p, c_void_p, P(c_int)]),
    "seed_debug_gemm": (c_int, [c_int, c_int, c_int, c_void_p, c_int, c_void_p, c_int,
                                c_void_p, c_int, c_int, c_void_p, c_void_p]),
}

EXPORTED = tuple(_SIGS)

_lib = None


class SeedError(RuntimeError):
    pass


def load():
    """Load the in-tree libseed.so.  Fails loudly when it is missing: there is
    no CPU or library fallback for any call."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SeedError(f"{LIB_PATH} is not built; run __graft_entry__.build() "
                            "(python -m paper_1910_06591_b200.build)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(status, what=""):
    if status != 0:
        msg = load().seed_status_string(status).decode()
        if status == 4:   # SEED_E_CUDA: the CUDA error behind it
            msg += f" [{load().seed_last_cuda_error().decode()}]"
        raise SeedError(f"{what}: {msg} ({status})")
