"""Python binding of the libseed C ABI (include/seed.h) over torch tensors.

Marshalling only: validates dtype / device / contiguity, passes raw pointers
and the current CUDA stream to the library.  No computation happens here.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

from . import _lib as L

NET_MLP, NET_ATARI_SHALLOW, NET_IMPALA_DEEP, NET_GFOOTBALL = 0, 1, 2, 3


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _need(t, dtype, name, device=True):
    if t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")
    if device and not t.is_cuda:
        raise ValueError(f"{name}: must be a CUDA tensor")


# --------------------------------------------------------------------------- V-trace
def vtrace(behaviour_logp, target_logp, rewards, discounts, values, bootstrap, rho_bar=1.0,
           c_bar=1.0, lam=1.0, vs=None, pg_advantages=None, nonfinite_flag=None, stream=None):
    """seed_vtrace: [B][T] float32 CUDA tensors -> (vs, pg_advantages)."""
    B, T = values.shape
    for n, t in (("behaviour_logp", behaviour_logp), ("target_logp", target_logp),
                 ("rewards", rewards), ("discounts", discounts), ("values", values)):
        _need(t, torch.float32, n)
        if tuple(t.shape) != (B, T):
            raise ValueError(f"{n}: shape {tuple(t.shape)} != {(B, T)}")
    _need(bootstrap, torch.float32, "bootstrap")
    if vs is None:
        vs = torch.empty_like(values)
    if pg_advantages is None:
        pg_advantages = torch.empty_like(values)
    st = L.load().seed_vtrace(T, B, _ptr(behaviour_logp), _ptr(target_logp), _ptr(rewards),
                              _ptr(discounts), _ptr(values), _ptr(bootstrap), float(rho_bar),
                              float(c_bar), float(lam), _ptr(vs), _ptr(pg_advantages),
                              _ptr(nonfinite_flag), _stream(stream))
    L.check(st, "seed_vtrace")
    return vs, pg_advantages


# --------------------------------------------------------------------------- R2D2
def r2d2_targets(q_online, q_target, actions, rewards, discounts, n=5, eta=0.9, rescale_eps=1e-3,
                 is_weights=None, loss_scale=1.0, want_grad=False, stream=None):
    """seed_r2d2_targets: q_online / q_target [B][T+1][A], actions [B][T+1] int32,
    rewards / discounts [B][T] -> (y, delta [B][T], priority [B], dq or None,
    loss_part or None)."""
    B, T1, A = q_online.shape
    T = T1 - 1
    _need(q_online, torch.float32, "q_online")
    _need(q_target, torch.float32, "q_target")
    _need(actions, torch.int32, "actions")
    _need(rewards, torch.float32, "rewards")
    _need(discounts, torch.float32, "discounts")
    if tuple(q_target.shape) != (B, T1, A) or tuple(actions.shape) != (B, T1) or \
            tuple(rewards.shape) != (B, T) or tuple(discounts.shape) != (B, T):
        raise ValueError("r2d2_targets: shapes")
    dev = q_online.device
    y = torch.empty(B, T, device=dev)
    delta = torch.empty(B, T, device=dev)
    prio = torch.empty(B, device=dev)
    dq = torch.empty(B, T1, A, device=dev) if want_grad else None
    loss = torch.empty(B, device=dev) if want_grad else None
    if is_weights is not None:
        _need(is_weights, torch.float32, "is_weights")
    L.check(L.load().seed_r2d2_targets(T, B, A, int(n), _ptr(q_online), _ptr(q_target),
                                       _ptr(actions), _ptr(rewards), _ptr(discounts), float(eta),
                                       float(rescale_eps), _ptr(is_weights), float(loss_scale),
                                       _ptr(y), _ptr(delta), _ptr(prio), _ptr(dq), _ptr(loss),
                                       _stream(stream)), "seed_r2d2_targets")
    return y, delta, prio, dq, loss


class PrioritizedReplay:
    """Learner-resident prioritized sequence replay in HBM (include/seed.h
    seed_replay_*): `slots` sequences of `record_bytes` each (the payload lives in
    self.data, one row per slot), a sum tree over p^alpha."""

    def __init__(self, slots, record_bytes, alpha=0.9, beta=0.6, device="cuda"):
        C = 1
        while C < slots:
            C *= 2
        self.slots, self.capacity, self.alpha, self.beta = slots, C, alpha, beta
        self.record_bytes = record_bytes
        z = lambda n, dt: torch.zeros(n, dtype=dt, device=device)
        self.tree = z(2 * C, torch.float32)
        self.max_priority = z(1, torch.float32)
        self.size = z(4, torch.int32)
        self.gen = z(slots, torch.int32)
        self.ticket = z(1, torch.int32)
        self.data = torch.zeros(slots, record_bytes, dtype=torch.uint8, device=device)
        self.c = L.Replay(C, slots, _ptr(self.tree), _ptr(self.max_priority), _ptr(self.size),
                          _ptr(self.gen), _ptr(self.ticket))
        L.check(L.load().seed_replay_check(self._cref()), "seed_replay_check")

    def _cref(self):
        return C.byref(self.c)

    def insert(self, records, stream=None):
        """records: uint8 [n][record_bytes] on the device -> (slots, gens)."""
        n = records.shape[0]
        slots = torch.empty(n, dtype=torch.int32, device=records.device)
        gens = torch.empty(n, dtype=torch.int32, device=records.device)
        L.check(L.load().seed_replay_insert(self._cref(), n, float(self.alpha), _ptr(slots),
                                            _ptr(gens), _stream(stream)), "seed_replay_insert")
        _need(records, torch.uint8, "records")
        L.check(L.load().seed_replay_scatter(_ptr(records), self.record_bytes, _ptr(slots), n,
                                             _ptr(self.data), _stream(stream)), "seed_replay_scatter")
        return slots, gens

    def update(self, slots, gens, priorities, stream=None):
        L.check(L.load().seed_replay_update(self._cref(), slots.numel(), _ptr(slots), _ptr(gens),
                                            _ptr(priorities), float(self.alpha), _stream(stream)),
                "seed_replay_update")

    def sample(self, B, uniforms=None, seed=0, counter=0, stream=None):
        dev = self.tree.device
        slots = torch.empty(B, dtype=torch.int32, device=dev)
        gens = torch.empty(B, dtype=torch.int32, device=dev)
        w = torch.empty(B, dtype=torch.float32, device=dev)
        L.check(L.load().seed_replay_sample(self._cref(), B, float(self.beta), _ptr(uniforms), seed,
                                            counter, _ptr(slots), _ptr(gens), _ptr(w),
                                            _stream(stream)), "seed_replay_sample")
        return slots, gens, w

    def gather(self, slots, out=None, stream=None):
        B = slots.numel()
        out = out if out is not None else torch.empty(B, self.record_bytes, dtype=torch.uint8,
                                                      device=self.data.device)
        L.check(L.load().seed_replay_gather(_ptr(self.data), self.record_bytes, _ptr(slots), B,
                                            _ptr(out), _stream(stream)), "seed_replay_gather")
        return out


def debug_gemm(A, B, a_t=False, b_t=False, bn=64, splits=1, out=None, stream=None):
    """Test hook: D = A @ B^T on the tcgen05 engine (bf16 in, fp32 out)."""
    _need(A, torch.bfloat16, "A")
    _need(B, torch.bfloat16, "B")
    M, K = (A.shape[1], A.shape[0]) if a_t else A.shape
    N = B.shape[1] if b_t else B.shape[0]
    D = out if out is not None else torch.empty(M, N, device=A.device, dtype=torch.float32)
    ws = torch.empty(max(abs(splits), 1) * M * N, device=A.device, dtype=torch.float32) \
        if abs(splits) > 1 else None
    st = L.load().seed_debug_gemm(M, N, K, _ptr(A), int(a_t), _ptr(B), int(b_t), _ptr(D), bn,
                                  splits, _ptr(ws), _stream(stream))
    L.check(st, "seed_debug_gemm")
    return D


# --------------------------------------------------------------------------- networks
@dataclass
class NetSpec:
    kind: int
    obs_h: int
    obs_w: int
    obs_c: int
    num_actions: int
    lstm_units: int = 256
    torso_width: int = 1

    def c(self):
        return L.NetSpec(self.kind, self.obs_h, self.obs_w, self.obs_c, self.num_actions,
                         self.lstm_units, self.torso_width)

    @property
    def obs_shape(self):
        return (self.obs_h * self.obs_w * self.obs_c,) if self.kind == NET_MLP else \
            (self.obs_h, self.obs_w, self.obs_c)

    @property
    def obs_dtype(self):
        return torch.float32 if self.kind == NET_MLP else torch.uint8


def spec_for_config(cfg):
    """BASELINE.json configs -> NetSpec (c1..c5; c4m / c4l the larger Football SMMs)."""
    return {
        "c1": NetSpec(NET_MLP, 1, 1, 16, 4, 0),
        "c2": NetSpec(NET_ATARI_SHALLOW, 84, 84, 4, 18, 256),
        "c3": NetSpec(NET_IMPALA_DEEP, 72, 96, 3, 15, 256),
        "c4": NetSpec(NET_GFOOTBALL, 72, 96, 16, 19, 256),
        "c5": NetSpec(NET_ATARI_SHALLOW, 84, 84, 4, 18, 256),
        # Football SMM Medium 120x90 / Large 144x108 (W x H)
        "c4m": NetSpec(NET_GFOOTBALL, 90, 120, 16, 19, 256),
        "c4l": NetSpec(NET_GFOOTBALL, 108, 144, 16, 19, 256),
        # DMLab ResNet "Medium 2x" filters (32, 64, 64)
        "c3m": NetSpec(NET_IMPALA_DEEP, 72, 96, 3, 15, 256, 2),
        # DMLab ResNet "Large 4x" filters (64, 128, 128)
        "c3l": NetSpec(NET_IMPALA_DEEP, 72, 96, 3, 15, 256, 4),
    }[cfg]


def net_param_count(spec):
    n = C.c_int64()
    L.check(L.load().seed_net_param_count(C.byref(spec.c()), C.byref(n)), "param_count")
    return n.value


def net_param_layout(spec):
    """[(name, shape)] in flat order, as the library defines it."""
    out = []
    lib = L.load()
    i = 0
    while True:
        name = C.create_string_buffer(64)
        nd = C.c_int()
        shape = (C.c_int64 * 4)()
        off = C.c_int64()
        st = lib.seed_net_param_tensor(C.byref(spec.c()), i, name, C.byref(nd), shape,
                                       C.byref(off))
        if st != 0:
            break
        out.append((name.value.decode(), tuple(shape[k] for k in range(nd.value))))
        i += 1
    return out


@dataclass
class HParams:
    discount: float = 0.99
    lam: float = 1.0
    rho_bar: float = 1.0
    c_bar: float = 1.0
    vf_coef: float = 0.5
    ent_coef: float = 0.01
    loss_scale: float = 1.0
    lr: float = 3e-4
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-5
    max_grad_norm: float = 40.0

    def c(self):
        return L.HParams(self.discount, self.lam, self.rho_bar, self.c_bar, self.vf_coef,
                         self.ent_coef, self.loss_scale, self.lr, self.beta1, self.beta2,
                         self.eps, self.max_grad_norm)

    def as_oracle(self):
        """The same hyper-parameters as the fp32 values the ABI receives (the
        oracle gets the same input bytes as the kernels)."""
        import struct
        f = lambda x: struct.unpack("f", struct.pack("f", x))[0]
        return dict(discount=f(self.discount), rho_bar=f(self.rho_bar), c_bar=f(self.c_bar),
                    vf_coef=f(self.vf_coef), ent_coef=f(self.ent_coef),
                    loss_scale=f(self.loss_scale), lr=f(self.lr), beta1=f(self.beta1),
                    beta2=f(self.beta2), eps=f(self.eps), max_grad_norm=f(self.max_grad_norm),
                    **{"lambda": f(self.lam)})


class Comm:
    """NCCL communicator owned by libseed; the unique id travels over the
    caller's torch.distributed process group (gloo or nccl)."""

    def __init__(self, rank, world, group=None):
        import torch.distributed as dist
        lib = L.load()
        buf = (C.c_uint8 * 128)()
        if rank == 0:
            L.check(lib.seed_comm_get_unique_id(buf), "seed_comm_get_unique_id")
        obj = [bytes(buf)]
        dist.broadcast_object_list(obj, src=0, group=group)
        C.memmove(buf, obj[0], 128)
        h = C.c_void_p()
        L.check(lib.seed_comm_init(buf, rank, world, C.byref(h)), "seed_comm_init")
        self.handle = h
        self.rank, self.world = rank, world
        self.group = group
        self.peer = False

    def enable_peer(self, max_floats):
        """Switch this communicator's allreduce to the peer-memory NVLink kernel
        (include/seed.h seed_comm_peer_*): exchange the CUDA IPC handles of every
        rank's buffer over the process group.  Collective; returns False (NCCL
        stays in use) when the GPUs cannot map each other's memory."""
        import torch.distributed as dist
        if self.world == 1 or self.peer:
            return self.peer
        lib = L.load()
        buf = (C.c_uint8 * 64)()
        ok = lib.seed_comm_peer_setup(self.handle, int(max_floats), buf) == 0
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(buf) if ok else None, group=self.group)
        if not all(h is not None for h in handles):
            return False
        allh = (C.c_uint8 * (64 * self.world)).from_buffer_copy(b"".join(handles))
        st = lib.seed_comm_peer_open(self.handle, allh)
        oks = [None] * self.world
        dist.all_gather_object(oks, st == 0, group=self.group)
        if not all(oks):
            raise L.SeedError(f"seed_comm_peer_open failed on some rank ({st})")
        self.peer = True
        return True

    def peer_status(self):
        L.check(L.load().seed_comm_peer_status(self.handle), "peer allreduce")

    def allreduce_(self, t, stream=None):
        _need(t, torch.float32, "allreduce buffer")
        L.check(L.load().seed_comm_allreduce_f32(self.handle, _ptr(t), t.numel(),
                                                 _stream(stream)), "allreduce")
        return t

    def close(self):
        if self.handle:
            L.load().seed_comm_destroy(self.handle)
            self.handle = None


class Learner:
    """Device-resident train state (fp32 master params, Adam moments, bf16
    operand image, version counter) + workspace for seed_learner_step."""

    def __init__(self, spec, T, B, params, hp=None, comm=None, device="cuda"):
        lib = L.load()
        self.spec, self.T, self.B = spec, T, B
        self.hp = hp or HParams()
        self.comm = comm
        n = net_param_count(spec)
        # opt-in peer-memory allreduce (NCCL measured faster inside the step);
        # SEED_PEER_MAX caps the bucket size (floats) it takes, larger buckets stay on NCCL
        if comm is not None and comm.world > 1 and os.environ.get("SEED_PEER", "0") == "1":
            comm.enable_peer(min(n, int(os.environ.get("SEED_PEER_MAX", n))))
        params = torch.as_tensor(params, dtype=torch.float32).reshape(-1)
        if params.numel() != n:
            raise ValueError(f"params has {params.numel()} values, net needs {n}")
        self.params = params.to(device).contiguous()
        self.grads = torch.zeros_like(self.params)
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        nb = C.c_size_t()
        L.check(lib.seed_net_lowp_bytes(C.byref(spec.c()), C.byref(nb)), "lowp_bytes")
        self.lowp = torch.zeros(max(nb.value, 16), dtype=torch.uint8, device=device)
        self.step_counter = torch.zeros(1, dtype=torch.int64, device=device)
        L.check(lib.seed_learner_workspace_size(C.byref(spec.c()), T, B, C.byref(nb)),
                "learner_workspace_size")
        self.ws = torch.empty(max(nb.value, 16), dtype=torch.uint8, device=device)
        self.metrics = torch.zeros(8, dtype=torch.float32, device=device)
        self._spec_c = spec.c()
        # caller-owned execution context (second stream + fork/join events) on this device
        h = C.c_void_p()
        with torch.cuda.device(self.params.device):
            L.check(lib.seed_exec_create(C.byref(h)), "seed_exec_create")
        self._exec = h
        self.refresh_lowp()

    def __del__(self):
        h = getattr(self, "_exec", None)
        if h is not None and h.value:
            try:
                L.load().seed_exec_destroy(h)
            except Exception:  # noqa: BLE001 (interpreter shutdown)
                pass
            self._exec = None

    def refresh_lowp(self, stream=None):
        L.check(L.load().seed_net_refresh_lowp(C.byref(self._spec_c), _ptr(self.params),
                                               _ptr(self.lowp), _stream(stream)), "refresh_lowp")

    def _batch(self, batch):
        B, T1 = self.B, self.T + 1
        _need(batch["obs"], self.spec.obs_dtype, "obs")
        if tuple(batch["obs"].shape[:2]) != (B, T1):
            raise ValueError("obs must be [B][T+1][...]")
        for k, dt in (("action", torch.int32), ("prev_action", torch.int32),
                      ("reward", torch.float32), ("done", torch.uint8),
                      ("behaviour_logp", torch.float32)):
            _need(batch[k], dt, k)
            if tuple(batch[k].shape) != (B, T1):
                raise ValueError(f"{k} must be [B][T+1]")
        h0 = batch.get("h0")
        c0 = batch.get("c0")
        if self.spec.lstm_units > 0:
            _need(h0, torch.float32, "h0")
            _need(c0, torch.float32, "c0")
        return L.Batch(*(_ptr(batch.get(k)) for k in ("obs", "action", "prev_action", "reward",
                                                      "done", "behaviour_logp", "h0", "c0")))

    def _train_state(self):
        return L.TrainState(_ptr(self.params), _ptr(self.grads), _ptr(self.m), _ptr(self.v),
                            _ptr(self.lowp), _ptr(self.step_counter))

    def step(self, batch, stream=None):
        """One seed_learner_step_ex (asynchronous); returns the device metrics[8]."""
        cb = self._batch(batch)
        ts = self._train_state()
        hp = self.hp.c()
        st = L.load().seed_learner_step_ex(C.byref(self._spec_c), self.T, self.B, C.byref(cb),
                                           C.byref(ts), C.byref(hp),
                                           self.comm.handle if self.comm else None, self._exec,
                                           _ptr(self.ws), self.ws.numel(), _ptr(self.metrics),
                                           _stream(stream))
        L.check(st, "seed_learner_step_ex")
        return self.metrics

    def publish(self, snapshot, stream=None):
        """seed_param_publish: hand the current parameters (version = step counter)
        to a ParamSnapshot's consumer, on `stream` after the step."""
        ts = self._train_state()
        L.check(L.load().seed_param_publish(C.byref(self._spec_c), C.byref(ts),
                                            C.byref(snapshot.c), _stream(stream)),
                "seed_param_publish")

    def debug_buffer(self, name, dtype, shape):
        """Test hook: a torch view of an internal workspace buffer (seed_learner_debug_buffer)."""
        ptr, nb = C.c_void_p(), C.c_size_t()
        L.check(L.load().seed_learner_debug_buffer(C.byref(self._spec_c), self.T, self.B,
                                                   _ptr(self.ws), name.encode(), C.byref(ptr),
                                                   C.byref(nb)), f"debug_buffer {name}")
        off = ptr.value - self.ws.data_ptr()
        return self.ws[off:off + nb.value].view(dtype).view(*shape)

    def outputs(self):
        """Views (logits, values, vs, pg_adv) into the workspace after a step."""
        ptrs = [C.c_void_p() for _ in range(4)]
        L.check(L.load().seed_learner_outputs(C.byref(self._spec_c), self.T, self.B,
                                              _ptr(self.ws), *[C.byref(p) for p in ptrs]),
                "learner_outputs")
        B, T1, A = self.B, self.T + 1, self.spec.num_actions
        base = self.ws.data_ptr()
        flat = self.ws.view(torch.float32) if self.ws.numel() % 4 == 0 else None

        def view(p, shape):
            off = (p.value - base) // 4
            n = 1
            for s in shape:
                n *= s
            return flat[off:off + n].view(*shape)
        return (view(ptrs[0], (B, T1, A)), view(ptrs[1], (B, T1)), view(ptrs[2], (B, T1 - 1)),
                view(ptrs[3], (B, T1 - 1)))


@dataclass
class R2d2HParams:
    """R2D2 hyper-parameters (P:586-622 table r2d2_params)."""
    discount: float = 0.997
    n: int = 5
    eta: float = 0.9
    rescale_eps: float = 1e-3
    loss_scale: float = 1.0
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-3
    max_grad_norm: float = 80.0

    def c(self):
        return L.R2d2HParams(self.discount, int(self.n), self.eta, self.rescale_eps,
                             self.loss_scale, self.lr, self.beta1, self.beta2, self.eps,
                             self.max_grad_norm)


class R2d2Learner(Learner):
    """Online network train state (Learner) + the target network's parameters
    (fp32 + bf16 image) and the workspace of seed_r2d2_learner_step."""

    def __init__(self, spec, burn_in, T, B, params, hp=None, comm=None, device="cuda"):
        super().__init__(spec, T, B, params, HParams(), comm=comm, device=device)
        self.burn_in = burn_in
        self.r2hp = hp or R2d2HParams()
        self.target_params = self.params.clone()
        self.target_lowp = self.lowp.clone()
        nb = C.c_size_t()
        L.check(L.load().seed_r2d2_workspace_size(C.byref(spec.c()), burn_in, T, B, C.byref(nb)),
                "seed_r2d2_workspace_size")
        self.ws = torch.empty(max(nb.value, 16), dtype=torch.uint8, device=device)
        self.priorities = torch.zeros(B, dtype=torch.float32, device=device)

    def sync_target(self, stream=None):
        """The target network takes the online parameters (every 2500 updates)."""
        self.target_params.copy_(self.params)
        self.target_lowp.copy_(self.lowp)

    def step(self, train, burn=None, is_weights=None, stream=None):
        """One seed_r2d2_learner_step; returns (metrics[8], priorities[B])."""
        ct = self._batch_r2d2(train, self.T + 1, need_h0=self.burn_in == 0)
        cb = self._batch_r2d2(burn, self.burn_in, need_h0=True) if self.burn_in > 0 else None
        ts = self._train_state()
        hp = self.r2hp.c()
        if is_weights is not None:
            _need(is_weights, torch.float32, "is_weights")
        st = L.load().seed_r2d2_learner_step(
            C.byref(self._spec_c), self.burn_in, self.T, self.B,
            C.byref(cb) if cb is not None else None, C.byref(ct), C.byref(ts),
            _ptr(self.target_params), _ptr(self.target_lowp), _ptr(is_weights), C.byref(hp),
            self.comm.handle if self.comm else None, self._exec, _ptr(self.ws), self.ws.numel(),
            _ptr(self.priorities), _ptr(self.metrics), _stream(stream))
        L.check(st, "seed_r2d2_learner_step")
        return self.metrics, self.priorities

    def _batch_r2d2(self, b, T1, need_h0):
        _need(b["obs"], self.spec.obs_dtype, "obs")
        if tuple(b["obs"].shape[:2]) != (self.B, T1):
            raise ValueError(f"obs must be [B][{T1}][...]")
        for k, dt in (("action", torch.int32), ("prev_action", torch.int32),
                      ("reward", torch.float32), ("done", torch.uint8)):
            if k in b:
                _need(b[k], dt, k)
        if need_h0:
            _need(b["h0"], torch.float32, "h0")
            _need(b["c0"], torch.float32, "c0")
        return L.Batch(*(_ptr(b.get(k)) for k in ("obs", "action", "prev_action", "reward", "done",
                                                  "behaviour_logp", "h0", "c0")))


class ParamSnapshot:
    """Device triple buffer for versioned parameter publication (include/seed.h
    seed_param_*): one producer (Learner.publish) and one consumer
    (InferenceServer with snapshot=...)."""

    def __init__(self, spec, device="cuda", stream=None):
        lib = L.load()
        nb = C.c_size_t()
        L.check(lib.seed_param_snapshot_bytes(C.byref(spec.c()), C.byref(nb)), "snapshot_bytes")
        self.slots = [torch.zeros(nb.value, dtype=torch.uint8, device=device) for _ in range(3)]
        self.state = torch.zeros(4, dtype=torch.int32, device=device)
        self.version = torch.zeros(3, dtype=torch.int64, device=device)
        self.c = L.ParamSnapshot((C.c_void_p * 3)(*[t.data_ptr() for t in self.slots]),
                                 _ptr(self.state), _ptr(self.version))
        L.check(lib.seed_param_snapshot_init(C.byref(self.c), _stream(stream)), "snapshot_init")


class InferenceServer:
    """Centralized batched inference (seed_infer) with the per-actor recurrent
    state table and the device unroll store."""

    def __init__(self, spec, num_actors, max_n, learner=None, T=None, ring_capacity=None,
                 device="cuda", snapshot=None):
        lib = L.load()
        self.spec, self.num_actors, self.max_n = spec, num_actors, max_n
        U = max(spec.lstm_units, 1)
        self.h = torch.zeros(num_actors, U, dtype=torch.float32, device=device)
        self.c = torch.zeros(num_actors, U, dtype=torch.float32, device=device)
        self.last_action = torch.full((num_actors,), -1, dtype=torch.int32, device=device)
        self.table = L.StateTable(_ptr(self.h), _ptr(self.c), _ptr(self.last_action), num_actors)
        nb = C.c_size_t()
        L.check(lib.seed_infer_workspace_size(C.byref(spec.c()), max_n, C.byref(nb)),
                "infer_workspace_size")
        self.ws = torch.empty(max(nb.value, 16), dtype=torch.uint8, device=device)
        self.learner = learner
        self._spec_c = spec.c()
        # concurrent serving: a private copy of the latest published parameters,
        # refreshed from the snapshot at the start of every call
        self.snapshot = snapshot
        if snapshot is not None:
            nb = C.c_size_t()
            L.check(lib.seed_net_lowp_bytes(C.byref(spec.c()), C.byref(nb)), "lowp_bytes")
            self.lowp = torch.zeros(max(nb.value, 16), dtype=torch.uint8, device=device)
            self.params = torch.zeros(net_param_count(spec), dtype=torch.float32, device=device)
            self.version = torch.full((1,), -1, dtype=torch.int64, device=device)
        self.store = None
        if T is not None:
            self._make_store(T, ring_capacity or 4 * num_actors, device)

    def _make_store(self, T, cap, device):
        NA, T1, U = self.num_actors, T + 1, max(self.spec.lstm_units, 1)
        obs_bytes = 1
        for s in self.spec.obs_shape:
            obs_bytes *= s
        self.obs_bytes = obs_bytes
        z = lambda *shape, dt: torch.zeros(*shape, dtype=dt, device=device)
        self.st = dict(obs=z(NA, 2, T1, obs_bytes, dt=torch.uint8),
                       action=z(NA, 2, T1, dt=torch.int32), prev_action=z(NA, 2, T1, dt=torch.int32),
                       reward=z(NA, 2, T1, dt=torch.float32), done=z(NA, 2, T1, dt=torch.uint8),
                       behaviour_logp=z(NA, 2, T1, dt=torch.float32),
                       h0=z(NA, 2, U, dt=torch.float32), c0=z(NA, 2, U, dt=torch.float32),
                       fill=z(NA, dt=torch.int32), cur=z(NA, dt=torch.int32),
                       ready_ring=z(cap, dt=torch.int32), ready_count=z(4, dt=torch.int32),
                       gen=z(NA, 2, dt=torch.int32), ready_gen=z(cap, dt=torch.int32))
        s = self.st
        self.T = T
        self.store = L.UnrollStore(T, NA, *(_ptr(s[k]) for k in (
            "obs", "action", "prev_action", "reward", "done", "behaviour_logp", "h0", "c0",
            "fill", "cur", "ready_ring", "ready_count")), cap, _ptr(s["gen"]), _ptr(s["ready_gen"]))

    def infer(self, actor_ids, obs, reward, done, uniforms=None, seed=0, counter=0,
              action_out=None, blp_out=None, logits_out=None, stream=None):
        n = actor_ids.numel()
        if n > self.max_n:
            raise ValueError("n > max_n")
        _need(actor_ids, torch.int32, "actor_ids")
        _need(obs, torch.uint8, "obs")
        _need(reward, torch.float32, "reward")
        _need(done, torch.uint8, "done")
        if uniforms is not None:
            _need(uniforms, torch.float32, "uniforms")
        dev = actor_ids.device
        a = action_out if action_out is not None else torch.empty(n, dtype=torch.int32, device=dev)
        blp = blp_out if blp_out is not None else torch.empty(n, dtype=torch.float32, device=dev)
        lib = L.load()
        if self.snapshot is not None:
            L.check(lib.seed_param_acquire(C.byref(self._spec_c), C.byref(self.snapshot.c),
                                           _ptr(self.lowp), _ptr(self.params), _ptr(self.version),
                                           0, _stream(stream)), "seed_param_acquire")
            lowp, params = self.lowp, self.params
        else:
            lowp, params = self.learner.lowp, self.learner.params
        st = lib.seed_infer(C.byref(self._spec_c), _ptr(lowp), _ptr(params),
                                 C.byref(self.table), n, _ptr(actor_ids), _ptr(obs), _ptr(reward),
                                 _ptr(done), _ptr(uniforms), seed, counter, _ptr(a), _ptr(blp),
                                 _ptr(logits_out), C.byref(self.store) if self.store else None,
                                 _ptr(self.ws), self.ws.numel(), _stream(stream))
        L.check(st, "seed_infer")
        return a, blp

    def infer_eps_greedy(self, actor_ids, obs, reward, done, uniforms=None, seed=0, counter=0,
                         eps_base=0.4, eps_alpha=7.0, num_actors_eps=None, action_out=None,
                         blp_out=None, q_out=None, stream=None):
        """R2D2 actors (seed_infer_eps_greedy): dueling Q from the net's
        A+1 outputs, per-actor epsilon-greedy; uniforms [n][2] (explore, action) or
        None (Philox).  num_actors_eps defaults to the state table's actor count."""
        n = actor_ids.numel()
        if n > self.max_n:
            raise ValueError("n > max_n")
        _need(actor_ids, torch.int32, "actor_ids")
        _need(obs, torch.uint8, "obs")
        _need(reward, torch.float32, "reward")
        _need(done, torch.uint8, "done")
        if uniforms is not None:
            _need(uniforms, torch.float32, "uniforms")
        dev = actor_ids.device
        a = action_out if action_out is not None else torch.empty(n, dtype=torch.int32, device=dev)
        blp = blp_out if blp_out is not None else torch.empty(n, dtype=torch.float32, device=dev)
        lib = L.load()
        if self.snapshot is not None:
            L.check(lib.seed_param_acquire(C.byref(self._spec_c), C.byref(self.snapshot.c),
                                           _ptr(self.lowp), _ptr(self.params), _ptr(self.version),
                                           0, _stream(stream)), "seed_param_acquire")
            lowp, params = self.lowp, self.params
        else:
            lowp, params = self.learner.lowp, self.learner.params
        st = lib.seed_infer_eps_greedy(
            C.byref(self._spec_c), _ptr(lowp), _ptr(params), C.byref(self.table), n, _ptr(actor_ids),
            _ptr(obs), _ptr(reward), _ptr(done), _ptr(uniforms), seed, counter, float(eps_base),
            float(eps_alpha), int(num_actors_eps or self.num_actors), _ptr(a), _ptr(blp), _ptr(q_out),
            C.byref(self.store) if self.store else None, _ptr(self.ws), self.ws.numel(), _stream(stream))
        L.check(st, "seed_infer_eps_greedy")
        return a, blp

    def stage_requests(self, obs_list, actor_ids, rewards, dones, threads=8, chunk=128,
                       stream=None, _ptrs=None):
        if getattr(self, "_stager", None) is None:
            h = C.c_void_p()
            L.check(L.load().seed_stager_create(threads, C.byref(h)), "seed_stager_create")
            self._stager = h
        return self._stage(obs_list, actor_ids, rewards, dones, chunk, stream, _ptrs)

    def __del__(self):
        h = getattr(self, "_stager", None)
        if h is not None and h.value:
            try:
                L.load().seed_stager_destroy(h)
            except Exception:  # noqa: BLE001
                pass
            self._stager = None

    def stage_requests_table(self, table, actor_ids, rewards, dones, threads=8, chunk=128,
                             stream=None):
        """stage_requests for frames held in one host table [num_actors][obs_bytes]
        (e.g. each actor's latest frame): request i's frame is table[actor_ids[i]].
        The n frame pointers are computed vectorised (no per-request Python work)."""
        import numpy as np
        ids = np.ascontiguousarray(actor_ids, np.int32)
        if table.ndim != 2 or table.strides[1] != table.itemsize:
            raise ValueError("table: [num_actors][frame] with contiguous rows")
        if ids.size and (ids.min() < 0 or ids.max() >= table.shape[0]):
            raise ValueError("actor id outside the table")
        ob = int(table.shape[1]) * table.itemsize
        base = table.__array_interface__["data"][0]
        ptrs = (base + ids.astype(np.uint64) * np.uint64(table.strides[0])).astype(np.uintp)
        return self.stage_requests(None, ids, rewards, dones, threads, chunk, stream,
                                   _ptrs=(ptrs, ob))

    def _stage(self, obs_list, actor_ids, rewards, dones, chunk, stream, _ptrs=None):
        """Host-fed requests (seed_stage_requests): obs_list = n host uint8 arrays
        (one per request, e.g. the actors' latest frames), actor_ids / rewards / dones
        host numpy arrays -> device (actor_ids, obs, reward, done) views of this
        server's staging buffers, filled asynchronously on `stream`."""
        import numpy as np
        if _ptrs is not None:
            ptr_arr, ob = _ptrs
            n = len(ptr_arr)
        else:
            n = len(obs_list)
            ob = int(obs_list[0].nbytes)
            ptr_arr = np.array([o.__array_interface__["data"][0] for o in obs_list], dtype=np.uintp)
        if getattr(self, "_stage_n", 0) < n or getattr(self, "_stage_ob", 0) != ob:
            self._pin_obs = torch.empty(n * ob, dtype=torch.uint8).pin_memory()
            self._pin_meta = torch.empty(9 * n + 16, dtype=torch.uint8).pin_memory()
            self._dev_obs = torch.empty(n * ob, dtype=torch.uint8, device=self.h.device)
            self._dev_meta = torch.empty(9 * n + 16, dtype=torch.uint8, device=self.h.device)
            self._stage_n, self._stage_ob = n, ob
        ptrs = C.c_void_p(ptr_arr.ctypes.data)
        ids = np.ascontiguousarray(actor_ids, np.int32)
        rw = np.ascontiguousarray(rewards, np.float32)
        dn = np.ascontiguousarray(dones, np.uint8)
        L.check(L.load().seed_stage_requests(self._stager, n, ptrs, ob, ids.ctypes.data,
                                             rw.ctypes.data, dn.ctypes.data, _ptr(self._pin_obs),
                                             _ptr(self._pin_meta), _ptr(self._dev_obs),
                                             _ptr(self._dev_meta), chunk, _stream(stream)),
                "seed_stage_requests")
        m = self._dev_meta
        return (m[:4 * n].view(torch.int32), self._dev_obs[:n * ob].view(n, ob),
                m[4 * n:8 * n].view(torch.float32), m[8 * n:9 * n])

    def assemble(self, B, out, stream=None):
        cb = L.Batch(*(_ptr(out.get(k)) for k in ("obs", "action", "prev_action", "reward",
                                                  "done", "behaviour_logp", "h0", "c0")))
        L.check(L.load().seed_assemble_batch(C.byref(self.store), self.obs_bytes,
                                             max(self.spec.lstm_units, 1), B, C.byref(cb),
                                             _stream(stream)), "seed_assemble_batch")
        return out
