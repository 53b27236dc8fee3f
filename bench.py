#!/usr/bin/env python
"""bench.py — SEED (arXiv 1910.06591) learner hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One "step" = one seed_learner_step (H0-H11 of SURVEY.md §8(a)) of the
BASELINE.json configs[1] workload — Atari IMPALA-shallow CNN + LSTM(256),
84x84x4 uint8 obs, 18 actions, T=20, B=32 per GPU — on synthetic seeded inputs
already resident in HBM; N>1 = one process per GPU (torchrun), data-parallel
with the NCCL gradient allreduce inside the step (weak scaling).
Metric: learner frames/s (frames = B*T*4, action repeat 4: P:163; C16).
The same JSON line carries the V-trace bandwidth leg (seed_vtrace at T=100,
B=2^17, 367 MB > L2), the per-phase breakdown, the roofline of the dominant
kernel, the e2e number through the public API with pinned H2D/D2H copies,
clocks, and the CPU oracle baseline.
--impl reference: the CPU oracle (oracle/, fp64 numpy) on a bounded sample of
the same workload (rank 0 only) — the reference arm for this tier.
"""
import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CFG = dict(name="c2", T=20, B=32, A=18, repeat=4)
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK = dict(hbm_gbs=6650.0, bf16_tflops=1590.0, bf16_tflops_sustained=1400.0)


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return dict(hbm_gbs=p["hbm_gbs"], bf16_tflops=p["bf16_tflops"],
                    bf16_tflops_sustained=p.get("bf16_tflops_sustained", p["bf16_tflops"]),
                    source="measured (MEASURED_PEAKS.json)")
    except Exception:
        return dict(FALLBACK, source="fallback (B200_PROFILING.md)")


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------- algorithmic work per phase
def phase_work(T, B, A):
    """Algorithmic FLOPs and bytes of each step phase.  Convs count
    the forward-equivalent MACs (no zero taps); bytes are compulsory HBM traffic
    (every input read once, every output written once)."""
    F = B * (T + 1)
    P1, P2 = F * 400, F * 81
    obs = F * 84 * 84 * 4
    a1, a2 = P1 * 16 * 2, P2 * 32 * 2
    Kxp, U = 288, 256
    X = F * Kxp * 2
    w = {}
    w["obs_s2d"] = (0, obs * 3)          # uint8 obs -> space-to-depth bf16 S0
    w["conv1_fwd"] = (2 * P1 * 16 * 256, obs * 2 + a1 + 16 * 256 * 2)
    w["conv2_fwd"] = (2 * P2 * 32 * 256, a1 + a2 + 32 * 256 * 2)
    w["fc_fwd"] = (2 * F * 256 * 2592, a2 + 256 * 2592 * 2 + F * 256 * 2)
    w["core_extras"] = (0, F * 32 * 2 + F * 9)
    w["xproj_fwd"] = (2 * F * 1024 * 275, X + 1024 * Kxp * 2 + F * 1024 * 4)
    w["lstm_fwd"] = (2 * F * 1024 * 256, F * 1024 * 4 + 1024 * 256 * 2 + F * (256 * 4 * 2 + 1024 * 4 + 256 * 2))
    # heads forward + policy loss + heads backward (one kernel + the weight-grad sum):
    # H read, logits/values/dlogits written, dH written, per-trajectory partials
    w["heads_loss"] = (6 * F * (A + 1) * 256,
                       2 * F * 256 * 4 + 2 * F * (A + 1) * 4 + F * 9 + B * T * 8 + 2 * B * (A + 1) * 257 * 4)
    w["lstm_bwd"] = (2 * F * 1024 * 256, F * (1024 * 4 + 256 * 4 * 2 + 256 * 4 + 1024 * 2))
    w["lstm_wgrad"] = (2 * 1024 * (275 + 1 + 256) * F, F * 1024 * 2 + X + F * 256 * 2 + 1024 * 532 * 4)
    w["dx_fc"] = (2 * F * 256 * 1024, F * 1024 * 2 + 1024 * Kxp * 2 + F * 256 * 2 * 2)
    w["fc_wgrad"] = (2 * 256 * 2593 * F, F * 256 * 2 + a2 + 256 * 2593 * 4)
    w["fc_dgrad"] = (2 * F * 2592 * 256, F * 256 * 2 + 256 * 2592 * 2 + 2 * a2)
    w["conv2_wgrad"] = (2 * 256 * 32 * P2, a1 + a2 + 257 * 32 * 4)   # + bias row
    w["conv2_dgrad"] = (2 * P2 * 32 * 256, a2 + 2 * a1 + 16 * 512 * 2)
    w["conv1_wgrad"] = (2 * 256 * 16 * P1, obs * 2 + a1 + 257 * 16 * 4)
    Pn = 1225795
    w["grad_norm"] = (0, Pn * 4)
    w["clip_adam"] = (0, Pn * 28)
    w["lowp_refresh"] = (0, Pn * 6)
    w["allreduce"] = (0, Pn * 4 * 2)
    w["allreduce_tail"] = (0, 12336 * 4 * 2)
    return w


# ---------------------------------------------------------------- committed ncu evidence
PHASE_KERNEL = {"obs_s2d": "s2d_obs_kernel", "conv1_fwd": "Conv1S2dEpi", "conv2_fwd": "Conv2S2dEpi",
                "fc_fwd": "FcFwd",
                "xproj_fwd": "XprojFwd", "lstm_fwd": "lstm_fwd_kernel", "lstm_bwd": "lstm_bwd_kernel",
                "lstm_wgrad": "LstmWgrad", "dx_fc": "DxFc", "fc_wgrad": "FcWgrad",
                "fc_dgrad": "FcDgrad", "conv2_wgrad": "win_wgrad_kernel<32>",
                "conv2_dgrad": "Conv2DgradS2dEpi", "conv1_wgrad": "win_wgrad_kernel<16>",
                "heads_loss": "heads_loss_kernel",
                "clip_adam": "adam_kernel"}


def ncu_traffic(phase):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the phase's main
    kernel from the committed `ncu --set full` capture (profiles/r01/ncu_full.json)."""
    key = PHASE_KERNEL.get(phase)
    path = os.path.join(ROOT, "profiles", "r01", "ncu_full.json")
    if not key or not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    for name, ents in d.items():
        if key in name and "splitk" not in name:
            v = [e["dram_bytes"] for e in ents if e.get("dram_bytes") is not None]
            return round(sum(v) / len(v)) if v else None
    return None


# ---------------------------------------------------------------- clocks (NVML)
class ClockSampler:
    def __init__(self, index):
        self.samples, self.reasons, self.stop_ev = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self.N = None
            self.err = str(e)

    def _run(self):
        N = self.N
        names = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                 "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4, "sync_boost": 0x10}
        while not self.stop_ev.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.N:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.N:
            self.stop_ev.set()
            self.t.join()

    def summary(self):
        if not self.N or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------- CPU oracle baseline
def oracle_step_time(B_sample, T, seed=0):
    import oracle as O
    import seedgen
    spec = O.spec_c2()
    params = seedgen.glorot_params(O.param_layout(spec), seed=seed)
    batch = seedgen.learner_batch((84, 84, 4), 18, B_sample, T, seed=seed)
    hp = dict(discount=0.99, rho_bar=1.0, c_bar=1.0, vf_coef=0.5, ent_coef=0.01,
              loss_scale=1.0 / (B_sample * T), lr=3e-4, beta1=0.9, beta2=0.999, eps=1e-5,
              max_grad_norm=40.0, **{"lambda": 1.0})
    z = np.zeros(params.size)
    t0 = time.perf_counter()
    O.learner_step(spec, params, z, z, 0, batch, hp)
    return time.perf_counter() - t0


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 1) for i in threadpool_info()]
        return max(n) if n else 1
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


def cpu_baseline(T):
    B_s = 4
    t = oracle_step_time(B_s, T)
    frames = B_s * T * CFG["repeat"]
    return {"value": round(frames / t, 2), "unit": "learner frames/s", "cores": blas_threads(),
            "kind": "oracle",
            "sample": f"1 oracle learner step (fp64 numpy) of the c2 workload at B={B_s} "
                      f"(of 32), T={T}: {t:.2f} s"}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    T = CFG["T"]
    B_s = 4
    for _ in range(args.warmup):
        oracle_step_time(B_s, T)
    ts = [oracle_step_time(B_s, T, seed=i) for i in range(args.steps)]
    t = sum(ts) / len(ts)
    frames = B_s * T * CFG["repeat"]
    v = frames / t
    line = {"impl": "reference", "metric": "learner frames/sec", "value": round(v, 3),
            "unit": "frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(t * 1e3, 2), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"c2 Atari IMPALA-shallow + LSTM256 learner step, T={T}, "
                                   f"B={B_s} sample of B=32 (CPU oracle)"},
            "cpu_baseline": {"value": round(v, 3), "unit": "frames/s", "cores": blas_threads(),
                             "kind": "oracle",
                             "sample": f"{args.steps} oracle steps at B={B_s}, T={T}"},
            "e2e": {"value": round(v, 3), "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- V-trace leg
def vtrace_leg(S, torch, T=100, B=1 << 17, iters=20):
    import seedgen
    x = seedgen.vtrace_inputs(B, T, seed=0)
    d = {k: torch.from_numpy(v).cuda() for k, v in x.items()}
    vs = torch.empty(B, T, device="cuda")
    pg = torch.empty(B, T, device="cuda")
    call = lambda: S.vtrace(d["behaviour_logp"], d["target_logp"], d["rewards"],
                            d["discounts"], d["values"], d["bootstrap"], 1.0, 1.0, 1.0,
                            vs=vs, pg_advantages=pg)
    for _ in range(3):
        call()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(iters):
            call()
    torch.cuda.synchronize()
    g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    nbytes = 28 * B * T + 4 * B
    return {"T": T, "B": B, "bytes": nbytes, "us": round(us, 2), "GBs": round(nbytes / us / 1e3, 1)}


# ---------------------------------------------------------------- inference leg (c5)
def inference_leg(S, torch, iters=20):
    """configs[4]: 4096 actors, per-actor LSTM state table, Atari net; one
    seed_infer call per step over n actor ids (device-resident requests, CUDA
    graph per n) and host-fed (pinned H2D of the n observations inside the timed
    region).  steps/s = n / call time."""
    import seedgen
    NA = 4096
    spec = S.spec_for_config("c5")
    params = seedgen.glorot_params(S.net_param_layout(spec), seed=0)
    learner = S.Learner(spec, 1, 1, params)
    srv = S.InferenceServer(spec, NA, 1024, learner=learner)
    out = {"actors": NA, "sweep": []}
    for n in (64, 128, 256, 512, 1024):
        req = seedgen.infer_requests((84, 84, 4), 18, NA, n, seed=0)
        d = {k: torch.from_numpy(v).cuda() for k, v in req.items()}
        a = torch.empty(n, dtype=torch.int32, device="cuda")
        blp = torch.empty(n, device="cuda")
        call = lambda st=None: srv.infer(d["actor_ids"], d["obs"], d["reward"], d["done"],
                                         d["uniforms"], action_out=a, blp_out=blp, stream=st)
        for _ in range(3):
            call()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            call(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            call(s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / iters
        row = {"n": n, "us_per_call": round(us, 2), "steps_per_s": round(n / us * 1e6, 1)}
        if n == 1024:   # host-fed: pinned H2D of the requests + D2H of the actions
            hobs = torch.from_numpy(req["obs"]).pin_memory()
            hact = torch.empty(n, dtype=torch.int32).pin_memory()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            tot = 0.0
            for _ in range(iters):
                t0.record()
                d["obs"].copy_(hobs, non_blocking=True)
                g.replay()
                hact.copy_(a, non_blocking=True)
                t1.record()
                torch.cuda.synchronize()
                tot += t0.elapsed_time(t1)
            hus = tot * 1e3 / iters
            row.update(host_fed_us=round(hus, 2), host_fed_steps_per_s=round(n / hus * 1e6, 1),
                       h2d_bytes=int(hobs.numel()))
        out["sweep"].append(row)
    return out


def other_configs_leg(S, torch, steps=3):
    """Learner-step timing of the other BASELINE.json configs (CUDA graph, L2
    flushed between steps): c1 MLP fp32 (T=20, B=8), c3 DMLab IMPALA-deep
    (T=100, B=32), c4 GRF SMM (T=32, B=128, repeat 1)."""
    import seedgen
    res = {}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for cfg, T, B, rep, kw in (("c1", 20, 8, 1, dict(float_obs=True, lstm_units=0)),
                               ("c3", 100, 32, 4, {}), ("c4", 32, 128, 1, dict(smm=True))):
        spec = S.spec_for_config(cfg)
        params = seedgen.glorot_params(S.net_param_layout(spec), seed=0,
                                       lstm_units=max(spec.lstm_units, 1))
        L = S.Learner(spec, T, B, params, S.HParams(loss_scale=1.0 / (B * T)))
        host = seedgen.learner_batch(spec.obs_shape, spec.num_actions, B, T, seed=1, **kw)
        dev = {k: torch.from_numpy(v).cuda() for k, v in host.items()}
        L.step(dev)
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            L.step(dev, stream=s)
        torch.cuda.synchronize()
        g.replay()
        ms = 0.0
        for _ in range(steps):
            flush.add_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ms += e0.elapsed_time(e1)
        ms /= steps
        res[cfg] = {"T": T, "B": B, "ms_per_step": round(ms, 3),
                    "learner_frames_per_s": round(B * T * rep / (ms / 1e3), 1),
                    "env_steps_per_s": round(B * T / (ms / 1e3), 1)}
        del L, dev, g
        torch.cuda.empty_cache()
    return res


# ---------------------------------------------------------------- ours
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1910_06591_b200 as S
    import seedgen
    from paper_1910_06591_b200 import _lib as L

    world, rank, local = dist_env()
    assert torch.cuda.is_available(), "bench.py needs a GPU"
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo", init_method="env://", rank=rank, world_size=world)
    T, B, A = CFG["T"], CFG["B"], CFG["A"]
    spec = S.spec_for_config("c2")
    layout = S.net_param_layout(spec)
    params = seedgen.glorot_params(layout, seed=0)  # identical on every rank
    hp = S.HParams(lam=1.0, loss_scale=1.0 / (world * B * T))
    comm = S.Comm(rank, world) if world > 1 else None
    learner = S.Learner(spec, T, B, params, hp, comm=comm)
    host = seedgen.learner_batch((84, 84, 4), A, B, T, seed=1000 + rank)
    pinned = {k: torch.from_numpy(v).pin_memory() for k, v in host.items()}
    dev = {k: v.cuda() for k, v in pinned.items()}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    # ---- warm-up (sets kernel attributes; eager)
    for _ in range(max(args.warmup, 3)):
        learner.step(dev)
    torch.cuda.synchronize()

    # ---- capture the traced step in a CUDA graph (events after every phase)
    MAXE = 64
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(MAXE)]
    for e in evs:
        e.record()
    torch.cuda.synchronize()
    ev_arr = (L.c_void_p * MAXE)(*[e.cuda_event for e in evs])
    names = (L.C.c_char_p * MAXE)()
    n_ev, n_launch = L.c_int(), L.c_int()
    import ctypes as C
    spec_c = spec.c()
    hp_c = hp.c()
    cb = learner._batch(dev)
    ts = L.TrainState(*(C.c_void_p(t.data_ptr()) for t in (learner.params, learner.grads,
                                                             learner.m, learner.v)),
                      C.c_void_p(learner.lowp.data_ptr()), C.c_void_p(learner.step_counter.data_ptr()))

    def traced(stream):
        st = L.load().seed_learner_step_traced(
            C.byref(spec_c), T, B, C.byref(cb), C.byref(ts), C.byref(hp_c),
            comm.handle if comm else None, C.c_void_p(learner.ws.data_ptr()), learner.ws.numel(),
            C.c_void_p(learner.metrics.data_ptr()), C.c_void_p(stream.cuda_stream), ev_arr, MAXE,
            names, C.byref(n_ev), C.byref(n_launch))
        L.check(st, "seed_learner_step_traced")

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        traced(s)   # eager once on the capture stream
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        traced(s)
    torch.cuda.synchronize()
    # the same step without event nodes (headline timing)
    plain = torch.cuda.CUDAGraph()
    with torch.cuda.graph(plain, stream=s):
        learner.step(dev, stream=s)
    torch.cuda.synchronize()
    nE = n_ev.value
    phase_names = [names[i].decode() for i in range(nE)]
    launches_per_step = n_launch.value
    for _ in range(2):
        graph.replay()
    torch.cuda.synchronize()

    # ---- timed region: K replays of the plain step graph, L2 flushed between
    K = args.steps
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    flush.random_()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(K):
            flush.add_(1)                      # L2 flush, outside the timed events
            e0[i].record()
            plain.replay()
            e1[i].record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in zip(e0, e1)]
    # ---- per-phase breakdown: the traced graph (an event node after every phase)
    phase_ms = {n: 0.0 for n in phase_names[1:]}
    traced_ms = 0.0
    for i in range(K):
        flush.add_(1)
        graph.replay()
        torch.cuda.synchronize()
        for j in range(1, nE):
            phase_ms[phase_names[j]] += evs[j - 1].elapsed_time(evs[j])
        traced_ms += evs[0].elapsed_time(evs[nE - 1])
    total_ms = sum(step_ms)
    t_local = torch.tensor([total_ms], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    total_ms = float(t_local.item())
    ms_per_step = total_ms / K
    frames = world * B * T * CFG["repeat"]
    value = frames / (ms_per_step / 1e3)

    # ---- e2e through the public API: every step copies its batch from pinned host
    # memory (H2D) and reads its metrics back (D2H) inside the timed region; the
    # batch is double-buffered on a copy stream so step i's H2D overlaps step
    # i-1's compute (the way a learner is fed: SEED's prefetch)
    h2d = sum(v.numel() * v.element_size() for v in pinned.values())
    d2h = 8 * 4
    torch.cuda.synchronize()
    ha, hb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ha.record()
    for _ in range(3):
        for k, v in pinned.items():
            dev[k].copy_(v, non_blocking=True)
    hb.record()
    torch.cuda.synchronize()
    h2d_alone_ms = ha.elapsed_time(hb) / 3
    Ke = max(4, min(K, 20))
    s_comp = torch.cuda.current_stream()
    s_copy = torch.cuda.Stream()
    devs = [dev, {k: torch.empty_like(v) for k, v in dev.items()}]
    outs = [torch.empty(8, dtype=torch.float32).pin_memory() for _ in range(2)]
    ready = [torch.cuda.Event() for _ in range(2)]
    freed = [torch.cuda.Event() for _ in range(2)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(s_comp)
    s_copy.wait_event(e0)
    for i in range(Ke):
        b = i % 2
        with torch.cuda.stream(s_copy):
            if i >= 2:
                s_copy.wait_event(freed[b])
            for k, v in pinned.items():
                devs[b][k].copy_(v, non_blocking=True)
            ready[b].record(s_copy)
        s_comp.wait_event(ready[b])
        m = learner.step(devs[b])
        outs[b].copy_(m, non_blocking=True)
        freed[b].record(s_comp)
    e1.record(s_comp)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / Ke
    t_e2e = torch.tensor([e2e_ms], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
    e2e_value = frames / (float(t_e2e.item()) / 1e3)

    if rank != 0:
        if world > 1:
            dist.barrier()
        return
    # ---- roofline of the dominant phase
    pk = peaks()
    work = phase_work(T, B, A)
    per_phase = {n: phase_ms[n] / K for n in phase_ms}
    dom = max(per_phase, key=per_phase.get)
    flops, nbytes = work.get(dom, (0, 0))
    ridge = pk["bf16_tflops_sustained"] * 1e12 / (pk["hbm_gbs"] * 1e9)
    t_s = per_phase[dom] / 1e3
    if flops and flops / max(nbytes, 1) >= ridge:
        roof = {"bound": "tensor", "achieved": round(flops / t_s / 1e12, 3),
                "peak": pk["bf16_tflops_sustained"], "unit": "TFLOP/s"}
    else:
        roof = {"bound": "hbm", "achieved": round(nbytes / t_s / 1e9, 2), "peak": pk["hbm_gbs"],
                "unit": "GB/s"}
    roof["frac"] = round(roof["achieved"] / roof["peak"], 4)
    roof["traffic"] = ncu_traffic(dom)
    roof["kernel"] = dom
    roof["us_per_launch"] = round(per_phase[dom] * 1e3, 2)
    roof["peak_source"] = pk["source"]
    kernels = []
    for n in phase_names[1:]:
        f, b = work.get(n, (0, 0))
        us = per_phase[n] * 1e3
        kernels.append({"phase": n, "us": round(us, 2), "share": round(per_phase[n] / ms_per_step, 4),
                        "TFLOPs": round(f / (us * 1e-6) / 1e12, 3) if f else None,
                        "GBs": round(b / (us * 1e-6) / 1e9, 1) if b else None})
    vt = vtrace_leg(S, torch)
    vt["frac"] = round(vt["GBs"] / pk["hbm_gbs"], 4)
    extra = {}
    if world == 1 and not args.no_extra:
        extra["inference"] = inference_leg(S, torch)
        extra["other_configs"] = other_configs_leg(S, torch)
    line = {
        "metric": "learner frames/sec", "value": round(value, 1), "unit": "frames/s",
        "n_gpus": world, "steps": K, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic",
        "config": {"workload": "c2 Atari IMPALA-shallow CNN + LSTM256 learner step "
                               "(BASELINE.json configs[1]): 84x84x4 uint8, A=18, T=20, B=32/GPU",
                   "global_batch": world * B, "seq_len": T + 1, "parallelism": f"dp{world}",
                   "frames_per_step": frames, "l2": "flushed (256 MiB write) between timed steps",
                   "timing": "CUDA-graph replay, CUDA events per step, max over ranks"},
        "env_steps_per_s": round(value / CFG["repeat"], 1),
        "gpu_launches": launches_per_step * K,
        "traced_ms_per_step": round(traced_ms / K, 4),
        "kernels": kernels,
        "roofline": roof,
        "vtrace": vt,
        "e2e": {"value": round(e2e_value, 1), "unit": "frames/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "api": "Learner.step (eager): pinned H2D of each step's batch on a copy stream, "
                       "double-buffered (overlaps the previous step), D2H of the metrics",
                "h2d_ms_alone": round(h2d_alone_ms, 4)},
        "clocks": clk.summary(),
        **extra,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(T)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the inference / other-config legs")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
