#!/usr/bin/env python
"""bench.py — SEED (arXiv 1910.06591) learner hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One "step" = one seed_learner_step (H0-H11 of SURVEY.md §8(a)) of the
headline workload, BASELINE.json configs[3] — Google Research Football SMM,
IMPALA-deep torso (16, 32, 32, 32) + LSTM(256), 72x96x16 uint8 obs, 19 actions,
T=32, B=128 per GPU (the largest single-GPU config, the one BASELINE.json
scales over 1/2/4/8 GPUs) — on synthetic seeded inputs already resident in HBM;
N>1 = one process per GPU (torchrun), data-parallel with the NCCL gradient
allreduce inside the step (weak scaling).
Metric: learner frames/s (frames = B*T*repeat; repeat 1 for GRF; 4 for
Atari / DMLab; C16).  The same JSON line carries the per-launch
breakdown, the roofline of the dominant kernel, the e2e number through the
public API (pinned H2D of every step's batch, D2H of the metrics), clocks, the
CPU oracle baseline, the V-trace bandwidth leg (T=100, B=2^17, 367 MB > L2),
inference steps/s (configs[4], on every rank), and the configs[1] / configs[2]
learner steps with their own rooflines.
--impl reference: the CPU oracle (oracle/, fp64 numpy) on a bounded sample of
the headline workload (rank 0 only) — the reference arm for this tier.
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

CONFIGS = {
    "c2": dict(T=20, B=32, A=18, repeat=4, batch_kw={},
               workload="c2 Atari IMPALA-shallow CNN + LSTM256 learner step (BASELINE.json "
                        "configs[1]): 84x84x4 uint8, A=18, T=20, B=32/GPU"),
    "c3": dict(T=100, B=32, A=15, repeat=4, batch_kw={},
               workload="c3 DMLab IMPALA-deep ResNet (16,32,32) + LSTM256 learner step "
                        "(BASELINE.json configs[2]): 72x96x3 uint8, A=15, T=100, B=32/GPU"),
    "c4": dict(T=32, B=128, A=19, repeat=1, batch_kw=dict(smm=True),
               workload="c4 Google Research Football SMM, IMPALA-deep (16,32,32,32) + LSTM256 "
                        "learner step (BASELINE.json configs[3]): 72x96x16 uint8, A=19, T=32, "
                        "B=128/GPU"),
}
# SURVEY §8(f) row 3 (larger torsos): reported as extra legs
CONFIGS["c3m"] = dict(T=100, B=32, A=15, repeat=4, batch_kw={},
                      workload="c3m DMLab IMPALA-deep Medium (2x filters: 32,64,64) + LSTM256 learner "
                               "step (P:411): 72x96x3 uint8, A=15, T=100, B=32/GPU")
CONFIGS["c3l"] = dict(T=100, B=32, A=15, repeat=4, batch_kw={},
                      workload="c3l DMLab IMPALA-deep Large (4x filters: 64,128,128; 128-channel "
                               "tensors as two 64-channel planes) + LSTM256 learner step (P:411, "
                               "P:434): 72x96x3 uint8, A=15, T=100, B=32/GPU")
CONFIGS["c4l"] = dict(T=32, B=128, A=19, repeat=1, batch_kw=dict(smm=True),
                      workload="c4l Google Research Football Large SMM 144x108 (P:358), IMPALA-deep "
                               "(16,32,32,32) + LSTM256 learner step: 108x144x16 uint8, A=19, T=32, "
                               "B=128/GPU")
HEAD = "c4"
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


# ---------------------------------------------------------------- algorithmic work per launch
def deep_geometry(cfg):
    """IMPALA-deep sections (C14): (H, W, cin, cin_rows, ch, H2, W2) per section."""
    H, W = (108, 144) if cfg == "c4l" else (72, 96)
    C = 3 if cfg.startswith("c3") else 16
    chans = {"c3m": (32, 64, 64), "c3l": (64, 128, 128)}.get(cfg, (16, 32, 32)) if cfg.startswith("c3") \
        else (16, 32, 32, 32)
    out, cin, cinp = [], C, 16
    for ch in chans:
        H2, W2 = (H + 1) // 2, (W + 1) // 2
        out.append((H, W, cin, cinp, ch, H2, W2))
        H, W, cin, cinp = H2, W2, ch, ch
    return out


def core_work(F, B, T, A, fc_in, P):
    """FC / LSTM / heads / optimizer launches: algorithmic FLOPs and
    compulsory HBM bytes (every input read once, every output written once)."""
    Kxp = ((256 + A + 1 + 1 + 31) // 32) * 32
    X = F * Kxp * 2
    w = {}
    w["core_extras"] = (0, F * (Kxp - 256) * 2 + F * 9)
    w["fc_fwd"] = (2 * F * 256 * fc_in, F * fc_in * 2 + 256 * fc_in * 2 + F * 256 * 2)
    w["xproj_fwd"] = (2 * F * 1024 * (256 + A + 1), X + 1024 * Kxp * 2 + F * 1024 * 4)
    w["lstm_fwd"] = (2 * F * 1024 * 256, F * 1024 * 4 + 1024 * 256 * 2 +
                     F * (256 * 4 * 2 + 1024 * 4 + 256 * 2))
    w["heads_loss"] = (6 * F * (A + 1) * 256, 2 * F * 256 * 4 + 2 * F * (A + 1) * 4 + F * 9 +
                       B * T * 8 + 2 * B * (A + 1) * 257 * 4)
    w["lstm_bwd"] = (2 * F * 1024 * 256, F * (1024 * 4 + 256 * 4 * 2 + 256 * 4 + 1024 * 2))
    w["lstm_wgrad"] = (2 * 1024 * (256 + A + 2 + 256) * F,
                       F * 1024 * 2 + X + F * 256 * 2 + 1024 * (Kxp + 256) * 4)
    w["dx_fc"] = (2 * F * 256 * 1024, F * 1024 * 2 + 1024 * Kxp * 2 + F * 256 * 2 * 2)
    w["fc_wgrad"] = (2 * 256 * (fc_in + 1) * F, F * 256 * 2 + F * fc_in * 2 + 256 * (fc_in + 1) * 4)
    w["fc_dgrad"] = (2 * F * fc_in * 256, F * 256 * 2 + 256 * fc_in * 2 + 2 * F * fc_in * 2)
    w["grad_norm"] = (0, P * 4)
    w["clip_adam"] = (0, P * 28)
    w["lowp_refresh"] = (0, P * 6)
    w["allreduce"] = (0, P * 4 * 2)
    w["allreduce_tail"] = (0, P * 4 * 2)
    return w


def launch_work(cfg, T, B, A, P, names):
    """(FLOPs, bytes) of every traced launch, in order.  Convolutions count the
    MACs of the definition (no padding taps); bytes are the op's compulsory
    traffic on unpadded tensors (bf16 activations, uint8 obs)."""
    F = B * (T + 1)
    out = []
    if cfg == "c2":
        P1, P2 = F * 400, F * 81
        obs = F * 84 * 84 * 4
        a1, a2 = P1 * 16 * 2, P2 * 32 * 2
        tw = {"obs_s2d": (0, obs * 3),
              "conv1_fwd": (2 * P1 * 16 * 256, obs * 2 + a1 + 16 * 256 * 2),
              "conv2_fwd": (2 * P2 * 32 * 256, a1 + a2 + 32 * 256 * 2),
              "conv2_wgrad": (2 * 256 * 32 * P2, a1 + a2 + 257 * 32 * 4),
              "conv2_dgrad": (2 * P2 * 32 * 256, a2 + 2 * a1 + 16 * 512 * 2),
              "conv1_wgrad": (2 * 256 * 16 * P1, obs * 2 + a1 + 257 * 16 * 4)}
        tw.update(core_work(F, B, T, A, 2592, P))
        return [tw.get(n, (0, 0)) for n in names]
    geo = deep_geometry(cfg)
    ns = len(geo)
    tw = core_work(F, B, T, A, geo[-1][5] * geo[-1][6] * geo[-1][4], P)
    # the (section, fraction of its work) of each launch of a phase name, in launch
    # order: sections ascending forward, descending backward; 128-channel sections
    # run as 64-channel plane pairs (learner.cu plane_section_*), each launch a
    # 1/(planes) share of the section's op
    fuse = os.environ.get("SEED_FUSE_POOL") != "0"
    seq = {}

    def add(name, s, n):
        seq.setdefault(name, []).extend([(s, 1.0 / n)] * n)
    for s, (H, W, cin, cinp, ch, H2, W2) in enumerate(geo):
        npo, npi = (2 if ch > 64 else 1), (2 if cinp > 64 else 1)
        fused = fuse and ch <= 32 and cinp <= 32
        if fused:
            add("deep_conv_pool", s, 1)
        else:
            add("deep_conv_fwd", s, npo * npi)
            add("deep_pool_fwd", s, npo)
        for _ in range(2):
            add("deep_res_fwd0", s, npo * npo)
            add("deep_res_fwd1", s, npo * npo)
    for s in range(ns - 1, -1, -1):
        H, W, cin, cinp, ch, H2, W2 = geo[s]
        npo, npi = (2 if ch > 64 else 1), (2 if cinp > 64 else 1)
        for _ in range(2):
            for nm in ("deep_res_wgrad1", "deep_res_dgrad1", "deep_res_wgrad0", "deep_res_dgrad0"):
                add(nm, s, npo * npo)
        add("deep_pool_bwd", s, npo)
        add("deep_conv_wgrad", s, npo * npi)
        if s > 0:
            add("deep_conv_dgrad", s, npo * npi)
    seen = {}
    for n in names:
        k = seen.get(n, 0)
        seen[n] = k + 1
        if not n.startswith("deep_") and n != "obs_bf16":
            out.append(tw.get(n, (0, 0)))
            continue
        if n == "obs_bf16":
            H, W, cin, cinp = geo[0][0], geo[0][1], geo[0][2], geo[0][3]
            out.append((0, F * H * W * (cin + cinp * 2)))
            continue
        if n not in seq or k >= len(seq[n]):
            out.append((0, 0))
            continue
        s, frac = seq[n][k]
        H, W, cin, cinp, ch, H2, W2 = geo[s]
        Ai, Ao = F * H * W, F * H2 * W2
        # section 0 reads the converted bf16 rows (obs_bf16: 16 planes, or DMLab's
        # x-im2col rows); with SEED_XF_U8=1 the GRF net reads the uint8 obs directly
        u8 = cfg == "c4" and os.environ.get("SEED_XF_U8") == "1"
        xin = Ai * (cin if u8 else cinp * 2) if s == 0 else Ai * cin * 2
        if n == "deep_conv_fwd":
            w = (2 * Ai * ch * 9 * cin, xin + Ai * ch * 2)
        elif n == "deep_conv_pool":    # fused: input read, pooled h, relu(h) + argmax written
            w = (2 * Ai * ch * 9 * cin, xin + 2 * Ao * ch * 2 + Ao * ch)
        elif n == "deep_pool_fwd":     # conv read, pooled h, relu(h) + argmax written
            w = (0, Ai * ch * 2 + 2 * Ao * ch * 2 + Ao * ch)
        elif n == "deep_res_fwd0":
            w = (2 * Ao * ch * 9 * ch, 2 * Ao * ch * 2)
        elif n == "deep_res_fwd1":     # u1 + residual read, h and relu(h) written
            w = (2 * Ao * ch * 9 * ch, 4 * Ao * ch * 2)
        elif n.startswith("deep_res_wgrad"):
            w = (2 * Ao * 9 * ch * ch, 2 * Ao * ch * 2)
        elif n == "deep_res_dgrad1":
            w = (2 * Ao * 9 * ch * ch, 3 * Ao * ch * 2)
        elif n == "deep_res_dgrad0":
            w = (2 * Ao * 9 * ch * ch, 4 * Ao * ch * 2)
        elif n == "deep_pool_bwd":
            w = (0, Ao * ch * 2 + Ao * ch + Ai * ch * 2)
        elif n == "deep_conv_wgrad":
            w = (2 * Ai * 9 * cin * ch, xin + Ai * ch * 2)
        elif n == "deep_conv_dgrad":
            w = (2 * Ai * 9 * cin * ch, Ai * ch * 2 + Ai * cin * 2)
        else:
            w = (0, 0)
        out.append((w[0] * frac, w[1] * frac))
    return out


# ---------------------------------------------------------------- committed ncu evidence
def ncu_traffic(label):
    """dram__bytes_read.sum + dram__bytes_write.sum of the launch `label` (phase#k)
    from the committed `ncu --set full` summary (profiles/r02/ncu_traffic.json)."""
    path = os.path.join(ROOT, "profiles", "r02", "ncu_traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    return d.get(HEAD, {}).get(label)


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
# (B, T) of one bounded oracle step: the reference arm times one such step per
# --steps (a few minutes for 25 steps); cpu_baseline one step of ORACLE_BASELINE
# (10-30 s of CPU work)
ORACLE_SAMPLE = dict(c2=(4, 20), c3=(1, 20), c4=(1, 32))
ORACLE_BASELINE = dict(c2=(32, 20), c3=(4, 20), c4=(8, 32))


def oracle_step_time(cfg, B_sample, T, seed=0):
    import oracle as O
    import seedgen
    spec = {"c2": O.spec_c2, "c3": O.spec_c3, "c4": O.spec_c4}[cfg]()
    obs_shape = (spec.obs_h, spec.obs_w, spec.obs_c)
    params = seedgen.glorot_params(O.param_layout(spec), seed=seed)
    batch = seedgen.learner_batch(obs_shape, spec.num_actions, B_sample, T, seed=seed,
                                  **CONFIGS[cfg]["batch_kw"])
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


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(cfg):
    B_s, T_s = ORACLE_BASELINE[cfg]
    t = oracle_step_time(cfg, B_s, T_s)
    frames = B_s * T_s * CONFIGS[cfg]["repeat"]
    out = {"value": round(frames / t, 2), "unit": "learner frames/s", "cores": blas_threads(),
           "host_cpus": os.cpu_count(), "cpu_model": cpu_model(), "kind": "oracle",
           "sample": f"1 oracle learner step (fp64 numpy) of the {cfg} network at B={B_s}, "
                     f"T={T_s} (of B={CONFIGS[cfg]['B']}, T={CONFIGS[cfg]['T']}): {t:.2f} s"}
    try:   # the same oracle on one core (BLAS limited to 1 thread), a B=1 sample
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1):
            t1 = oracle_step_time(cfg, 1, T_s)
        out["value_1thread"] = round(1 * T_s * CONFIGS[cfg]["repeat"] / t1, 2)
        out["sample_1thread"] = f"B=1, T={T_s}, 1 BLAS thread: {t1:.2f} s"
    except Exception as e:  # noqa: BLE001
        out["value_1thread"] = None
        out["sample_1thread"] = f"unavailable: {e}"
    return out


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = HEAD
    B_s, T_s = ORACLE_SAMPLE[cfg]
    for _ in range(args.warmup):
        oracle_step_time(cfg, B_s, T_s)
    ts = [oracle_step_time(cfg, B_s, T_s, seed=i) for i in range(args.steps)]
    t = sum(ts) / len(ts)
    frames = B_s * T_s * CONFIGS[cfg]["repeat"]
    v = frames / t
    line = {"impl": "reference", "metric": "learner frames/sec", "value": round(v, 3),
            "unit": "frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(t * 1e3, 2), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIGS[cfg]["workload"] +
                       f" — CPU oracle on a B={B_s}, T={T_s} sample per step"},
            "cpu_baseline": {"value": round(v, 3), "unit": "frames/s", "cores": blas_threads(),
                             "host_cpus": os.cpu_count(), "cpu_model": cpu_model(),
                             "kind": "oracle",
                             "sample": f"{args.steps} oracle steps at B={B_s}, T={T_s}"},
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
    return {"T": T, "B": B, "bytes": nbytes, "us": round(us, 2), "GBs": round(nbytes / us / 1e3, 1),
            "working_set": "367.5 MB > 126 MB L2 (20 back-to-back calls in one graph)"}


# ---------------------------------------------------------------- R2D2 leg
def wire_leg(S, torch, actors=16, envs=2, steps=30):
    """f4: actors (threads, one TCP connection each, SEEDWire v1
    uint8 StepRequests) -> the library's batching server (max batch 32, 1 ms
    deadline) -> seed_infer on the configs[4] net -> ActionResponses routed back.
    Reports env steps/s through the whole loop and the actor-observed round-trip
    latency (send -> action) percentiles.  Host networking on loopback; the actors
    are Python threads, so this measures the library's path under a light load."""
    import threading
    import numpy as np
    import seedgen
    from paper_1910_06591_b200 import wire as Wr
    spec = S.spec_for_config("c5")
    params = seedgen.glorot_params(S.net_param_layout(spec), seed=0)
    learner = S.Learner(spec, 1, 1, params)
    rows = actors * envs
    srv = S.InferenceServer(spec, rows, 32, learner=learner)
    obs_bytes = 84 * 84 * 4
    ws = Wr.WireServer(obs_bytes, rows, max_batch=32, max_wait_us=1000)
    lat, errors = [], []
    frame = np.random.default_rng(0).integers(0, 256, obs_bytes, dtype=np.uint8)

    def actor(aid):
        try:
            c = Wr.ActorClient(ws.port, aid, envs)
            for step in range(steps):
                t0 = time.perf_counter()
                for e in range(envs):
                    c.send_step(e, 0.0, step == 0, frame)
                for _ in range(envs):
                    c.recv()
                lat.append((time.perf_counter() - t0) * 1e3)
            c.close()
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))
    dev = {k: torch.empty(32, dtype=dt, device="cuda") for k, dt in
           (("ids", torch.int32), ("rew", torch.float32), ("done", torch.uint8), ("u", torch.float32))}
    dobs = torch.empty(32, 84, 84, 4, dtype=torch.uint8, device="cuda")
    dev["u"].uniform_()
    threads = [threading.Thread(target=actor, args=(i,)) for i in range(actors)]
    t0 = time.perf_counter()
    for t in threads:
        t.start()
    served, batches = 0, 0
    while served < rows * steps and time.perf_counter() - t0 < 120:
        obs, ids, rew, done = ws.next_batch(timeout_us=100000)
        n = len(ids)
        if n == 0:
            continue
        dobs[:n].copy_(torch.from_numpy(obs.reshape(n, 84, 84, 4)))
        dev["ids"][:n].copy_(torch.from_numpy(ids))
        dev["rew"][:n].copy_(torch.from_numpy(rew))
        dev["done"][:n].copy_(torch.from_numpy(done))
        a, _ = srv.infer(dev["ids"][:n], dobs[:n], dev["rew"][:n], dev["done"][:n], dev["u"][:n])
        ws.reply(ids, a.cpu().numpy())
        served += n
        batches += 1
    dt = time.perf_counter() - t0
    for t in threads:
        t.join(timeout=30)
    st = ws.stats()
    ws.close()
    lat = np.sort(np.asarray(lat)) if lat else np.zeros(1)
    return {"actors": actors, "envs_per_actor": envs, "steps": served, "batches": batches,
            "mean_batch": round(served / max(batches, 1), 2), "env_steps_per_s": round(served / dt, 1),
            "round_trip_ms_p50_p99": [round(float(np.percentile(lat, 50)), 3),
                                      round(float(np.percentile(lat, 99)), 3)],
            "batch_triggers": {k: st[k] for k in ("by_size", "by_deadline", "by_timeout")},
            "errors": errors[:3]}


def r2d2_leg(S, torch, iters=20):
    """seed_r2d2_targets at the paper's trained-sequence shape (80 steps after the
    40-step burn-in of 120; 18 actions; n = 5) over B = 2^14 sequences
    (> L2), as HBM GB/s of its compulsory traffic; and the replay at the paper's
    10^5 sequences: one training iteration's sample (B = 64) +
    priority update (+ tree rebuilds), device time per iteration."""
    B, T, A = 1 << 14, 80, 18
    g = torch.Generator(device="cuda").manual_seed(0)
    qo = torch.randn(B, T + 1, A, device="cuda", generator=g)
    qt = torch.randn(B, T + 1, A, device="cuda", generator=g)
    a = torch.randint(0, A, (B, T + 1), device="cuda", dtype=torch.int32, generator=g)
    r = torch.randn(B, T, device="cuda", generator=g)
    disc = torch.full((B, T), 0.997, device="cuda")
    w = torch.rand(B, device="cuda", generator=g)
    call = lambda: S.r2d2_targets(qo, qt, a, r, disc, n=5, is_weights=w, want_grad=True)
    for _ in range(3):
        call()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        call()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    # compulsory bytes: q_online read + q_target rows read (~1/A of it: one value per
    # step, but whole rows for the argmax are q_online's) + actions, rewards,
    # discounts, weights read; y, delta, priority, loss written; dq written
    nbytes = 4 * (B * (T + 1) * A + B * (T + 1) + 2 * B * T + B + B * (T + 1) * A +
                  2 * B * T + 2 * B) + 4 * B * T
    out = {"targets": {"B": B, "T": T, "A": A, "n": 5, "us": round(us, 2),
                       "GBs": round(nbytes / us / 1e3, 1), "bytes": nbytes}}
    N, Bs = 100000, 64
    R = S.PrioritizedReplay(N, 16)
    recs = torch.zeros(1024, 16, dtype=torch.uint8, device="cuda")
    for k in range(0, N, 1024):
        R.insert(recs[:min(1024, N - k)])
    torch.cuda.synchronize()
    pr = torch.rand(Bs, device="cuda", generator=g)
    e0.record()
    for i in range(iters):
        sl, gn, ww = R.sample(Bs, seed=1, counter=i)
        R.update(sl, gn, pr)
    e1.record()
    torch.cuda.synchronize()
    out["replay"] = {"sequences": N, "tree_leaves": R.capacity, "batch": Bs,
                     "us_per_sample_and_update": round(e0.elapsed_time(e1) * 1e3 / iters, 2),
                     "launches_per_iteration": 3}
    del R, qo, qt
    torch.cuda.empty_cache()
    # one R2D2 learner update at the paper's shape: 64 sequences of
    # 120 Atari frames, the first 40 burn-in, on the configs[1] network with dueling
    # heads; CUDA-graph replays, L2 flushed between them
    import seedgen
    spec = S.spec_for_config("c2")
    Bq, bi, Tq = 64, 40, 79
    params = seedgen.glorot_params(S.net_param_layout(spec), seed=0)
    Lq = S.R2d2Learner(spec, bi, Tq, Bq, params, S.R2d2HParams(loss_scale=1.0 / (Bq * Tq)))
    full = seedgen.learner_batch(spec.obs_shape, spec.num_actions, Bq, bi + Tq, seed=5)
    L1 = bi + Tq + 1
    cut = lambda a, b: {k: torch.from_numpy(np.ascontiguousarray(v[:, a:b] if v.ndim >= 2 and v.shape[1] == L1
                                                                  else v)).cuda() for k, v in full.items()}
    burn, train = cut(0, bi), cut(bi, L1)
    w = torch.rand(Bq, device="cuda", generator=g)
    for _ in range(3):
        Lq.step(train, burn=burn, is_weights=w)
    sq = torch.cuda.Stream()
    sq.wait_stream(torch.cuda.current_stream())
    gq = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gq, stream=sq):
        Lq.step(train, burn=burn, is_weights=w, stream=sq)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    tot = 0.0
    for _ in range(iters):
        flush.add_(1)
        e0.record()
        gq.replay()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    ms = tot / iters
    out["learner_step"] = {"net": "configs[1] Atari net + LSTM256, dueling heads", "B": Bq,
                           "burn_in": bi, "trained_steps": Tq, "ms_per_update": round(ms, 4),
                           "updates_per_s": round(1e3 / ms, 1),
                           "trained_frames_per_s": round(Bq * Tq * 4 / (ms / 1e3), 1)}
    del Lq, gq, flush
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------- inference leg (c5)
def inference_leg(S, torch, world, rank, dist, iters=20):
    """configs[4]: 4096 actors per GPU, per-actor LSTM state table, Atari net; one
    seed_infer call per step over n actor ids (device-resident requests, CUDA graph
    per n) and host-fed (pinned H2D of the n observations + D2H of the actions
    inside the timed region).  steps/s = N * n / (max over ranks of the call time)."""
    import seedgen
    NA = 4096
    spec = S.spec_for_config("c5")
    params = seedgen.glorot_params(S.net_param_layout(spec), seed=0)
    learner = S.Learner(spec, 1, 1, params)
    srv = S.InferenceServer(spec, NA, 1024, learner=learner)
    out = {"actors_per_gpu": NA, "n_gpus": world, "sweep": []}

    def tmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    for n in (64, 128, 256, 512, 1024):
        req = seedgen.infer_requests((84, 84, 4), 18, NA, n, seed=rank)
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
        us = tmax(e0.elapsed_time(e1) * 1e3 / iters)
        row = {"n": n, "us_per_call": round(us, 2), "steps_per_s": round(world * n / us * 1e6, 1)}
        if n == 1024:
            # host-fed: the actors' latest frames sit in per-actor host buffers; every
            # call packs the n requests into pinned staging (seed_stage_requests: the
            # library's host worker threads, chunked copies overlapping the packing),
            # runs the inference graph on the staged buffers and reads the actions back
            frames = np.random.default_rng(rank).integers(0, 256, size=(NA, 84 * 84 * 4),
                                                          dtype=np.uint8)
            ids = req["actor_ids"]
            hact = torch.empty(n, dtype=torch.int32).pin_memory()
            sd = srv.stage_requests_table(frames, ids, req["reward"], req["done"], threads=8,
                                          chunk=128, stream=s)
            torch.cuda.synchronize()
            g2 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g2, stream=s):
                srv.infer(sd[0], sd[1], sd[2], sd[3], d["uniforms"], action_out=a, blp_out=blp,
                          stream=s)
            torch.cuda.synchronize()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            # same-job pinned H2D probe of the same bytes: the PCIe denominator
            hobs = torch.from_numpy(frames[ids].reshape(req["obs"].shape)).pin_memory()
            tp0, tp1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            d["obs"].copy_(hobs, non_blocking=True)
            torch.cuda.synchronize()
            tp0.record()
            for _ in range(iters):
                d["obs"].copy_(hobs, non_blocking=True)
            tp1.record()
            torch.cuda.synchronize()
            h2d_us = tp0.elapsed_time(tp1) * 1e3 / iters
            cur = torch.cuda.current_stream()
            tot = 0.0
            host = 0.0
            for _ in range(iters):
                t0.record(cur)
                th = time.perf_counter()
                srv.stage_requests_table(frames, ids, req["reward"], req["done"], stream=cur)
                host += time.perf_counter() - th
                g2.replay()
                hact.copy_(a, non_blocking=True)
                t1.record(cur)
                torch.cuda.synchronize()
                tot += t0.elapsed_time(t1)
            hus = tmax(tot * 1e3 / iters)
            row.update(host_fed_us=round(hus, 2), host_stage_call_us=round(host * 1e6 / iters, 2),
                       host_fed_steps_per_s=round(world * n / hus * 1e6, 1),
                       h2d_bytes=int(hobs.numel()), h2d_probe_us=round(h2d_us, 2),
                       host_fed_api="InferenceServer.stage_requests_table (seed_stage_requests: 8 "
                                    "host threads pack per-actor frames into pinned staging, "
                                    "128-request chunks copied as packed) + graph replay + "
                                    "D2H of the actions",
                       h2d_probe_GBs=round(hobs.numel() / h2d_us / 1e3, 2),
                       host_fed_vs_probe=round(hus / max(h2d_us + us, 1e-9), 3))
        out["sweep"].append(row)
    del srv, learner
    return out


# ---------------------------------------------------------------- one learner config
def make_learner(S, torch, cfg, world, rank, comm):
    import seedgen
    c = CONFIGS[cfg]
    spec = S.spec_for_config(cfg)
    params = seedgen.glorot_params(S.net_param_layout(spec), seed=0)   # identical on every rank
    hp = S.HParams(lam=1.0, loss_scale=1.0 / (world * c["B"] * c["T"]))
    L = S.Learner(spec, c["T"], c["B"], params, hp, comm=comm)
    host = seedgen.learner_batch(spec.obs_shape, spec.num_actions, c["B"], c["T"],
                                 seed=1000 + rank, **c["batch_kw"])
    pinned = {k: torch.from_numpy(v).pin_memory() for k, v in host.items()}
    dev = {k: v.cuda() for k, v in pinned.items()}
    return spec, L, pinned, dev


def traced_graph(S, torch, L, spec, dev, comm, maxe=160):
    """A CUDA graph of the step with an event node after every launch group
    (seed_learner_step_traced) -> per-launch times; the plain graph is separate."""
    import ctypes as C
    from paper_1910_06591_b200 import _lib as Lb
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(maxe)]
    for e in evs:
        e.record()
    torch.cuda.synchronize()
    ev_arr = (Lb.c_void_p * maxe)(*[e.cuda_event for e in evs])
    names = (Lb.C.c_char_p * maxe)()
    n_ev, n_launch = Lb.c_int(), Lb.c_int()
    spec_c, hp_c = spec.c(), L.hp.c()
    cb = L._batch(dev)
    ts = L._train_state()

    def traced(stream):
        st = Lb.load().seed_learner_step_traced(
            C.byref(spec_c), L.T, L.B, C.byref(cb), C.byref(ts), C.byref(hp_c),
            comm.handle if comm else None, C.c_void_p(L.ws.data_ptr()), L.ws.numel(),
            C.c_void_p(L.metrics.data_ptr()), C.c_void_p(stream.cuda_stream), ev_arr, maxe,
            names, C.byref(n_ev), C.byref(n_launch), None)
        Lb.check(st, "seed_learner_step_traced")

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        traced(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        traced(s)
    torch.cuda.synchronize()
    nE = n_ev.value
    return g, evs, [names[i].decode() for i in range(nE)], n_launch.value


def measure_learner(S, torch, dist, cfg, steps, warmup, world, rank, local, comm, clocks=True,
                    e2e=True):
    c = CONFIGS[cfg]
    T, B, A = c["T"], c["B"], c["A"]
    spec, L, pinned, dev = make_learner(S, torch, cfg, world, rank, comm)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2
    for _ in range(max(warmup, 3)):
        L.step(dev)
    torch.cuda.synchronize()
    tgraph, evs, names, launches = traced_graph(S, torch, L, spec, dev, comm)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    plain = torch.cuda.CUDAGraph()
    with torch.cuda.graph(plain, stream=s):
        L.step(dev, stream=s)
    torch.cuda.synchronize()
    # warm replays (first replays of a graph with NCCL inside carry one-time setup);
    # every rank replays the same count, in step
    for _ in range(2):
        tgraph.replay()
    for _ in range(max(warmup, 3)):
        plain.replay()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # ---- timed region: K replays of the plain step graph, L2 flushed between
    K = steps
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    flush.random_()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local) if clocks else None
    if clk:
        clk.__enter__()
    for i in range(K):
        flush.add_(1)                      # L2 flush, outside the timed events
        e0[i].record()
        plain.replay()
        e1[i].record()
    torch.cuda.synchronize()
    if clk:
        clk.__exit__()
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in zip(e0, e1)]
    total = torch.tensor([sum(step_ms)], dtype=torch.float64)
    per_rank = [sum(step_ms) / K]
    if world > 1:
        allr = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allr, total)
        per_rank = [float(x.item()) / K for x in allr]
        dist.all_reduce(total, op=dist.ReduceOp.MAX)
    ms_per_step = float(total.item()) / K
    # ---- per-launch breakdown from the traced graph (event node after every launch group)
    nE = len(names)
    Kt = max(2, min(K, 10))
    per = [0.0] * nE
    for _ in range(Kt):
        flush.add_(1)
        tgraph.replay()
        torch.cuda.synchronize()
        for j in range(1, nE):
            per[j] += evs[j - 1].elapsed_time(evs[j])
    per = [p / Kt for p in per]
    work = launch_work(cfg, T, B, A, int(L.params.numel()), names[1:])
    seen, kernels = {}, []
    for j in range(1, nE):
        n = names[j]
        k = seen.get(n, 0) + 1
        seen[n] = k
        f, b = work[j - 1]
        us = per[j] * 1e3
        kernels.append({"launch": f"{n}#{k}", "us": round(us, 2),
                        "share": round(per[j] / ms_per_step, 4),
                        "TFLOPs": round(f / (us * 1e-6) / 1e12, 2) if f and us > 0 else None,
                        "GBs": round(b / (us * 1e-6) / 1e9, 1) if b and us > 0 else None,
                        "flops": f, "bytes": b})
    frames = world * B * T * c["repeat"]
    out = {"cfg": cfg, "ms_per_step": ms_per_step, "frames_per_step": frames,
           "value": frames / (ms_per_step / 1e3), "env_steps_per_s": world * B * T / (ms_per_step / 1e3),
           "gpu_launches_per_step": launches, "kernels": kernels,
           "traced_ms_per_step": sum(per[1:]),
           "clocks": clk.summary() if clk else None,
           "step_ms_p10_p50_p90": [round(float(np.percentile(step_ms, q)), 4) for q in (10, 50, 90)],
           "ms_per_step_per_rank": [round(x, 4) for x in per_rank]}
    out["roofline"] = roofline_of(kernels, cfg)
    # the step's roofline floor: every launch at max(FLOPs / sustained bf16, bytes / HBM)
    pk = peaks()
    floor_us = sum(max(k["flops"] / (pk["bf16_tflops_sustained"] * 1e6),
                       k["bytes"] / (pk["hbm_gbs"] * 1e3)) for k in kernels)
    out["step_floor"] = {"ms": round(floor_us / 1e3, 4),
                         "frac_of_measured": round(floor_us / 1e3 / ms_per_step, 4),
                         "model": "sum over launches of max(algorithmic FLOPs / sustained bf16 "
                                  "peak, algorithmic bytes / measured HBM) — ignores the serial "
                                  "LSTM latency and per-MMA issue floors"}
    if e2e:
        out["e2e"] = e2e_leg(torch, dist, L, dev, pinned, steps, world, frames)
    del L, dev, pinned, tgraph, plain, flush
    torch.cuda.empty_cache()
    return out


def roofline_of(kernels, cfg):
    """Roofline of the dominant launch: algorithmic FLOPs (or bytes) ÷ its measured
    average duration, against the measured tensor-core (or HBM) peak."""
    pk = peaks()
    dom = max(kernels, key=lambda k: k["us"])
    ridge = pk["bf16_tflops_sustained"] * 1e12 / (pk["hbm_gbs"] * 1e9)
    t_s = dom["us"] * 1e-6
    f, b = dom["flops"], dom["bytes"]
    if f and f / max(b, 1) >= ridge:
        roof = {"bound": "tensor", "achieved": round(f / t_s / 1e12, 3),
                "peak": pk["bf16_tflops_sustained"], "unit": "TFLOP/s"}
    else:
        roof = {"bound": "hbm", "achieved": round(b / t_s / 1e9, 2), "peak": pk["hbm_gbs"],
                "unit": "GB/s"}
    roof["frac"] = round(roof["achieved"] / roof["peak"], 4)
    roof["traffic"] = ncu_traffic(dom["launch"]) if cfg == HEAD else None
    roof["kernel"] = dom["launch"]
    roof["us_per_launch"] = dom["us"]
    roof["algorithmic"] = {"flops": f, "bytes": b}
    roof["peak_source"] = pk["source"] + (" sustained bf16" if roof["bound"] == "tensor" else "")
    return roof


def e2e_leg(torch, dist, L, dev, pinned, steps, world, frames):
    """The same metric through the public API (Learner.step, eager): every step
    copies its batch from pinned host memory (H2D) and reads its metrics back
    (D2H) inside the timed region; the batch is double-buffered on a copy stream
    so step i's H2D overlaps step i-1's compute (the way a learner is fed:
    SEED's prefetch)."""
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
    Ke = max(4, min(steps, 20))
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
        m = L.step(devs[b])
        outs[b].copy_(m, non_blocking=True)
        freed[b].record(s_comp)
    e1.record(s_comp)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / Ke
    t = torch.tensor([e2e_ms], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    del devs
    return {"value": round(frames / (float(t.item()) / 1e3), 1), "unit": "frames/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": round(float(t.item()), 4),
            "api": "Learner.step (eager): pinned H2D of each step's batch on a copy stream, "
                   "double-buffered (overlaps the previous step), D2H of the metrics",
            "h2d_ms_alone": round(h2d_alone_ms, 4),
            "h2d_GBs_alone": round(h2d / (h2d_alone_ms * 1e-3) / 1e9, 2)}


# ---------------------------------------------------------------- ours
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1910_06591_b200 as S

    world, rank, local = dist_env()
    assert torch.cuda.is_available(), "bench.py needs a GPU"
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo", init_method="env://", rank=rank, world_size=world)
    comm = S.Comm(rank, world) if world > 1 else None
    head = measure_learner(S, torch, dist, HEAD, args.steps, args.warmup, world, rank, local,
                           comm)
    extra = {}
    if not args.no_extra:
        # the other learner configs (fewer timed steps) and inference, on every rank
        for cfg, k in (("c2", max(20, min(args.steps, 100))), ("c3", max(5, min(args.steps, 20))),
                       ("c3m", 5), ("c3l", 3), ("c4l", 5)):
            r = measure_learner(S, torch, dist, cfg, k, 3, world, rank, local, comm, clocks=False,
                                e2e=False)
            extra[cfg] = {"workload": CONFIGS[cfg]["workload"], "steps": k,
                          "ms_per_step": round(r["ms_per_step"], 4),
                          "learner_frames_per_s": round(r["value"], 1),
                          "env_steps_per_s": round(r["env_steps_per_s"], 1),
                          "gpu_launches_per_step": r["gpu_launches_per_step"],
                          "roofline": r["roofline"], "step_floor": r["step_floor"],
                          "top_kernels": sorted(r["kernels"], key=lambda x: -x["us"])[:8]}
        inf = inference_leg(S, torch, world, rank, dist)
        r2 = r2d2_leg(S, torch) if rank == 0 else None
        wl = wire_leg(S, torch) if rank == 0 else None
    c = CONFIGS[HEAD]
    if rank == 0:
        vt = vtrace_leg(S, torch)
        vt["frac"] = round(vt["GBs"] / peaks()["hbm_gbs"], 4)
        line = {
            "metric": "learner frames/sec", "value": round(head["value"], 1), "unit": "frames/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(head["ms_per_step"], 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": {"workload": c["workload"], "global_batch": world * c["B"],
                       "seq_len": c["T"] + 1, "parallelism": f"dp{world}",
                       "frames_per_step": head["frames_per_step"],
                       "l2": "flushed (256 MiB write) between timed steps; the 467 MB obs batch "
                             "alone exceeds the 126 MB L2",
                       "timing": "CUDA-graph replay, CUDA events per step, max over ranks"},
            "env_steps_per_s": round(head["env_steps_per_s"], 1),
            "gpu_launches": head["gpu_launches_per_step"] * args.steps,
            "step_ms_p10_p50_p90": head["step_ms_p10_p50_p90"],
            "ms_per_step_per_rank": head["ms_per_step_per_rank"],
            "traced_ms_per_step": round(head["traced_ms_per_step"], 4),
            "roofline": head["roofline"],
            "step_floor": head["step_floor"],
            "e2e": head["e2e"],
            "clocks": head["clocks"],
            "kernels": [{k: v for k, v in x.items() if k not in ("flops", "bytes")}
                        for x in head["kernels"]],
            "vtrace": vt,
        }
        if not args.no_extra:
            line["other_configs"] = extra
            line["inference"] = inf
            line["r2d2"] = r2
            line["actor_transport"] = wl
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(HEAD)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the other-config / inference legs")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
