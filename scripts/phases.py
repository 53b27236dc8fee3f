"""Per-phase breakdown of one learner step for any config (traced CUDA graph:
an event node after every phase, L2 flushed between replays).

usage: CFG=c3 python scripts/phases.py [reps]"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import seedgen  # noqa: E402
import paper_1910_06591_b200 as S  # noqa: E402
from paper_1910_06591_b200 import _lib as L  # noqa: E402

cfg = os.environ.get("CFG", "c3")
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
T, B, kw = {"c1": (20, 8, dict(float_obs=True, lstm_units=0)), "c2": (20, 32, {}),
            "c3": (100, 32, {}), "c4": (32, 128, dict(smm=True)), "c3m": (100, 32, {}),
            "c4m": (32, 128, dict(smm=True)), "c4l": (32, 128, dict(smm=True)), "c3l": (100, 32, {})}[cfg]
T = int(os.environ.get("T", T))
B = int(os.environ.get("B", B))
spec = S.spec_for_config(cfg)
params = seedgen.glorot_params(S.net_param_layout(spec), seed=0, lstm_units=max(spec.lstm_units, 1))
learner = S.Learner(spec, T, B, params, S.HParams(loss_scale=1.0 / (B * T)))
host = seedgen.learner_batch(spec.obs_shape, spec.num_actions, B, T, seed=1, **kw)
dev = {k: torch.from_numpy(v).cuda() for k, v in host.items()}
learner.step(dev)
torch.cuda.synchronize()

MAXE = 128
evs = [torch.cuda.Event(enable_timing=True) for _ in range(MAXE)]
for e in evs:
    e.record()
torch.cuda.synchronize()
ev_arr = (L.c_void_p * MAXE)(*[e.cuda_event for e in evs])
names = (L.C.c_char_p * MAXE)()
n_ev, n_launch = L.c_int(), L.c_int()
spec_c, hp_c = spec.c(), learner.hp.c()
cb = learner._batch(dev)
ts = L.TrainState(*(C.c_void_p(t.data_ptr()) for t in (learner.params, learner.grads, learner.m,
                                                        learner.v)),
                  C.c_void_p(learner.lowp.data_ptr()), C.c_void_p(learner.step_counter.data_ptr()))


def traced(stream):
    L.check(L.load().seed_learner_step_traced(
        C.byref(spec_c), T, B, C.byref(cb), C.byref(ts), C.byref(hp_c), None,
        C.c_void_p(learner.ws.data_ptr()), learner.ws.numel(),
        C.c_void_p(learner.metrics.data_ptr()), C.c_void_p(stream.cuda_stream), ev_arr, MAXE,
        names, C.byref(n_ev), C.byref(n_launch), None), "traced")


s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    traced(s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    traced(s)
plain = torch.cuda.CUDAGraph()
with torch.cuda.graph(plain, stream=s):
    learner.step(dev, stream=s)
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
nE = n_ev.value
pn = [names[i].decode() for i in range(nE)]
acc = {}
order = []
tot = 0.0
for _ in range(reps):
    flush.add_(1)
    g.replay()
    torch.cuda.synchronize()
    seen = {}
    for j in range(1, nE):
        k = pn[j]
        if os.environ.get("PER_LAUNCH"):
            seen[k] = seen.get(k, 0) + 1
            k = f"{k}#{seen[k]}"
        if k not in acc:
            acc[k] = 0.0
            order.append(k)
        acc[k] += evs[j - 1].elapsed_time(evs[j])
    tot += evs[0].elapsed_time(evs[nE - 1])
ms = 0.0
for _ in range(reps):
    flush.add_(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    plain.replay()
    e1.record()
    torch.cuda.synchronize()
    ms += e0.elapsed_time(e1)
out = {"cfg": cfg, "T": T, "B": B, "plain_ms": round(ms / reps, 4), "traced_ms": round(tot / reps, 4),
       "launches": n_launch.value,
       "phases_us": {n: round(acc[n] / reps * 1e3, 2) for n in order}}
print(json.dumps(out))
