"""One eager traced learner step (seed_learner_step_traced: events after every
phase, all kernels on one stream, in launch order) after a warm-up step, for an
ncu launch list; writes the phase labels and their kernel counts to
gpurun_out/<cfg>_phase_names.json (scripts/ncu_traffic.py maps the two).

usage: CFG=c4 ncu --launch-skip-before-match ... python scripts/traced_step.py"""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import seedgen  # noqa: E402
import paper_1910_06591_b200 as S  # noqa: E402
from paper_1910_06591_b200 import _lib as L  # noqa: E402

cfg = os.environ.get("CFG", "c4")
T, B, kw = {"c2": (20, 32, {}), "c3": (100, 32, {}), "c4": (32, 128, dict(smm=True))}[cfg]
spec = S.spec_for_config(cfg)
params = seedgen.glorot_params(S.net_param_layout(spec), seed=0)
learner = S.Learner(spec, T, B, params, S.HParams(loss_scale=1.0 / (B * T)))
host = seedgen.learner_batch(spec.obs_shape, spec.num_actions, B, T, seed=1, **kw)
dev = {k: torch.from_numpy(v).cuda() for k, v in host.items()}
MAXE = 192
evs = [torch.cuda.Event(enable_timing=True) for _ in range(MAXE)]
for e in evs:   # torch creates the CUDA event at its first record
    e.record()
torch.cuda.synchronize()
ev_arr = (L.c_void_p * MAXE)(*[e.cuda_event for e in evs])
names = (L.C.c_char_p * MAXE)()
counts = (C.c_int * MAXE)()
n_ev, n_launch = L.c_int(), L.c_int()
spec_c, hp_c = spec.c(), learner.hp.c()
cb = learner._batch(dev)
ts = learner._train_state()
s = torch.cuda.current_stream()
for _ in range(2):   # the first step sets kernel attributes; the second is the profiled one
    torch.cuda.synchronize()
    L.check(L.load().seed_learner_step_traced(
        C.byref(spec_c), T, B, C.byref(cb), C.byref(ts), C.byref(hp_c), None,
        C.c_void_p(learner.ws.data_ptr()), learner.ws.numel(),
        C.c_void_p(learner.metrics.data_ptr()), C.c_void_p(s.cuda_stream), ev_arr, MAXE,
        names, C.byref(n_ev), C.byref(n_launch), counts), "traced")
torch.cuda.synchronize()
seen, out = {}, []
for i in range(1, n_ev.value):
    n = names[i].decode()
    seen[n] = seen.get(n, 0) + 1
    out.append((f"{n}#{seen[n]}", counts[i]))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open(f"gpurun_out/{cfg}_phase_names.json", "w"))
print("launches per step", n_launch.value, "phases", len(out))
