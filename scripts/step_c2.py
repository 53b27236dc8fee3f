"""Run K eager c2 learner steps at the bench configuration (B=32, T=20) — a
small driver for ncu launch lists / captures of the learner step kernels."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import seedgen  # noqa: E402
import paper_1910_06591_b200 as S  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 3
B, T = int(os.environ.get("B", 32)), int(os.environ.get("T", 20))
cfg = os.environ.get("CFG", "c2")
spec = S.spec_for_config(cfg)
n = S.net_param_count(spec)
params = np.random.default_rng(0).standard_normal(n).astype(np.float32) * 0.02
obs_shape = {"c2": (84, 84, 4), "c3": (72, 96, 3), "c4": (72, 96, 16)}[cfg]
batch = seedgen.learner_batch(obs_shape, spec.num_actions, B, T, seed=0, done_p=0.02)
L = S.Learner(spec, T, B, params, S.HParams(loss_scale=1.0 / (B * T)))
bt = {k: torch.from_numpy(v).cuda() for k, v in batch.items()}
for _ in range(K):
    L.step(bt)
torch.cuda.synchronize()
print("ok", float(L.metrics[0]))
