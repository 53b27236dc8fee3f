"""Run a few seed_infer calls at configs[4] (4096 actors, n requests per call) —
a small driver for ncu launch lists of the inference kernels.  usage: N=1024 python scripts/infer_c5.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import seedgen  # noqa: E402
import paper_1910_06591_b200 as S  # noqa: E402

n = int(os.environ.get("N", 1024))
spec = S.spec_for_config("c5")
params = seedgen.glorot_params(S.net_param_layout(spec), seed=0)
learner = S.Learner(spec, 1, 1, params)
srv = S.InferenceServer(spec, 4096, 1024, learner=learner)
req = seedgen.infer_requests((84, 84, 4), 18, 4096, n, seed=0)
d = {k: torch.from_numpy(v).cuda() for k, v in req.items()}
a = torch.empty(n, dtype=torch.int32, device="cuda")
blp = torch.empty(n, device="cuda")
for _ in range(3):
    srv.infer(d["actor_ids"], d["obs"], d["reward"], d["done"], d["uniforms"], action_out=a, blp_out=blp)
torch.cuda.synchronize()
print("ok", int(a[0]))
