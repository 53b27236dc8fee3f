"""A few seed_infer calls at n (env N, default 64) on the configs[4] server, for an
ncu launch list of the inference path.  usage: N=64 ncu ... python scripts/infer_once.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import seedgen  # noqa: E402
import paper_1910_06591_b200 as S  # noqa: E402

n = int(os.environ.get("N", "64"))
NA = 4096
spec = S.spec_for_config("c5")
params = seedgen.glorot_params(S.net_param_layout(spec), seed=0)
learner = S.Learner(spec, 1, 1, params)
srv = S.InferenceServer(spec, NA, 1024, learner=learner)
req = seedgen.infer_requests((84, 84, 4), 18, NA, n, seed=0)
d = {k: torch.from_numpy(v).cuda() for k, v in req.items()}
a = torch.empty(n, dtype=torch.int32, device="cuda")
blp = torch.empty(n, device="cuda")
for _ in range(3):
    srv.infer(d["actor_ids"], d["obs"], d["reward"], d["done"], d["uniforms"], action_out=a, blp_out=blp)
torch.cuda.synchronize()
print("ok", n)
