"""Device-resident inference sweep (configs[4] server, 4096 actors, CUDA graph per
n, L2 warm): us per seed_infer call at n = 64 .. 1024 (the bench's inference leg
without the host-fed part).  usage: python scripts/infer_sweep.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import seedgen  # noqa: E402
import paper_1910_06591_b200 as S  # noqa: E402

NA = 4096
spec = S.spec_for_config("c5")
params = seedgen.glorot_params(S.net_param_layout(spec), seed=0)
learner = S.Learner(spec, 1, 1, params)
srv = S.InferenceServer(spec, NA, 1024, learner=learner)
out = {}
for n in (1, 16, 64, 128, 256, 512, 1024):
    req = seedgen.infer_requests((84, 84, 4), 18, NA, n, seed=0)
    d = {k: torch.from_numpy(v).cuda() for k, v in req.items()}
    a = torch.empty(n, dtype=torch.int32, device="cuda")
    blp = torch.empty(n, device="cuda")
    call = lambda st=None: srv.infer(d["actor_ids"], d["obs"], d["reward"], d["done"], d["uniforms"],
                                     action_out=a, blp_out=blp, stream=st)
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
    for _ in range(50):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    out[n] = round(e0.elapsed_time(e1) * 1e3 / 50, 2)
print(json.dumps({"us_per_call": out}))
