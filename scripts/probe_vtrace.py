"""Quick V-trace bandwidth sweep (CUDA events, inputs >> L2)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1910_06591_b200 as S  # noqa: E402

res = []
for T in (20, 32, 100):
    for lb in (14, 17, 20):
        B = 1 << lb
        if B * T * 28 > 8e9:
            continue
        t = {k: torch.randn(B, T, device="cuda") for k in ("blp", "tlp", "r", "d", "v")}
        t["d"].uniform_(0.9, 0.99)
        boot = torch.randn(B, device="cuda")
        vs = torch.empty(B, T, device="cuda")
        pg = torch.empty(B, T, device="cuda")
        for _ in range(3):
            S.vtrace(t["blp"], t["tlp"], t["r"], t["d"], t["v"], boot, vs=vs, pg_advantages=pg)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        n = 20
        e0.record()
        for _ in range(n):
            S.vtrace(t["blp"], t["tlp"], t["r"], t["d"], t["v"], boot, vs=vs, pg_advantages=pg)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / n * 1e3
        gbs = (28 * B * T + 4 * B) / us / 1e3
        res.append(dict(T=T, B=B, us=round(us, 2), GBs=round(gbs, 1), MB=round((28 * B * T + 4 * B) / 1e6, 1)))
        print(res[-1], flush=True)
        del t, vs, pg
json.dump(res, open("gpurun_out/vtrace_sweep.json", "w"), indent=1)
