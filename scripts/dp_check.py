"""torchrun --nproc-per-node N scripts/dp_check.py OUTDIR: one learner step per rank on
its shard with the NCCL allreduce inside seed_learner_step; rank 0 then runs the
1-GPU step on the concatenated batch and compares (DP equivalence, H10)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_1910_06591_b200 as S  # noqa: E402
import seedgen  # noqa: E402

out = sys.argv[1]
world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("gloo")
cfg = os.environ.get("CFG", "c2")
T, B = (5, 4) if cfg == "c2" else (4, 2)
spec = S.spec_for_config(cfg)
ospec = {"c2": O.spec_c2, "c3": O.spec_c3, "c4": O.spec_c4}[cfg]()
params = seedgen.glorot_params(O.param_layout(ospec), seed=2, bias_std=0.1)
shards = [seedgen.learner_batch(spec.obs_shape, spec.num_actions, B, T, seed=60 + r, done_p=0.1,
                                smm=(cfg == "c4")) for r in range(world)]
hp = S.HParams(lam=0.95, loss_scale=1.0 / (world * B * T), lr=1e-3)
comm = S.Comm(rank, world)
L = S.Learner(spec, T, B, params, hp, comm=comm)
m = L.step({k: torch.from_numpy(v).cuda() for k, v in shards[rank].items()})
torch.cuda.synchronize()
if comm.peer:
    comm.peer_status()   # raises if a peer wait timed out
np.save(os.path.join(out, f"grads{rank}.npy"), L.grads.cpu().numpy())
np.save(os.path.join(out, f"params{rank}.npy"), L.params.cpu().numpy())
np.save(os.path.join(out, f"metrics{rank}.npy"), m.cpu().numpy())
dist.barrier()
if rank == 0:
    full = {k: np.concatenate([s[k] for s in shards], 0) for k in shards[0]}
    L1 = S.Learner(spec, T, world * B, params, hp)
    L1.step({k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in full.items()})
    torch.cuda.synchronize()
    np.save(os.path.join(out, "grads_full.npy"), L1.grads.cpu().numpy())
    np.save(os.path.join(out, "params_full.npy"), L1.params.cpu().numpy())
dist.barrier()
comm.close()
dist.destroy_process_group()
