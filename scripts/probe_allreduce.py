"""torchrun --nproc-per-node N scripts/probe_allreduce.py: device time of the
seed_comm allreduce for the c2 gradient buckets (graph of back-to-back calls)."""
import os
import sys
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_06591_b200 as S  # noqa: E402

world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("gloo")
comm = S.Comm(rank, world)
if os.environ.get("PEER", "0") == "1":
    assert comm.enable_peer(1225795 + 16)
for n in [12336, 663808, 549651, 1225795]:
    x = torch.arange(n, device="cuda", dtype=torch.float32) * (rank + 1) % 977
    ref = torch.arange(n, device="cuda", dtype=torch.float32)
    ref = sum(ref * (r + 1) % 977 for r in range(world))
    comm.allreduce_(x)
    torch.cuda.synchronize()
    err = (x - ref).abs().max().item()
    if rank == 0:
        print(f"check n={n}: max err {err}", flush=True)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            comm.allreduce_(x, stream=s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(20):
                comm.allreduce_(x, stream=s)
        torch.cuda.synchronize()
        dist.barrier()
        g.replay()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / 20
    if comm.peer and os.environ.get("SEED_PEER_DEBUG"):
        comm.peer_status()
    if rank == 0:
        print(f"allreduce {n} floats ({n*4/1e6:.2f} MB): {us:.1f} us  busbw {2*(world-1)/world*n*4/us/1e3:.1f} GB/s", flush=True)
if comm.peer:
    comm.peer_status()
comm.close()
