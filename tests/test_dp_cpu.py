"""Data-parallel host logic on CPU (gloo, world_size 2): the unique-id broadcast
the NCCL communicator uses, and the DP semantics of the learner step (C20): the
sum over ranks of per-shard gradients scaled by 1/(N B T) equals the
single-process gradient on the concatenated batch (oracle, fp64)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import seedgen


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec = O.spec_c1()
    B, T = 3, 4
    flat = seedgen.glorot_params(O.param_layout(spec), seed=3, bias_std=0.1)
    shard = seedgen.learner_batch((16,), 4, B, T, seed=40 + rank, lstm_units=0, float_obs=True)
    hp = dict(discount=0.99, rho_bar=1.0, c_bar=1.0, vf_coef=0.5, ent_coef=0.01,
              loss_scale=1.0 / (world * B * T), lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-5,
              max_grad_norm=40.0, **{"lambda": 0.95})
    z = np.zeros(flat.size)
    g = torch.tensor(O.learner_step(spec, flat, z, z, 0, shard, hp)["grads"])
    dist.all_reduce(g)                              # the DP exchange step (H10)
    # unique-id broadcast as seed_comm uses it (128 opaque bytes from rank 0)
    obj = [bytes(range(128)) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    assert obj[0] == bytes(range(128))
    np.save(os.path.join(out_dir, f"g{rank}.npy"), g.numpy())
    dist.destroy_process_group()


def test_dp_allreduce_equals_full_batch(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    g0, g1 = (np.load(tmp_path / f"g{r}.npy") for r in range(world))
    np.testing.assert_array_equal(g0, g1)            # every rank holds the same sum
    spec = O.spec_c1()
    B, T = 3, 4
    flat = seedgen.glorot_params(O.param_layout(spec), seed=3, bias_std=0.1)
    shards = [seedgen.learner_batch((16,), 4, B, T, seed=40 + r, lstm_units=0, float_obs=True)
              for r in range(world)]
    full = {k: np.concatenate([s[k] for s in shards], 0) for k in shards[0]}
    hp = dict(discount=0.99, rho_bar=1.0, c_bar=1.0, vf_coef=0.5, ent_coef=0.01,
              loss_scale=1.0 / (world * B * T), lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-5,
              max_grad_norm=40.0, **{"lambda": 0.95})
    z = np.zeros(flat.size)
    ref = O.learner_step(spec, flat, z, z, 0, full, hp)["grads"]
    np.testing.assert_allclose(g0, ref, rtol=1e-12, atol=1e-15)


def test_nccl_unique_id_is_128_bytes():
    """The library's NCCL binding (dlopen) produces the opaque id the ranks exchange."""
    import paper_1910_06591_b200 as S
    import ctypes as C
    lib = S.load()
    buf = (C.c_uint8 * 128)()
    st = lib.seed_comm_get_unique_id(buf)
    if st == 5:
        pytest.skip("NCCL not loadable on this host")
    assert st == 0 and any(bytes(buf))
