"""GPU tests of versioned parameter publication (include/seed.h seed_param_*;
SURVEY §8(f) row 2: inference concurrent with training, P:98, P:111, P:125,
P:238; S:37-42 version, S:109 / S:465 single-copy semantics).

The property is integer / byte work, so it is checked bit-exactly: every
parameter set the consumer acquires is exactly the learner's parameters of the
version it reports (never a mix of two updates), versions never go backwards,
and an acquire after a publish sees that publish or a later one."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle as O
import seedgen

pytestmark = pytest.mark.gpu


def _setup(B=2, T=3):
    import paper_1910_06591_b200 as S
    spec = S.spec_for_config("c2")
    params = seedgen.glorot_params(O.param_layout(O.spec_c2()), seed=61, bias_std=0.1)
    L = S.Learner(spec, T, B, params, S.HParams(lr=1e-3, loss_scale=1.0 / (B * T)))
    batch = seedgen.learner_batch((84, 84, 4), 18, B, T, seed=62)
    gb = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in batch.items()}
    return S, spec, L, gb


def _acquire(S, spec, snap, lowp, params, version, stream, force=0):
    from paper_1910_06591_b200 import _lib
    spec_c = spec.c()
    _lib.check(_lib.load().seed_param_acquire(
        C.byref(spec_c), C.byref(snap.c), C.c_void_p(lowp.data_ptr()), C.c_void_p(params.data_ptr()),
        C.c_void_p(version.data_ptr()), force, C.c_void_p(stream.cuda_stream)), "acquire")


def test_publish_acquire_sequential():
    S, spec, L, gb = _setup()
    snap = S.ParamSnapshot(spec)
    lowp = torch.zeros_like(L.lowp)
    params = torch.zeros_like(L.params)
    ver = torch.zeros(1, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    _acquire(S, spec, snap, lowp, params, ver, s)
    torch.cuda.synchronize()
    assert int(ver.item()) == -1                       # nothing published yet
    L.step(gb)
    L.publish(snap)
    _acquire(S, spec, snap, lowp, params, ver, s)
    torch.cuda.synchronize()
    assert int(ver.item()) == 1
    assert torch.equal(params, L.params) and torch.equal(lowp, L.lowp)
    p1 = L.params.clone()
    # no new publish: the held version stays, the private copy is not rewritten
    params.zero_()
    _acquire(S, spec, snap, lowp, params, ver, s)
    torch.cuda.synchronize()
    assert int(ver.item()) == 1 and not params.any()
    _acquire(S, spec, snap, lowp, params, ver, s, force=1)
    torch.cuda.synchronize()
    assert torch.equal(params, p1)
    # two publishes before an acquire: the consumer gets the latest
    for _ in range(2):
        L.step(gb)
        L.publish(snap)
    _acquire(S, spec, snap, lowp, params, ver, s)
    torch.cuda.synchronize()
    assert int(ver.item()) == 3 and int(L.step_counter.item()) == 3
    assert torch.equal(params, L.params) and torch.equal(lowp, L.lowp)


def test_concurrent_training_and_acquire_never_torn():
    """Learner (step + publish) on one stream, consumer (acquire + record) on
    another, enqueued interleaved so they overlap on the device."""
    S, spec, L, gb = _setup()
    snap = S.ParamSnapshot(spec)
    K, M = 24, 160
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    hist_p = torch.zeros(K + 1, L.params.numel(), device="cuda")
    hist_l = torch.zeros(K + 1, L.lowp.numel(), dtype=torch.uint8, device="cuda")
    rec_p = torch.zeros(M, L.params.numel(), device="cuda")
    rec_v = torch.zeros(M, dtype=torch.int64, device="cuda")
    lowp = torch.zeros_like(L.lowp)
    params = torch.zeros_like(L.params)
    rec_l = torch.zeros(M, L.lowp.numel(), dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    with torch.cuda.stream(sa):
        L.publish(snap, stream=sa)                    # version 0 = the initial parameters
        hist_p[0].copy_(L.params)
        hist_l[0].copy_(L.lowp)
    k = 0
    for i in range(M):
        if i % (M // K) == 0 and k < K:
            with torch.cuda.stream(sa):
                L.step(gb, stream=sa)
                L.publish(snap, stream=sa)
                k += 1
                hist_p[k].copy_(L.params)
                hist_l[k].copy_(L.lowp)
        with torch.cuda.stream(sb):
            _acquire(S, spec, snap, lowp, params, rec_v[i:i + 1], sb)
            rec_p[i].copy_(params)
            rec_l[i].copy_(lowp)
    torch.cuda.synchronize()
    v = rec_v.cpu().numpy()
    assert np.all(v >= 0) and np.all(v <= K) and np.all(np.diff(v) >= 0), v
    hp, hl = hist_p.cpu().numpy(), hist_l.cpu().numpy()
    rp, rl = rec_p.cpu().numpy(), rec_l.cpu().numpy()
    for i in range(M):
        np.testing.assert_array_equal(rp[i], hp[v[i]], err_msg=f"acquire {i} (version {v[i]}) torn")
        np.testing.assert_array_equal(rl[i], hl[v[i]], err_msg=f"acquire {i} image torn")
    assert len(np.unique(v)) > 2, v                    # the consumer really saw several versions
    # after the learner finished, an acquire sees the last version and its image
    _acquire(S, spec, snap, lowp, params, rec_v[:1], torch.cuda.current_stream())
    torch.cuda.synchronize()
    assert int(rec_v[0].item()) == K
    assert torch.equal(lowp, hist_l[K]) and torch.equal(params, hist_p[K])


def test_inference_server_serves_published_parameters():
    """InferenceServer(snapshot=...) acquires before every call: its actions and
    logits equal those of a server reading the learner's parameters directly."""
    S, spec, L, gb = _setup()
    snap = S.ParamSnapshot(spec)
    L.step(gb)
    L.publish(snap)
    NA, n = 64, 16
    a_srv = S.InferenceServer(spec, NA, n, snapshot=snap)
    b_srv = S.InferenceServer(spec, NA, n, learner=L)
    req = seedgen.infer_requests((84, 84, 4), 18, NA, n, seed=63)
    d = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in req.items()}
    la = torch.empty(n, 18, device="cuda")
    lb = torch.empty(n, 18, device="cuda")
    aa, ba = a_srv.infer(d["actor_ids"], d["obs"], d["reward"], d["done"], d["uniforms"],
                         logits_out=la)
    ab, bb = b_srv.infer(d["actor_ids"], d["obs"], d["reward"], d["done"], d["uniforms"],
                         logits_out=lb)
    torch.cuda.synchronize()
    assert int(a_srv.version.item()) == 1
    assert torch.equal(la, lb) and torch.equal(aa, ab) and torch.equal(ba, bb)
