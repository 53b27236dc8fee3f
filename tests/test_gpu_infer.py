"""GPU parity of seed_infer / seed_assemble_batch (H12, H13) against the oracle
(bf16-emulated network, C26), the state-table semantics, the unroll
store accounting (C17, C19) and the behaviour-fidelity self-consistency."""
import numpy as np
import pytest
import torch

import oracle as O
import seedgen

pytestmark = pytest.mark.gpu
NA, T, A = 48, 4, 18


def _setup(seed=0, store=True, max_n=16):
    import paper_1910_06591_b200 as S
    spec = S.spec_for_config("c5")
    ospec = O.spec_c2()
    params = seedgen.glorot_params(O.param_layout(ospec), seed=seed + 3, bias_std=0.1)
    learner = S.Learner(spec, T, 2, params)
    srv = S.InferenceServer(spec, NA, max_n, learner=learner, T=T if store else None)
    g = seedgen.rng(seed + 100)
    h = (0.5 * g.standard_normal((NA, 256))).astype(np.float32)
    c = (0.5 * g.standard_normal((NA, 256))).astype(np.float32)
    la = g.integers(-1, A, NA).astype(np.int32)
    srv.h.copy_(torch.from_numpy(h))
    srv.c.copy_(torch.from_numpy(c))
    srv.last_action.copy_(torch.from_numpy(la))
    return S, srv, ospec, params


def _call(srv, req, uniforms=True, seed=0, counter=0):
    d = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in req.items()}
    logits = torch.empty(len(req["actor_ids"]), A, device="cuda")
    a, blp = srv.infer(d["actor_ids"], d["obs"], d["reward"], d["done"],
                       d["uniforms"] if uniforms else None, seed=seed, counter=counter,
                       logits_out=logits)
    torch.cuda.synchronize()
    return a.cpu().numpy(), blp.cpu().numpy(), logits.cpu().numpy()


def _relL2(x, y):
    return np.linalg.norm(np.asarray(x, np.float64) - y) / max(np.linalg.norm(y), 1e-30)


def _near_boundary(logits, u, tol=2e-3):
    p = np.exp(O.log_softmax(np.asarray(logits, np.float64)))
    cdf = np.cumsum(p, axis=-1)
    return np.any(np.abs(cdf - u[:, None]) < tol, axis=-1)


@pytest.mark.parametrize("n", [1, 7, 16])
def test_infer_parity_and_table(n):
    S, srv, ospec, params = _setup(store=False)
    th, tc, tla = (srv.h.cpu().numpy(), srv.c.cpu().numpy(), srv.last_action.cpu().numpy())
    req = seedgen.infer_requests((84, 84, 4), A, NA, n, seed=5)
    req["done"][: min(2, n)] = 1
    a, blp, logits = _call(srv, req)
    ra, rblp, rlg, rth, rtc, rtla = O.infer(ospec, params, th, tc, tla, req["actor_ids"],
                                            req["obs"], req["reward"], req["done"],
                                            req["uniforms"], emu=True)
    assert _relL2(logits, rlg) < 2e-2
    nb = _near_boundary(rlg, req["uniforms"].astype(np.float64))
    assert np.all((a == ra) | nb), (a, ra)
    ok = a == ra
    np.testing.assert_allclose(blp[ok], rblp[ok], atol=2e-2 * max(1.0, np.abs(rblp).max()))
    ids = req["actor_ids"]
    assert _relL2(srv.h.cpu().numpy()[ids], rth[ids]) < 2e-2
    assert _relL2(srv.c.cpu().numpy()[ids], rtc[ids]) < 2e-2
    others = np.setdiff1d(np.arange(NA), ids)
    np.testing.assert_array_equal(srv.h.cpu().numpy()[others], th[others])   # untouched, bitwise
    np.testing.assert_array_equal(srv.c.cpu().numpy()[others], tc[others])
    np.testing.assert_array_equal(srv.last_action.cpu().numpy()[ids], a)
    np.testing.assert_array_equal(srv.last_action.cpu().numpy()[others], tla[others])


def test_infer_philox_stream():
    S, srv, ospec, params = _setup(store=False)
    th, tc, tla = (srv.h.cpu().numpy(), srv.c.cpu().numpy(), srv.last_action.cpu().numpy())
    req = seedgen.infer_requests((84, 84, 4), A, NA, 16, seed=9)
    a, blp, logits = _call(srv, req, uniforms=False, seed=1234567, counter=42)
    u = O.philox_uniforms(1234567, 42, req["actor_ids"])
    ra, *_ = O.infer(ospec, params, th, tc, tla, req["actor_ids"], req["obs"], req["reward"],
                     req["done"], u, emu=True)
    p = np.exp(O.log_softmax(logits.astype(np.float64)))
    cdf = np.cumsum(p, axis=-1)
    expect = (u[:, None] < cdf).argmax(-1)      # GPU logits, oracle uniforms
    nb = _near_boundary(logits, u)
    assert np.all((a == expect) | nb)
    assert np.all((a == ra) | _near_boundary(logits, u, 2e-2))


def _batch_bufs(B, flat_obs=True):
    shape = (B, T + 1, 84 * 84 * 4) if flat_obs else (B, T + 1, 84, 84, 4)
    return dict(obs=torch.empty(*shape, dtype=torch.uint8, device="cuda"),
                action=torch.empty(B, T + 1, dtype=torch.int32, device="cuda"),
                prev_action=torch.empty(B, T + 1, dtype=torch.int32, device="cuda"),
                reward=torch.empty(B, T + 1, device="cuda"),
                done=torch.empty(B, T + 1, dtype=torch.uint8, device="cuda"),
                behaviour_logp=torch.empty(B, T + 1, device="cuda"),
                h0=torch.empty(B, 256, device="cuda"), c0=torch.empty(B, 256, device="cuda"))


def test_unroll_store_and_assemble():
    """Two unroll rounds over all actors: completed unrolls, overlap slot, h0
    (C17, C19), deterministic ready-ring order, seed_assemble_batch (an unroll is
    consumed before its buffer is reused T steps later)."""
    S, srv, ospec, params = _setup(store=True, max_n=NA)
    ref = O.UnrollStore(T=T, num_actors=NA)
    completed = []          # (key, snapshot of slots, h0, c0) in completion order
    consumed = 0
    call = 0
    for rnd in range(2):
        ncalls = T + 1 if rnd == 0 else T
        for _ in range(ncalls):
            req = seedgen.infer_requests((84, 84, 4), A, NA, NA, seed=3, call_index=call)
            call += 1
            hpre = srv.h.cpu().numpy()[req["actor_ids"]]
            cpre = srv.c.cpu().numpy()[req["actor_ids"]]
            prev = srv.last_action.cpu().numpy()[req["actor_ids"]]
            a, blp, _ = _call(srv, req)
            for i, act in enumerate(req["actor_ids"]):
                rec = dict(obs=req["obs"][i], action=a[i], prev=prev[i], reward=req["reward"][i],
                           done=req["done"][i], blp=blp[i])
                before = len(ref.ready)
                ref.record(int(act), rec, hpre[i], cpre[i])
                if len(ref.ready) > before:
                    key = ref.ready[-1]
                    st = ref.steps[key]
                    completed.append((key, list(st["slots"]), st["h0"].copy(), st["c0"].copy()))
        cnt = srv.st["ready_count"].cpu().numpy()
        assert cnt[0] == len(completed) == NA * (rnd + 1)
        ring = srv.st["ready_ring"].cpu().numpy()[consumed: cnt[0]]
        assert [(e >> 1, e & 1) for e in ring] == [k for k, *_ in completed[consumed:]]
        B = NA
        out = _batch_bufs(B)
        srv.assemble(B, out)
        torch.cuda.synchronize()
        assert srv.st["ready_count"].cpu().numpy()[1] == consumed + B
        for b in range(B):
            key, slots, h0, c0 = completed[consumed + b]
            assert len(slots) == T + 1
            np.testing.assert_array_equal(out["obs"][b].cpu().numpy(),
                                          np.stack([s["obs"].reshape(-1) for s in slots]))
            for f, k in (("action", "action"), ("prev_action", "prev"), ("done", "done"),
                         ("reward", "reward"), ("behaviour_logp", "blp")):
                np.testing.assert_array_equal(out[f][b].cpu().numpy(), [s[k] for s in slots])
            np.testing.assert_array_equal(out["h0"][b].cpu().numpy(), h0)
            np.testing.assert_array_equal(out["c0"][b].cpu().numpy(), c0)
        consumed += B


def test_behaviour_fidelity_self_consistency():
    """S:466 / SURVEY §4.4: with frozen params, the learner forward on an assembled
    unroll reproduces the behaviour log-probs recorded at inference (ratio == 1)."""
    S, srv, ospec, params = _setup(store=True, max_n=NA)
    for call in range(T + 1):
        req = seedgen.infer_requests((84, 84, 4), A, NA, NA, seed=11, call_index=call)
        _call(srv, req)
    B = NA
    out = _batch_bufs(B, flat_obs=False)
    srv.assemble(B, out)
    L = S.Learner(S.spec_for_config("c2"), T, B, params, S.HParams(lr=0.0))
    L.step(out)
    torch.cuda.synchronize()
    logits = L.outputs()[0].cpu().numpy().astype(np.float64)
    logp = O.log_softmax(logits)
    act = out["action"].cpu().numpy()
    tlp = np.take_along_axis(logp, act[:, :, None], 2)[:, :, 0]
    blp = out["behaviour_logp"].cpu().numpy()
    assert np.max(np.abs(tlp - blp)) < 1e-4, np.max(np.abs(tlp - blp))


def test_infer_bench_shape_n1024_store():
    """The bench's c5 shape: 4096 actors, n = 1024 requests per call (the split-K /
    tiling of the big-n path), unroll store on.  Logits, actions, log-probs and the
    state table against the emulated oracle; actors not in the call untouched
    (bitwise); every called actor's first unroll slot and h0 / c0 recorded exactly."""
    import paper_1910_06591_b200 as S
    NA4, n = 4096, 1024
    spec = S.spec_for_config("c5")
    ospec = O.spec_c2()
    params = seedgen.glorot_params(O.param_layout(ospec), seed=51, bias_std=0.1)
    learner = S.Learner(spec, T, 2, params)
    srv = S.InferenceServer(spec, NA4, n, learner=learner, T=T)
    g = seedgen.rng(52)
    th = (0.5 * g.standard_normal((NA4, 256))).astype(np.float32)
    tc = (0.5 * g.standard_normal((NA4, 256))).astype(np.float32)
    tla = g.integers(-1, A, NA4).astype(np.int32)
    srv.h.copy_(torch.from_numpy(th))
    srv.c.copy_(torch.from_numpy(tc))
    srv.last_action.copy_(torch.from_numpy(tla))
    req = seedgen.infer_requests((84, 84, 4), A, NA4, n, seed=53)
    a, blp, logits = _call(srv, req)
    ra, rblp, rlg, rth, rtc, rtla = O.infer(ospec, params, th, tc, tla, req["actor_ids"],
                                            req["obs"], req["reward"], req["done"],
                                            req["uniforms"], emu=True)
    assert _relL2(logits, rlg) < 2e-2
    nb = _near_boundary(rlg, req["uniforms"].astype(np.float64))
    assert np.all((a == ra) | nb), np.nonzero((a != ra) & ~nb)
    ok = a == ra
    np.testing.assert_allclose(blp[ok], rblp[ok], atol=2e-2 * max(1.0, np.abs(rblp).max()))
    ids = req["actor_ids"]
    h_gpu, c_gpu = srv.h.cpu().numpy(), srv.c.cpu().numpy()
    assert _relL2(h_gpu[ids], rth[ids]) < 2e-2
    assert _relL2(c_gpu[ids], rtc[ids]) < 2e-2
    others = np.setdiff1d(np.arange(NA4), ids)
    np.testing.assert_array_equal(h_gpu[others], th[others])
    np.testing.assert_array_equal(c_gpu[others], tc[others])
    np.testing.assert_array_equal(srv.last_action.cpu().numpy()[ids], a)
    np.testing.assert_array_equal(srv.last_action.cpu().numpy()[others], tla[others])
    # unroll store: slot 0 of buffer 0 of each called actor (C17, C19)
    st = {k: v.cpu().numpy() for k, v in srv.st.items()}
    np.testing.assert_array_equal(st["fill"][ids], 1)
    np.testing.assert_array_equal(st["fill"][others], 0)
    np.testing.assert_array_equal(st["obs"][ids, 0, 0], req["obs"].reshape(n, -1))
    np.testing.assert_array_equal(st["action"][ids, 0, 0], a)
    np.testing.assert_array_equal(st["behaviour_logp"][ids, 0, 0], blp)
    np.testing.assert_array_equal(st["reward"][ids, 0, 0], req["reward"])
    np.testing.assert_array_equal(st["done"][ids, 0, 0], req["done"])
    np.testing.assert_array_equal(st["prev_action"][ids, 0, 0], tla[ids])
    np.testing.assert_array_equal(st["h0"][ids, 0], th[ids])
    np.testing.assert_array_equal(st["c0"][ids, 0], tc[ids])


def test_infer_out_of_range_actor_ids():
    """An actor id outside [0, num_actors) is reported on the device (action -1,
    NaN log-prob and logits), reads and writes nothing; the valid requests of the
    same call are unaffected."""
    S, srv, ospec, params = _setup(store=True, max_n=16)
    th, tc, tla = (srv.h.cpu().numpy(), srv.c.cpu().numpy(), srv.last_action.cpu().numpy())
    req = seedgen.infer_requests((84, 84, 4), A, NA, 8, seed=71)
    bad = np.array([3, 5])
    req["actor_ids"][3] = NA + 5
    req["actor_ids"][5] = -2
    a, blp, logits = _call(srv, req)
    assert np.all(a[bad] == -1) and np.all(np.isnan(blp[bad])) and np.all(np.isnan(logits[bad]))
    ok = np.setdiff1d(np.arange(8), bad)
    ids = req["actor_ids"][ok]
    sub = {k: v[ok] for k, v in req.items()}
    ra, rblp, rlg, rth, rtc, _ = O.infer(ospec, params, th, tc, tla, ids, sub["obs"], sub["reward"],
                                         sub["done"], sub["uniforms"], emu=True)
    assert _relL2(logits[ok], rlg) < 2e-2
    nb = _near_boundary(rlg, sub["uniforms"].astype(np.float64))
    assert np.all((a[ok] == ra) | nb)
    others = np.setdiff1d(np.arange(NA), ids)
    np.testing.assert_array_equal(srv.h.cpu().numpy()[others], th[others])
    np.testing.assert_array_equal(srv.last_action.cpu().numpy()[others], tla[others])
    fill = srv.st["fill"].cpu().numpy()
    np.testing.assert_array_equal(fill[ids], 1)
    np.testing.assert_array_equal(fill[others], 0)


def test_store_stale_and_short_assemble_reported():
    """an unroll whose buffer was reused before it was assembled
    (the actor completed its next unroll) is counted in ready_count[2]; asking for
    more unrolls than are pushed and unconsumed is counted in ready_count[3]."""
    S, srv, ospec, params = _setup(store=True, max_n=NA)
    call = 0
    for _ in range(T + 1):                        # every actor completes unroll 0
        _call(srv, seedgen.infer_requests((84, 84, 4), A, NA, NA, seed=72, call_index=call))
        call += 1
    out = _batch_bufs(NA // 2)
    srv.assemble(NA // 2, out)                    # fresh: nothing stale
    torch.cuda.synchronize()
    assert srv.st["ready_count"].cpu().numpy()[2:].tolist() == [0, 0]
    for _ in range(T):                            # unroll 1 completes: unroll 0 buffers reused
        _call(srv, seedgen.infer_requests((84, 84, 4), A, NA, NA, seed=72, call_index=call))
        call += 1
    srv.assemble(NA // 2, out)                    # the other half of unroll 0: all stale
    torch.cuda.synchronize()
    rc = srv.st["ready_count"].cpu().numpy()
    assert rc[2] == NA // 2 and rc[3] == 0, rc
    big = _batch_bufs(NA + 1)
    srv.assemble(NA + 1, big)                     # NA pushed and unconsumed (unroll 1) < NA + 1
    torch.cuda.synchronize()
    rc = srv.st["ready_count"].cpu().numpy()
    assert rc[3] == 1, rc


def test_stage_requests_host_fed_equals_device_fed():
    """H12 host side (seed_stage_requests): the requests' observations gathered from
    per-actor host buffers into pinned staging by the stager's threads and copied in
    chunks give exactly the device-fed call's results (bit-exact staging)."""
    S, srv, ospec, params = _setup(store=False, max_n=16)
    S2, srv2, _, _ = _setup(store=False, max_n=16)
    g = seedgen.rng(81)
    frames = g.integers(0, 256, size=(NA, 84 * 84 * 4), dtype=np.uint8)   # the actors' latest obs
    req = seedgen.infer_requests((84, 84, 4), A, NA, 16, seed=82)
    ids = req["actor_ids"]
    ids_d, obs_d, rw_d, dn_d = srv.stage_requests([frames[i] for i in ids], ids, req["reward"],
                                                  req["done"], threads=4, chunk=5)
    u = torch.from_numpy(req["uniforms"]).cuda()
    a1, b1 = srv.infer(ids_d, obs_d, rw_d, dn_d, u)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(obs_d.cpu().numpy(), frames[ids])
    np.testing.assert_array_equal(ids_d.cpu().numpy(), ids)
    np.testing.assert_array_equal(rw_d.cpu().numpy(), req["reward"])
    np.testing.assert_array_equal(dn_d.cpu().numpy(), req["done"])
    dev = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in req.items()}
    a2, b2 = srv2.infer(dev["actor_ids"], torch.from_numpy(frames[ids]).cuda(), dev["reward"],
                        dev["done"], u)
    torch.cuda.synchronize()
    assert torch.equal(a1, a2) and torch.equal(b1, b2)
    assert torch.equal(srv.h, srv2.h) and torch.equal(srv.c, srv2.c)
    # the table form (frames indexed by actor id, pointers computed vectorised) stages
    # the same bytes
    ids_t, obs_t, rw_t, dn_t = srv.stage_requests_table(frames, ids, req["reward"], req["done"])
    torch.cuda.synchronize()
    np.testing.assert_array_equal(obs_t.cpu().numpy(), frames[ids])
    np.testing.assert_array_equal(ids_t.cpu().numpy(), ids)
    np.testing.assert_array_equal(rw_t.cpu().numpy(), req["reward"])
    np.testing.assert_array_equal(dn_t.cpu().numpy(), req["done"])


def test_wire_actors_to_inference_and_back():
    """f4: actors stream uint8 frames over SEEDWire to the
    library's batching server; each batch runs through seed_infer and the actions
    go back to the originating connections.  The actions every actor received equal
    those of a replay of the same batches (rows, frames, rewards, dones, uniforms) on
    a fresh server with the same parameters and state table — bit-exact."""
    import threading
    from paper_1910_06591_b200 import wire as Wr
    NACT, NENV, STEPS, OBS = 6, 2, 4, 84 * 84 * 4
    S, srv, _, params = _setup(seed=5, store=False, max_n=8)
    S2, srv2, _, _ = _setup(seed=5, store=False, max_n=8)     # the replay target (same init)
    ws = Wr.WireServer(OBS, NA, max_batch=8, max_wait_us=2000)
    received, errors = {}, []

    def actor(aid):
        try:
            c = Wr.ActorClient(ws.port, aid, NENV)
            rng = np.random.default_rng(aid)
            for step in range(STEPS):
                for e in range(NENV):
                    c.send_step(e, float(rng.normal()), step == 0, rng.integers(0, 256, OBS, dtype=np.uint8))
                for _ in range(NENV):
                    t, (env, act) = c.recv()
                    received.setdefault((aid, env), []).append(act)
            c.close()
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    threads = [threading.Thread(target=actor, args=(i,)) for i in range(NACT)]
    for t in threads:
        t.start()
    log, served, g = [], 0, np.random.default_rng(99)
    t_end = __import__("time").time() + 120
    while served < NACT * NENV * STEPS and __import__("time").time() < t_end:
        obs, rows, rew, done = ws.next_batch(timeout_us=200000)
        n = len(rows)
        if n == 0:
            continue
        u = g.random(n).astype(np.float32)
        req = dict(actor_ids=rows.copy(), obs=obs.reshape(n, 84, 84, 4).copy(), reward=rew.copy(),
                   done=done.copy(), uniforms=u)
        a, _, _ = _call(srv, req)
        ws.reply(rows, a)
        log.append((req, a.copy()))
        served += n
    for t in threads:
        t.join(timeout=60)
    ws.close()
    assert not errors, errors
    assert served == NACT * NENV * STEPS
    # rows were assigned per Hello in connection order; map them back via the log
    per_row = {}
    for req, a in log:
        for r, act in zip(req["actor_ids"].tolist(), a.tolist()):
            per_row.setdefault(r, []).append(act)
    assert sorted(len(v) for v in per_row.values()) == [STEPS] * (NACT * NENV)
    assert sorted(map(tuple, per_row.values())) == sorted(map(tuple, received.values()))
    for req, a in log:   # replay on the fresh server: the same actions, bit for bit
        a2, _, _ = _call(srv2, req)
        np.testing.assert_array_equal(a2, a)


def test_infer_eps_greedy_r2d2_actors():
    """R2D2 actors (seed_infer_eps_greedy; P:591 dueling heads, P:614 per-actor
    epsilon-greedy): Q vs the oracle (C22), the explore / greedy decisions bit-exact
    (greedy = first maximum of the kernel's own Q; explore = floor(u1 * A)), the
    behaviour log-probs and the state table against the oracle; the Philox path is
    reproducible."""
    S, srv, ospec, params = _setup(store=False)
    th, tc, tla = (srv.h.cpu().numpy(), srv.c.cpu().numpy(), srv.last_action.cpu().numpy())
    n = 16
    req = seedgen.infer_requests((84, 84, 4), A, NA, n, seed=11)
    req["done"][:2] = 1
    g = np.random.default_rng(3)
    u = np.stack([np.where(np.arange(n) % 2 == 0, 0.0, 1.0), g.random(n)], axis=1).astype(np.float32)
    d = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in req.items()}
    q = torch.empty(n, A, device="cuda")
    a, blp = srv.infer_eps_greedy(d["actor_ids"], d["obs"], d["reward"], d["done"],
                                  torch.from_numpy(u).cuda(), num_actors_eps=NA, q_out=q)
    torch.cuda.synchronize()
    a, blp, q = a.cpu().numpy(), blp.cpu().numpy(), q.cpu().numpy()
    ra, rblp, rq, rth, rtc, rtla = O.infer_eps_greedy(ospec, params, th, tc, tla, req["actor_ids"],
                                                       req["obs"], req["reward"], req["done"], u, NA,
                                                       emu=True)
    assert _relL2(q, rq) < 2e-2
    ids = req["actor_ids"]
    explore = u[:, 0] < np.array([O.actor_epsilon(int(i), NA) for i in ids])
    assert explore.sum() == n // 2
    np.testing.assert_array_equal(a[explore], np.minimum(np.floor(u[explore, 1] * A), A - 1))
    np.testing.assert_array_equal(a[~explore], np.argmax(q[~explore], axis=1))   # first maximum
    np.testing.assert_array_equal(a, ra)
    eps = np.array([O.actor_epsilon(int(i), NA) for i in ids])
    greedy = np.argmax(q, axis=1)
    np.testing.assert_allclose(blp, np.log(eps / A + (1 - eps) * (a == greedy)), rtol=1e-5, atol=1e-6)
    assert _relL2(srv.h.cpu().numpy()[ids], rth[ids]) < 2e-2
    np.testing.assert_array_equal(srv.last_action.cpu().numpy()[ids], a)
    # Philox draws: same (seed, counter, state) -> same actions
    S2, srv2, _, _ = _setup(store=False)
    S3, srv3, _, _ = _setup(store=False)
    outs = []
    for s in (srv2, srv3):
        aa, _ = s.infer_eps_greedy(d["actor_ids"], d["obs"], d["reward"], d["done"], None, seed=5,
                                   counter=9, num_actors_eps=NA)
        outs.append(aa.cpu().numpy())
    np.testing.assert_array_equal(outs[0], outs[1])
