"""Actor transport: SEEDWire v1 framing
 and the library's server-side batcher (include/seed.h
seed_wire_*): golden frames from the SPEC's examples, fuzzed round trips and
byte-at-a-time reassembly, the size and deadline triggers, exactly-once routed
replies with per-connection order under concurrent actors, and protocol errors.
Host only (TCP on 127.0.0.1)."""
import socket
import struct
import threading
import time

import numpy as np
import pytest

from paper_1910_06591_b200 import wire as Wr


def _server(obs_bytes=8, rows=64, B=4, wait_us=1000):
    return Wr.WireServer(obs_bytes, rows, max_batch=B, max_wait_us=wait_us)


def test_golden_frames():
    # S:391-392 (byte-for-byte examples of the SPEC)
    assert Wr.encode_hello(1, 2) == bytes.fromhex("09000000 01 01000000 02000000".replace(" ", ""))
    assert Wr.encode_step(0, 0.0, 1, np.zeros(0, np.float32)) == bytes.fromhex(
        "0E000000 02 00000000 00000000 01 00000000".replace(" ", ""))
    assert Wr.encode_action(3, 7) == struct.pack("<IBII", 9, 3, 3, 7)


def test_roundtrip_fuzz_and_fragmentation():
    rng = np.random.default_rng(0)
    msgs, raw = [], b""
    for _ in range(2000):
        k = int(rng.integers(0, 4))
        if k == 0:
            a, e = int(rng.integers(0, 2 ** 32)), int(rng.integers(0, 2 ** 32))
            msgs.append((Wr.HELLO, (a, e)))
            raw += Wr.encode_hello(a, e)
        elif k == 1:
            env, rew, done = int(rng.integers(0, 2 ** 32)), float(np.float32(rng.normal())), int(rng.integers(0, 2))
            obs = rng.normal(size=int(rng.integers(0, 9))).astype(np.float32)
            msgs.append((Wr.STEP, (env, np.float32(rew), done, obs)))
            raw += Wr.encode_step(env, rew, done, obs)
        elif k == 2:
            env, rew, done = int(rng.integers(0, 2 ** 32)), float(np.float32(rng.normal())), int(rng.integers(0, 2))
            obs = rng.integers(0, 256, size=int(rng.integers(0, 9)), dtype=np.uint8)
            msgs.append((Wr.STEP_U8, (env, np.float32(rew), done, obs)))
            raw += Wr.encode_step(env, rew, done, obs)
        else:
            e, act = int(rng.integers(0, 2 ** 32)), int(rng.integers(0, 2 ** 32))
            msgs.append((Wr.ACTION, (e, act)))
            raw += Wr.encode_action(e, act)

    def same(a, b):
        if a[0] != b[0]:
            return False
        if a[0] in (Wr.STEP, Wr.STEP_U8):
            return (a[1][0] == b[1][0] and np.float32(a[1][1]) == np.float32(b[1][1]) and a[1][2] == b[1][2]
                    and np.array_equal(a[1][3], b[1][3]))
        return tuple(a[1]) == tuple(b[1])
    whole = Wr.Decoder().feed(raw)
    d = Wr.Decoder()
    bytewise = []
    for i in range(len(raw)):
        bytewise.extend(d.feed(raw[i:i + 1]))
    assert len(whole) == len(bytewise) == len(msgs)
    assert all(same(a, b) for a, b in zip(whole, msgs))
    assert all(same(a, b) for a, b in zip(bytewise, msgs))
    with pytest.raises(ValueError):
        Wr.Decoder().feed(struct.pack("<IB", Wr.MAX_FRAME + 1, 2))


def test_size_trigger_and_rows():
    srv = _server(B=4, wait_us=10 ** 6)
    try:
        a = Wr.ActorClient(srv.port, actor_id=7, num_envs=4)
        for e in range(4):
            a.send_step(e, float(e), e == 0, np.full(8, e, np.uint8))
        t0 = time.time()
        obs, rows, rew, done = srv.next_batch(timeout_us=5 * 10 ** 6)
        assert time.time() - t0 < 0.5                       # size trigger, not the 1 s deadline
        assert len(rows) == 4 and sorted(rows.tolist()) == [0, 1, 2, 3]
        for i, r in enumerate(rows):
            assert obs[i].tolist() == [r] * 8 and rew[i] == float(r) and done[i] == (r == 0)
        srv.reply(rows, rows * 10)
        got = sorted(a.recv()[1] for _ in range(4))
        assert got == [(e, 10 * e) for e in range(4)]
        st = srv.stats()
        assert st["batches"] == 1 and st["by_size"] == 1 and st["requests"] == 4 and st["rows"] == 4
        a.close()
    finally:
        srv.close()


def test_deadline_trigger():
    srv = _server(B=4, wait_us=20000)
    try:
        a = Wr.ActorClient(srv.port, actor_id=0, num_envs=2)
        a.send_step(0, 0.0, 1, np.zeros(8, np.uint8))
        a.send_step(1, 0.0, 1, np.zeros(8, np.uint8))
        t0 = time.time()
        obs, rows, _, _ = srv.next_batch(timeout_us=2 * 10 ** 6)
        dt = time.time() - t0
        assert len(rows) == 2 and 0.01 <= dt < 1.0          # released by the 20 ms deadline
        assert srv.stats()["by_deadline"] == 1
        srv.reply(rows, [1, 2])
        a.recv(), a.recv()
        # an empty poll times out with n = 0
        obs, rows, _, _ = srv.next_batch(timeout_us=20000)
        assert len(rows) == 0
        a.close()
    finally:
        srv.close()


def test_float_observations_converted():
    srv = _server(obs_bytes=4, B=1)
    try:
        a = Wr.ActorClient(srv.port, 0, 1)
        a.send_step(0, 1.5, 0, np.array([0.0, 17.4, 254.6, 300.0], np.float32))
        obs, rows, rew, done = srv.next_batch(timeout_us=10 ** 6)
        assert obs[0].tolist() == [0, 17, 255, 255] and rew[0] == 1.5 and done[0] == 0
        srv.reply(rows, [3])
        assert a.recv() == (Wr.ACTION, (0, 3))
        a.close()
    finally:
        srv.close()


def test_exactly_once_routed_in_order_concurrent_actors():
    """1000 requests over 10 connections (4 environments each, lock-step),
    B = 32 — every request answered exactly once, to its own connection, in order."""
    NA, NE, STEPS, A = 10, 4, 25, 18
    srv = _server(obs_bytes=8, rows=NA * NE, B=32, wait_us=2000)
    errors = []

    def policy(row, step):
        return (row * 7 + step) % A

    def actor(aid):
        try:
            c = Wr.ActorClient(srv.port, aid, NE)
            for step in range(STEPS):
                for e in range(NE):
                    c.send_step(e, float(step), step == 0, np.full(8, step, np.uint8))
                got = {}
                for _ in range(NE):
                    t, (env, act) = c.recv()
                    assert t == Wr.ACTION and env not in got
                    got[env] = act
                # rows of this actor are consecutive; the learner's action encodes (row, step)
                acts = [got[e] for e in range(NE)]
                base = [r for r in range(NA * NE) if all(policy(r + e, step) == acts[e] for e in range(NE))]
                assert base, (aid, step, acts)
            c.close()
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    threads = [threading.Thread(target=actor, args=(i,)) for i in range(NA)]
    for t in threads:
        t.start()
    seen = {}
    served = 0
    deadline = time.time() + 60
    while served < NA * NE * STEPS and time.time() < deadline:
        obs, rows, _, _ = srv.next_batch(timeout_us=100000)
        if len(rows) == 0:
            continue
        steps = obs[:, 0].astype(int)
        for r, s in zip(rows.tolist(), steps.tolist()):
            assert seen.get(r, -1) == s - 1, (r, s, seen.get(r))   # per-row order, no loss / dup
            seen[r] = s
        srv.reply(rows, [policy(r, s) for r, s in zip(rows.tolist(), steps.tolist())])
        served += len(rows)
    for t in threads:
        t.join(timeout=30)
    assert not errors, errors
    assert served == NA * NE * STEPS
    st = srv.stats()
    assert st["requests"] == served and st["errors"] == 0
    assert all(v == STEPS - 1 for v in seen.values()) and len(seen) == NA * NE
    srv.close()


def test_fragmented_stream():
    srv = _server(obs_bytes=8, B=1)
    try:
        s = socket.create_connection(("127.0.0.1", srv.port))
        raw = Wr.encode_hello(5, 1) + Wr.encode_step(0, 2.0, 1, np.arange(8, dtype=np.uint8))
        for i in range(len(raw)):
            s.sendall(raw[i:i + 1])
            time.sleep(0.001)
        obs, rows, rew, done = srv.next_batch(timeout_us=2 * 10 ** 6)
        assert rows.tolist() == [0] and obs[0].tolist() == list(range(8)) and rew[0] == 2.0 and done[0] == 1
        srv.reply(rows, [4])
        assert Wr.Decoder().feed(s.recv(64)) == [(Wr.ACTION, (0, 4))]
        s.close()
    finally:
        srv.close()


@pytest.mark.parametrize("bad", ["type", "before_hello", "duplicate", "length", "wrong_size"])
def test_protocol_errors(bad):
    srv = _server(obs_bytes=8, B=8, wait_us=10 ** 6)
    try:
        s = socket.create_connection(("127.0.0.1", srv.port))
        if bad == "type":
            s.sendall(Wr.encode_hello(0, 1) + Wr.frame(0x7F, b"x"))
        elif bad == "before_hello":
            s.sendall(Wr.encode_step(0, 0.0, 0, np.zeros(8, np.uint8)))
        elif bad == "duplicate":
            s.sendall(Wr.encode_hello(0, 1) + Wr.encode_step(0, 0.0, 0, np.zeros(8, np.uint8)) * 2)
        elif bad == "length":
            s.sendall(Wr.encode_hello(0, 1) + struct.pack("<IB", Wr.MAX_FRAME + 1, 2))
        else:
            s.sendall(Wr.encode_hello(0, 1) + Wr.encode_step(0, 0.0, 0, np.zeros(5, np.uint8)))
        s.settimeout(5)
        data = b""
        while True:   # an Error frame, then the server closes the connection
            chunk = s.recv(4096)
            if not chunk:
                break
            data += chunk
        msgs = Wr.Decoder().feed(data)
        assert msgs and msgs[-1][0] == Wr.ERROR
        assert srv.stats()["errors"] == 1
        s.close()
    finally:
        srv.close()
