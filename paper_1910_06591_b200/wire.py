"""Actor transport: the learner-side
server is `WireServer` over libseed's seed_wire_* (include/seed.h: SEEDWire v1
framing, server-side batching by size or deadline, exactly-once routed replies);
this module also has the actor side — SEEDWire v1 frame encoding / incremental
decoding and a blocking `ActorClient` — which is plain host
networking (no GPU work)."""
import ctypes as C
import socket
import struct

import numpy as np

from . import _lib as L

HELLO, STEP, ACTION, ERROR, STEP_U8 = 0x01, 0x02, 0x03, 0x00, 0x04
MAX_FRAME = 16 << 20


def frame(msg_type, payload=b""):
    """u32 LE length (of type byte + payload) | u8 type | payload."""
    return struct.pack("<IB", 1 + len(payload), msg_type) + payload


def encode_hello(actor_id, num_envs):
    return frame(HELLO, struct.pack("<II", actor_id, num_envs))


def encode_step(env_id, reward, done, obs):
    """StepRequest: f32 observations; uint8 arrays go as StepRequest-u8 (0x04)."""
    obs = np.asarray(obs)
    if obs.dtype == np.uint8:
        return frame(STEP_U8, struct.pack("<IfBI", env_id, reward, int(bool(done)), obs.size) + obs.tobytes())
    o = obs.astype("<f4").ravel()
    return frame(STEP, struct.pack("<IfBI", env_id, reward, int(bool(done)), o.size) + o.tobytes())


def encode_action(env_id, action):
    return frame(ACTION, struct.pack("<II", env_id, action))


def encode_error(code, msg):
    m = msg.encode()
    return frame(ERROR, struct.pack("<HH", code, len(m)) + m)


class Decoder:
    """Incremental frame decoder: feed arbitrary fragments, get whole messages
    (type, fields) in order; a truncated frame waits for more bytes."""

    def __init__(self):
        self.buf = b""

    def feed(self, data):
        self.buf += data
        out = []
        while len(self.buf) >= 4:
            (n,) = struct.unpack_from("<I", self.buf)
            if n < 1 or n > MAX_FRAME:
                raise ValueError("bad frame length")
            if len(self.buf) < 4 + n:
                break
            t, p = self.buf[4], self.buf[5:4 + n]
            self.buf = self.buf[4 + n:]
            if t == HELLO:
                out.append((t, struct.unpack("<II", p)))
            elif t == ACTION:
                out.append((t, struct.unpack("<II", p)))
            elif t in (STEP, STEP_U8):
                env, rew, done, cnt = struct.unpack_from("<IfBI", p)
                obs = np.frombuffer(p[13:], dtype="<f4" if t == STEP else np.uint8)
                assert obs.size == cnt
                out.append((t, (env, rew, done, obs)))
            elif t == ERROR:
                code, ln = struct.unpack_from("<HH", p)
                out.append((t, (code, p[4:4 + ln].decode())))
            else:
                raise ValueError(f"unknown message type {t}")
        return out


class ActorClient:
    """One actor: a persistent connection, Hello once, then lock-step
    StepRequest / ActionResponse per environment."""

    def __init__(self, port, actor_id, num_envs, host="127.0.0.1"):
        self.sock = socket.create_connection((host, port))
        self.sock.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
        self.dec = Decoder()
        self.inbox = []
        self.sock.sendall(encode_hello(actor_id, num_envs))

    def send_step(self, env_id, reward, done, obs):
        self.sock.sendall(encode_step(env_id, reward, done, obs))

    def recv(self):
        while not self.inbox:
            data = self.sock.recv(1 << 16)
            if not data:
                raise ConnectionError("server closed the connection")
            self.inbox.extend(self.dec.feed(data))
        return self.inbox.pop(0)

    def close(self):
        self.sock.close()


class WireServer:
    """Learner side: seed_wire_server (accepts actors, batches their requests)."""

    def __init__(self, obs_bytes, max_rows, max_batch=32, max_wait_us=1000, port=0):
        self.lib = L.load()
        self.obs_bytes, self.max_batch = obs_bytes, max_batch
        h, pt = C.c_void_p(), C.c_int()
        L.check(self.lib.seed_wire_server_create(port, max_batch, max_wait_us, obs_bytes, max_rows,
                                                 C.byref(h), C.byref(pt)), "wire_server_create")
        self.h, self.port = h, pt.value
        self.obs = np.zeros((max_batch, obs_bytes), dtype=np.uint8)
        self.rows = np.zeros(max_batch, dtype=np.int32)
        self.reward = np.zeros(max_batch, dtype=np.float32)
        self.done = np.zeros(max_batch, dtype=np.uint8)

    def next_batch(self, timeout_us=100000):
        """(obs [n][obs_bytes] uint8, rows int32, reward f32, done u8) views, n may be 0."""
        n = C.c_int()
        L.check(self.lib.seed_wire_next_batch(self.h, timeout_us, self.obs.ctypes.data, self.rows.ctypes.data,
                                              self.reward.ctypes.data, self.done.ctypes.data, C.byref(n)),
                "wire_next_batch")
        k = n.value
        return self.obs[:k], self.rows[:k], self.reward[:k], self.done[:k]

    def reply(self, rows, actions):
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        actions = np.ascontiguousarray(actions, dtype=np.int32)
        L.check(self.lib.seed_wire_reply(self.h, len(rows), rows.ctypes.data, actions.ctypes.data), "wire_reply")

    def stats(self):
        s = (C.c_int64 * 6)()
        r = C.c_int()
        L.check(self.lib.seed_wire_server_stats(self.h, s, C.byref(r)), "wire_stats")
        keys = ("batches", "requests", "by_size", "by_deadline", "by_timeout", "errors")
        return dict(zip(keys, list(s))) | {"rows": r.value}

    def close(self):
        if self.h:
            self.lib.seed_wire_server_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
