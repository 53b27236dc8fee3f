// wire.cu — actor transport and server-side batching (
// P:95-96 "streaming gRPC ... the connection from actor to learner is kept open
// and metadata sent only once", "a batching module that efficiently batches
// multiple actor inference calls together"; wire format SEEDWire v1, SPEC.md
// S:350-414).  Host code only: it feeds the inference batch (seed_infer via the
// caller) and routes the actions back.
//
// One I/O thread owns every socket (poll over the listener and the connections):
// it accepts, reassembles length-prefixed frames from arbitrary fragments, and
// turns Hello (actor id, number of environments: the once-only metadata) into a
// block of state-table rows, StepRequest into a pending entry of the batcher.
// seed_wire_next_batch blocks until max_batch entries are pending or the oldest
// has waited max_wait_us, copies them (observation, row, reward, done)
// into the caller's host buffers, and seed_wire_reply sends ActionResponse frames
// to the originating connections (exactly once per request, per-connection
// order preserved: a connection's entries are taken in arrival order).
#include <arpa/inet.h>
#include <errno.h>
#include <fcntl.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <poll.h>
#include <string.h>
#include <sys/socket.h>
#include <unistd.h>
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <deque>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>
#include "common.cuh"

namespace {

constexpr uint32_t WIRE_MAX_FRAME = 16u << 20;
enum : uint8_t { W_ERROR = 0x00, W_HELLO = 0x01, W_STEP = 0x02, W_ACTION = 0x03, W_STEP_U8 = 0x04 };
using Clock = std::chrono::steady_clock;

struct Conn {
  int fd = -1;
  int actor_id = -1, num_envs = 0, row_base = -1;
  std::vector<uint8_t> rbuf;
  std::vector<uint8_t> inflight;   // per env: a request waiting for its action
  bool dead = false;
  std::mutex wmu;                  // response writes are serialised per connection
};

struct Entry {
  std::shared_ptr<Conn> conn;
  int env, row;
  float reward;
  uint8_t done;
  std::vector<uint8_t> obs;
  Clock::time_point t;
};

uint32_t rd32(const uint8_t* p) { uint32_t v; memcpy(&v, p, 4); return v; }   // little-endian host
void wr32(std::vector<uint8_t>& b, uint32_t v) { const uint8_t* p = (const uint8_t*)&v; b.insert(b.end(), p, p + 4); }

bool send_all(int fd, const uint8_t* p, size_t n) {
  while (n) {
    const ssize_t k = send(fd, p, n, MSG_NOSIGNAL);
    if (k < 0) {
      if (errno == EINTR) continue;
      if (errno == EAGAIN || errno == EWOULDBLOCK) {
        pollfd pf{fd, POLLOUT, 0};
        poll(&pf, 1, 100);
        continue;
      }
      return false;
    }
    p += k;
    n -= (size_t)k;
  }
  return true;
}

}  // namespace

struct seed_wire_server {
  int listen_fd = -1, port = 0;
  int max_batch = 32, max_wait_us = 1000, obs_bytes = 0, max_rows = 0;
  std::thread io;
  std::atomic<bool> stop{false};
  std::mutex mu;
  std::condition_variable cv;
  std::vector<std::shared_ptr<Conn>> conns;          // I/O thread only
  std::deque<Entry> pending;                         // guarded by mu
  std::vector<std::pair<std::shared_ptr<Conn>, int>> owner;   // row -> (connection, env); guarded by mu
  int next_row = 0;                                  // guarded by mu
  int64_t stats[6] = {0, 0, 0, 0, 0, 0};             // batches, requests, size / deadline / timeout polls, errors

  void error_close(const std::shared_ptr<Conn>& c, uint16_t code, const char* msg) {
    std::vector<uint8_t> f;
    const uint16_t ml = (uint16_t)strlen(msg);
    wr32(f, 1 + 4 + ml);
    f.push_back(W_ERROR);
    f.insert(f.end(), (const uint8_t*)&code, (const uint8_t*)&code + 2);
    f.insert(f.end(), (const uint8_t*)&ml, (const uint8_t*)&ml + 2);
    f.insert(f.end(), (const uint8_t*)msg, (const uint8_t*)msg + ml);
    {
      std::lock_guard<std::mutex> g(c->wmu);
      send_all(c->fd, f.data(), f.size());
    }
    std::lock_guard<std::mutex> g(mu);
    c->dead = true;
    ++stats[5];
  }

  // one frame (type + payload of `len` bytes); false: protocol error (connection closed)
  bool frame(const std::shared_ptr<Conn>& c, const uint8_t* p, uint32_t len) {
    const uint8_t type = p[0];
    const uint8_t* q = p + 1;
    const uint32_t pl = len - 1;
    if (type == W_HELLO) {
      if (pl != 8 || c->actor_id >= 0) { error_close(c, 2, "bad Hello"); return false; }
      const int actor = (int)rd32(q), envs = (int)rd32(q + 4);
      {
        std::lock_guard<std::mutex> g(mu);
        if (envs >= 1 && next_row + envs <= max_rows) {
          c->actor_id = actor; c->num_envs = envs; c->row_base = next_row;
          c->inflight.assign(envs, 0);
          for (int e = 0; e < envs; ++e) owner.emplace_back(c, e);
          next_row += envs;
          return true;
        }
      }
      error_close(c, 7, "no state-table rows left for this actor");
      return false;
    }
    if (type == W_STEP || type == W_STEP_U8) {
      if (c->actor_id < 0 || pl < 13) { error_close(c, 3, "StepRequest before Hello"); return false; }
      const uint32_t env = rd32(q), cnt = rd32(q + 9);
      float reward;
      memcpy(&reward, q + 4, 4);
      const uint8_t done = q[8];
      const size_t esz = type == W_STEP ? 4 : 1;
      if ((int)env >= c->num_envs || (size_t)pl != 13 + (size_t)cnt * esz || (int)cnt != obs_bytes) {
        error_close(c, 4, "bad StepRequest");
        return false;
      }
      Entry e;
      e.conn = c; e.env = (int)env; e.row = c->row_base + (int)env; e.reward = reward; e.done = done;
      e.obs.resize(obs_bytes);
      if (type == W_STEP_U8) {
        memcpy(e.obs.data(), q + 13, obs_bytes);
      } else {   // f32 observations (SEEDWire v1): pixel values rounded and clamped to 0..255
        for (int i = 0; i < obs_bytes; ++i) {
          float v;
          memcpy(&v, q + 13 + 4 * (size_t)i, 4);
          e.obs[i] = (uint8_t)std::min(255.f, std::max(0.f, std::nearbyint(v)));
        }
      }
      e.t = Clock::now();
      {
        std::lock_guard<std::mutex> g(mu);
        if (!c->inflight[env]) {   // actors are lock-step per environment
          c->inflight[env] = 1;
          pending.push_back(std::move(e));
          ++stats[1];
          if ((int)pending.size() >= max_batch) cv.notify_all();
          return true;
        }
      }
      error_close(c, 5, "duplicate in-flight request");
      return false;
    }
    if (type == W_ERROR) {
      std::lock_guard<std::mutex> g(mu);
      c->dead = true;
      return false;
    }
    error_close(c, 1, "unknown message type");
    return false;
  }

  void run() {
    std::vector<uint8_t> tmp(1 << 16);
    while (!stop.load()) {
      std::vector<pollfd> pf;
      pf.push_back({listen_fd, POLLIN, 0});
      for (auto& c : conns) pf.push_back({c->fd, POLLIN, 0});
      const int r = poll(pf.data(), pf.size(), 1);
      if (r < 0 && errno != EINTR) break;
      {   // deadline trigger: wake a waiting next_batch when the oldest entry is due
        std::lock_guard<std::mutex> g(mu);
        if (!pending.empty() &&
            Clock::now() - pending.front().t >= std::chrono::microseconds(max_wait_us))
          cv.notify_all();
      }
      if (r <= 0) continue;
      if (pf[0].revents & POLLIN) {
        const int fd = accept(listen_fd, nullptr, nullptr);
        if (fd >= 0) {
          const int one = 1;
          setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &one, sizeof(one));
          auto c = std::make_shared<Conn>();
          c->fd = fd;
          conns.push_back(c);
        }
      }
      for (size_t i = 1; i < pf.size(); ++i) {
        auto& c = conns[i - 1];
        if (!(pf[i].revents & (POLLIN | POLLHUP | POLLERR))) continue;
        const ssize_t k = recv(c->fd, tmp.data(), tmp.size(), 0);
        if (k <= 0) {
          if (k < 0 && (errno == EINTR || errno == EAGAIN)) continue;
          std::lock_guard<std::mutex> g(mu);
          c->dead = true;
          continue;
        }
        c->rbuf.insert(c->rbuf.end(), tmp.data(), tmp.data() + k);
        size_t off = 0;
        bool ok = true;
        while (ok && c->rbuf.size() - off >= 4) {   // reassemble frames
          const uint32_t len = rd32(c->rbuf.data() + off);
          if (len < 1 || len > WIRE_MAX_FRAME) { error_close(c, 6, "bad frame length"); ok = false; break; }
          if (c->rbuf.size() - off < 4 + (size_t)len) break;   // incomplete: await more bytes
          ok = frame(c, c->rbuf.data() + off + 4, len);
          off += 4 + len;
        }
        c->rbuf.erase(c->rbuf.begin(), c->rbuf.begin() + off);
      }
      // drop closed connections (their pending entries are still answered, to a dead socket)
      for (size_t i = 0; i < conns.size();) {
        bool dead;
        {
          std::lock_guard<std::mutex> g(mu);
          dead = conns[i]->dead;
        }
        if (dead) {
          std::lock_guard<std::mutex> w(conns[i]->wmu);   // not while a reply is being written
          close(conns[i]->fd);
          conns[i]->fd = -1;
          conns.erase(conns.begin() + i);
        } else {
          ++i;
        }
      }
    }
  }
};

extern "C" {

seed_status seed_wire_server_create(int port, int max_batch, int max_wait_us, int obs_bytes, int max_rows,
                                    seed_wire_server** out, int* port_out) {
  if (!out || max_batch < 1 || max_wait_us < 0 || obs_bytes < 1 || max_rows < 1 || port < 0 || port > 65535)
    return SEED_E_ARG;
  auto* s = new seed_wire_server();
  s->max_batch = max_batch; s->max_wait_us = max_wait_us; s->obs_bytes = obs_bytes; s->max_rows = max_rows;
  s->listen_fd = socket(AF_INET, SOCK_STREAM, 0);
  const int one = 1;
  setsockopt(s->listen_fd, SOL_SOCKET, SO_REUSEADDR, &one, sizeof(one));
  sockaddr_in a{};
  a.sin_family = AF_INET;
  a.sin_port = htons((uint16_t)port);
  a.sin_addr.s_addr = htonl(INADDR_LOOPBACK);
  socklen_t al = sizeof(a);
  if (s->listen_fd < 0 || bind(s->listen_fd, (sockaddr*)&a, sizeof(a)) != 0 || listen(s->listen_fd, 256) != 0 ||
      getsockname(s->listen_fd, (sockaddr*)&a, &al) != 0) {
    if (s->listen_fd >= 0) close(s->listen_fd);
    delete s;
    return SEED_E_ARG;
  }
  s->port = ntohs(a.sin_port);
  if (port_out) *port_out = s->port;
  s->io = std::thread([s] { s->run(); });
  *out = s;
  return SEED_OK;
}

seed_status seed_wire_server_destroy(seed_wire_server* s) {
  if (!s) return SEED_OK;
  s->stop.store(true);
  if (s->io.joinable()) s->io.join();
  for (auto& c : s->conns)
    if (c->fd >= 0) close(c->fd);
  close(s->listen_fd);
  delete s;
  return SEED_OK;
}

seed_status seed_wire_next_batch(seed_wire_server* s, int timeout_us, uint8_t* obs_out, int32_t* rows_out,
                                 float* reward_out, uint8_t* done_out, int* n_out) {
  if (!s || !obs_out || !rows_out || !reward_out || !done_out || !n_out) return SEED_E_ARG;
  std::unique_lock<std::mutex> g(s->mu);
  const auto t_end = Clock::now() + std::chrono::microseconds(timeout_us);
  int trigger = 4;   // 2 size, 3 deadline, 4 timeout
  for (;;) {
    if ((int)s->pending.size() >= s->max_batch) { trigger = 2; break; }
    const auto now = Clock::now();
    if (!s->pending.empty() && now - s->pending.front().t >= std::chrono::microseconds(s->max_wait_us)) {
      trigger = 3;
      break;
    }
    if (now >= t_end) break;
    auto until = t_end;
    if (!s->pending.empty())
      until = std::min(until, s->pending.front().t + std::chrono::microseconds(s->max_wait_us));
    s->cv.wait_until(g, until);
  }
  const int n = std::min<int>((int)s->pending.size(), s->max_batch);
  for (int i = 0; i < n; ++i) {
    Entry& e = s->pending[i];
    memcpy(obs_out + (size_t)i * s->obs_bytes, e.obs.data(), s->obs_bytes);
    rows_out[i] = e.row; reward_out[i] = e.reward; done_out[i] = e.done;
  }
  s->pending.erase(s->pending.begin(), s->pending.begin() + n);
  if (n > 0) { ++s->stats[0]; ++s->stats[trigger]; }
  *n_out = n;
  return SEED_OK;
}

seed_status seed_wire_reply(seed_wire_server* s, int n, const int32_t* rows, const int32_t* actions) {
  if (!s || n < 0 || (n > 0 && (!rows || !actions))) return SEED_E_ARG;
  for (int i = 0; i < n; ++i) {
    std::shared_ptr<Conn> c;
    int env;
    {
      std::lock_guard<std::mutex> g(s->mu);
      if (rows[i] < 0 || rows[i] >= (int)s->owner.size()) return SEED_E_ARG;
      c = s->owner[rows[i]].first;
      env = s->owner[rows[i]].second;
      if (!c->inflight[env]) return SEED_E_ARG;   // no request waiting on that row
      c->inflight[env] = 0;
      if (c->dead) continue;
    }
    std::vector<uint8_t> f;
    wr32(f, 9);
    f.push_back(W_ACTION);
    wr32(f, (uint32_t)env);
    wr32(f, (uint32_t)actions[i]);
    std::lock_guard<std::mutex> g(c->wmu);
    if (c->fd >= 0) send_all(c->fd, f.data(), f.size());
  }
  return SEED_OK;
}

seed_status seed_wire_server_stats(seed_wire_server* s, int64_t* stats6, int* rows_assigned) {
  if (!s || !stats6) return SEED_E_ARG;
  std::lock_guard<std::mutex> g(s->mu);
  for (int k = 0; k < 6; ++k) stats6[k] = s->stats[k];
  if (rows_assigned) *rows_assigned = s->next_row;
  return SEED_OK;
}

}  // extern "C"
