// host_stage.cu — host side of the inference batch assembly (
// P:96 "streaming ... batching", P:125 the inference batch): the n
// requests' observations, wherever the actor transport left them in host memory
// (one buffer per actor), are packed by a caller-owned pool of worker threads
// (seed_stager) into contiguous pinned staging and copied to the device with one
// cudaMemcpyAsync per chunk, issued as soon as that chunk is packed — the copy of
// chunk k overlaps the packing of the chunks after it.  The request metadata
// (actor id, reward, done) goes in one small copy in seed_infer's layouts.
#include <string.h>
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <vector>
#include "common.cuh"

struct seed_stager {
  std::vector<std::thread> workers;
  std::mutex mu;
  std::condition_variable cv;
  bool quit = false;
  uint64_t job_id = 0;
  // the current job (valid while job_id is odd... see run())
  int n = 0, chunk = 0, slice = 0, ntasks = 0;
  const uint8_t* const* ptrs = nullptr;
  size_t obs_bytes = 0;
  uint8_t* dst = nullptr;
  std::atomic<int> next_task{0};
  std::atomic<int> active{0};
  std::vector<std::atomic<int>> packed;   // requests packed per chunk

  void work(int i0, int i1) {
    for (int i = i0; i < i1; ++i) memcpy(dst + (size_t)i * obs_bytes, ptrs[i], obs_bytes);
  }
  // tasks = (chunk, slice of it), taken in order so early chunks finish first
  void drain() {
    const int per_chunk = (chunk + slice - 1) / slice;
    for (;;) {
      const int t = next_task.fetch_add(1);
      if (t >= ntasks) break;
      const int c = t / per_chunk, s = t % per_chunk;
      const int c0 = c * chunk, c1 = std::min(n, c0 + chunk);
      const int i0 = c0 + s * slice, i1 = std::min(c1, i0 + slice);
      if (i0 < i1) {
        work(i0, i1);
        packed[c].fetch_add(i1 - i0, std::memory_order_release);
      }
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return quit || job_id != seen; });
        if (quit) return;
        seen = job_id;
        active.fetch_add(1);
      }
      drain();
      active.fetch_sub(1, std::memory_order_release);
    }
  }
};

using namespace seed;

extern "C" seed_status seed_stager_create(int threads, seed_stager** out) {
  if (!out || threads < 1 || threads > 64) return SEED_E_ARG;
  seed_stager* s = new seed_stager();
  for (int t = 0; t < threads; ++t) s->workers.emplace_back([s] { s->loop(); });
  *out = s;
  return SEED_OK;
}

extern "C" seed_status seed_stager_destroy(seed_stager* s) {
  if (!s) return SEED_OK;
  {
    std::lock_guard<std::mutex> lk(s->mu);
    s->quit = true;
  }
  s->cv.notify_all();
  for (auto& t : s->workers) t.join();
  delete s;
  return SEED_OK;
}

extern "C" seed_status seed_stage_requests(seed_stager* sg, int n, const uint8_t* const* obs_ptrs,
                                           size_t obs_bytes, const int32_t* actor_ids,
                                           const float* rewards, const uint8_t* dones,
                                           uint8_t* pinned_obs, uint8_t* pinned_meta, uint8_t* dev_obs,
                                           uint8_t* dev_meta, int chunk, void* stream) {
  if (!sg || n < 1 || !obs_ptrs || obs_bytes == 0 || !pinned_obs || !dev_obs) return SEED_E_ARG;
  if ((actor_ids || rewards || dones) && (!actor_ids || !rewards || !dones || !pinned_meta || !dev_meta))
    return SEED_E_ARG;
  for (int i = 0; i < n; ++i)
    if (!obs_ptrs[i]) return SEED_E_ARG;
  chunk = chunk > 0 ? std::min(chunk, n) : std::min(128, n);
  cudaStream_t st = (cudaStream_t)stream;
  // metadata, one small copy: int32 actor ids at byte 0, fp32 rewards at 4n, uint8
  // dones at 8n (the seed_infer argument layouts)
  if (actor_ids) {
    memcpy(pinned_meta, actor_ids, (size_t)n * 4);
    memcpy(pinned_meta + (size_t)4 * n, rewards, (size_t)n * 4);
    memcpy(pinned_meta + (size_t)8 * n, dones, (size_t)n);
    SEED_CUDA_TRY(cudaMemcpyAsync(dev_meta, pinned_meta, (size_t)9 * n, cudaMemcpyHostToDevice, st));
  }
  const int nchunks = (n + chunk - 1) / chunk;
  const int slice = std::max(1, chunk / (int)sg->workers.size());
  {
    std::lock_guard<std::mutex> lk(sg->mu);
    sg->n = n;
    sg->chunk = chunk;
    sg->slice = slice;
    sg->ptrs = obs_ptrs;
    sg->obs_bytes = obs_bytes;
    sg->dst = pinned_obs;
    sg->ntasks = nchunks * ((chunk + slice - 1) / slice);
    sg->packed = std::vector<std::atomic<int>>(nchunks);
    for (auto& p : sg->packed) p.store(0);
    sg->next_task.store(0);
    sg->job_id++;
  }
  sg->cv.notify_all();
  seed_status rc = SEED_OK;
  for (int c = 0; c < nchunks; ++c) {
    const int c0 = c * chunk, c1 = std::min(n, c0 + chunk);
    while (sg->packed[c].load(std::memory_order_acquire) < c1 - c0) std::this_thread::yield();
    if (rc == SEED_OK &&
        cudaMemcpyAsync(dev_obs + (size_t)c0 * obs_bytes, pinned_obs + (size_t)c0 * obs_bytes,
                        (size_t)(c1 - c0) * obs_bytes, cudaMemcpyHostToDevice, st) != cudaSuccess)
      rc = SEED_E_CUDA;
  }
  // every task is done (all chunks packed); wait for the workers to leave drain()
  // before the job's arrays can be reused
  while (sg->active.load(std::memory_order_acquire) > 0) std::this_thread::yield();
  return rc;
}
