// run.cpp — collaboration strategy: two pinned host pools; the
// sampler threads fill one while the trainer pushes and trains the other.
// "With the collaboration strategy, the synchronization cost between CPUs
// and GPUs is reduced and the speed of our hybrid system is almost doubled."
#include <cuda_runtime.h>

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>

#include "engine.hpp"

namespace {

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

struct HostPool {
  uint32_t* pairs = nullptr;
  uint64_t count = 0;
  bool ready = false;  // filled, not yet pushed
};

}  // namespace

extern "C" gv_status gv_run(gv_ctx* c, const gv_augment_cfg* cfg, uint64_t total_samples,
                            gv_run_report* report) {
  if (!c || !cfg) return gv::fail(c, GV_ERR_INVALID_ARG, "null context or config");
  if (!c->loaded) return gv::fail(c, GV_ERR_STATE, "gv_load_edges has not been called");
  if (cfg->pool_samples == 0 || cfg->threads == 0)
    return gv::fail(c, GV_ERR_INVALID_ARG, "pool_samples and threads must be > 0");
  const uint64_t P = cfg->pool_samples;
  const uint64_t npools = (total_samples + P - 1) / P;
  gv_run_report rep;
  std::memset(&rep, 0, sizeof(rep));
  auto pool_count = [&](uint64_t k) { return std::min<uint64_t>(P, total_samples - k * P); };
  auto t0 = Clock::now();
  gv_status status = GV_OK;
  gv_episode_stats st;
  if (cfg->device) {
    // GPU-resident pipeline (NEXT-1): pool k+1 is generated on the copy
    // stream while pool k trains on the compute stream.
    // Pools are generated raw and bucketed by the trainer; GV_AUG_BLOCKS=1
    // buckets them inside the sampler (gv_augment_device_blocks) when the
    // shape allows it. Measured on C2 (profiles/r02_q_*): 2.52 / 2.13 /
    // 1.78e9 vs 2.61 / 2.11 / 1.92e9 at n = 1 / 4 / 16 — the sampler's two
    // passes (walk cache + per-tile counts, then placement) cost about as
    // much as one raw pool write plus the trainer's bucketing pass.
    const char* env = getenv("GV_AUG_BLOCKS");
    const bool blocks = env && atoi(env) != 0 &&
                        gv_augment_device_blocks(c, cfg->walk_len, cfg->s, cfg->threads,
                                                 pool_count(0), cfg->seed, GV_SHUFFLE_PSEUDO) == GV_OK;
    auto produce = [&](uint64_t k) {
      return blocks ? gv_augment_device_blocks(c, cfg->walk_len, cfg->s, cfg->threads,
                                               pool_count(k), cfg->seed + k, GV_SHUFFLE_PSEUDO)
                    : gv_augment_device(c, cfg->walk_len, cfg->s, cfg->threads, pool_count(k),
                                        cfg->seed + k);
    };
    if (!blocks) status = produce(0);
    for (uint64_t k = 0; k < npools && status == GV_OK; ++k) {
      status = gv_train_episode(c, nullptr);
      if (status == GV_OK && k + 1 < npools) status = produce(k + 1);
      if (status == GV_OK) status = gv_read_stats(c, &st);  // pool k (pool k+1 already generating)
      if (status == GV_OK) rep.loss_sum += st.loss_sum;
      if (status == GV_OK && !cfg->collaborate) status = gv_synchronize(c);
    }
    if (status == GV_OK) status = gv_synchronize(c);
    rep.pools = npools;
    rep.samples = total_samples;
    rep.wall_ms = ms_since(t0);
    if (report) *report = rep;
    return status;
  }
  HostPool pool[2];
  for (auto& p : pool)
    if (cudaMallocHost(&p.pairs, 2 * P * sizeof(uint32_t)) != cudaSuccess) {
      for (auto& q : pool)
        if (q.pairs) cudaFreeHost(q.pairs);
      return GV_ERR_NOMEM;
    }
  t0 = Clock::now();  // wall_ms excludes the one-time pinning of the two host pools
  if (!cfg->collaborate) {
    for (uint64_t k = 0; k < npools && status == GV_OK; ++k) {
      const auto tp = Clock::now();
      status = gv_augment(c, cfg->walk_len, cfg->s, cfg->threads, pool_count(k), cfg->seed + k,
                          pool[0].pairs);
      rep.produce_ms += ms_since(tp);
      if (status == GV_OK) status = gv_push_sample_pool(c, pool[0].pairs, pool_count(k));
      if (status == GV_OK) status = gv_train_episode(c, &st);  // waits: fill-then-train
      if (status == GV_OK) rep.loss_sum += st.loss_sum;
    }
  } else {
    std::mutex mu;
    std::condition_variable cv;
    bool stop = false;
    gv_status prod_status = GV_OK;
    std::thread producer([&] {
      for (uint64_t k = 0; k < npools; ++k) {
        HostPool& hp = pool[k % 2];
        {
          const auto tw = Clock::now();
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&] { return !hp.ready || stop; });
          rep.producer_wait_ms += ms_since(tw);
          if (stop) return;
        }
        const auto tp = Clock::now();
        gv_status s = gv_augment(c, cfg->walk_len, cfg->s, cfg->threads, pool_count(k),
                                 cfg->seed + k, hp.pairs);
        rep.produce_ms += ms_since(tp);
        std::lock_guard<std::mutex> lk(mu);
        if (s != GV_OK) {
          prod_status = s;
          stop = true;
          cv.notify_all();
          return;
        }
        hp.count = pool_count(k);
        hp.ready = true;
        cv.notify_all();
      }
    });
    for (uint64_t k = 0; k < npools; ++k) {
      HostPool& hp = pool[k % 2];
      {
        const auto tw = Clock::now();
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return hp.ready || stop; });
        rep.train_wait_ms += ms_since(tw);
        if (stop) break;
      }
      status = gv_push_sample_pool(c, hp.pairs, hp.count);  // H2D overlaps training of pool k-1
      {
        std::lock_guard<std::mutex> lk(mu);
        hp.ready = false;
        cv.notify_all();
      }
      // pool k-1's loss, read once pool k is staged (the GPU idles only for
      // the few microseconds between this sync and the next enqueue)
      if (status == GV_OK && k > 0) {
        status = gv_read_stats(c, &st);
        if (status == GV_OK) rep.loss_sum += st.loss_sum;
      }
      if (status == GV_OK) status = gv_train_episode(c, nullptr);
      if (status != GV_OK) {
        std::lock_guard<std::mutex> lk(mu);
        stop = true;
        cv.notify_all();
        break;
      }
    }
    producer.join();
    if (status == GV_OK) status = prod_status;
    if (status == GV_OK) status = gv_read_stats(c, &st);  // the last pool (synchronizes)
    if (status == GV_OK) rep.loss_sum += st.loss_sum;
  }
  rep.pools = npools;
  rep.samples = total_samples;
  rep.wall_ms = ms_since(t0);
  for (auto& p : pool) cudaFreeHost(p.pairs);
  if (report) *report = rep;
  return status;
}
