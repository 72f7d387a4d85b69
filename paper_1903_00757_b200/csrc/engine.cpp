// engine.cpp — pool preparation, episode scheduler, statistics and the C ABI
// (include/gv.h). State: engine.hpp; exchanges between ranks: transport.hpp;
// host-resident partitions: outofcore.cpp.
//
// One gv_ctx per process. It drives D ranks of Alg. 3: either
// the single rank of this process (world_size = D, IpcTransport between
// processes) or D virtual ranks on this process's GPU (virtual_ranks = D,
// LocalTransport).
// Rank d owns vertex partitions [d m, (d+1) m), m = n / D, and at offset
// step t holds the context window (d m + t + g) mod n, g = 0..m-1. After it
// trains its first block of step t (context (d m + t) mod n) it sends that
// partition to rank d-1, which needs it for the LAST block of step t+1, so
// the transfer overlaps the rank's remaining m-1 blocks.
// With m = 1 this is Alg. 3's train -> rotate -> train ring.
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "engine.hpp"
#include "transport.hpp"

using gv::DevBuf;
using gv::fail;
using gv::HpMat;
using gv::PoolState;
using gv::psize;
using gv::Rank;
using gv::elapsed;
using gv::new_event;
using gv::NvtxRange;
using gv::sync_all;

#define CK GV_CK

namespace {
thread_local std::string g_last_error;
}  // namespace

namespace gv {

gv_status fail(gv_ctx* c, gv_status s, const std::string& msg) {
  if (c) {
    std::lock_guard<std::mutex> lk(c->err_mu);
    c->err = msg;
  }
  g_last_error = msg;
  return s;
}

cudaEvent_t new_event(bool timing) {
  cudaEvent_t e = nullptr;
  cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming);
  return e;
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) return 0.f;
  return ms;
}

gv_status sync_all(gv_ctx* c) {
  for (auto& r : c->ranks) {
    CK(cudaStreamSynchronize(r.compute));
    CK(cudaStreamSynchronize(r.comm));
  }
  if (c->copy_stream) CK(cudaStreamSynchronize(c->copy_stream));
  if (c->hp_h2d) CK(cudaStreamSynchronize(c->hp_h2d));
  if (c->hp_d2h) CK(cudaStreamSynchronize(c->hp_d2h));
  return GV_OK;
}

}  // namespace gv

namespace {

float lr_at(const gv_ctx* c, uint64_t s_before) {
  if (c->alpha.kind == GV_LR_CONSTANT || c->alpha.total_samples == 0) return c->lr0;
  double r = 1.0 - static_cast<double>(s_before) / static_cast<double>(c->alpha.total_samples);
  if (r < c->alpha.floor_ratio) r = c->alpha.floor_ratio;
  return static_cast<float>(static_cast<double>(c->lr0) * r);
}

// --------------------------------------------------------------- prepare
// a5 + a6 fused (D > 1, virtual ranks or CUDA-IPC processes): every local
// rank s scatters its pool segment straight into the receive buffers of the
// owners of the block rows. Block (i, j) of owner d = concatenation over
// source ranks 0..D-1 of their sub-blocks (i, j) in pool order — the global
// stable counting sort (R-BUCKET) — so source s writes its sub-block (i, j)
// at final_off_d[(i, j)] + (samples of (i, j) in ranks < s).
gv_status place_fused(gv_ctx* c, const std::vector<std::vector<uint64_t>>& bc) {
  const uint32_t n = c->n, m = c->m, bins = n * n, bpr = m * n;
  const int D = c->D;
  // final layout of every rank's rows (all ranks: sources need the owners')
  std::vector<std::vector<uint64_t>> final_off(D, std::vector<uint64_t>(bpr + 1, 0));
  for (int d = 0; d < D; ++d)
    for (uint32_t q = 0; q < bpr; ++q)
      final_off[d][q + 1] = final_off[d][q] + c->global_counts[d * bpr + q];
  // receive buffers, then every rank's, addressable from this process
  for (auto& r : c->ranks)
    if (gv_status st = c->tr->reserve_blocks(c, r, final_off[r.d][bpr])) return st;
  std::vector<uint2*> outs(D, nullptr);
  if (gv_status st = c->tr->scatter_targets(c, outs)) return st;
  for (auto& r : c->ranks) {
    std::vector<uint64_t> args(bins + D);
    for (uint32_t q = 0; q < bins; ++q) {
      const uint32_t d = q / bpr;
      uint64_t off = final_off[d][q - d * bpr];
      for (int s2 = 0; s2 < r.d; ++s2) off += bc[s2][q];
      args[q] = off;
    }
    for (int d = 0; d < D; ++d) args[bins + d] = reinterpret_cast<uint64_t>(outs[d]);
    CK(r.place_args.ensure(args.size()));
    CK(cudaMemcpyAsync(r.place_args.p, args.data(), args.size() * sizeof(uint64_t),
                       cudaMemcpyHostToDevice, r.compute));  // pageable: staged before return
    const gv::IdMap ids{c->d_packed, c->relabeled() ? c->d_part_off : nullptr, c->nv,
                        c->part.pbits};
    CK(gv::launch_bucket_place(c->raw.p + r.seg_begin, r.seg_count, ids, r.plan, r.scratch.p,
                               r.place_args.p,
                               reinterpret_cast<uint2* const*>(r.place_args.p + bins), bpr,
                               reinterpret_cast<uint32_t*>(r.counts.p + bins + 1), r.compute,
                               &r.kernel_launches));
    CK(cudaEventRecord(r.ev_bucket, r.compute));
    CK(cudaEventRecord(r.ev_exch_sent, r.compute));
  }
  // an owner trains its rows only after every source has placed its samples
  return c->tr->scatter_done(c);
}

// a3-a6: bucket every local rank's pool segment, exchange block rows.
gv_status prepare(gv_ctx* c) {
  if (c->state == PoolState::Prepared) return GV_OK;
  NvtxRange nv_range("gv:prepare (bucket + exchange)");
  const bool from_fused = c->fused_pending;  // NEXT-1: already bucketed on the device
  {
    std::lock_guard<std::mutex> lk(c->mu);
    if (from_fused) {
      c->pool_P = c->fused_count;
      c->fused_pending = false;
    } else {
      if (c->raw_count == 0) return fail(c, GV_ERR_EMPTY, "no pending samples");
      c->pool_P = c->raw_count;
      c->raw_count = 0;
      c->raw_busy = true;  // pushes wait until raw_free is recorded below
    }
    c->have_last = false;
  }
  // whatever way prepare ends, pushes must not wait forever
  struct RawGuard {
    gv_ctx* c;
    ~RawGuard() {
      std::lock_guard<std::mutex> lk(c->mu);
      if (c->raw_busy) {  // an error path: let the kernels that read the pool finish
        for (auto& r : c->ranks) cudaStreamSynchronize(r.compute);
        cudaEventRecord(c->raw_free, c->copy_stream);
        c->raw_busy = false;
        c->raw_cv.notify_all();
      }
    }
  } raw_guard{c};
  const uint32_t n = c->n, bins = n * n;
  const uint64_t P = c->pool_P;
  // D > 1 (virtual ranks, CUDA-IPC processes): the scatter of a5 writes every
  // sample straight into the receive buffer of the rank that owns its block
  // row (a6 fused into a5); it runs after the counts are known
  const bool fused = c->D > 1;
  const gv::IdMap ids{c->d_packed, c->relabeled() ? c->d_part_off : nullptr, c->nv, c->part.pbits};
  const bool swap = c->swap_mode();
  // 1) bucketing per rank (a3-a5)
  for (auto& r : c->ranks) {
    r.kernel_launches = 0;
    r.sgd_launches = 0;
    if (c->opt.world_size > 1) {
      r.seg_begin = 0;
      r.seg_count = P;
    } else {
      r.seg_begin = P * static_cast<uint64_t>(r.d) / c->D;
      r.seg_count = P * static_cast<uint64_t>(r.d + 1) / c->D - r.seg_begin;
    }
    CK(cudaStreamWaitEvent(r.compute, c->raw_ready, 0));
    CK(cudaEventRecord(r.ev_start, r.compute));
    r.plan = gv::make_bucket_plan(n, r.seg_count);
    CK(r.scratch.ensure(gv::bucket_scratch_bytes(r.plan)));
    CK(cudaMemsetAsync(r.counts.p + bins + 1, 0, sizeof(uint64_t), r.compute));
    uint32_t* err = reinterpret_cast<uint32_t*>(r.counts.p + bins + 1);
    if (from_fused) {
      // the device sampler wrote the blocks and their offsets: swap them in;
      // the previous pool's SGD (enqueued before) is the last reader of the
      // buffer that becomes blocks_alt
      CK(cudaStreamWaitEvent(r.compute, c->fused_ready, 0));
      CK(cudaMemcpyAsync(r.counts.p, c->fused_off.p, sizeof(uint64_t) * (bins + 2),
                         cudaMemcpyDeviceToDevice, r.compute));
      std::swap(r.blocks, r.blocks_alt);
      CK(cudaEventRecord(c->alt_free, r.compute));
      CK(cudaEventRecord(r.ev_bucket, r.compute));
    } else if (swap) {
      // relabelled pool, n = 1: range check where the pool lies, then the
      // raw buffer becomes the block buffer (no copy); the old block buffer
      // becomes the raw buffer once the previous pool's SGD, enqueued before
      // this check on the same stream, has read it (raw_free below)
      const uint2* pool = c->pending_in_blocks ? r.blocks.p : c->raw.p;
      CK(gv::launch_validate(pool, P, c->nv, r.counts.p, err, r.compute, &r.kernel_launches));
      CK(cudaEventRecord(r.ev_bucket, r.compute));
      if (!c->pending_in_blocks) std::swap(c->raw, r.blocks);
      c->pending_in_blocks = false;
    } else if (fused) {
      CK(gv::launch_bucket_count(c->raw.p + r.seg_begin, r.seg_count, ids, r.plan, r.scratch.p,
                                 r.counts.p, err, r.compute, &r.kernel_launches));
    } else {
      CK(r.blocks.ensure(r.seg_count));
      CK(gv::launch_bucket(c->raw.p + r.seg_begin, r.seg_count, ids, r.plan, r.scratch.p,
                           r.blocks.p, r.counts.p, err, r.compute, &r.kernel_launches));
      CK(cudaEventRecord(r.ev_bucket, r.compute));
    }
  }
  // the raw buffer may be refilled once every rank has bucketed (and, fused,
  // placed) it
  auto release_raw = [&]() -> gv_status {
    for (auto& r : c->ranks) CK(cudaStreamWaitEvent(c->copy_stream, r.ev_bucket, 0));
    CK(cudaEventRecord(c->raw_free, c->copy_stream));
    std::lock_guard<std::mutex> lk(c->mu);
    c->raw_busy = false;
    c->have_last = true;
    c->last_count = P;
    c->raw_cv.notify_all();
    return GV_OK;
  };
  if (!fused && !from_fused)
    if (gv_status st = release_raw()) return st;
  // 2) counts of every rank to the host (a4)
  std::vector<std::vector<uint64_t>> cnt(c->D, std::vector<uint64_t>(bins + 2, 0));
  if (gv_status st = c->tr->gather_counts(c, cnt)) return st;
  bool bad = false;
  for (int q = 0; q < c->D; ++q) bad |= cnt[q][bins + 1] != 0;
  if (bad) {
    c->state = PoolState::Idle;
    if (fused)
      if (gv_status st = release_raw()) return st;
    return fail(c, GV_ERR_OUT_OF_RANGE, "sample pool contains a node id >= num_nodes");
  }
  // per-rank bin counts from block offsets
  std::vector<std::vector<uint64_t>> bc(c->D, std::vector<uint64_t>(bins));
  c->global_counts.assign(bins, 0);
  c->pool_P_global = 0;
  for (int q = 0; q < c->D; ++q)
    for (uint32_t b = 0; b < bins; ++b) {
      bc[q][b] = cnt[q][b + 1] - cnt[q][b];
      c->global_counts[b] += bc[q][b];
    }
  for (uint32_t b = 0; b < bins; ++b) {
    c->pool_P_global += c->global_counts[b];
    if (c->global_counts[b] > 0xFFFFFFFFull) {
      c->state = PoolState::Idle;
      if (fused)
        if (gv_status st = release_raw()) return st;
      return fail(c, GV_ERR_CAPACITY, "a block holds more than 2^32-1 samples");
    }
  }
  // 3) final layout of each local rank's block rows; exchange (a6)
  const uint32_t m = c->m;
  for (auto& r : c->ranks) {
    r.local_off.assign(cnt[r.d].begin(), cnt[r.d].begin() + bins + 1);
    r.final_off.assign(static_cast<size_t>(m) * n + 1, 0);
    const uint32_t b0 = r.d * m * n;
    for (uint32_t q = 0; q < m * n; ++q) r.final_off[q + 1] = r.final_off[q] + c->global_counts[b0 + q];
  }
  if (fused) {
    if (gv_status st = place_fused(c, bc)) return st;
    if (gv_status st = release_raw()) return st;
  }
  // R-VTILE: each block of the rank's rows in vertex-tile order (after the
  // exchange: an owner's block holds every source's samples by then)
  if (c->opt.vertex_tile > 0)
    for (auto& r : c->ranks) {
      const uint32_t nseg = m * n;
      std::vector<uint64_t> rows(nseg);
      for (uint32_t q = 0; q < nseg; ++q) rows[q] = psize(c, r.d * m + q / n);
      const uint32_t b = static_cast<uint32_t>(c->opt.vertex_tile);
      CK(r.tile_tmp.ensure(r.final_off[nseg]));
      CK(r.tile_scratch.ensure(gv::tile_sort_scratch_bytes(r.final_off.data(), rows.data(), nseg, b)));
      CK(gv::launch_tile_sort(r.blocks.p, r.tile_tmp.p, r.final_off.data(), rows.data(), nseg,
                              b, r.tile_scratch.p,
                              r.compute, &r.kernel_launches));
      if (!fused) CK(cudaEventRecord(r.ev_bucket, r.compute));  // counted in ms_bucket
    }
  for (auto& r : c->ranks) CK(cudaEventRecord(r.ev_exch, r.compute));
  c->state = PoolState::Prepared;
  return GV_OK;
}

// ---------------------------------------------------------------- steps
// a7-a8 for the prepared pool.
gv_status run_steps(gv_ctx* c) {
  NvtxRange nv_range("gv:offset steps (block-SGD + rotation)");
  const uint32_t n = c->n, m = c->m;
  const uint32_t e = static_cast<uint32_t>(c->pool_index);
  const uint32_t key0 = static_cast<uint32_t>(c->opt.seed), key1 = static_cast<uint32_t>(c->opt.seed >> 32);
  // orthogonality of every offset step (Def. 1 / P:229): over all D
  // ranks the step's blocks use each vertex and each context partition once
  for (uint32_t t = 0; t < n; ++t) {
    std::vector<uint8_t> vi(n, 0), cj(n, 0);
    for (int d = 0; d < c->D; ++d) {
      gv_step_plan pl;
      gv_plan_step(n, c->D, d, t, &pl);
      for (uint32_t g = 0; g < pl.n_blocks; ++g) {
        if (vi[pl.vpart[g]]++ || cj[pl.cpart[g]]++)
          return fail(c, GV_ERR_STATE, "internal: offset step " + std::to_string(t) +
                                           " is not orthogonal");
      }
    }
  }
  // lr per offset step from the global sample counts (R-LR)
  std::vector<float> lr(n);
  uint64_t s_before = c->samples_done;
  for (uint32_t t = 0; t < n; ++t) {
    lr[t] = lr_at(c, s_before);
    for (uint32_t i = 0; i < n; ++i) s_before += c->global_counts[i * n + (i + t) % n];
  }
  // descriptors: D == 1 -> one launch per step over all n blocks;
  //              D > 1  -> one launch per block (g), so the first block of a
  //              step can release its context partition early.
  // GV_BLOCK_LAUNCH=1 (measurement): one launch per block on one rank too —
  // the kernel then sees one block's rows at a time, as a GPU of a D = n
  // grid does (hot-row density n times that of n = 1)
  static const bool per_block = getenv("GV_BLOCK_LAUNCH") && atoi(getenv("GV_BLOCK_LAUNCH")) != 0;
  const bool step_launch = c->D == 1 && !c->hp() && !per_block;
  gv::HpPlan hp;  // out-of-core: residency order, slots, loads and write-backs
  if (c->hp()) gv::hp_plan(c, &hp);
  for (auto& r : c->ranks) {
    std::vector<gv::BlockDesc> desc(static_cast<size_t>(n) * m);
    // slot bookkeeping is simulated here exactly as the rotation will move data
    std::vector<int> slot_of = r.slot_of;
    int free_slot = r.free_slot;
    for (uint32_t t = 0; t < n; ++t) {
      uint64_t prefix = 0;
      gv_step_plan plan;
      gv_plan_step(n, c->D, r.d, t, &plan);
      for (uint32_t g = 0; g < m; ++g) {
        const uint32_t i = plan.vpart[g], j = plan.cpart[g];
        gv::BlockDesc& d = desc[t * m + g];
        d.sample_off = r.final_off[g * n + j];
        d.count_lo = static_cast<uint32_t>(r.final_off[g * n + j + 1] - r.final_off[g * n + j]);
        d.prefix = step_launch ? prefix : 0;
        prefix += d.count_lo;
        d.vrow0 = static_cast<uint32_t>(c->part.off[i] - r.vrow_first);
        d.crow0 = static_cast<uint32_t>(c->D == 1 ? c->part.off[j]
                                                  : static_cast<uint64_t>(slot_of[j]) * r.slot_rows);
        if (c->hp()) {
          d.vrow0 = static_cast<uint32_t>(hp.use[0][hp.pos[t * n + i]].s * r.slot_rows);
          d.crow0 = static_cast<uint32_t>(hp.use[1][hp.pos[t * n + i]].s * r.slot_rows);
        }
        d.alias0 = static_cast<uint32_t>(c->part.off[j]);
        d.m = static_cast<uint32_t>(psize(c, j));
        d.ij = (i << 16) | j;
      }
      if (c->D > 1) {  // after step t: send_part leaves, recv_part arrives
        const uint32_t out_p = plan.send_part, in_p = plan.recv_part;
        const int s_out = slot_of[out_p];
        slot_of[in_p] = free_slot;
        slot_of[out_p] = -1;
        free_slot = s_out;
      }
    }
    CK(r.desc.ensure(desc.size()));
    CK(cudaMemcpyAsync(r.desc.p, desc.data(), desc.size() * sizeof(gv::BlockDesc),
                       cudaMemcpyHostToDevice, r.compute));
    // (pageable source: the copy is staged before cudaMemcpyAsync returns)
    if (c->opt.compute_loss) CK(cudaMemsetAsync(r.loss.p, 0, sizeof(double), r.compute));
    const size_t need = static_cast<size_t>(2) * (step_launch ? n : n * m);
    while (r.ev_sgd.size() < need) r.ev_sgd.push_back(new_event(true));
  }
  // enqueue the steps
  auto launch_blocks = [&](Rank& r, uint32_t t, uint32_t g0, uint32_t cnt_blk) -> gv_status {
    gv::SgdArgs a{};
    a.samples = r.blocks.p;
    a.vertex = r.vertex;
    a.context = r.context;
    a.alias = c->d_alias;
    a.stride = c->stride;
    a.lr = lr[t];
    a.neg_weight = c->opt.neg_weight;
    a.pool_index = e;
    a.key0 = key0;
    a.key1 = key1;
    a.loss_acc = c->opt.compute_loss ? r.loss.p : nullptr;
    a.hot_rows = c->hot_rows;
    a.chunk_ctr = c->ring_dynamic ? r.chunk_ctr.p : nullptr;
    a.vertex_keep = (c->vtile_hint && c->opt.vertex_tile > 0) ? static_cast<uint32_t>(c->vtile_hint) : 0u;
    gv_step_plan plan;
    gv_plan_step(n, c->D, r.d, t, &plan);
    a.desc = r.desc.p + t * m + g0;
    a.nblk = static_cast<int>(cnt_blk);
    uint64_t tot = 0;
    for (uint32_t g = g0; g < g0 + cnt_blk; ++g)
      tot += r.final_off[g * n + plan.cpart[g] + 1] - r.final_off[g * n + plan.cpart[g]];
    a.total = tot;
    cudaEvent_t eb = r.ev_sgd[2 * r.sgd_launches], ee = r.ev_sgd[2 * r.sgd_launches + 1];
    CK(cudaEventRecord(eb, r.compute));
    if (c->opt.ordered)
      CK(gv::launch_sgd_ordered(a, c->dim, c->K, r.compute));
    else
      CK(gv::launch_sgd_hogwild(a, c->dim, c->K, c->sms, r.compute));
    CK(cudaEventRecord(ee, r.compute));
    r.sgd_launches++;
    r.kernel_launches++;
    return GV_OK;
  };
  if (c->hp()) {
    // out-of-core (Alg. 3): before block (i, j), its vertex and
    // context partitions are loaded into device slots; the load and
    // write-back streams run ahead of the compute stream
    Rank& r = c->ranks[0];
    gv_status st = gv::hp_enqueue(c, hp, [&](uint32_t t, uint32_t i) { return launch_blocks(r, t, i, 1); });
    if (st) return st;
  }
  for (uint32_t t = 0; t < n && !c->hp(); ++t) {
    for (auto& r : c->ranks) {
      gv_step_plan plan;
      gv_plan_step(n, c->D, r.d, t, &plan);
      auto launch = [&](uint32_t g0, uint32_t cnt_blk) { return launch_blocks(r, t, g0, cnt_blk); };
      if (step_launch) {
        gv_status st = launch(0, m);
        if (st) return st;
        continue;
      }
      for (uint32_t g = 0; g < m; ++g) {
        if (g == plan.wait_block) {
          // this block's context arrived by the previous rotation
          if (t > 0) CK(cudaStreamWaitEvent(r.compute, r.ev_recv[t - 1], 0));
          else if (r.have_last_recv) CK(cudaStreamWaitEvent(r.compute, r.ev_last_recv, 0));
        }
        gv_status st = launch(g, 1);
        if (st) return st;
        if (g == 0 && c->D > 1) {
          CK(cudaEventRecord(r.ev_first_done[t], r.compute));
          if (gv_status st2 = c->tr->first_block_done(c, r, t)) return st2;
        }
      }
    }
    if (c->D == 1) continue;
    // rotation of step t (a8): rank d sends partition (d m + t) to rank d-1
    if (gv_status st = c->tr->rotate(c, t)) return st;
  }
  for (auto& r : c->ranks) {
    if (c->D > 1) {
      // the pool ends after the last rotation (Alg. 3 order); the next pool's
      // step-0 last block and the next rotation wait on it
      CK(cudaStreamWaitEvent(r.compute, r.ev_recv[n - 1], 0));
      CK(cudaEventRecord(r.ev_last_recv, r.compute));
      r.have_last_recv = true;
    }
    CK(cudaEventRecord(r.ev_end, r.compute));
  }
  c->samples_done = s_before;
  c->pool_index++;
  c->state = PoolState::Idle;
  return GV_OK;
}

gv_status collect_stats(gv_ctx* c, gv_episode_stats* out) {
  gv_status st = sync_all(c);
  if (st) return st;
  std::memset(out, 0, sizeof(*out));
  out->pool_index = c->pool_index - 1;
  out->samples_global = c->pool_P_global;
  out->n_steps = c->n;
  uint64_t before = c->samples_done - c->pool_P_global;
  out->lr_first = lr_at(c, before);
  uint64_t s = before;
  for (uint32_t t = 0; t + 1 < c->n; ++t)
    for (uint32_t i = 0; i < c->n; ++i) s += c->global_counts[i * c->n + (i + t) % c->n];
  out->lr_last = lr_at(c, s);
  for (auto& r : c->ranks) {
    out->samples += r.final_off.empty() ? 0 : r.final_off.back();
    r.ms_bucket = elapsed(r.ev_start, r.ev_bucket);
    r.ms_exchange = elapsed(r.ev_bucket, r.ev_exch);
    r.ms_total = elapsed(r.ev_start, r.ev_end);
    double sgd = 0;
    for (int k = 0; k < r.sgd_launches; ++k) sgd += elapsed(r.ev_sgd[2 * k], r.ev_sgd[2 * k + 1]);
    r.ms_sgd = sgd;
    out->ms_bucket = std::max(out->ms_bucket, r.ms_bucket);
    out->ms_exchange = std::max(out->ms_exchange, r.ms_exchange);
    out->ms_sgd = std::max(out->ms_sgd, r.ms_sgd);
    out->ms_total = std::max(out->ms_total, r.ms_total);
    out->sgd_launches += r.sgd_launches;
    out->kernel_launches += r.kernel_launches;
    if (c->opt.compute_loss) {
      double l = 0;
      CK(cudaMemcpy(&l, r.loss.p, sizeof(double), cudaMemcpyDeviceToHost));
      out->loss_sum += l;
    }
  }
  out->ms_rotate = std::max(0.0, out->ms_total - out->ms_bucket - out->ms_exchange - out->ms_sgd);
  // per-rank device times; processes exchange theirs through
  // the transport, so every rank reports all D ranks and their maximum
  out->n_ranks = static_cast<uint32_t>(c->D);
  auto put = [&](int d, const double* v) {
    out->ms_total_rank[d] = v[0];
    out->ms_bucket_rank[d] = v[1];
    out->ms_exchange_rank[d] = v[2];
    out->ms_sgd_rank[d] = v[3];
    out->ms_rotate_rank[d] = v[4];
  };
  std::vector<std::array<double, 5>> v(c->D, std::array<double, 5>{});
  for (auto& r : c->ranks)
    v[r.d] = {r.ms_total, r.ms_bucket, r.ms_exchange, r.ms_sgd,
              std::max(0.0, r.ms_total - r.ms_bucket - r.ms_exchange - r.ms_sgd)};
  if (gv_status st2 = c->tr->exchange_stats(c, v)) return st2;
  for (int d = 0; d < c->D; ++d) put(d, v[d].data());
  for (int d = 0; d < c->D; ++d) out->ms_device_max = std::max(out->ms_device_max, out->ms_total_rank[d]);
  return GV_OK;
}

gv_status setup_device(gv_ctx* c) {
  const uint32_t nv = c->nv, n = c->n, m = c->m;
  CK(cudaMalloc(&c->d_packed, sizeof(uint32_t) * nv));
  CK(cudaMalloc(&c->d_alias, sizeof(uint2) * nv));
  CK(cudaMalloc(&c->d_inv_perm, sizeof(uint32_t) * nv));
  CK(cudaMalloc(&c->d_part_off, sizeof(uint64_t) * (n + 1)));
  CK(cudaMemcpy(c->d_part_off, c->part.off.data(), sizeof(uint64_t) * (n + 1), cudaMemcpyHostToDevice));
  static_assert(sizeof(gv::ProbAlias) == sizeof(uint2), "alias slots upload as uint2");
  CK(cudaMemcpy(c->d_packed, c->part.packed.data(), sizeof(uint32_t) * nv, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_alias, c->nalias.data(), sizeof(uint2) * nv, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_inv_perm, c->part.inv_perm.data(), sizeof(uint32_t) * nv,
                cudaMemcpyHostToDevice));
  CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  c->raw_ready = new_event(false);
  c->raw_free = new_event(false);
  c->fused_ready = new_event(false);
  c->alt_free = new_event(false);
  c->raw.host = c->opt.host_pool != 0;
  const uint32_t key0 = static_cast<uint32_t>(c->opt.init_seed);
  const uint32_t key1 = static_cast<uint32_t>(c->opt.init_seed >> 32);
  const uint64_t max_part = c->part.max_part();
  for (auto& r : c->ranks) {
    CK(cudaStreamCreateWithFlags(&r.compute, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&r.comm, cudaStreamNonBlocking));
    r.vrow_first = c->part.off[r.d * m];
    r.vrows = c->part.off[(r.d + 1) * m] - r.vrow_first;
    if (c->hp()) {
      // out-of-core: host arrays in relabelled order, device slots
      if (gv_status st = gv::hp_setup(c, r)) return st;
    } else {
    CK(cudaMalloc(&r.vertex, sizeof(float) * std::max<uint64_t>(r.vrows, 1) * c->stride));
    CK(cudaMemsetAsync(r.vertex, 0, sizeof(float) * r.vrows * c->stride, r.compute));
    CK(gv::launch_init_vertex(r.vertex, c->stride, c->dim, r.vrow_first, r.vrows, c->d_inv_perm,
                              key0, key1, r.compute));
    if (c->D == 1) {
      r.crows = nv;
      r.slot_rows = 0;
    } else {
      r.slot_rows = max_part;
      r.crows = (m + 1) * max_part;
      r.slot_of.assign(n, -1);
      for (uint32_t g = 0; g < m; ++g) r.slot_of[r.d * m + g] = static_cast<int>(g);
      r.free_slot = static_cast<int>(m);
      r.ev_first_done.resize(n);
      r.ev_recv.resize(n);
      r.ev_sent.resize(n);
      for (uint32_t t = 0; t < n; ++t) {
        r.ev_first_done[t] = new_event(false);
        r.ev_recv[t] = new_event(false);
        r.ev_sent[t] = new_event(false);
      }
      r.ev_last_recv = new_event(false);
    }
    CK(cudaMalloc(&r.context, sizeof(float) * r.crows * c->stride));
    CK(cudaMemsetAsync(r.context, 0, sizeof(float) * r.crows * c->stride, r.compute));
    }  // !hp
    CK(r.counts.ensure(n * n + 2));
    CK(r.loss.ensure(1));
    CK(r.chunk_ctr.ensure(1));
    CK(cudaMallocHost(&r.counts_host, sizeof(uint64_t) * (n * n + 2) * c->D));
    r.ev_start = new_event(true);
    r.ev_bucket = new_event(true);
    r.ev_exch = new_event(true);
    r.ev_end = new_event(true);
    r.ev_exch_sent = new_event(false);
  }
  gv_status st = sync_all(c);
  if (st) return st;
  return c->tr->connect(c);
}

// Graph preparation (gv_load_edges): ingest (R-INGEST), zig-zag partition
// (R-ZIGZAG), the partitions' negative alias tables over deg^0.75 (P:231,
// P:392; R-ALIAS) and the walk tables of the augmentation.
template <class Lap>
gv_status prepare_graph(gv_ctx* c, const uint32_t* src, const uint32_t* dst, const float* weight,
                        uint64_t num_edges, Lap& lap) {
  std::string msg;
  int rc = gv::build_graph(c->nv, src, dst, weight, num_edges, c->threads, &c->graph, &msg);
  if (rc) return fail(c, static_cast<gv_status>(rc), msg);
  lap("graph");
  rc = gv::build_partitioning(c->graph, c->n, &c->part, &msg);
  if (rc) return fail(c, static_cast<gv_status>(rc), msg);
  lap("zig-zag partition");
  // negative tables: deg^0.75 over each partition in local order
  c->nalias.assign(c->nv, gv::ProbAlias{0, 0});
  std::vector<double> w(c->nv);
  gv::parallel_for(c->nv, c->threads, [&](uint64_t b, uint64_t e) {
    for (uint64_t k = b; k < e; ++k) w[k] = std::pow(c->graph.deg[c->part.inv_perm[k]], 0.75);
  });
  std::vector<int> prc(c->n, 0);
  gv::parallel_for(c->n, c->n >= 2 ? std::min<int>(c->threads, static_cast<int>(c->n)) : 1,
                   [&](uint64_t b, uint64_t e) {
    for (uint64_t p = b; p < e; ++p)
      prc[p] = gv::build_alias(w.data() + c->part.off[p], static_cast<uint32_t>(psize(c, p)),
                               c->nalias.data() + c->part.off[p]);
  });
  for (uint32_t p = 0; p < c->n; ++p)
    if (prc[p]) return fail(c, GV_ERR_EMPTY, "context partition " + std::to_string(p) + " has zero noise mass");
  lap("negative alias tables");
  rc = gv::build_walk_tables(c->graph, c->threads, &c->walks);
  if (rc) return fail(c, static_cast<gv_status>(rc), "departure table has zero mass");
  c->graph.w.release();  // merged weights: only the alias tables needed them
  lap("walk alias tables");
  return GV_OK;
}

gv_status check_ctx(gv_ctx* c, bool need_loaded) {
  if (!c) return fail(nullptr, GV_ERR_INVALID_ARG, "null context");
  if (need_loaded && !c->loaded) return fail(c, GV_ERR_STATE, "gv_load_edges has not been called");
  return GV_OK;
}

}  // namespace

// ====================================================================== ABI
extern "C" {

void gv_default_options(gv_options* o) {
  std::memset(o, 0, sizeof(*o));
  o->seed = 5;
  o->init_seed = 4;
  o->neg_weight = 5.0f;
  o->device = 0;
  o->rank = 0;
  o->world_size = 1;
  o->virtual_ranks = 1;
  o->ordered = 0;
  o->compute_loss = 1;
  o->host_threads = 0;
  o->max_pool_samples = 0;
  o->host_partitions = 0;
}

int gv_abi_version(void) { return GV_ABI_VERSION; }

const char* gv_status_string(gv_status s) {
  switch (s) {
    case GV_OK: return "GV_OK";
    case GV_ERR_INVALID_ARG: return "GV_ERR_INVALID_ARG";
    case GV_ERR_STATE: return "GV_ERR_STATE";
    case GV_ERR_OUT_OF_RANGE: return "GV_ERR_OUT_OF_RANGE";
    case GV_ERR_EMPTY: return "GV_ERR_EMPTY";
    case GV_ERR_CAPACITY: return "GV_ERR_CAPACITY";
    case GV_ERR_NOMEM: return "GV_ERR_NOMEM";
    case GV_ERR_CUDA: return "GV_ERR_CUDA";
    case GV_ERR_COMM: return "GV_ERR_COMM";
  }
  return "unknown";
}

const char* gv_last_error(const gv_ctx* c) { return c ? c->err.c_str() : g_last_error.c_str(); }

gv_status gv_create(uint32_t num_nodes, uint32_t dim, uint32_t n_partitions,
                    uint32_t num_negatives, float lr0, const gv_lr_schedule* alpha,
                    const gv_options* opt, gv_ctx** out) {
  gv_ctx* c = nullptr;
  if (!out) return fail(nullptr, GV_ERR_INVALID_ARG, "out is null");
  gv_options o;
  if (opt) o = *opt; else gv_default_options(&o);
  if (num_nodes == 0 || dim == 0 || dim % 4 != 0 || dim > 512)
    return fail(nullptr, GV_ERR_INVALID_ARG, "num_nodes > 0 and dim in {4, 8, ..., 512} required");
  if (num_negatives == 0 || num_negatives > 8)
    return fail(nullptr, GV_ERR_INVALID_ARG, "num_negatives must be in [1, 8]");
  if (n_partitions == 0 || n_partitions > num_nodes || n_partitions > 64)
    return fail(nullptr, GV_ERR_INVALID_ARG, "n_partitions must be in [1, min(64, num_nodes)]");
  if (!(lr0 >= 0.0f)) return fail(nullptr, GV_ERR_INVALID_ARG, "lr0 must be >= 0");
  if (o.world_size < 1 || o.virtual_ranks < 1 || o.rank < 0 || o.rank >= o.world_size ||
      (o.world_size > 1 && o.virtual_ranks != 1))
    return fail(nullptr, GV_ERR_INVALID_ARG, "bad rank / world_size / virtual_ranks");
  const int D = o.world_size * o.virtual_ranks;
  if (n_partitions % D != 0)
    return fail(nullptr, GV_ERR_INVALID_ARG, "n_partitions must be a multiple of the rank count");
  if (o.host_partitions && (o.world_size * o.virtual_ranks != 1 || n_partitions < 2))
    return fail(nullptr, GV_ERR_INVALID_ARG, "host_partitions needs one rank and n_partitions >= 2");
  if (o.vertex_tile < 0 || o.vertex_tile > 31)
    return fail(nullptr, GV_ERR_INVALID_ARG, "vertex_tile must be in [0, 31]");
  if (o.pool_ids != GV_IDS_ORIGINAL && o.pool_ids != GV_IDS_RELABELED)
    return fail(nullptr, GV_ERR_INVALID_ARG, "pool_ids must be GV_IDS_ORIGINAL or GV_IDS_RELABELED");
  if (alpha && (alpha->kind != GV_LR_CONSTANT && alpha->kind != GV_LR_LINEAR))
    return fail(nullptr, GV_ERR_INVALID_ARG, "bad lr schedule kind");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(nullptr, GV_ERR_CUDA, "no CUDA device");
  if (o.device < 0 || o.device >= ndev) return fail(nullptr, GV_ERR_INVALID_ARG, "bad device");
  if (cudaSetDevice(o.device) != cudaSuccess) return fail(nullptr, GV_ERR_CUDA, "cudaSetDevice failed");
  c = new gv_ctx();
  c->nv = num_nodes;
  c->dim = dim;
  c->n = n_partitions;
  c->K = num_negatives;
  c->lr0 = lr0;
  if (alpha) c->alpha = *alpha;
  c->opt = o;
  c->D = D;
  c->local = o.virtual_ranks;
  c->m = n_partitions / D;
  c->stride = (dim + 3) / 4 * 4;
  c->threads = o.host_threads > 0 ? o.host_threads : gv::default_threads();
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, o.device);
  // L2 retention hints (hot rows evict_last, cold rows evict_first) are OFF:
  // measured on C2 they evict a cold line between its cp.async read and its
  // red.global.add write-back (DRAM reads +29%, -19% samples/s; profiles/).
  // GV_HOT_ROWS=<local-id threshold> enables them for experiments.
  if (const char* e = getenv("GV_HOT_ROWS")) c->hot_rows = static_cast<uint32_t>(atol(e));
  if (const char* e = getenv("GV_RING_DYN")) c->ring_dynamic = atoi(e) != 0;
  if (const char* e = getenv("GV_VTILE_HINT")) c->vtile_hint = atoi(e);  // 1: vertex kept, context first out; 2: vertex kept
  c->ranks.resize(c->local);
  for (int v = 0; v < c->local; ++v) c->ranks[v].d = (o.world_size > 1) ? o.rank : v;
  if (o.world_size == 1) c->tr = gv::make_local_transport();  // processes: gv_comm_init
  *out = c;
  return GV_OK;
}

gv_status gv_comm_unique_id(uint8_t id_out[128]) {
  FILE* f = fopen("/dev/urandom", "rb");
  if (!f || fread(id_out, 1, 128, f) != 128) {
    if (f) fclose(f);
    return fail(nullptr, GV_ERR_COMM, "no /dev/urandom for a unique id");
  }
  fclose(f);
  return GV_OK;
}

gv_status gv_comm_init(gv_ctx* c, const uint8_t id[128]) {
  if (gv_status s = check_ctx(c, false)) return s;
  if (c->opt.world_size <= 1) return fail(c, GV_ERR_STATE, "gv_comm_init needs world_size > 1");
  if (c->loaded || c->tr) return fail(c, GV_ERR_STATE, "call gv_comm_init before gv_load_edges, once");
  CK(cudaSetDevice(c->opt.device));
  return gv::make_ipc_transport(c, id, &c->tr);
}

gv_status gv_load_edges(gv_ctx* c, const uint32_t* src, const uint32_t* dst, const float* weight,
                        uint64_t num_edges) {
  if (gv_status s = check_ctx(c, false)) return s;
  if (c->loaded) return fail(c, GV_ERR_STATE, "gv_load_edges called twice");
  if (!c->tr) return fail(c, GV_ERR_STATE, "gv_comm_init first");
  // multi-process: rank 0 prepares the graph once for the node and shares it
  const bool builder = !c->ipc() || c->opt.rank == 0;
  if (builder && num_edges && (!src || !dst)) return fail(c, GV_ERR_INVALID_ARG, "null edge arrays");
  CK(cudaSetDevice(c->opt.device));
  NvtxRange nv_range("gv:load_edges");
  const bool timing = getenv("GV_INGEST_TIMING") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[load_edges] %s %.0f ms\n", what,
            std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  gv_status st = c->tr->load_graph(c, [&] { return prepare_graph(c, src, dst, weight, num_edges, lap); });
  if (st) return st;
  lap(builder ? "graph ready" : "attach the node-shared graph");
  st = setup_device(c);
  if (st) return st;
  lap("device setup");
  c->loaded = true;
  return GV_OK;
}

// a2, batched transfer ("we transfer the sample block by a small
// granularity"): pairs are appended to the raw pool in chunks of
// kPushChunk samples on the copy stream. With host_pool the raw pool itself
// lives in pinned, mapped host memory (the bucketing kernels read it over
// PCIe), so edge samples cost no device memory beyond the bucketed blocks.
constexpr uint64_t kPushChunk = uint64_t(1) << 23;  // 64 MiB of pairs

// Makes room for `count` more pending samples: waits (host) while a
// prepare holds the pool; orders the copy stream (or, host_pool, the host)
// after the bucketing kernels that read the buffer last; grows the buffer,
// keeping the samples already pending. Returns the pending count.
static gv_status reserve_raw(gv_ctx* c, std::unique_lock<std::mutex>& lk, uint64_t count,
                             uint64_t* have_out) {
  c->raw_cv.wait(lk, [&] { return !c->raw_busy; });
  if (c->pending_in_blocks)
    return fail(c, GV_ERR_STATE, "a replayed pool is pending: train it before pushing");
  const uint64_t have = c->raw_count;
  if (c->opt.max_pool_samples && have + count > c->opt.max_pool_samples)
    return fail(c, GV_ERR_CAPACITY, "pending pool would exceed max_pool_samples");
  if (c->raw.host) CK(cudaEventSynchronize(c->raw_free));
  else CK(cudaStreamWaitEvent(c->copy_stream, c->raw_free, 0));
  if (have + count > c->raw.cap) {
    DevBuf<uint2> bigger;
    bigger.host = c->raw.host;
    CK(bigger.ensure(std::max<uint64_t>(have + count, c->raw.cap + c->raw.cap / 2)));
    if (have) CK(cudaMemcpyAsync(bigger.p, c->raw.p, have * sizeof(uint2), cudaMemcpyDefault,
                                 c->copy_stream));
    CK(cudaStreamSynchronize(c->copy_stream));
    c->raw.release();
    c->raw = bigger;
  }
  c->have_last = false;  // the buffer is being refilled: no replay of the last pool
  *have_out = have;
  return GV_OK;
}

static gv_status push_impl(gv_ctx* c, const uint32_t* pairs, uint64_t count, bool from_device) {
  if (gv_status s = check_ctx(c, true)) return s;
  if (count == 0) return GV_OK;
  if (!pairs) return fail(c, GV_ERR_INVALID_ARG, "null pairs");
  CK(cudaSetDevice(c->opt.device));
  std::unique_lock<std::mutex> lk(c->mu);
  uint64_t have = 0;
  if (gv_status st = reserve_raw(c, lk, count, &have)) return st;
  const uint2* src = reinterpret_cast<const uint2*>(pairs);
  uint2* dst = c->raw.p + have;
  if (c->raw.host && !from_device) {
    // host pool: a plain parallel copy into the pinned buffer
    gv::parallel_for(count, std::min(c->threads, 16), [&](uint64_t b, uint64_t e) {
      std::memcpy(dst + b, src + b, (e - b) * sizeof(uint2));
    });
  } else {
    for (uint64_t off = 0; off < count; off += kPushChunk)
      CK(cudaMemcpyAsync(dst + off, src + off, std::min(kPushChunk, count - off) * sizeof(uint2),
                         cudaMemcpyDefault, c->copy_stream));
  }
  CK(cudaEventRecord(c->raw_ready, c->copy_stream));
  CK(cudaStreamSynchronize(c->copy_stream));  // the caller may reuse `pairs` on return
  c->raw_count = have + count;
  return GV_OK;
}

gv_status gv_push_sample_pool(gv_ctx* c, const uint32_t* pairs, uint64_t count) {
  return push_impl(c, pairs, count, false);
}

gv_status gv_push_sample_pool_device(gv_ctx* c, const uint32_t* pairs_dev, uint64_t count) {
  return push_impl(c, pairs_dev, count, true);
}

gv_status gv_replay_pool(gv_ctx* c) {
  if (gv_status s = check_ctx(c, true)) return s;
  std::lock_guard<std::mutex> lk(c->mu);
  if (c->state == PoolState::Prepared || !c->have_last || c->raw_busy || c->raw_count != 0)
    return fail(c, GV_ERR_STATE, "no trained pool to replay, or a pool is pending");
  c->raw_count = c->last_count;
  c->pending_in_blocks = c->swap_mode();  // swap mode: the last pool lies in the block buffer
  return GV_OK;
}

gv_status gv_prepare_episode(gv_ctx* c) {
  if (gv_status s = check_ctx(c, true)) return s;
  CK(cudaSetDevice(c->opt.device));
  return prepare(c);
}

gv_status gv_train_episode(gv_ctx* c, gv_episode_stats* out) {
  if (gv_status s = check_ctx(c, true)) return s;
  CK(cudaSetDevice(c->opt.device));
  gv_status st = prepare(c);
  if (st) return st;
  st = run_steps(c);
  if (st) return st;
  if (out) return collect_stats(c, out);
  return GV_OK;
}

gv_status gv_read_stats(gv_ctx* c, gv_episode_stats* out) {
  if (gv_status s = check_ctx(c, true)) return s;
  if (!out) return fail(c, GV_ERR_INVALID_ARG, "null out");
  if (c->pool_index == 0) return fail(c, GV_ERR_STATE, "no pool trained yet");
  CK(cudaSetDevice(c->opt.device));
  return collect_stats(c, out);
}

gv_status gv_synchronize(gv_ctx* c) {
  if (gv_status s = check_ctx(c, false)) return s;
  return sync_all(c);
}

static gv_status embeddings_io(gv_ctx* c, bool context, float* out, const float* in,
                               uint64_t len) {
  if (gv_status s = check_ctx(c, true)) return s;
  if (len != static_cast<uint64_t>(c->nv) * c->dim)
    return fail(c, GV_ERR_INVALID_ARG, "buffer length must be num_nodes * dim");
  if (c->state == PoolState::Prepared)
    return fail(c, GV_ERR_STATE, "a prepared pool is pending training");
  CK(cudaSetDevice(c->opt.device));
  gv_status st = sync_all(c);
  if (st) return st;
  const uint32_t dim = c->dim, stride = c->stride, m = c->m;
  if (c->hp()) return gv::hp_embeddings_io(c, context, out, in);
  std::vector<float> buf;
  for (auto& r : c->ranks) {
    // list of (device base row, first new id, rows)
    struct Span { uint64_t dev_row, id0, rows; };
    std::vector<Span> spans;
    float* base = context ? r.context : r.vertex;
    if (!context) {
      spans.push_back({0, r.vrow_first, r.vrows});
    } else if (c->D == 1) {
      spans.push_back({0, 0, c->nv});
    } else {
      for (uint32_t g = 0; g < m; ++g) {
        const uint32_t j = r.d * m + g;
        spans.push_back({static_cast<uint64_t>(r.slot_of[j]) * r.slot_rows, c->part.off[j], psize(c, j)});
      }
    }
    for (const Span& sp : spans) {
      buf.resize(sp.rows * stride);
      if (out) {
        CK(cudaMemcpy(buf.data(), base + sp.dev_row * stride, sp.rows * stride * sizeof(float),
                      cudaMemcpyDeviceToHost));
        for (uint64_t q = 0; q < sp.rows; ++q)
          std::memcpy(out + static_cast<uint64_t>(c->part.inv_perm[sp.id0 + q]) * dim,
                      buf.data() + q * stride, dim * sizeof(float));
      } else {
        std::fill(buf.begin(), buf.end(), 0.0f);
        for (uint64_t q = 0; q < sp.rows; ++q)
          std::memcpy(buf.data() + q * stride,
                      in + static_cast<uint64_t>(c->part.inv_perm[sp.id0 + q]) * dim,
                      dim * sizeof(float));
        CK(cudaMemcpy(base + sp.dev_row * stride, buf.data(), sp.rows * stride * sizeof(float),
                      cudaMemcpyHostToDevice));
      }
    }
  }
  return GV_OK;
}

gv_status gv_get_vertex_embeddings(gv_ctx* c, float* out, uint64_t len) {
  if (!out) return fail(c, GV_ERR_INVALID_ARG, "null out");
  return embeddings_io(c, false, out, nullptr, len);
}
gv_status gv_get_context_embeddings(gv_ctx* c, float* out, uint64_t len) {
  if (!out) return fail(c, GV_ERR_INVALID_ARG, "null out");
  return embeddings_io(c, true, out, nullptr, len);
}
gv_status gv_set_vertex_embeddings(gv_ctx* c, const float* in, uint64_t len) {
  if (!in) return fail(c, GV_ERR_INVALID_ARG, "null in");
  return embeddings_io(c, false, nullptr, in, len);
}
gv_status gv_set_context_embeddings(gv_ctx* c, const float* in, uint64_t len) {
  if (!in) return fail(c, GV_ERR_INVALID_ARG, "null in");
  return embeddings_io(c, true, nullptr, in, len);
}

gv_status gv_get_progress(gv_ctx* c, uint64_t* pool_index, uint64_t* samples_done) {
  if (gv_status s = check_ctx(c, false)) return s;
  if (pool_index) *pool_index = c->pool_index;
  if (samples_done) *samples_done = c->samples_done;
  return GV_OK;
}

gv_status gv_set_progress(gv_ctx* c, uint64_t pool_index, uint64_t samples_done) {
  if (gv_status s = check_ctx(c, false)) return s;
  if (c->state == PoolState::Prepared) return fail(c, GV_ERR_STATE, "a prepared pool is pending");
  if (c->tr)
    if (gv_status st = c->tr->set_progress(c, pool_index)) return st;
  c->pool_index = pool_index;
  c->samples_done = samples_done;
  return GV_OK;
}

gv_status gv_get_stream(gv_ctx* c, int vrank, uintptr_t* stream_out) {
  if (gv_status s = check_ctx(c, true)) return s;
  if (vrank < 0 || vrank >= static_cast<int>(c->ranks.size()) || !stream_out)
    return fail(c, GV_ERR_INVALID_ARG, "bad vrank");
  *stream_out = reinterpret_cast<uintptr_t>(c->ranks[vrank].compute);
  return GV_OK;
}

gv_status gv_augment(gv_ctx* c, uint32_t walk_len, uint32_t s, uint32_t threads, uint64_t count,
                     uint64_t seed, uint32_t* out_pairs) {
  if (gv_status st = check_ctx(c, true)) return st;
  if (walk_len == 0 || s == 0 || s > walk_len || threads == 0)
    return fail(c, GV_ERR_INVALID_ARG, "need walk_len > 0, 0 < s <= walk_len, threads > 0");
  if (count && !out_pairs) return fail(c, GV_ERR_INVALID_ARG, "null out_pairs");
  gv::augment(c->walks, walk_len, s, threads, count, seed, out_pairs,
              c->relabeled() ? c->part.perm.data() : nullptr);
  return GV_OK;
}

gv_status gv_augment_device(gv_ctx* c, uint32_t walk_len, uint32_t s, uint32_t segments,
                            uint64_t count, uint64_t seed) {
  return gv_augment_device_ex(c, walk_len, s, segments, count, seed, GV_SHUFFLE_PSEUDO);
}

// The device copy of the samplers' tables (CSR, alias tables; perm for
// relabelled pools), uploaded on first use.
static gv_status walk_tables_on_device(gv_ctx* c, gv::WalkDev* wd) {
  if (!c->d_woff) {  // upload the CSR and the alias tables the host sampler uses
    const gv::HostGraph& g = c->graph;
    const size_t ne = g.nbr.size();
    CK(cudaMalloc(&c->d_woff, sizeof(uint64_t) * (g.nv + 1)));
    CK(cudaMalloc(&c->d_wnbr, sizeof(uint32_t) * std::max<size_t>(ne, 1)));
    CK(cudaMalloc(&c->d_walias, sizeof(uint2) * std::max<size_t>(ne, 1)));
    CK(cudaMalloc(&c->d_dalias, sizeof(uint2) * g.nv));
    CK(cudaMemcpy(c->d_woff, g.off.data(), sizeof(uint64_t) * (g.nv + 1), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_wnbr, g.nbr.data(), sizeof(uint32_t) * ne, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_walias, c->walks.edge.data(), sizeof(uint2) * ne, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_dalias, c->walks.departure.data(), sizeof(uint2) * g.nv,
                  cudaMemcpyHostToDevice));
  }
  if (c->relabeled() && !c->d_perm) {
    CK(cudaMalloc(&c->d_perm, sizeof(uint32_t) * c->nv));
    CK(cudaMemcpy(c->d_perm, c->part.perm.data(), sizeof(uint32_t) * c->nv, cudaMemcpyHostToDevice));
  }
  *wd = gv::WalkDev{c->d_woff, c->d_wnbr, c->d_walias, c->d_dalias, c->nv,
                    c->relabeled() ? c->d_perm : nullptr};
  return GV_OK;
}

gv_status gv_augment_device_blocks(gv_ctx* c, uint32_t walk_len, uint32_t s, uint32_t segments,
                                   uint64_t count, uint64_t seed, int shuffle) {
  if (gv_status st = check_ctx(c, true)) return st;
  if (shuffle != GV_SHUFFLE_PSEUDO && shuffle != GV_SHUFFLE_NONE)
    return fail(c, GV_ERR_INVALID_ARG, "shuffle must be GV_SHUFFLE_PSEUDO or _NONE");
  if (walk_len == 0 || walk_len > 1000 || s == 0 || s > walk_len || segments == 0 || count == 0)
    return fail(c, GV_ERR_INVALID_ARG, "need 0 < walk_len <= 1000, 0 < s <= walk_len, segments, count > 0");
  if (c->D != 1) return fail(c, GV_ERR_STATE, "gv_augment_device_blocks needs one rank");
  const size_t scratch = gv::augment_blocks_scratch_bytes(
      walk_len, s, shuffle == GV_SHUFFLE_NONE ? 1 : 0, c->n, segments, count);
  if (scratch == 0)
    return fail(c, GV_ERR_INVALID_ARG, "shape not eligible for bucketing in the sampler "
                                       "(s > 32, count >= 2^32 or n^2 * s too large)");
  if (c->opt.max_pool_samples && count > c->opt.max_pool_samples)
    return fail(c, GV_ERR_CAPACITY, "pool would exceed max_pool_samples");
  CK(cudaSetDevice(c->opt.device));
  gv::WalkDev wd;
  if (gv_status st = walk_tables_on_device(c, &wd)) return st;
  std::lock_guard<std::mutex> lk(c->mu);
  if (c->raw_count != 0 || c->fused_pending || c->pending_in_blocks || c->state == PoolState::Prepared)
    return fail(c, GV_ERR_STATE, "a pool is pending: train it first");
  Rank& r = c->ranks[0];
  const uint32_t bins = c->n * c->n;
  CK(c->aug_scratch.ensure(scratch));
  CK(c->fused_off.ensure(bins + 2));
  CK(cudaStreamWaitEvent(c->copy_stream, c->alt_free, 0));  // the previous reader of blocks_alt
  if (count > r.blocks_alt.cap) {
    CK(cudaStreamSynchronize(c->copy_stream));  // the old buffer is no longer read
    CK(r.blocks_alt.ensure(count));
  }
  CK(cudaMemsetAsync(c->fused_off.p + bins + 1, 0, sizeof(uint64_t), c->copy_stream));
  const gv::IdMap ids{c->d_packed, c->relabeled() ? c->d_part_off : nullptr, c->nv, c->part.pbits};
  CK(gv::launch_augment_blocks(wd, walk_len, s, segments, count, seed,
                               shuffle == GV_SHUFFLE_NONE ? 1 : 0, ids, c->n, c->aug_scratch.p,
                               c->fused_off.p, reinterpret_cast<uint32_t*>(c->fused_off.p + bins + 1),
                               r.blocks_alt.p, c->copy_stream, nullptr));
  CK(cudaEventRecord(c->fused_ready, c->copy_stream));
  c->fused_pending = true;
  c->fused_count = count;
  c->have_last = false;
  return GV_OK;
}

gv_status gv_augment_device_ex(gv_ctx* c, uint32_t walk_len, uint32_t s, uint32_t segments,
                               uint64_t count, uint64_t seed, int shuffle) {
  if (gv_status st = check_ctx(c, true)) return st;
  if (shuffle != GV_SHUFFLE_PSEUDO && shuffle != GV_SHUFFLE_NONE && shuffle != GV_SHUFFLE_RANDOM)
    return fail(c, GV_ERR_INVALID_ARG, "shuffle must be GV_SHUFFLE_PSEUDO, _NONE or _RANDOM");
  if (walk_len == 0 || walk_len > 1000 || s == 0 || s > walk_len || segments == 0)
    return fail(c, GV_ERR_INVALID_ARG, "need 0 < walk_len <= 1000, 0 < s <= walk_len, segments > 0");
  if (count == 0) return GV_OK;
  if (count > (UINT64_MAX / segments)) return fail(c, GV_ERR_CAPACITY, "count * segments overflows");
  CK(cudaSetDevice(c->opt.device));
  gv::WalkDev wd;
  if (gv_status st = walk_tables_on_device(c, &wd)) return st;
  std::unique_lock<std::mutex> lk(c->mu);
  uint64_t have = 0;
  if (gv_status st = reserve_raw(c, lk, count, &have)) return st;
  if (shuffle == GV_SHUFFLE_RANDOM) {  // walk order into scratch, then a keyed permutation
    CK(c->shuf_tmp.ensure(count));
    CK(gv::launch_augment(wd, walk_len, s, segments, count, seed, 1, c->shuf_tmp.p,
                          c->copy_stream));
    CK(gv::launch_random_permute(c->shuf_tmp.p, count, seed, c->raw.p + have, c->copy_stream));
  } else {
    CK(gv::launch_augment(wd, walk_len, s, segments, count, seed,
                          shuffle == GV_SHUFFLE_NONE ? 1 : 0, c->raw.p + have, c->copy_stream));
  }
  CK(cudaEventRecord(c->raw_ready, c->copy_stream));
  c->raw_count = have + count;
  return GV_OK;
}

gv_status gv_debug_get_pending(gv_ctx* c, uint32_t* out, uint64_t cap, uint64_t* count) {
  if (gv_status st = check_ctx(c, true)) return st;
  CK(cudaSetDevice(c->opt.device));
  std::lock_guard<std::mutex> lk(c->mu);
  if (count) *count = c->raw_count;
  if (!out) return GV_OK;
  if (cap < c->raw_count) return fail(c, GV_ERR_CAPACITY, "cap < pending pool size");
  CK(cudaStreamSynchronize(c->copy_stream));
  const uint2* pool = c->pending_in_blocks ? c->ranks[0].blocks.p : c->raw.p;
  CK(cudaMemcpy(out, pool, sizeof(uint2) * c->raw_count, cudaMemcpyDefault));
  return GV_OK;
}

gv_status gv_get_partition(gv_ctx* c, uint32_t* perm, uint64_t* part_off) {
  if (gv_status s = check_ctx(c, true)) return s;
  if (perm) std::memcpy(perm, c->part.perm.data(), sizeof(uint32_t) * c->nv);
  if (part_off) std::memcpy(part_off, c->part.off.data(), sizeof(uint64_t) * (c->n + 1));
  return GV_OK;
}

gv_status gv_get_alias(gv_ctx* c, uint32_t p, uint32_t* prob, uint32_t* alias, uint64_t cap) {
  if (gv_status s = check_ctx(c, true)) return s;
  if (p == UINT32_MAX) {
    if (cap < c->nv) return fail(c, GV_ERR_CAPACITY, "cap < num_nodes");
    for (uint32_t k = 0; k < c->nv; ++k) {
      prob[k] = c->walks.departure[k].prob;
      alias[k] = c->walks.departure[k].alias;
    }
    return GV_OK;
  }
  if (p >= c->n) return fail(c, GV_ERR_INVALID_ARG, "bad partition");
  const uint64_t b = c->part.off[p], sz = psize(c, p);
  if (cap < sz) return fail(c, GV_ERR_CAPACITY, "cap < partition size");
  for (uint64_t k = 0; k < sz; ++k) {
    prob[k] = c->nalias[b + k].prob;
    alias[k] = c->nalias[b + k].alias;
  }
  return GV_OK;
}

gv_status gv_debug_get_buckets(gv_ctx* c, uint32_t* pairs_out, uint64_t cap, uint64_t* block_off) {
  if (gv_status s = check_ctx(c, true)) return s;
  if (c->state != PoolState::Prepared) return fail(c, GV_ERR_STATE, "call gv_prepare_episode first");
  CK(cudaSetDevice(c->opt.device));
  if (gv_status s = sync_all(c)) return s;
  const uint32_t n = c->n, m = c->m;
  std::vector<uint64_t> off(n * n + 1, 0);
  for (uint32_t b = 0; b < n * n; ++b) off[b + 1] = off[b] + c->global_counts[b];
  if (block_off) std::memcpy(block_off, off.data(), sizeof(uint64_t) * off.size());
  if (!pairs_out) return GV_OK;
  if (cap < off.back()) return fail(c, GV_ERR_CAPACITY, "cap < pool size");
  for (auto& r : c->ranks) {
    const uint64_t first = off[r.d * m * n], len = r.final_off.back();
    CK(cudaMemcpy(pairs_out + 2 * first, r.blocks.p, len * sizeof(uint2), cudaMemcpyDeviceToHost));
  }
  return GV_OK;
}

gv_status gv_debug_get_negatives(gv_ctx* c, uint32_t i, uint32_t j, uint32_t* out, uint64_t cap) {
  if (gv_status s = check_ctx(c, true)) return s;
  if (c->state != PoolState::Prepared) return fail(c, GV_ERR_STATE, "call gv_prepare_episode first");
  if (i >= c->n || j >= c->n) return fail(c, GV_ERR_INVALID_ARG, "bad block");
  CK(cudaSetDevice(c->opt.device));
  const uint32_t owner = i / c->m;
  Rank* r = nullptr;
  for (auto& x : c->ranks)
    if (static_cast<uint32_t>(x.d) == owner) r = &x;
  if (!r) return fail(c, GV_ERR_INVALID_ARG, "block row not owned by this process");
  const uint32_t g = i - owner * c->m;
  gv::BlockDesc d{};
  d.sample_off = r->final_off[g * c->n + j];
  d.count_lo = static_cast<uint32_t>(r->final_off[g * c->n + j + 1] - d.sample_off);
  d.alias0 = static_cast<uint32_t>(c->part.off[j]);
  d.m = static_cast<uint32_t>(psize(c, j));
  d.ij = (i << 16) | j;
  if (cap < static_cast<uint64_t>(d.count_lo) * c->K) return fail(c, GV_ERR_CAPACITY, "cap too small");
  DevBuf<uint32_t> tmp;
  CK(tmp.ensure(static_cast<size_t>(d.count_lo) * c->K));
  CK(gv::launch_negatives(d, c->d_alias, static_cast<uint32_t>(c->pool_index),
                          static_cast<uint32_t>(c->opt.seed), static_cast<uint32_t>(c->opt.seed >> 32),
                          c->K, tmp.p, r->compute));
  CK(cudaStreamSynchronize(r->compute));
  CK(cudaMemcpy(out, tmp.p, sizeof(uint32_t) * d.count_lo * c->K, cudaMemcpyDeviceToHost));
  tmp.release();
  return GV_OK;
}

gv_status gv_train_explicit(gv_ctx* c, const uint32_t* u, const uint32_t* v, const uint32_t* negs,
                            uint64_t count, float lr) {
  if (gv_status s = check_ctx(c, true)) return s;
  if (c->D != 1 || c->hp())
    return fail(c, GV_ERR_STATE, "gv_train_explicit needs a single rank with resident matrices");
  if (count == 0) return GV_OK;
  CK(cudaSetDevice(c->opt.device));
  const uint32_t K = c->K;
  std::vector<uint32_t> vrow(count), crow(count * (K + 1));
  for (uint64_t q = 0; q < count; ++q) {
    if (u[q] >= c->nv || v[q] >= c->nv) return fail(c, GV_ERR_OUT_OF_RANGE, "id >= num_nodes");
    vrow[q] = c->part.perm[u[q]];
    crow[q * (K + 1)] = c->part.perm[v[q]];
    for (uint32_t k = 0; k < K; ++k) {
      if (negs[q * K + k] >= c->nv) return fail(c, GV_ERR_OUT_OF_RANGE, "negative id >= num_nodes");
      crow[q * (K + 1) + 1 + k] = c->part.perm[negs[q * K + k]];
    }
  }
  Rank& r = c->ranks[0];
  DevBuf<uint32_t> dv, dc;
  CK(dv.ensure(count));
  CK(dc.ensure(crow.size()));
  CK(cudaMemcpy(dv.p, vrow.data(), sizeof(uint32_t) * count, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dc.p, crow.data(), sizeof(uint32_t) * crow.size(), cudaMemcpyHostToDevice));
  gv::ExplicitArgs a{dv.p, dc.p, count, r.vertex, r.context, c->stride, lr, c->opt.neg_weight};
  CK(gv::launch_sgd_explicit(a, c->dim, c->K, r.compute));
  CK(cudaStreamSynchronize(r.compute));
  dv.release();
  dc.release();
  return GV_OK;
}

gv_status gv_plan_step(uint32_t n, uint32_t D, uint32_t d, uint32_t t, gv_step_plan* out) {
  gv_ctx* c = nullptr;
  if (!out || n == 0 || n > 64 || D == 0 || n % D != 0 || d >= D || t >= n)
    return fail(c, GV_ERR_INVALID_ARG, "gv_plan_step: bad arguments");
  const uint32_t m = n / D;
  std::memset(out, 0, sizeof(*out));
  out->n_blocks = m;
  for (uint32_t g = 0; g < m; ++g) {
    out->vpart[g] = d * m + g;
    out->cpart[g] = (d * m + g + t) % n;
  }
  if (D == 1) {
    out->send_part = out->recv_part = UINT32_MAX;
    out->send_to = out->recv_from = 0;
    out->wait_block = UINT32_MAX;
  } else {
    out->send_part = (d * m + t) % n;        // = cpart[0]: free after block 0
    out->send_to = (d + D - 1) % D;
    out->recv_part = ((d + 1) * m + t) % n;  // = cpart[m-1] of step t+1
    out->recv_from = (d + 1) % D;
    out->wait_block = m - 1;
  }
  return GV_OK;
}

gv_status gv_device_bytes(gv_ctx* c, uint64_t* bytes) {
  if (gv_status s = check_ctx(c, true)) return s;
  uint64_t b = static_cast<uint64_t>(c->nv) * (4 + 8 + 4);
  if (!c->raw.host) b += c->raw.bytes_total();
  for (auto& r : c->ranks) {
    b += (r.vrows + r.crows) * c->stride * 4;
    b += r.blocks.bytes_total() + r.blocks_alt.bytes_total() + r.scratch.bytes_total();
    b += r.tile_tmp.bytes_total() + r.tile_scratch.bytes_total();
  }
  b += c->aug_scratch.bytes_total();
  *bytes = b;
  return GV_OK;
}

void gv_destroy(gv_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->opt.device);
  for (auto& r : c->ranks) {
    if (r.compute) cudaStreamSynchronize(r.compute);
    if (r.comm) cudaStreamSynchronize(r.comm);
  }
  if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
  if (c->tr) c->tr->close(c);  // peers may read this rank's exported memory until here
  for (auto& r : c->ranks) {
    cudaFree(r.vertex);
    cudaFree(r.context);
    r.blocks.release(); r.blocks_alt.release(); r.scratch.release();
    r.tile_tmp.release(); r.tile_scratch.release();
    r.counts.release(); r.desc.release(); r.loss.release(); r.chunk_ctr.release();
    if (r.counts_host) cudaFreeHost(r.counts_host);
    for (cudaEvent_t e : {r.ev_start, r.ev_bucket, r.ev_exch, r.ev_end,
                          r.ev_exch_sent, r.ev_last_recv})
      if (e) cudaEventDestroy(e);
    for (auto* v : {&r.ev_first_done, &r.ev_recv, &r.ev_sent, &r.ev_sgd})
      for (cudaEvent_t e : *v) cudaEventDestroy(e);
    if (r.compute) cudaStreamDestroy(r.compute);
    if (r.comm) cudaStreamDestroy(r.comm);
  }
  c->raw.release();
  if (c->raw_ready) cudaEventDestroy(c->raw_ready);
  if (c->fused_ready) cudaEventDestroy(c->fused_ready);
  if (c->alt_free) cudaEventDestroy(c->alt_free);
  c->fused_off.release();
  c->aug_scratch.release();
  if (c->raw_free) cudaEventDestroy(c->raw_free);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  gv::hp_destroy(c);
  cudaFree(c->d_packed);
  cudaFree(c->d_alias);
  cudaFree(c->d_woff);
  cudaFree(c->d_wnbr);
  cudaFree(c->d_walias);
  cudaFree(c->d_dalias);
  cudaFree(c->d_inv_perm);
  cudaFree(c->d_part_off);
  cudaFree(c->d_perm);
  gv::graph_share_unmap(&c->graph_map);
  delete c;
}

}  // extern "C"
