// augment.cpp — parallel online augmentation (Alg. 2).
//
// Each sampler thread owns a private segment of the pool ("each thread is
// allocated with an independent sample pool in advance"). It draws a
// departure node proportional to degree, walks walk_len edges choosing each
// neighbour proportional to the edge weight, emits the pairs of walk
// positions within distance s, and finally pseudo-shuffles its
// segment: pair k goes to sub-block k mod s, sub-blocks concatenated
// (P:198-199). Random numbers come from Philox with counter
// {walk, step, thread, 'WALK'} and key = seed (DESIGN.md R-AUG), so a pool is
// a pure function of (graph, seed, threads) whatever the thread timing.
#include "augment.hpp"

#include <algorithm>
#include <atomic>
#include <thread>

#include "../../include/gv.h"
#include "philox.cuh"

namespace gv {

int build_walk_tables(const HostGraph& g, int threads, WalkTables* t) {
  t->g = &g;
  t->departure.resize(g.nv);
  int rc = build_alias(g.deg.data(), g.nv, t->departure.data());
  if (rc) return rc;
  t->edge.assign(g.nbr.size(), ProbAlias{0, 0});
  // rows in interleaved blocks: hub rows (up to thousands of entries) sit at
  // random ids, so contiguous thread ranges would be unbalanced
  std::atomic<uint64_t> next{0};
  constexpr uint64_t kRows = 4096;
  std::vector<std::thread> pool;
  for (int th = 0; th < std::max(1, threads); ++th)
    pool.emplace_back([&] {
      for (uint64_t b; (b = next.fetch_add(kRows)) < g.nv;) {
        const uint64_t e = std::min<uint64_t>(g.nv, b + kRows);
        for (uint64_t v = b; v < e; ++v) {
          const uint64_t o = g.off[v], m = g.off[v + 1] - o;
          if (m == 0 || !(g.deg[v] > 0.0)) continue;  // unreachable by any walk
          build_alias(g.w.data() + o, static_cast<uint32_t>(m), t->edge.data() + o);
        }
      }
    });
  for (auto& x : pool) x.join();
  return GV_OK;
}

namespace {

inline uint32_t draw(const ProbAlias* t, uint32_t m, const u32x4& r) {
  const uint32_t slot = slot_of((static_cast<uint64_t>(r.x) << 32) | r.y, m);
  return alias_pick(t[slot].prob, t[slot].alias, slot, r.z);
}

// Walks are generated kBatch at a time, one step of every walk of the batch
// per round, in two phases: (1) read the current node's CSR range, draw the
// Philox numbers and the alias slot, prefetch the slot's table entries and
// neighbour; (2) resolve the draw and prefetch the next node's CSR offsets.
// The batch's independent random accesses are thus in flight together (the
// walk is a chain of dependent cache misses otherwise). Pairs are emitted in
// walk order and written straight to their pseudo-shuffled positions, so the
// segment is exactly the serial definition (R-AUG): walk w, step k draws
// Philox {w, k, thread, 'WALK'} whatever the batching.
constexpr uint32_t kBatch = 16;

void fill_segment(const WalkTables& t, uint32_t walk_len, uint32_t s, uint32_t thread,
                  uint64_t cap, uint64_t seed, const uint32_t* relabel, uint32_t* out) {
  const HostGraph& g = *t.g;
  const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
  const uint32_t W = walk_len + 1;
  std::vector<uint32_t> walks(static_cast<size_t>(kBatch) * W);
  std::vector<uint64_t> sub_start(s);  // pseudo shuffle: pair k -> sub_start[k % s] + k / s
  uint64_t acc = 0;
  for (uint32_t j = 0; j < s; ++j) {
    sub_start[j] = acc;
    acc += cap > j ? (cap - j + s - 1) / s : 0;
  }
  const uint64_t* off = g.off.data();
  const uint32_t* nbr = g.nbr.data();
  const ProbAlias* et = t.edge.data();
  uint64_t o[kBatch], slot[kBatch];
  uint32_t rz[kBatch];
  uint64_t filled = 0;
  for (uint32_t w0 = 0; filled < cap; w0 += kBatch) {
    for (uint32_t i = 0; i < kBatch; ++i) {
      const u32x4 r = philox4x32_10(u32x4{w0 + i, 0u, thread, kTagWalk}, k0, k1);
      const uint32_t x = draw(t.departure.data(), g.nv, r);
      walks[i * W] = x;
      __builtin_prefetch(off + x);
      if (relabel) __builtin_prefetch(relabel + x);
    }
    for (uint32_t k = 1; k <= walk_len; ++k) {
      for (uint32_t i = 0; i < kBatch; ++i) {
        const uint32_t x = walks[i * W + k - 1];
        o[i] = off[x];
        const uint32_t m = static_cast<uint32_t>(off[x + 1] - o[i]);
        const u32x4 r = philox4x32_10(u32x4{w0 + i, k, thread, kTagWalk}, k0, k1);
        slot[i] = slot_of((static_cast<uint64_t>(r.x) << 32) | r.y, m);
        rz[i] = r.z;
        __builtin_prefetch(et + o[i] + slot[i]);
        __builtin_prefetch(nbr + o[i] + slot[i]);
      }
      for (uint32_t i = 0; i < kBatch; ++i) {
        const uint64_t q = o[i] + slot[i];
        const uint32_t pick = alias_pick(et[q].prob, et[q].alias, static_cast<uint32_t>(slot[i]), rz[i]);
        const uint32_t x = nbr[o[i] + pick];
        walks[i * W + k] = x;
        __builtin_prefetch(off + x);
        if (relabel) __builtin_prefetch(relabel + x);  // mapped after the batch, from cache
      }
    }
    if (relabel)  // pairs in the pool's id space (a bijection: w_a != w_b is unchanged)
      for (uint32_t q = 0; q < kBatch * W; ++q) walks[q] = relabel[walks[q]];
    // pairs within distance s, walk by walk, by increasing start then end position
    for (uint32_t i = 0; i < kBatch && filled < cap; ++i) {
      const uint32_t* walk = walks.data() + static_cast<size_t>(i) * W;
      for (uint32_t a = 0; a <= walk_len && filled < cap; ++a) {
        const uint32_t last = a + s < walk_len ? a + s : walk_len;
        for (uint32_t b = a + 1; b <= last && filled < cap; ++b) {
          if (walk[a] == walk[b]) continue;
          const uint64_t pos = sub_start[filled % s] + filled / s;
          out[2 * pos] = walk[a];
          out[2 * pos + 1] = walk[b];
          ++filled;
        }
      }
    }
  }
}

}  // namespace

void augment(const WalkTables& t, uint32_t walk_len, uint32_t s, uint32_t threads,
             uint64_t count, uint64_t seed, uint32_t* out, const uint32_t* relabel) {
  std::vector<std::thread> pool;
  for (uint32_t th = 0; th < threads; ++th) {
    const uint64_t b = static_cast<uint64_t>((static_cast<unsigned __int128>(count) * th) / threads);
    const uint64_t e =
        static_cast<uint64_t>((static_cast<unsigned __int128>(count) * (th + 1)) / threads);
    pool.emplace_back(fill_segment, std::cref(t), walk_len, s, th, e - b, seed, relabel,
                      out + 2 * b);
  }
  for (auto& x : pool) x.join();
}

}  // namespace gv
