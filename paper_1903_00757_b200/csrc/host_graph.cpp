// host_graph.cpp — graph preparation (ingest, degree, zig-zag, alias).
// Semantics follow DESIGN.md readings R-INGEST, R-ZIGZAG, R-ALIAS
// (SURVEY §8(c) steps 1-3). Written independently of oracle/.
#include "host_graph.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <memory>
#include <numeric>

#include "../../include/gv.h"

namespace gv {

int default_threads() {
  unsigned h = std::thread::hardware_concurrency();
  return h ? static_cast<int>(h) : 1;
}

uint64_t Partitioning::max_part() const {
  uint64_t m = 0;
  for (uint32_t p = 0; p < n; ++p) m = std::max(m, off[p + 1] - off[p]);
  return m;
}

// P:392 undirected; self-loops dropped; duplicates summed in input order;
// rows sorted by neighbour id; degree summed in that order.
int build_graph(uint32_t nv, const uint32_t* src, const uint32_t* dst, const float* w,
                uint64_t ne, int threads, HostGraph* g, std::string* msg) {
  const bool timing = getenv("GV_INGEST_TIMING") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[ingest] %s %.0f ms\n", what,
            std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  if (nv == 0) return GV_ERR_INVALID_ARG;
  if (ne >= (uint64_t(1) << 32)) {
    *msg = "at most 2^32-1 input edges";
    return GV_ERR_CAPACITY;
  }
  // 1) validation and row counts of the symmetrised multigraph (parallel;
  //    atomic counters). The first invalid edge (lowest k) is reported.
  std::vector<std::atomic<uint32_t>> deg_cnt(nv);
  for (auto& x : deg_cnt) x.store(0, std::memory_order_relaxed);
  std::atomic<uint64_t> bad_range{UINT64_MAX}, bad_weight{UINT64_MAX};
  auto lower_to = [](std::atomic<uint64_t>& a, uint64_t k) {
    uint64_t cur = a.load(std::memory_order_relaxed);
    while (k < cur && !a.compare_exchange_weak(cur, k, std::memory_order_relaxed)) {
    }
  };
  parallel_for(ne, threads, [&](uint64_t b, uint64_t e) {
    for (uint64_t k = b; k < e; ++k) {
      const uint32_t a = src[k], c = dst[k];
      if (a >= nv || c >= nv) {
        lower_to(bad_range, k);
        continue;
      }
      if (w && (!std::isfinite(w[k]) || w[k] < 0.0f)) lower_to(bad_weight, k);
      if (a == c) continue;
      deg_cnt[a].fetch_add(1, std::memory_order_relaxed);
      deg_cnt[c].fetch_add(1, std::memory_order_relaxed);
    }
  });
  if (bad_range.load() != UINT64_MAX || bad_weight.load() != UINT64_MAX) {
    if (bad_range.load() <= bad_weight.load()) {
      *msg = "edge " + std::to_string(bad_range.load()) + " has a node id >= num_nodes";
      return GV_ERR_OUT_OF_RANGE;
    }
    *msg = "edge " + std::to_string(bad_weight.load()) + " has a negative or non-finite weight";
    return GV_ERR_INVALID_ARG;
  }
  lap("validate + count");
  std::vector<uint64_t> cnt(static_cast<size_t>(nv) + 1, 0);
  for (uint32_t v = 0; v < nv; ++v) cnt[v + 1] = cnt[v] + deg_cnt[v].load(std::memory_order_relaxed);
  const uint64_t total = cnt[nv];
  if (total == 0) {
    *msg = "graph has no edge besides self-loops";
    return GV_ERR_EMPTY;
  }
  // 2) scatter (col, input index) entries into their rows
  struct Ent {  // 8 bytes: C5 has 3.6e9 directed entries
    uint32_t col;
    uint32_t k;  // input index: duplicates are summed in input order
  };
  std::unique_ptr<Ent[]> ent(new Ent[total]);
  {
    // parallel over the edges; each entry takes the next slot of its row
    // (atomic cursor). The order inside a row depends on the thread timing;
    // the per-row sort below by (column, input index) makes it canonical.
    std::vector<std::atomic<uint64_t>> cursor(nv);
    for (uint32_t v = 0; v < nv; ++v) cursor[v].store(cnt[v], std::memory_order_relaxed);
    parallel_for(ne, threads, [&](uint64_t b, uint64_t e) {
      for (uint64_t k = b; k < e; ++k) {
        const uint32_t a = src[k], c = dst[k];
        if (a == c) continue;
        ent[cursor[a].fetch_add(1, std::memory_order_relaxed)] = Ent{c, static_cast<uint32_t>(k)};
        ent[cursor[c].fetch_add(1, std::memory_order_relaxed)] = Ent{a, static_cast<uint32_t>(k)};
      }
    });
  }
  lap("scatter");
  // 3) per row: sort by (column, input index) — deterministic whatever the
  //    scatter order — and count the merged entries; rows are independent
  std::vector<uint64_t> merged(nv, 0);
  parallel_for(nv, threads, [&](uint64_t b, uint64_t e) {
    for (uint64_t v = b; v < e; ++v) {
      Ent* first = ent.get() + cnt[v];
      Ent* last = ent.get() + cnt[v + 1];
      std::sort(first, last, [](const Ent& x, const Ent& y) {
        return x.col != y.col ? x.col < y.col : x.k < y.k;
      });
      uint64_t u = 0;
      for (Ent* it = first; it != last; ++it)
        if (it == first || (it - 1)->col != it->col) ++u;
      merged[v] = u;
    }
  });
  lap("row sort");
  g->nv = nv;
  g->off.assign(static_cast<size_t>(nv) + 1, 0);
  for (uint32_t v = 0; v < nv; ++v) g->off[v + 1] = g->off[v] + merged[v];
  g->nbr.resize(g->off[nv]);
  g->w.resize(g->off[nv]);
  g->deg.assign(nv, 0.0);
  parallel_for(nv, threads, [&](uint64_t b, uint64_t e) {
    for (uint64_t v = b; v < e; ++v) {
      const Ent* first = ent.get() + cnt[v];
      const Ent* last = ent.get() + cnt[v + 1];
      uint64_t o = g->off[v] - 1;
      uint32_t prev = 0;
      bool have = false;
      for (const Ent* it = first; it != last; ++it) {
        const double wk = w ? static_cast<double>(w[it->k]) : 1.0;
        if (!have || it->col != prev) {
          ++o;
          g->nbr[o] = it->col;
          g->w[o] = wk;
          prev = it->col;
          have = true;
        } else {
          g->w[o] += wk;
        }
      }
      double s = 0.0;
      for (uint64_t q = g->off[v]; q < g->off[v + 1]; ++q) s += g->w[q];
      g->deg[v] = s;
    }
  });
  lap("merge + degree");
  return GV_OK;
}

// Zig-zag (R-ZIGZAG): rank nodes by (degree desc, id asc); rank r goes to
// part r%n on even rounds r/n and n-1-r%n on odd rounds; local id = r/n.
int build_partitioning(const HostGraph& g, uint32_t n, Partitioning* p, std::string* msg) {
  const uint32_t nv = g.nv;
  if (n == 0 || n > nv) {
    *msg = "n_partitions must be in [1, num_nodes]";
    return GV_ERR_INVALID_ARG;
  }
  std::vector<uint32_t> order(nv);
  std::iota(order.begin(), order.end(), 0u);
  std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
    if (g.deg[a] != g.deg[b]) return g.deg[a] > g.deg[b];
    return a < b;
  });
  p->n = n;
  p->off.assign(n + 1, 0);
  for (uint32_t q = 0; q < n; ++q) {
    // partition q receives ranks r with zig-zag position q: one per full round
    // plus one in the last partial round if it reaches q
    const uint64_t rounds = nv / n, rem = nv % n;
    const uint64_t last_round = rounds;  // index of the partial round
    const bool even = (last_round % 2) == 0;
    const uint64_t pos_in_round = even ? q : n - 1 - q;
    p->off[q + 1] = rounds + (pos_in_round < rem ? 1 : 0);
  }
  for (uint32_t q = 0; q < n; ++q) p->off[q + 1] += p->off[q];
  p->perm.resize(nv);
  p->inv_perm.resize(nv);
  for (uint32_t r = 0; r < nv; ++r) {
    const uint32_t round = r / n, pos = r % n;
    const uint32_t part = (round & 1u) ? (n - 1 - pos) : pos;
    const uint32_t nid = static_cast<uint32_t>(p->off[part] + round);
    p->perm[order[r]] = nid;
    p->inv_perm[nid] = order[r];
  }
  // packed ids: partition in the top pbits bits, local id below
  uint32_t pbits = 0;
  while ((1u << pbits) < n) ++pbits;
  p->pbits = pbits;
  const uint64_t local_limit = pbits ? (uint64_t(1) << (32 - pbits)) : (uint64_t(1) << 32);
  if (p->max_part() > local_limit) {
    *msg = "partition too large for the packed id range";
    return GV_ERR_CAPACITY;
  }
  p->packed.resize(nv);
  for (uint32_t q = 0; q < n; ++q)
    for (uint64_t id = p->off[q]; id < p->off[q + 1]; ++id) {
      const uint32_t local = static_cast<uint32_t>(id - p->off[q]);
      p->packed[p->inv_perm[id]] = pbits ? ((q << (32 - pbits)) | local) : local;
    }
  return GV_OK;
}

// Integer Vose (R-ALIAS): a_i = trunc(w_i m 2^32 / W); the residual
// m 2^32 - sum(a) goes to the first maximal a_i; FIFO worklists of
// under-full (< 2^32) and over-full slots in index order.
int build_alias(const double* w, uint32_t m, ProbAlias* out) {
  if (m == 0) return GV_ERR_EMPTY;
  double total = 0.0;
  for (uint32_t i = 0; i < m; ++i) total += w[i];
  if (!(total > 0.0)) return GV_ERR_EMPTY;
  constexpr uint64_t kOne = uint64_t(1) << 32;
  const double scale = static_cast<double>(m) * 4294967296.0 / total;
  // per-thread scratch: the walk tables build one table per node (65.6 M on
  // the Friendster-shaped graph), so no allocation per table
  thread_local std::vector<uint64_t> a;
  thread_local std::vector<uint32_t> under, over;  // FIFO queues: [head, tail)
  if (a.size() < m) {
    a.resize(m);
    under.resize(m);
    over.resize(m);
  }
  uint64_t sum = 0;
  uint32_t top = 0;
  for (uint32_t i = 0; i < m; ++i) {
    a[i] = static_cast<uint64_t>(w[i] * scale);
    sum += a[i];
    if (a[i] > a[top]) top = i;
  }
  a[top] += (static_cast<uint64_t>(m) << 32) - sum;
  uint32_t uh = 0, ut = 0, oh = 0, ot = 0;
  for (uint32_t i = 0; i < m; ++i) {
    if (a[i] < kOne) under[ut++] = i;
    else over[ot++] = i;
  }
  while (uh < ut && oh < ot) {
    const uint32_t s = under[uh++];
    const uint32_t l = over[oh];
    out[s] = ProbAlias{static_cast<uint32_t>(a[s]), l};
    a[l] -= kOne - a[s];
    if (a[l] < kOne) {
      ++oh;
      under[ut++] = l;  // at most m entries are ever queued: ut <= m
    }
  }
  while (uh < ut) {
    const uint32_t s = under[uh++];
    out[s] = ProbAlias{0xFFFFFFFFu, s};
  }
  while (oh < ot) {
    const uint32_t l = over[oh++];
    out[l] = ProbAlias{0xFFFFFFFFu, l};
  }
  return GV_OK;
}

}  // namespace gv
