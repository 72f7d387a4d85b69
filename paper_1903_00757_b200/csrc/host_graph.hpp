// host_graph.hpp — host-side graph preparation of the product path (L0):
// ingest/symmetrise, degree, zig-zag partition + relabel, integer alias
// tables. Multi-threaded C++17; independent of the oracle.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace gv {

// Undirected graph, CSR over ORIGINAL ids.
struct HostGraph {
  uint32_t nv = 0;
  std::vector<uint64_t> off;  // nv + 1
  std::vector<uint32_t> nbr;  // 2|E| entries, ascending per row
  std::vector<double> w;      // merged weights
  std::vector<double> deg;    // weighted degree
  uint64_t undirected_edges() const { return nbr.size() / 2; }
};

// Zig-zag partition + relabel (fig:zig-zag_partition).
struct Partitioning {
  uint32_t n = 1;
  std::vector<uint32_t> perm;      // orig -> new
  std::vector<uint32_t> inv_perm;  // new -> orig
  std::vector<uint64_t> off;       // n + 1, partition p owns new ids [off[p], off[p+1])
  uint32_t pbits = 0;              // bits of the partition field of a packed id
  std::vector<uint32_t> packed;    // orig -> (part << (32-pbits)) | local
  uint64_t max_part() const;
};

// Integer alias table: slot k accepts itself when r < prob[k], else alias[k].
struct AliasU32 {
  std::vector<uint32_t> prob, alias;
};

// Returns 0 or a gv_status code; msg receives a description on error.
int build_graph(uint32_t nv, const uint32_t* src, const uint32_t* dst, const float* w,
                uint64_t ne, int threads, HostGraph* g, std::string* msg);
int build_partitioning(const HostGraph& g, uint32_t n, Partitioning* p, std::string* msg);
// Integer Vose over weights w[0..m) (reading R-ALIAS); writes into
// prob/alias (size m). Returns 0 or GV_ERR_EMPTY when the total mass is 0.
int build_alias(const double* w, uint32_t m, uint32_t* prob, uint32_t* alias);

// Runs f(begin, end) over [0, n) split across `threads` std::threads.
template <class F>
void parallel_for(uint64_t n, int threads, F f);

int default_threads();

}  // namespace gv

#include <thread>
namespace gv {
template <class F>
void parallel_for(uint64_t n, int threads, F f) {
  if (threads <= 1 || n < 4096) {
    f(uint64_t(0), n);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    uint64_t b = n * t / threads, e = n * (t + 1) / threads;
    pool.emplace_back([=] { f(b, e); });
  }
  for (auto& th : pool) th.join();
}
}  // namespace gv
