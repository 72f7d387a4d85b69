// host_graph.hpp — host-side graph preparation of the product path (L0):
// ingest/symmetrise, degree, zig-zag partition + relabel, integer alias
// tables. Multi-threaded C++17; independent of the oracle.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

namespace gv {

// An array that either owns its elements (a std::vector) or views memory it
// does not own — the node-shared graph segment that the ranks of a
// multi-process run map instead of each preparing the graph (graph_share.hpp).
template <class T>
class Arr {
 public:
  Arr() = default;
  Arr(const Arr&) = delete;
  Arr& operator=(const Arr&) = delete;
  Arr(Arr&& o) noexcept { *this = std::move(o); }
  Arr& operator=(Arr&& o) noexcept {
    const bool owned = o.p_ == o.own_.data();
    own_ = std::move(o.own_);
    p_ = owned ? own_.data() : o.p_;
    n_ = o.n_;
    o.p_ = nullptr;
    o.n_ = 0;
    return *this;
  }
  void assign(size_t n, const T& v) {
    own_.assign(n, v);
    p_ = own_.data();
    n_ = n;
  }
  void resize(size_t n) {
    own_.resize(n);
    p_ = own_.data();
    n_ = n;
  }
  void view(const T* p, size_t n) {  // drop owned storage, look at p[0..n)
    std::vector<T>().swap(own_);
    p_ = const_cast<T*>(p);
    n_ = n;
  }
  void release() { view(nullptr, 0); }
  T* data() { return p_; }
  const T* data() const { return p_; }
  size_t size() const { return n_; }
  T& operator[](size_t i) { return p_[i]; }
  const T& operator[](size_t i) const { return p_[i]; }
  T* begin() { return p_; }
  T* end() { return p_ + n_; }
  const T* begin() const { return p_; }
  const T* end() const { return p_ + n_; }

 private:
  std::vector<T> own_;
  T* p_ = nullptr;
  size_t n_ = 0;
};

// Undirected graph, CSR over ORIGINAL ids.
struct HostGraph {
  uint32_t nv = 0;
  Arr<uint64_t> off;  // nv + 1
  Arr<uint32_t> nbr;  // 2|E| entries, ascending per row
  Arr<double> w;      // merged weights (released once the walk tables are built)
  Arr<double> deg;    // weighted degree
  uint64_t undirected_edges() const { return nbr.size() / 2; }
};

// Zig-zag partition + relabel (fig:zig-zag_partition).
struct Partitioning {
  uint32_t n = 1;
  Arr<uint32_t> perm;      // orig -> new
  Arr<uint32_t> inv_perm;  // new -> orig
  Arr<uint64_t> off;       // n + 1, partition p owns new ids [off[p], off[p+1])
  uint32_t pbits = 0;      // bits of the partition field of a packed id
  Arr<uint32_t> packed;    // orig -> (part << (32-pbits)) | local
  uint64_t max_part() const;
};

// One slot of an integer alias table: slot k accepts itself when r < prob,
// else alias (layout of CUDA's uint2, so tables upload as they are).
struct ProbAlias {
  uint32_t prob, alias;
};

// Returns 0 or a gv_status code; msg receives a description on error.
int build_graph(uint32_t nv, const uint32_t* src, const uint32_t* dst, const float* w,
                uint64_t ne, int threads, HostGraph* g, std::string* msg);
int build_partitioning(const HostGraph& g, uint32_t n, Partitioning* p, std::string* msg);
// Integer Vose over weights w[0..m) (reading R-ALIAS); writes into
// out[0..m). Returns 0 or GV_ERR_EMPTY when the total mass is 0.
int build_alias(const double* w, uint32_t m, ProbAlias* out);

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
